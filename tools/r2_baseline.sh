#!/bin/bash
# Round-2 measurement on one B200: full GPU test suite, smoke, bench lines (R18, R50, reference arm),
# GRU probe, warm launch list of the R18 step. Outputs under gpurun_out/ (TAG prefix).
TAG=${1:-r2a}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfs -x --timeout 600 > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench_r18.log 2>&1; tail -1 gpurun_out/${TAG}_bench_r18.log | cut -c1-400
timeout 600 python bench.py --model resnet50 --steps 10 > gpurun_out/${TAG}_bench_r50.log 2>&1; tail -1 gpurun_out/${TAG}_bench_r50.log | cut -c1-300
timeout 300 python tools/probe_gru.py > gpurun_out/${TAG}_gru.log 2>&1; tail -2 gpurun_out/${TAG}_gru.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/${TAG}_launches_r18.csv python tools/probe_step.py 256 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_launches_r18.csv > gpurun_out/${TAG}_launches_r18_summary.txt 2>&1
head -25 gpurun_out/${TAG}_launches_r18_summary.txt
