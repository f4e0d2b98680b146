#!/bin/bash
# Iteration run on one B200: selected GPU tests, R18 bench line, warm launch list of the R18 step.
#   bash tools/r2_iter.sh TAG "pytest args"
TAG=${1:-r2x}
TESTS=${2:-tests -m gpu}
mkdir -p gpurun_out
timeout 1500 python -m pytest $TESTS -q -rfs -x --timeout 600 > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench_r18.log 2>&1; tail -1 gpurun_out/${TAG}_bench_r18.log | cut -c1-330
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/${TAG}_launches_r18.csv python tools/probe_step.py 256 > gpurun_out/${TAG}_probe.log 2>&1
tail -2 gpurun_out/${TAG}_probe.log
python tools/ncu_summary.py gpurun_out/${TAG}_launches_r18.csv > gpurun_out/${TAG}_launches_r18_summary.txt 2>&1
head -22 gpurun_out/${TAG}_launches_r18_summary.txt
