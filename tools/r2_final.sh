#!/bin/bash
# Round-2 closing measurement on one B200: full GPU suite, smoke, default bench line (R18 + C4/C3 sub-runs), warm
# launch lists of the R18 and GRU steps. Outputs under gpurun_out/r2final_*.
mkdir -p gpurun_out
T=r2final
timeout 2400 python -m pytest tests -m gpu -q -rfs --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; tail -1 gpurun_out/${T}_bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/${T}_launches_r18.csv python tools/probe_step.py 256 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${T}_launches_r18.csv > gpurun_out/${T}_launches_r18_summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/${T}_launches_gru.csv python tools/probe_gru.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${T}_launches_gru.csv > gpurun_out/${T}_launches_gru_summary.txt 2>&1
head -6 gpurun_out/${T}_launches_r18_summary.txt
B=64 T=128 timeout 300 python tools/trace_gru.py > gpurun_out/${T}_gru_trace_fwd.txt 2>&1
BWD=1 B=64 T=128 timeout 300 python tools/trace_gru.py > gpurun_out/${T}_gru_trace_bwd.txt 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_reference.log 2>&1; tail -1 gpurun_out/${T}_bench_reference.log | cut -c1-300
