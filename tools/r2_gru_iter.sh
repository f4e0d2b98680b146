timeout 900 python -m pytest tests/test_gpu_gru.py -q -x 2>&1 | tail -3
timeout 300 python tools/probe_gru.py 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v_launches_gru.csv python tools/probe_gru.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r2v_launches_gru.csv 2>&1 | head -16
