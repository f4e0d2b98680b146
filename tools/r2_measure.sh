mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_parity_c2.py tests/test_gpu_models.py -q -rf -x > gpurun_out/r2g_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2g_pytest.log
timeout 300 python tools/probe_gru.py > gpurun_out/r2g_gru.log 2>&1; tail -2 gpurun_out/r2g_gru.log
NSK_GRU_TC=0 timeout 300 python tools/probe_gru.py > gpurun_out/r2g_gru_simt.log 2>&1; tail -2 gpurun_out/r2g_gru_simt.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches_gru.csv python tools/probe_gru.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r2g_launches_gru.csv > gpurun_out/r2g_launches_gru_summary.txt 2>&1; head -20 gpurun_out/r2g_launches_gru_summary.txt
timeout 300 python bench.py > gpurun_out/r2g_bench.log 2>&1; tail -1 gpurun_out/r2g_bench.log | cut -c1-600
