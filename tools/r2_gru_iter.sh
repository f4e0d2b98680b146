timeout 300 python tools/trace_gru.py 2>&1 | tail -12
timeout 300 python tools/probe_gru.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_gru.py -q -x 2>&1 | tail -2
