mkdir -p gpurun_out
T=32 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gru_fwd_tc -s 2 -c 1 -o gpurun_out/r2p_gru_fwd python tools/probe_gru.py > gpurun_out/r2p_ncu_fwd.log 2>&1
ls -la gpurun_out | grep r2p
