# GRU C3 step: warm launch list (ncu per-launch durations, serialised) -> gpurun_out/<tag>_launches_gru.csv + summary
tag=${1:-r2x}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${tag}_launches_gru.csv python bench.py --model gru --steps 3 --warmup 3 --no-sub \
  > gpurun_out/${tag}_ncu_gru.log 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_launches_gru.csv > gpurun_out/${tag}_launches_gru_summary.txt 2>&1
head -30 gpurun_out/${tag}_launches_gru_summary.txt
