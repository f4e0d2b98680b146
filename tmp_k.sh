for kv in "X=0" "NSK_GRID_CAP=32" "NSK_GRID_CAP=24" "NSK_GRID_CAP=12"; do
  echo "== $kv"; env $kv timeout 300 python tools/probe_step.py 2>&1 | grep -o "[0-9.]* ms/step"; env $kv timeout 300 python tools/probe_step.py --r50 2>&1 | grep -o "[0-9.]* ms/step"
  env $kv timeout 300 python bench.py --model gru --steps 20 --warmup 5 --no-sub 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*'
done
