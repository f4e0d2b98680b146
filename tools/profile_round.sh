#!/bin/bash
# Run on the GPU box (gpurun): launch list of the bench step + one full ncu capture of the dominant kernel.
set -x
mkdir -p gpurun_out
TAG=${1:-r1}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 > gpurun_out/bench_under_ncu_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 \
    -o gpurun_out/conv_fprop_${TAG} python tools/probe_conv.py fprop 256 32 64 64 3 1 1 > gpurun_out/ncu_full_${TAG}.log 2>&1
ncu --set full --clock-control none -k regex:bn_apply -s 2 -c 1 -o gpurun_out/bn_apply_${TAG} \
    python tools/probe_step.py 64 --eager > gpurun_out/ncu_bn_${TAG}.log 2>&1
ls -la gpurun_out
