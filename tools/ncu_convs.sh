#!/bin/bash
# ncu --set full captures of representative conv passes (run on the GPU box via gpurun).
mkdir -p gpurun_out
TAG=${1:-r1c}
run() {  # name kind n hw c k r st pad
  ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 \
      -o gpurun_out/${TAG}_$1 python tools/probe_conv.py $2 $3 $4 $5 $6 $7 $8 $9 > gpurun_out/${TAG}_$1.log 2>&1
}
run fprop32 fprop 256 32 64 64 3 1 1
run wgrad32 wgrad 256 32 64 64 3 1 1
run dgrad32 dgrad 256 32 64 64 3 1 1
run wgrad4 wgrad 256 4 512 512 3 1 1
run fprop8 fprop 256 8 256 256 3 1 1
run fprop56 fprop 64 56 64 64 3 1 1
ls -la gpurun_out | grep $TAG
