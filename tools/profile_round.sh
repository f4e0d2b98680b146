#!/bin/bash
# Run on the GPU box (gpurun): launch lists of the ResNet-18 / ResNet-50 / GRU steps (warm cache) and one full
# ncu capture of the dominant conv kernel. Summaries: python tools/ncu_summary.py gpurun_out/launches_<tag>_*.csv
mkdir -p gpurun_out
TAG=${1:-r1}
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/launches_${TAG}_r18.csv python tools/probe_step.py 256 > gpurun_out/probe_${TAG}_r18.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_${TAG}_r18.csv > gpurun_out/launches_${TAG}_r18_summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv -c 3000 \
    --log-file gpurun_out/launches_${TAG}_r50.csv python bench.py --model resnet50 --steps 2 --warmup 3 \
    > gpurun_out/probe_${TAG}_r50.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_${TAG}_r50.csv > gpurun_out/launches_${TAG}_r50_summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/launches_${TAG}_gru.csv python tools/probe_gru.py > gpurun_out/probe_${TAG}_gru.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_${TAG}_gru.csv > gpurun_out/launches_${TAG}_gru_summary.txt
ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 \
    -o gpurun_out/${TAG}_conv_fprop python tools/probe_conv.py fprop 256 32 64 64 3 1 1 > /dev/null 2>&1
ls -la gpurun_out | grep ${TAG}
