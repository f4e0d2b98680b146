#!/bin/bash
# A/B two builds of libnskb (compile-time variants) on the R18 conv table, alternating processes:
#   tools/ab_lib.sh abl/libnskb_<tag>.so [rounds] [model] [batch]
B=$1; R=${2:-2}; M=${3:-resnet18}; N=${4:-256}
for i in $(seq 1 $R); do
  echo "== A (in-tree) round $i"; timeout 300 python tools/conv_table.py $M $N | tail -1
  echo "== B ($B) round $i"; NSK_LIB=$B timeout 300 python tools/conv_table.py $M $N | tail -1
done
