#!/bin/bash
# ncu --set full of the short-sentence attention kernels (tools/nn_bench.py attention shapes)
O=gpurun_out/${1:-attn_ncu}; mkdir -p $O
for k in fwd_k bwd_small_k; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:"^$k\$" -s 5 -c 1 -o $O/$k python tools/nn_bench.py attention > $O/$k.log 2>&1
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/$k.raw.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page source --csv > $O/$k.source.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page source --csv --print-source=cuda,sass > $O/$k.cuda.csv 2>/dev/null
  rm -f $O/$k.ncu-rep
  python tools/ncu_summary.py $O/$k.raw.csv
done
