#!/bin/bash
# ncu --set full of selected kernels inside tools/nn_bench.py [MODE]
# Usage: bash tools/kern_ncu.sh TAG "MODE|-" kernel_base_name...
O=gpurun_out/${1:-kern_ncu}; MODE=${2:--}; shift 2; mkdir -p $O
[ "$MODE" = "-" ] && MODE=""
for k in "$@"; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:"^$k\$" -s 5 -c 1 -o $O/$k python tools/nn_bench.py $MODE > $O/$k.log 2>&1
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/$k.raw.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page source --csv --print-source=cuda,sass > $O/$k.cuda.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page details --csv > $O/$k.details.csv 2>/dev/null
  rm -f $O/$k.ncu-rep
  python tools/ncu_summary.py $O/$k.raw.csv
done
