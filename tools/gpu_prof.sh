#!/bin/bash
# ncu --set full captures of the non-GEMM kernel classes of a C4 sub-batch
# (two steady-state launches each), exported as raw CSV for profiles/.
# Usage (under gpurun): bash tools/gpu_prof.sh TAG "regex1 regex2 ..."
TAG=${1:-prof}; O=gpurun_out/$TAG; mkdir -p $O
KS=${2:-"ln_fwd_v ln_dx_v colred_k fa::fwd_k fa::bwd_small_k fa::bwd_dq_k fa::bwd_dkv_k xent_v adam4_k nonfinite_k embed_fwd_v"}
for k in $KS; do
  n=$(echo $k | tr -c 'a-zA-Z0-9_\n' '_')
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 6 -c 2 -o $O/$n \
    python tools/step_once.py --accum 2 --warmup 1 > $O/$n.log 2>&1
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>/dev/null
  python tools/ncu_summary.py $O/$n.raw.csv >> $O/summary.txt 2>&1
done
cat $O/summary.txt
