#!/bin/bash
# ncu --set full captures of kernel classes of a C4 step (two launches each,
# after `skip` launches of that kernel), exported as raw CSV + one summary line
# per launch. Usage (under gpurun): bash tools/gpu_prof.sh TAG "name:skip ..."
# (names are ncu's base kernel names, e.g. fwd_k, bwd_small_k, ln_fwd_v)
TAG=${1:-prof}; O=gpurun_out/$TAG; mkdir -p $O
KS=${2:-"ln_fwd_v:6 ln_dx_v:6 colred_k:6 fwd_k:6 bwd_small_k:6 bwd_dq_k:2 bwd_dkv_k:2 xent_v:0 adam4_k:2 nonfinite_k:0"}
for ks in $KS; do
  k=${ks%%:*}; s=${ks##*:}
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -s $s -c 2 -o $O/$k \
    python tools/step_once.py --accum 2 --warmup 1 > $O/$k.log 2>&1
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/$k.raw.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page source --csv > $O/$k.source.csv 2>/dev/null; rm -f $O/$k.ncu-rep
  python tools/ncu_summary.py $O/$k.raw.csv >> $O/summary.txt 2>&1
done
cat $O/summary.txt
