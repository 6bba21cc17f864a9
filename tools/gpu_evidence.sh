#!/bin/bash
# Evidence run on one B200: bench (default), per-class ncu metrics of one
# 2-sub-batch C4 step, ncu --set full of GEMM launches of each class.
TAG=${1:-evidence}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 5 > $O/bench.jsonl 2> $O/bench.err; cut -c1-300 $O/bench.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file $O/step_metrics.csv python tools/step_once.py --accum 2 --warmup 1 > $O/ncu_metrics.log 2>&1
python tools/ncu_classes.py $O/step_metrics.csv > $O/classes.txt 2>&1; cat $O/classes.txt
for k in gemm_tc2; do
  timeout 900 ncu --set full --clock-control none -k regex:gemm_tc2 -s ${GEMM_SKIP:-300} -c ${GEMM_COUNT:-24} -o $O/gemm_full python tools/step_once.py --accum ${GEMM_ACCUM:-4} --warmup 1 > $O/ncu_full.log 2>&1
  ncu -i $O/gemm_full.ncu-rep --page raw --csv > $O/gemm_full.raw.csv 2>/dev/null; rm -f $O/gemm_full.ncu-rep
  python tools/ncu_summary.py $O/gemm_full.raw.csv > $O/gemm_full.txt; cat $O/gemm_full.txt
done
