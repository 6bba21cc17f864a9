#!/bin/bash
# One GPU session: parity tests, bench, GEMM microbench, ncu launch list + full capture.
# Usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag]
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
GB_BACK2BACK=1 timeout 300 python tools/gemm_bench.py > $O/gemm_bench.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python tools/step_once.py --accum 2 --warmup 1 > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc --launch-skip 300 -c 4 \
  -o $O/gemm_step python tools/step_once.py --accum 1 --warmup 1 > $O/ncu_full.log 2>&1
echo done
