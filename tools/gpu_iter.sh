#!/bin/bash
# Iteration loop on the GPU box: parity suite, GEMM calibration, bench.
O=gpurun_out/${1:-iter}
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
if [ "${SKIP_CALIB:-0}" != "1" ]; then timeout 300 python tools/gemm_calib.py > $O/calib.txt 2>&1; fi
timeout 600 python bench.py --no-cpu-baseline > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
cat $O/bench.jsonl | cut -c1-400
if [ -n "$NCU_LAUNCH" ]; then timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python tools/step_once.py --accum 2 --warmup 1 > $O/ncu_launch.log 2>&1; fi
echo done
