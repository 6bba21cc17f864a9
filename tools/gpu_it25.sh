#!/bin/bash
O=gpurun_out/it25; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > $O/pytest_a.log 2>&1; echo "rc=$?" >> $O/pytest_a.log; tail -2 $O/pytest_a.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
for r in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 6 > $O/b.jsonl 2>/dev/null; cut -c180-250 $O/b.jsonl; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/step_once.py --accum 2 --warmup 1 > $O/ncu_launch.log 2>&1
echo done
