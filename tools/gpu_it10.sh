#!/bin/bash
O=gpurun_out/it10; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "bias_grad or gemm or colsum" > $O/pytest_k.log 2>&1; echo "rc=$?" >> $O/pytest_k.log; tail -2 $O/pytest_k.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.jsonl 2> $O/bench.err; cut -c100-200 $O/bench.jsonl
SQF_DEBUG_SKIP=16 timeout 600 python bench.py --no-cpu-baseline --steps 3 > $O/bench_unfused.jsonl 2>/dev/null; cut -c100-200 $O/bench_unfused.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/step_once.py --accum 2 --warmup 1 > $O/ncu_launch.log 2>&1
echo done
