#!/bin/bash
O=gpurun_out/it7; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "stream_k" > $O/pytest_sk.log 2>&1; echo "rc=$?" >> $O/pytest_sk.log
tail -3 $O/pytest_sk.log
for sk in 0 1 2; do SQF_GEMM_STREAM_K=$sk timeout 600 python bench.py --no-cpu-baseline --steps 4 > $O/bench_sk$sk.jsonl 2> $O/bench_sk$sk.err; echo "sk=$sk"; cut -c100-200 $O/bench_sk$sk.jsonl; done
echo done
