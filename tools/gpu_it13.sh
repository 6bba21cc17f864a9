#!/bin/bash
O=gpurun_out/it13; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
for pr in 1 0; do SQF_STREAM_PRIO=$pr timeout 600 python bench.py --no-cpu-baseline > $O/bench_p$pr.jsonl 2>/dev/null; echo "prio=$pr $(cut -c100-200 $O/bench_p$pr.jsonl)"; done
echo done
