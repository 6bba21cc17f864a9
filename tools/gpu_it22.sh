#!/bin/bash
O=gpurun_out/it22; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.jsonl 2>$O/bench.err; cut -c180-250 $O/bench.jsonl
echo done
