#!/bin/bash
O=gpurun_out/it18; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "layernorm" > $O/pytest_k.log 2>&1; echo "rc=$?" >> $O/pytest_k.log; tail -2 $O/pytest_k.log
for v in "SQF_X=0" "SQF_LN_FUSED=0"; do env $v timeout 600 python bench.py --no-cpu-baseline --steps 4 > $O/b.jsonl 2>/dev/null; echo "$v $(cut -c180-250 $O/b.jsonl)"; done
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
echo done
