#!/bin/bash
O=gpurun_out/it6; mkdir -p $O
timeout 300 python tools/gemm_scale.py > $O/scale.txt 2>&1; cat $O/scale.txt
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "stream_k or gemm" > $O/pytest_sk.log 2>&1; echo "rc=$?" >> $O/pytest_sk.log
tail -3 $O/pytest_sk.log
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.jsonl 2> $O/bench.err; cut -c1-300 $O/bench.jsonl
timeout 300 python tools/gemm_calib.py > $O/calib.txt 2>&1
echo done
