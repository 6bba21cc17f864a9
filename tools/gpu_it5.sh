#!/bin/bash
O=gpurun_out/it5; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "stream_k or gemm" > $O/pytest_sk.log 2>&1; echo "rc=$?" >> $O/pytest_sk.log
tail -3 $O/pytest_sk.log
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.jsonl 2> $O/bench.err; cut -c1-300 $O/bench.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/step_once.py --accum 2 --warmup 1 > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_small --launch-skip 20 -c 1 -o $O/attn_bwd python tools/step_once.py --accum 1 --warmup 1 > $O/ncu_attn.log 2>&1
echo done
