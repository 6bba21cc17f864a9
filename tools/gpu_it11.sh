#!/bin/bash
O=gpurun_out/it11; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_trainer.py -x -q -k "dropout" > $O/pytest_d.log 2>&1; echo "rc=$?" >> $O/pytest_d.log; tail -2 $O/pytest_d.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.jsonl 2> $O/bench.err; cut -c100-200 $O/bench.jsonl
SQF_WGRAD_TILE=0 timeout 600 python bench.py --no-cpu-baseline > $O/bench_t0.jsonl 2>/dev/null; cut -c100-200 $O/bench_t0.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc --launch-skip 40 -c 6 -o $O/gemm_full python tools/step_once.py --accum 1 --warmup 1 > $O/ncu_full.log 2>&1
echo done
