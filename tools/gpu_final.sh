#!/bin/bash
# Round-end evidence run on one B200: parity suite, bench (with the CPU
# reference baseline), ncu launch list of a 2-sub-batch step, ncu --set full of
# six GEMM launches inside a sub-batch.
O=gpurun_out/final; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_full.jsonl 2> $O/bench_full.err; cut -c1-150 $O/bench_full.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/step_once.py --accum 2 --warmup 1 > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc --launch-skip 40 -c 6 -o $O/gemm_full python tools/step_once.py --accum 1 --warmup 1 > $O/ncu_full.log 2>&1
echo done
