#!/bin/bash
O=gpurun_out/it19; mkdir -p $O
timeout 900 python bench.py > $O/bench_full.jsonl 2> $O/bench_full.err; cut -c1-150 $O/bench_full.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/step_once.py --accum 2 --warmup 1 > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc --launch-skip 40 -c 6 -o $O/gemm_full python tools/step_once.py --accum 1 --warmup 1 > $O/ncu_full.log 2>&1
echo done
