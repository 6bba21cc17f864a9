#!/bin/bash
O=gpurun_out/it16; mkdir -p $O
for v in "SQF_X=0" "SQF_LN_PARAMS_MAIN=1" "SQF_DEBUG_SKIP=2" "SQF_DEBUG_SKIP=4" "SQF_DEBUG_SKIP=8"; do env $v timeout 600 python bench.py --no-cpu-baseline --steps 4 > $O/b.jsonl 2>/dev/null; echo "$v $(cut -c180-250 $O/b.jsonl)"; done
timeout 900 python bench.py > $O/bench_full.jsonl 2> $O/bench_full.err; cut -c1-200 $O/bench_full.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/step_once.py --accum 2 --warmup 1 > $O/ncu_launch.log 2>&1
echo done
