#!/bin/bash
O=gpurun_out/it14; mkdir -p $O
for v in "SQF_STREAM_PRIO=0" "SQF_STREAM_PRIO=2" "SQF_PAIR=1" "SQF_GEMM_STREAM_K=0"; do env $v timeout 600 python bench.py --no-cpu-baseline --steps 4 > $O/b.jsonl 2>/dev/null; echo "$v $(cut -c180-250 $O/b.jsonl)"; done
echo done
