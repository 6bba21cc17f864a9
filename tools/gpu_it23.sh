#!/bin/bash
O=gpurun_out/it23; mkdir -p $O
for r in 1 2; do for v in "SQF_ACC_INPLACE=0" "SQF_ACC_INPLACE=1"; do env $v timeout 600 python bench.py --no-cpu-baseline --steps 6 > $O/b.jsonl 2>/dev/null; echo "$v $(cut -c180-250 $O/b.jsonl)"; done; done
echo done
