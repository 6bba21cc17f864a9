#!/bin/bash
O=gpurun_out/it15; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
for v in "SQF_STREAM_PRIO=0" "SQF_STREAM_PRIO=2" "SQF_PAIR=1" "SQF_PAIR=1 SQF_STREAM_PRIO=2" "SQF_PAIR=1 SQF_STREAM_PRIO=1"; do env $v timeout 600 python bench.py --no-cpu-baseline --steps 4 > $O/b.jsonl 2>/dev/null; echo "$v $(cut -c180-250 $O/b.jsonl)"; done
echo done
