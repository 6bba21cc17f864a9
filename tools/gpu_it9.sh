#!/bin/bash
O=gpurun_out/it9; mkdir -p $O
timeout 600 python -m pytest tests/test_checkpoint.py tests/test_gpu_trainer.py -x -q > $O/pytest_ck.log 2>&1; echo "rc=$?" >> $O/pytest_ck.log
tail -2 $O/pytest_ck.log
for m in 0 1 2 3 4 8 15; do SQF_DEBUG_SKIP=$m timeout 300 python bench.py --no-cpu-baseline --steps 3 > $O/skip$m.jsonl 2>/dev/null; echo "skip=$m $(cut -c100-190 $O/skip$m.jsonl)"; done
echo done
