#!/bin/bash
O=gpurun_out/it21; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.jsonl 2> $O/ref.err; echo "ref rc=$?"; cut -c1-300 $O/ref.jsonl
timeout 900 python bench.py --config C3 --no-cpu-baseline > $O/c3.jsonl 2> $O/c3.err; echo "c3 rc=$?"; cut -c1-250 $O/c3.jsonl
timeout 900 python bench.py --config C2 --no-cpu-baseline > $O/c2.jsonl 2> $O/c2.err; echo "c2 rc=$?"; cut -c1-250 $O/c2.jsonl
echo done
