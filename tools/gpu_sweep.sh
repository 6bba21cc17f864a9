#!/bin/bash
# C5-style sweep on one GPU: Transformer-big fp16, per-GPU max_tokens 1k..16k, update_freq 1
O=gpurun_out/sweep; mkdir -p $O
[ "${SKIP_TESTS:-0}" = "1" ] || { timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log; }
for mt in 1024 2048 4096 8192 16384; do
  timeout 600 python bench.py --no-cpu-baseline --max-tokens $mt --accum 1 --steps 20 --warmup 5 > $O/c5_$mt.jsonl 2> $O/c5_$mt.err
  python -c "import json;d=json.loads(open('$O/c5_$mt.jsonl').readline());print($mt, round(d['value']), round(d['ms_per_step'],2), d['roofline']['frac'])"
done
timeout 600 python bench.py --no-cpu-baseline --steps 4 > $O/c4.jsonl 2>/dev/null; cut -c180-250 $O/c4.jsonl
echo done
