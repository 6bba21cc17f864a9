#!/bin/bash
# Step time of the C4 bench under scheduling knobs (env settings), one line each.
# Usage (under gpurun): bash tools/knob_sweep.sh TAG "ENV1=a,ENV2=b  ENV3=c ..."  ("-" = defaults)
TAG=${1:-knobs}; O=gpurun_out/$TAG; mkdir -p $O
for set in ${2:-"-"}; do
  envs=$(echo "$set" | tr ',' ' '); [ "$set" = "-" ] && envs=""
  env $envs timeout 600 python bench.py --no-cpu-baseline --steps ${STEPS:-6} --warmup 3 > $O/b.jsonl 2> $O/b.err
  python -c "import json;d=json.loads(open('$O/b.jsonl').readline());print('$set', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), {k: round(v,1) for k,v in d['profile_ms_per_step'].items()})" || tail -3 $O/b.err
done
