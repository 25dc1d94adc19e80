#!/bin/bash
# C4 device-timed A/B: each argument is an env assignment list (comma-separated), "-" = defaults.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
B="python bench.py --config ${CFG:-C4} --no-cpu-baseline --no-e2e --no-roofline --steps ${STEPS:-1} --warmup 1 ${EXTRA}"
for kv in "$@"; do
  envs=$(echo "$kv" | tr ',' ' '); [ "$kv" = "-" ] && envs=""
  env $envs $B > $O/ab_run.jsonl 2>>$O/ab_run.err
  python -c "
import json; d=json.loads(open('$O/ab_run.jsonl').read().strip().splitlines()[-1]); print('$kv', round(d['value'],3), round(d['ms_per_step'],1))"
done
