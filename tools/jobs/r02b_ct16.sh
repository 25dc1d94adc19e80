#!/bin/bash
# fp16 screening of the full passes: GPU suite, then C4 / C3 device-timed lines with SPKM_CT16=1 (default) and 0.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/h_gputest.log 2>&1; echo "pytest rc=$?" >> $O/h_gputest.log
tail -4 $O/h_gputest.log
for cfg in C4 C3; do
for v in 1 0; do
  SPKM_CT16=$v python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $O/h_${cfg}_$v.jsonl 2> $O/h_${cfg}_$v.err
  python -c "
import json; d=json.loads(open('$O/h_${cfg}_$v.jsonl').read().strip().splitlines()[-1])
pk=d['roofline'].get('per_kernel',{})
print('$cfg ct16=$v', round(d['value'],3), round(d['ms_per_step'],1), {k:v2['ms'] for k,v2 in pk.items() if v2['ms']>5})"
done; done
