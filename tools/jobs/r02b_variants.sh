#!/bin/bash
# C4: one device-timed fit of every variant (quick form) -> per-variant seconds per fit.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
for v in standard elkan simp_elkan hamerly simp_hamerly yinyang; do
  python bench.py --config C4 --variants $v --no-cpu-baseline --no-e2e --no-roofline --steps 2 --warmup 1 > $O/v_$v.jsonl 2> $O/v_$v.err
  python -c "
import json; d=json.loads(open('$O/v_$v.jsonl').read().strip().splitlines()[-1]); pv=d['per_variant']['$v']
print('$v', round(d['ms_per_step']/1e3,3), 's/fit', round(d['value'],2), 'it/s', pv['iterations'], 'its', round(pv['pruned_frac'],4), 'pruned', pv['objective'])"
done
