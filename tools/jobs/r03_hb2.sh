#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
for t in base hb6 hb8; do
  L=""; [ $t != base ] && L="SPKM_LIB=$PWD/paper_2107_04074_b200/libspkm_$t.so"
  env $L python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 --variants hamerly > $O/hb2_$t.jsonl 2> $O/hb2_$t.err
  python -c "
import json; d=json.loads(open('$O/hb2_$t.jsonl').read().strip().splitlines()[-1]); print('$t', round(d['value'],3), d['roofline']['per_kernel']['spkm_hamerly_bounds'])" 2>&1 | tail -1
done
