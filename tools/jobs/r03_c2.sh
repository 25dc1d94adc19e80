#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
for t in new prev new2 prev2; do
  L=""; case $t in prev*) L="SPKM_LIB=$PWD/paper_2107_04074_b200/libspkm_prev.so";; esac
  env $L python bench.py --config C2 --k 100 --no-cpu-baseline --no-e2e --no-roofline --steps 20 --warmup 5 > $O/c2_$t.jsonl 2> $O/c2_$t.err
  python -c "
import json; d=json.loads(open('$O/c2_$t.jsonl').read().strip().splitlines()[-1]); print('C2 $t', round(d['value'],1))" 2>&1 | tail -1
done
