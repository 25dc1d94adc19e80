#!/bin/bash
# A/B of the gathers' L2 eviction hints and the cluster ordering at C4 (device-timed value only).
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
B="python bench.py --config C4 --no-cpu-baseline --no-e2e --no-roofline --steps 1 --warmup 1"
$B > $O/ab_hot64.jsonl 2>$O/ab.err
SPKM_HOT_MB=0 $B > $O/ab_hot0.jsonl 2>>$O/ab.err
SPKM_HOT_MB=110 $B > $O/ab_hot110.jsonl 2>>$O/ab.err
SPKM_ORDER=0 $B > $O/ab_order0.jsonl 2>>$O/ab.err
SPKM_HOT_MB=32 $B > $O/ab_hot32.jsonl 2>>$O/ab.err
for f in $O/ab_*.jsonl; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],3), round(d['ms_per_step'],1))"; done
