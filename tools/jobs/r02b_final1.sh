#!/bin/bash
# Default bench line (C4) + reference arm (timed), then A/Bs: row pass occupancy at C4, EB=4 Elkan scan at C2.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
( time python bench.py ) > $O/f_bench.jsonl 2> $O/f_bench.err; tail -3 $O/f_bench.err
python -c "
import json; d=json.loads(open('$O/f_bench.jsonl').read().strip().splitlines()[-1]); print('BENCH', round(d['value'],3), d['e2e'], d['roofline'].get('kernel'), d['roofline'].get('frac'), d['clocks'])"
( time python bench.py --impl reference --steps 3 --warmup 1 ) > $O/f_ref.jsonl 2> $O/f_ref.err; tail -3 $O/f_ref.err; cut -c1-300 $O/f_ref.jsonl
bash tools/jobs/r02b_ab2.sh rp1 rp2=SPKM_LIB=lib:rp2 rp2u3=SPKM_LIB=lib:rp2u3
CFG=C2 STEPS=5 EXTRA="--warmup 3" bash tools/jobs/r02b_ab2.sh c2 c2ek4m1=SPKM_LIB=lib:ek4m1
