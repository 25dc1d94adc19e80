#!/bin/bash
# Default bench line + reference arm at HEAD, per-variant C4 fits, fused-Elkan A/B at C4.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
( time python bench.py ) > $O/g_bench.jsonl 2> $O/g_bench.err; tail -3 $O/g_bench.err
( time python bench.py --impl reference ) > $O/g_ref.jsonl 2> $O/g_ref.err; tail -3 $O/g_ref.err
python -c "
import json; d=json.loads(open('$O/g_bench.jsonl').read().strip().splitlines()[-1]); print('BENCH', d['value'], d['e2e'], d['clocks'])
r=json.loads(open('$O/g_ref.jsonl').read().strip().splitlines()[-1]); print('REF', r['value'], r['cpu_baseline']['cores'])"
bash tools/jobs/r02b_variants.sh
bash tools/jobs/r02b_ab2.sh nofuse fuse=SPKM_ELKAN_FUSE=1 ebm4=SPKM_LIB=lib:ebm4
