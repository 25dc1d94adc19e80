#!/bin/bash
# C2 (5 variants, k = 100): round-1 tree, start-of-round-2 tree and HEAD on the same box, interleaved.
O=$PWD/gpurun_out
for rep in 1 2; do
for t in 35da942 82e2bd2 HEAD; do
  if [ $t = HEAD ]; then d=$PWD; else d=$PWD/baseline/_old/$t; fi
  (cd $d && python bench.py --config C2 --k 100 --variants standard,elkan,simp_elkan,hamerly,simp_hamerly --steps 20 --warmup 5 --no-cpu-baseline > $O/o_$t.jsonl 2> $O/o_$t.err)
  python -c "
import json; d=json.loads(open('$O/o_$t.jsonl').read().strip().splitlines()[-1]); print('$t', round(d['value'],1), round(d['ms_per_step'],3), d.get('e2e',{}).get('value') if isinstance(d.get('e2e'),dict) else d.get('e2e'))"
done; done
