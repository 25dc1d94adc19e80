#!/bin/bash
# GPU suite, then C2 (5 variants, 20 steps): HEAD vs A/B builds vs the round-1 tree; C4 quick line.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=$PWD/gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/x_gputest.log 2>&1; echo "pytest rc=$?" >> $O/x_gputest.log; tail -3 $O/x_gputest.log
CFG=C2 STEPS=20 EXTRA="--warmup 5 --k 100 --variants standard,elkan,simp_elkan,hamerly,simp_hamerly" bash tools/jobs/r02b_ab2.sh head hintall=SPKM_LIB=lib:hintall ekr1off=SPKM_LIB=lib:ekr1off head2
(cd baseline/_old/35da942 && python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > $O/x_old.jsonl 2> $O/x_old.err)
python -c "
import json; d=json.loads(open('$O/x_old.jsonl').read().strip().splitlines()[-1]); print('r01 tree', round(d['value'],1))"
bash tools/jobs/r02b_ab2.sh c4
