#!/bin/bash
# Re-entry check at HEAD: GPU suite + smoke + default bench line.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/q_smi.txt
timeout 1800 python -m pytest tests -m gpu -x -q --durations=5 > $O/q_gputest.log 2>&1; echo "pytest rc=$?" >> $O/q_gputest.log; tail -3 $O/q_gputest.log
python __graft_entry__.py smoke > $O/q_smoke.log 2>&1; tail -1 $O/q_smoke.log
( time python bench.py ) > $O/q_bench.jsonl 2> $O/q_bench.err; tail -3 $O/q_bench.err
python -c "
import json; d=json.loads(open('$O/q_bench.jsonl').read().strip().splitlines()[-1]); print('BENCH', round(d['value'],3), d['e2e'], d['roofline'].get('kernel'), d['roofline'].get('frac'), d['clocks'])
print({k:(v['ms'],v.get('frac')) for k,v in d['roofline']['per_kernel'].items()})"
