#!/bin/bash
# GPU suite, then bench lines at C2 (20 steps), C3, C5 (with e2e) and a quick C4 line.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/c_gputest.log 2>&1; echo "pytest rc=$?" >> $O/c_gputest.log; tail -3 $O/c_gputest.log
python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > $O/c_C2.jsonl 2> $O/c_C2.err
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/c_C3.jsonl 2> $O/c_C3.err
python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $O/c_C5.jsonl 2> $O/c_C5.err
python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 > $O/c_C4.jsonl 2> $O/c_C4.err
for c in C2 C3 C5 C4; do python -c "
import json; d=json.loads(open('$O/c_$c.jsonl').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['value'],2), d.get('e2e',{}).get('value'), r.get('kernel'), r.get('frac'), d['clocks'].get('reasons'))"; done
