#!/bin/bash
# GPU test suite + smoke, then a C4 bench of the current code (ordering on) and an A/B with SPKM_ORDER=0.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/r02_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02_gputest.log
python __graft_entry__.py smoke > $O/r02_smoke.log 2>&1
B="python bench.py --config C4 --k 1000 --no-cpu-baseline --variants hamerly,simp_elkan"
$B --steps 2 --warmup 1 > $O/r02_c4_order.jsonl 2> $O/r02_c4_order.err
