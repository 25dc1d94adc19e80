#!/bin/bash
# Session re-entry check: GPU suite + smoke, then the default bench line (C4) and the reference arm.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/s_gputest.log 2>&1; echo "pytest rc=$?" >> $O/s_gputest.log
tail -3 $O/s_gputest.log
python __graft_entry__.py smoke > $O/s_smoke.log 2>&1; tail -1 $O/s_smoke.log
( time python bench.py ) > $O/s_bench.jsonl 2> $O/s_bench.err; tail -4 $O/s_bench.err
( time python bench.py --impl reference --steps 1 --warmup 0 ) > $O/s_ref.jsonl 2> $O/s_ref.err; tail -4 $O/s_ref.err
