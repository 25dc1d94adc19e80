#!/bin/bash
# Yin-Yang tests, then C4 per-variant device-timed fits (quick form).
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_yinyang.py -x -q > $O/y_tests.log 2>&1; echo "pytest rc=$?" >> $O/y_tests.log
tail -15 $O/y_tests.log
for v in yinyang simp_elkan hamerly; do
  python bench.py --config C4 --variants $v --no-cpu-baseline --no-e2e --no-roofline --steps 1 --warmup 1 > $O/y_c4_$v.jsonl 2> $O/y_c4_$v.err
  python -c "
import json; d=json.loads(open('$O/y_c4_$v.jsonl').read().strip().splitlines()[-1]); print('$v', round(d['value'],3), round(d['ms_per_step'],1), d['per_variant'])"
done
