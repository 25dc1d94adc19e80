#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q > $O/c3h_tests.log 2>&1; echo "pytest rc=$?"; tail -4 $O/c3h_tests.log
CFG=C3 STEPS=5 bash tools/jobs/r02b_ab2.sh c3new c3old=SPKM_EK_HEAVY_MINK=257
python bench.py --config C3 --no-cpu-baseline --steps 5 --warmup 3 > $O/c3h_bench.jsonl 2> $O/c3h_bench.err
python -c "
import json; d=json.loads(open('$O/c3h_bench.jsonl').read().strip().splitlines()[-1]); print('C3', round(d['value'],2), round(d['e2e']['value'],2), d['per_variant'])"
bash tools/jobs/r02b_ab2.sh c4check
