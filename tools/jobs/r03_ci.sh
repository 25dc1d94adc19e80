#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q -k "sparse_center or heavy or config or checks or yinyang" > $O/ci_tests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/ci_tests.log
bash tools/jobs/r02b_ab2.sh ci1 ci2
python -c "
import json; d=json.loads(open('$O/ab2_ci1.jsonl').read().strip().splitlines()[-1]); print(d['roofline']['time_share'])"
