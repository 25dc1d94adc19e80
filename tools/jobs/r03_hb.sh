#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q > $O/hb_tests.log 2>&1; echo "pytest rc=$?"; tail -4 $O/hb_tests.log
bash tools/jobs/r02b_ab2.sh hb1
python -c "
import json; d=json.loads(open('$O/ab2_hb1.jsonl').read().strip().splitlines()[-1]); print(d['roofline']['per_kernel']['spkm_hamerly_bounds'])"
