#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q -k "elkan or audit or parity or golden or config" > $O/eb_tests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/eb_tests.log
bash tools/jobs/r02b_ab2.sh eb1 eb2
