#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q > $O/ah_tests.log 2>&1; echo "pytest rc=$?"; tail -4 $O/ah_tests.log
bash tools/jobs/r02b_ab2.sh ah1 ah0=SPKM_EK_ALLHEAVY=0 ah1b
