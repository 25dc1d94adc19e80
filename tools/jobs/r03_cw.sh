#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q > $O/cw_tests.log 2>&1; echo "pytest rc=$?"; tail -4 $O/cw_tests.log
bash tools/jobs/r02b_ab2.sh cw1 m5=SPKM_LIB=lib:m5 m6=SPKM_LIB=lib:m6 cw2
