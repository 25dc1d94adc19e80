#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py -x -q -k "heavy or sparse_center_index" > $O/pr_tests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pr_tests.log
bash tools/jobs/r02b_ab2.sh pair1 pair0=SPKM_LIB=lib:pair0 pair1b pair0b=SPKM_LIB=lib:pair0
