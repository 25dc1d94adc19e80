#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_validation.py -x -q -k "heavy or sparse_center_index or audit" > $O/d_tests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/d_tests.log
bash tools/jobs/r02b_ab2.sh base d2=SPKM_CI_DIV=2 d3=SPKM_CI_DIV=3 d6=SPKM_CI_DIV=6 d8=SPKM_CI_DIV=8 d16=SPKM_CI_DIV=16
