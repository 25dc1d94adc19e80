#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
SPKM_LIB=$PWD/paper_2107_04074_b200/libspkm_lead1.so timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sparse_center or heavy" > $O/ld_tests.log 2>&1; echo "pytest rc=$?"; tail -2 $O/ld_tests.log
bash tools/jobs/r02b_ab2.sh base lead1=SPKM_LIB=lib:lead1 lead2=SPKM_LIB=lib:lead2
