#!/bin/bash
# Elkan heavy-row pass: tests, then C4 A/B over SPKM_EK_HEAVY_PCT.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py -x -q -k "heavy or sparse_center_index" > $O/h_tests.log 2>&1; echo "pytest rc=$?"; tail -5 $O/h_tests.log
PRETEST="" bash tools/jobs/r02b_ab2.sh "$@"
