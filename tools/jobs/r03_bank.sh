#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q -k "sparse_center or heavy or config or checks" > $O/bk_tests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/bk_tests.log
bash tools/jobs/r02b_ab2.sh bank1 bank2
