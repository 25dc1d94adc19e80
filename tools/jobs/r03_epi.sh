#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q > $O/ep_tests.log 2>&1; echo "pytest rc=$?"; tail -4 $O/ep_tests.log
bash tools/jobs/r02b_ab2.sh epi1 epi2
CFG=C2 EXTRA="--k 100" STEPS=10 bash tools/jobs/r02b_ab2.sh c2a c2b
CFG=C3 STEPS=5 bash tools/jobs/r02b_ab2.sh c3a
