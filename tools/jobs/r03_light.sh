#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q -k "elkan or audit or config or checks or loopback" > $O/lt_tests.log 2>&1; echo "pytest rc=$?"; tail -5 $O/lt_tests.log
bash tools/jobs/r02b_ab2.sh light1 light0=SPKM_EK_LIGHT=0 light1b
