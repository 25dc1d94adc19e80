#!/bin/bash
# New GPU tests (config parity, loopback ranks, device corpus layout, dense Elkan), then the C4
# locality experiment, then compute-sanitizer.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
free -g | head -2 > $O/n_free.txt; nproc >> $O/n_free.txt
timeout 1500 python -m pytest tests/test_gpu_prepare.py tests/test_gpu_loopback.py tests/test_gpu_config_parity.py \
   "tests/test_gpu_parity.py::test_c5_dense_subsample_parity" -x -q --durations=15 > $O/n_tests.log 2>&1
echo "pytest rc=$?" >> $O/n_tests.log; tail -25 $O/n_tests.log
timeout 1200 python tools/c4_locality.py > $O/n_locality.jsonl 2> $O/n_locality.err; echo "locality rc=$?"
cat $O/n_locality.jsonl | cut -c1-600
bash tools/jobs/r02b_sanitize.sh
cat $O/san_summary.txt
