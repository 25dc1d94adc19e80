#!/bin/bash
# Round-2 C4 baseline: bench line, launch list, ncu --set full of the C4 gather / bound / center kernels.
set -x
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
B="python bench.py --config C4 --k 1000 --no-cpu-baseline"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r02_smi.txt
$B --variants hamerly,simp_elkan --steps 2 --warmup 1 > $O/r02_c4_base.jsonl 2> $O/r02_c4_base.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_c4_launches.csv \
   $B --variants hamerly,simp_elkan --profile-only > $O/r02_c4_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_row_pass|k_hamerly_bounds|k_hamerly_tighten" \
   --launch-skip 15 --launch-count 3 -f -o $O/r02_c4_hamerly $B --variants hamerly --profile-only > $O/r02_c4_ncu_h.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_elkan" \
   --launch-skip 10 --launch-count 2 -f -o $O/r02_c4_elkan $B --variants simp_elkan --profile-only > $O/r02_c4_ncu_e.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_center|k_apply|k_finalize" \
   --launch-skip 40 --launch-count 6 -f -o $O/r02_c4_center $B --variants hamerly --profile-only > $O/r02_c4_ncu_c.log 2>&1
ls -la $O
