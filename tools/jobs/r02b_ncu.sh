#!/bin/bash
# Full GPU suite (incl. the new C3/C4/C5 parity, loopback, device layout tests), then at C4:
# the ncu launch list of one profile-only bench step and ncu --set full of the top kernels.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=20 > $O/q_gputest.log 2>&1
echo "pytest rc=$?" >> $O/q_gputest.log; tail -30 $O/q_gputest.log
B="python bench.py --config C4 --no-cpu-baseline --profile-only"
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/q_c4_launches.csv $B > $O/q_c4_launches.log 2>&1
python tools/ncu_launches.py $O/q_c4_launches.csv > $O/q_c4_launches.txt; head -30 $O/q_c4_launches.txt
F="$NCU --set full --import-source on -f"
$F -k regex:"k_row_pass|k_hamerly_bounds" --launch-skip 12 --launch-count 3 -o $O/q_c4_h $B --variants hamerly > $O/q_ncu_h.log 2>&1
$F -k regex:"k_elkan" --launch-skip 8 --launch-count 3 -o $O/q_c4_e $B --variants simp_elkan > $O/q_ncu_e.log 2>&1
$F -k regex:"k_center|k_apply|k_gram|k_row_max" --launch-skip 40 --launch-count 9 -o $O/q_c4_c $B --variants hamerly > $O/q_ncu_c.log 2>&1
for r in h e c; do python tools/ncu_summary.py $O/q_c4_$r.ncu-rep > $O/q_c4_$r.txt 2>&1; cat $O/q_c4_$r.txt; done
ls -la $O/*.ncu-rep
