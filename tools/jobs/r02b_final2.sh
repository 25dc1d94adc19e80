#!/bin/bash
# Final round-2 evidence at HEAD: default bench line, reference arm, ncu launch list of the default
# command, ncu --set full of the C4 kernels (hamerly, simp_elkan, center pipeline, yinyang).
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/g_smi.txt
( time python bench.py ) > $O/g_bench.jsonl 2> $O/g_bench.err; tail -3 $O/g_bench.err
( time python bench.py --impl reference ) > $O/g_ref.jsonl 2> $O/g_ref.err; tail -3 $O/g_ref.err
B="python bench.py --config C4 --no-cpu-baseline --profile-only"
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/g_launches.csv $B > $O/g_launches.log 2>&1
python tools/ncu_launches.py $O/g_launches.csv > $O/g_launches.txt; head -24 $O/g_launches.txt
F="$NCU --set full --import-source on -f"
$F -k regex:"k_row_pass|k_hamerly_bounds" --launch-skip 12 --launch-count 3 -o /tmp/g_c4_h $B --variants hamerly > $O/g_ncu_h.log 2>&1
$F -k regex:"k_elkan" --launch-skip 8 --launch-count 3 -o /tmp/g_c4_e $B --variants simp_elkan > $O/g_ncu_e.log 2>&1
$F -k regex:"k_center|k_apply|k_gram|k_row_max" --launch-skip 40 --launch-count 9 -o /tmp/g_c4_c $B --variants hamerly > $O/g_ncu_c.log 2>&1
$F -k regex:"k_yy|k_row_pass" --launch-skip 8 --launch-count 3 -o /tmp/g_c4_y $B --variants yinyang > $O/g_ncu_y.log 2>&1
for r in h e c y; do python tools/ncu_summary.py /tmp/g_c4_$r.ncu-rep > $O/g_c4_$r.txt 2>&1; cat $O/g_c4_$r.txt; done
rm -f $O/g_c4_*.ncu-rep.tmp
ls -la $O/g_*
