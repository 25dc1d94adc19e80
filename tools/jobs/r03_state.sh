#!/bin/bash
# Round-2 re-entry state at HEAD: GPU suite + smoke, default bench line, reference arm, C4 launch list,
# ncu --set full of the C4 gather passes (sparse rescan, Elkan scan) and the Elkan bound pass.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/s_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > $O/s_gputest.log 2>&1; echo "pytest rc=$?" >> $O/s_gputest.log; tail -3 $O/s_gputest.log
python __graft_entry__.py smoke > $O/s_smoke.log 2>&1; tail -1 $O/s_smoke.log
( time python bench.py ) > $O/s_bench.jsonl 2> $O/s_bench.err; tail -3 $O/s_bench.err
python -c "
import json; d=json.loads(open('$O/s_bench.jsonl').read().strip().splitlines()[-1]); print('BENCH', round(d['value'],3), d['e2e'], d['roofline'].get('kernel'), d['roofline'].get('frac'), d['clocks'])
print({k:(v['ms'],v.get('frac')) for k,v in d['roofline']['per_kernel'].items()})"
( time python bench.py --impl reference ) > $O/s_ref.jsonl 2> $O/s_ref.err; tail -3 $O/s_ref.err; cut -c1-200 $O/s_ref.jsonl
B="python bench.py --config C4 --no-cpu-baseline --profile-only"
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/s_launches.csv $B > $O/s_launches.log 2>&1
python tools/ncu_launches.py $O/s_launches.csv > $O/s_launches.txt; head -24 $O/s_launches.txt
F="$NCU --set full --import-source on -f"
$F -k regex:"k_row_pass|k_ci_|k_hamerly_bounds" --launch-skip 20 --launch-count 5 -o /tmp/s_c4_h $B --variants hamerly > $O/s_ncu_h.log 2>&1
$F -k regex:"k_elkan" --launch-skip 8 --launch-count 3 -o /tmp/s_c4_e $B --variants simp_elkan > $O/s_ncu_e.log 2>&1
for r in h e; do python tools/ncu_summary.py /tmp/s_c4_$r.ncu-rep > $O/s_c4_$r.txt 2>&1; cat $O/s_c4_$r.txt; cp /tmp/s_c4_$r.ncu-rep $O/; done
ls -la $O/s_*
