#!/bin/bash
# Round-2 final evidence at HEAD: GPU suite + smoke, default bench line, reference arm, other configs,
# C4 launch list, ncu --set full of the C4 kernels.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/f_smi.txt
timeout 1800 python -m pytest tests -m gpu -x -q --durations=5 > $O/f_gputest.log 2>&1; echo "pytest rc=$?" >> $O/f_gputest.log; tail -3 $O/f_gputest.log
python __graft_entry__.py smoke > $O/f_smoke.log 2>&1; tail -1 $O/f_smoke.log
( time python bench.py ) > $O/f_bench.jsonl 2> $O/f_bench.err; tail -3 $O/f_bench.err
python -c "
import json; d=json.loads(open('$O/f_bench.jsonl').read().strip().splitlines()[-1]); print('BENCH', round(d['value'],3), d['e2e'], d['roofline'].get('kernel'), d['roofline'].get('frac'), d['clocks'])
print({k:(v['ms'],v.get('frac')) for k,v in d['roofline']['per_kernel'].items()})"
( time python bench.py --impl reference ) > $O/f_ref.jsonl 2> $O/f_ref.err; tail -3 $O/f_ref.err; cut -c1-200 $O/f_ref.jsonl
for cfg in "C2 --k 100" "C2 --k 20" "C3" "C5"; do
  set -- $cfg; tag=$(echo $cfg | tr -d ' -')
  python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > $O/f_bench_$tag.jsonl 2> $O/f_bench_$tag.err
  python -c "
import json; d=json.loads(open('$O/f_bench_$tag.jsonl').read().strip().splitlines()[-1]); print('$tag', round(d['value'],2), round(d['e2e']['value'],2), d['config']['workload'][:60])" 2>&1 | tail -1
done
python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 --variants standard,elkan,simp_elkan,hamerly,simp_hamerly,yinyang > $O/f_bench_C4_all.jsonl 2> $O/f_bench_C4_all.err
python -c "
import json; d=json.loads(open('$O/f_bench_C4_all.jsonl').read().strip().splitlines()[-1]); print('C4 all', round(d['value'],2), d['per_variant'])" 2>&1 | tail -1
B="python bench.py --config C4 --no-cpu-baseline --profile-only"
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/f_launches.csv $B > $O/f_launches.log 2>&1
python tools/ncu_launches.py $O/f_launches.csv > $O/f_launches.txt; head -24 $O/f_launches.txt
F="$NCU --set full --import-source on -f"
$F -k regex:"k_row_pass|k_ci_|k_hamerly_bounds|k_center_write|k_gram_mn" --launch-skip 40 --launch-count 8 -o /tmp/f_c4_h $B --variants hamerly > $O/f_ncu_h.log 2>&1
$F -k regex:"k_elkan|k_row_pass" --launch-skip 24 --launch-count 6 -o /tmp/f_c4_e $B --variants simp_elkan > $O/f_ncu_e.log 2>&1
for r in h e; do python tools/ncu_summary.py /tmp/f_c4_$r.ncu-rep > $O/f_c4_$r.txt 2>&1; cat $O/f_c4_$r.txt; cp /tmp/f_c4_$r.ncu-rep $O/; done
ls -la $O/f_*
