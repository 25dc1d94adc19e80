#!/bin/bash
# C4 (CFG) A/B: each argument is name=ENV1=V1,ENV2=V2 (lib builds via SPKM_LIB=lib:<tag>); prints per-entry ms.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
CFG=${CFG:-C4}
B="python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps ${STEPS:-1} --warmup 1 ${EXTRA}"
[ -n "$PRETEST" ] && { timeout 1800 python -m pytest $PRETEST -x -q > $O/ab2_tests.log 2>&1; echo "pytest rc=$?"; tail -3 $O/ab2_tests.log; }
for item in "$@"; do
  name=${item%%=*}; envs=${item#*=}; [ "$envs" = "$item" ] && envs=""
  envs=$(echo "$envs" | tr ',' ' ' | sed "s#SPKM_LIB=lib:\([a-z0-9_]*\)#SPKM_LIB=$PWD/paper_2107_04074_b200/libspkm_\1.so#")
  env $envs $B > $O/ab2_$name.jsonl 2> $O/ab2_$name.err
  python -c "
import json; d=json.loads(open('$O/ab2_$name.jsonl').read().strip().splitlines()[-1])
pk=d['roofline'].get('per_kernel',{})
print('$CFG $name', round(d['value'],3), round(d['ms_per_step'],1), {k:v['ms'] for k,v in pk.items() if v['ms']>5})" 2>&1 | tail -1
done
