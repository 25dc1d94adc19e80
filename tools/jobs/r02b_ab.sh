#!/bin/bash
# YY tests, then C4 A/B of alternative builds (SPKM_LIB) with per-entry CUDA-event times.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_yinyang.py -q > $O/ab_yy_tests.log 2>&1; echo "pytest rc=$?" >> $O/ab_yy_tests.log
tail -5 $O/ab_yy_tests.log
B="python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 1 --warmup 1"
for tag in default "$@"; do
  if [ "$tag" = default ]; then lib=""; else lib="SPKM_LIB=$PWD/paper_2107_04074_b200/libspkm_$tag.so"; fi
  env $lib $B > $O/ab_$tag.jsonl 2> $O/ab_$tag.err
  python -c "
import json; d=json.loads(open('$O/ab_$tag.jsonl').read().strip().splitlines()[-1])
pk=d['roofline'].get('per_kernel',{})
print('$tag', round(d['value'],3), round(d['ms_per_step'],1), {k:(v['ms'],v['frac']) for k,v in pk.items() if v['ms']>100})"
done
