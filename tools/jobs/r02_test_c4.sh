#!/bin/bash
# GPU suite, then the C4 device-timed line (quick form) and optional A/B env settings given as args.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/t_gputest.log 2>&1; echo "pytest rc=$?" >> $O/t_gputest.log
tail -3 $O/t_gputest.log
B="python bench.py --config C4 --no-cpu-baseline --no-e2e --no-roofline --steps 1 --warmup 1"
$B > $O/t_c4.jsonl 2>$O/t_c4.err
python -c "
import json; d=json.loads(open('$O/t_c4.jsonl').read().strip().splitlines()[-1]); print('C4', round(d['value'],3), round(d['ms_per_step'],1), d['per_variant'])"
for kv in "$@"; do
  env $kv $B > $O/t_c4_ab.jsonl 2>>$O/t_c4.err
  python -c "
import json; d=json.loads(open('$O/t_c4_ab.jsonl').read().strip().splitlines()[-1]); print('$kv', round(d['value'],3), round(d['ms_per_step'],1))"
done
