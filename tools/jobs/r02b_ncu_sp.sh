#!/bin/bash
# ncu --set full of the sparse-gather rescan and the index build at C4 (hamerly fit); reps stay in /tmp.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
B="python bench.py --config C4 --no-cpu-baseline --profile-only --variants hamerly"
ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $O/sp_launches.csv $B > /dev/null 2>&1
python tools/ncu_launches.py $O/sp_launches.csv | head -16
ncu --clock-control none --set full --import-source on -f -k regex:"k_row_pass|k_ci_" --launch-skip 20 --launch-count 4 -o /tmp/sp_h $B > $O/sp_ncu.log 2>&1
python tools/ncu_summary.py /tmp/sp_h.ncu-rep
ncu -i /tmp/sp_h.ncu-rep --page source --csv --print-source sass 2>/dev/null | head -1 > /dev/null
