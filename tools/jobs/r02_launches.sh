#!/bin/bash
# ncu launch list (gpu__time_duration only) of one untimed C4 fit per variant given; env passthrough.
export SPKM_DATA_CACHE=/tmp/spkm_data
O=gpurun_out
tag=${TAG:-x}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_$tag.csv \
   python bench.py --config ${CFG:-C4} --no-cpu-baseline --variants ${VARS:-hamerly,simp_elkan} --profile-only > $O/launch_$tag.log 2>&1
python tools/ncu_launches.py $O/launch_$tag.csv | head -25
