#!/bin/bash
# (1) heavy threshold below 1% of k; (2) timing probe of register accumulation for dense term rows (hamerly only)
export SPKM_DATA_CACHE=/tmp/spkm_data
bash tools/jobs/r02b_ab2.sh p01=SPKM_EK_HEAVY_PCT=0.1 p03=SPKM_EK_HEAVY_PCT=0.3 p05=SPKM_EK_HEAVY_PCT=0.5 p1=SPKM_EK_HEAVY_PCT=1
EXTRA="--variants hamerly" bash tools/jobs/r02b_ab2.sh hbase e4=SPKM_LIB=lib:e4 e3=SPKM_LIB=lib:e3 e2=SPKM_LIB=lib:e2
