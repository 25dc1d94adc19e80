#!/bin/bash
export SPKM_DATA_CACHE=/tmp/spkm_data
STEPS=2 bash tools/jobs/r02b_ab2.sh base ph=SPKM_LIB=lib:ph base2 ph2=SPKM_LIB=lib:ph
