#!/bin/bash
# A/B builds: tools/build_ab.sh TAG -DFLAG=V ... -> paper_2107_04074_b200/libspkm_TAG.so (use with SPKM_LIB=...)
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC "$@" \
  -I include -o paper_2107_04074_b200/libspkm_$tag.so paper_2107_04074_b200/csrc/spkm.cu paper_2107_04074_b200/csrc/ingest.cpp
echo built paper_2107_04074_b200/libspkm_$tag.so
