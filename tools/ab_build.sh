#!/bin/bash
# A/B builds for same-box timing comparisons (dev tool):
#   tools/debug/lib_base.so  from git REF (default HEAD)
#   tools/debug/lib_new.so   from the working tree
# (NEW_FLAGS="-DPF_BITS_CTAS=4" adds compile flags to lib_new)
# then on the GPU box:  python tools/ab_time.py c5_lem c4_aco_x64 ...
set -e
cd "$(dirname "$0")/.."
REF=${1:-HEAD}
mkdir -p tools/debug
TMP=$(mktemp -d)
git archive "$REF" paper_1412_4933_b200/csrc include | tar -x -C "$TMP"
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off"
nvcc $FLAGS -I "$TMP/include" -shared -o tools/debug/lib_base.so $(ls "$TMP"/paper_1412_4933_b200/csrc/*.cu "$TMP"/paper_1412_4933_b200/csrc/*.cpp) &
nvcc $FLAGS $NEW_FLAGS -I include -shared -o tools/debug/lib_new.so $(ls paper_1412_4933_b200/csrc/*.cu paper_1412_4933_b200/csrc/*.cpp) &
wait
rm -rf "$TMP"
echo "built tools/debug/lib_base.so ($REF) and tools/debug/lib_new.so (working tree)"
