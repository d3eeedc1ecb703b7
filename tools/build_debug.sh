#!/bin/bash
# Debug variant of the library (dev tool): the small shared-memory ring
# (one window + the next tile, no cross-item prefetch), so that code path is
# exercised by the parity tests too (run them with
# PEDFLOW_B200_LIB=tools/debug/libpedflow_b200_smallring.so). The scalar work
# lists are bounded by the unit count and have no overflow path to force.
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/debug
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  -I include -DPF_BITS_SMALL_RING -shared -o tools/debug/libpedflow_b200_smallring.so \
  paper_1412_4933_b200/csrc/pf_kernels.cu paper_1412_4933_b200/csrc/pf_bitstep.cu paper_1412_4933_b200/csrc/pf_bitstep_ns8.cu paper_1412_4933_b200/csrc/pf_bitstep_ns10.cu paper_1412_4933_b200/csrc/pf_bitstep_small.cu \
  paper_1412_4933_b200/csrc/pf_context.cu paper_1412_4933_b200/csrc/pf_setup.cpp
