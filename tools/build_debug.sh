#!/bin/bash
# Debug variants of the library (dev tool): tiny work-queue / deposit-queue
# capacities so the overflow paths of the bit kernel are exercised by the
# parity tests (run them with PEDFLOW_B200_LIB=tools/debug/libpedflow_b200_q4.so).
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/debug
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  -I include -DPF_BITS_QCAP=4 -DPF_BITS_DCAP=4 -shared -o tools/debug/libpedflow_b200_q4.so \
  paper_1412_4933_b200/csrc/pf_kernels.cu paper_1412_4933_b200/csrc/pf_bitstep.cu \
  paper_1412_4933_b200/csrc/pf_context.cu paper_1412_4933_b200/csrc/pf_setup.cpp
