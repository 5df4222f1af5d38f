#!/bin/bash
# builds scripts/native/qr_timing (links the in-tree library objects except qr.o)
set -e
cd "$(dirname "$0")/../.."
O=paper_2001_11619_b200/build_obj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DSKB_QR_TIMING \
  -I paper_2001_11619_b200/csrc scripts/native/qr_timing.cu $O/gemm.o $O/lu.o $O/misc.o $O/assemble.o $O/matvec.o \
  -o scripts/native/qr_timing
