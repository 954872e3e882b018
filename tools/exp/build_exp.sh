#!/bin/bash
# Experiment builds of liboqr (NOT product): e.g. -DOQR_EXP_NODMMA (data supply only),
# -DOQR_EXP_NOLOAD (compute + sync only), -DOQR_EXP_NOA / NOZ (one stream only).
# Used as OQR_LIB=tools/exp/liboqr_<name>.so python tools/time_k1.py m n
set -e
cd "$(dirname "$0")/../.."
SRC="paper_1401_5171_b200/csrc/*.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
build() { /usr/local/cuda/bin/nvcc $F $2 -o tools/exp/liboqr_$1.so $SRC; }
build NODMMA "-DOQR_EXP_NODMMA" &
build NOLOAD "-DOQR_EXP_NOLOAD" &
build NOCONTRACT "-DOQR_EXP_NOCONTRACT" &
wait
