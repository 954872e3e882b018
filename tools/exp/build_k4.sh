#!/bin/bash
# Experiment builds of liboqr for the K4 family (NOT product): units per warp / warps per part.
#   OQR_LIB=tools/exp/liboqr_<name>.so python tools/prof_k4t.py m n reps mode
set -e
cd "$(dirname "$0")/../.."
SRC="paper_1401_5171_b200/csrc/*.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
build() { /usr/local/cuda/bin/nvcc $F $2 -o tools/exp/liboqr_$1.so $SRC; }
build k4_c10_w8 "-DOQR_EXP_UP_MAXC=10 -DOQR_EXP_UP_WARPS=8" &
build k4_c8_w11 "-DOQR_EXP_UP_MAXC=8 -DOQR_EXP_UP_WARPS=11" &
build k4_c6_w16 "-DOQR_EXP_UP_MAXC=6 -DOQR_EXP_UP_WARPS=16" &
build k4_nodmma "-DOQR_EXP_NODMMA" &
wait
