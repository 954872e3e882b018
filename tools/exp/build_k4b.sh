#!/bin/bash
# Experiment builds of liboqr for the K4 family (NOT product): data supply only / ring depth.
set -e
cd "$(dirname "$0")/../.."
SRC="paper_1401_5171_b200/csrc/*.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
build() { /usr/local/cuda/bin/nvcc $F $2 -o tools/exp/liboqr_$1.so $SRC; }
build k4_nocons "-DOQR_EXP_K4_NOCONSUME" &
build k4_nocons_s2 "-DOQR_EXP_K4_NOCONSUME -DOQR_EXP_K4_STAGES=2" &
build k4_s2 "-DOQR_EXP_K4_STAGES=2" &
build k4_s4 "-DOQR_EXP_K4_STAGES=4" &
wait
