#!/bin/bash
# K3 experiment builds (NOT product): one-warp kernel with prefetch distance 2 / 6, the warp-pair
# kernel with DMMA or DFMA critical update and prefetch distance 2 / 4 / 6 own tiles.
set -e
cd "$(dirname "$0")/../.."
SRC="paper_1401_5171_b200/csrc/*.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
build() { /usr/local/cuda/bin/nvcc $F $2 -o tools/exp/liboqr_$1.so $SRC; }
build K3ONE_PD2 "-DOQR_EXP_TRSM_ONEWARP -DOQR_EXP_TRSM_PD=2" &
build K3ONE_PD4 "-DOQR_EXP_TRSM_ONEWARP -DOQR_EXP_TRSM_PD=4" &
build K3PAIR_DMMA_PD4 "-DOQR_EXP_TP_DMMA_CRIT -DOQR_EXP_TP_PD=4" &
build K3PAIR_FMA_PD2 "-DOQR_EXP_TP_PD=2" &
build K3PAIR_FMA_PD6 "-DOQR_EXP_TP_PD=6" &
wait
