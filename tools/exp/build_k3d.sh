#!/bin/bash
# K3 timing-only diagnostic builds (NOT product; most give a wrong Q): which part of the per-tile
# step (diagonal chain, DMMA batch, Z loads, Q stores) a warp waits for.
set -e
cd "$(dirname "$0")/../.."
SRC="paper_1401_5171_b200/csrc/*.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
build() { /usr/local/cuda/bin/nvcc $F $2 -o tools/exp/liboqr_$1.so $SRC 2>/dev/null; }
for v in "$@"; do
case $v in
  nochain) build k3_nochain "-DOQR_EXP_TRSM_NOCHAIN" & ;;
  fmaonly) build k3_fmaonly "-DOQR_EXP_TRSM_FMAONLY" & ;;
  nobatch) build k3_nobatch "-DOQR_EXP_TRSM_NOBATCH" & ;;
  t128) build k3_t128 "-DOQR_EXP_TRSM_THREADS=128" & ;;
  t256) build k3_t256 "-DOQR_EXP_TRSM_THREADS=256" & ;;
  noldg) build k3_noldg "-DOQR_EXP_TRSM_NOLDG" & ;;
  nostg) build k3_nostg "-DOQR_EXP_TRSM_NOSTG" & ;;
  nomem) build k3_nomem "-DOQR_EXP_TRSM_NOLDG -DOQR_EXP_TRSM_NOSTG" & ;;
  nomem_nobatch) build k3_nomem_nobatch "-DOQR_EXP_TRSM_NOLDG -DOQR_EXP_TRSM_NOSTG -DOQR_EXP_TRSM_NOBATCH" & ;;
  nomem_nochain) build k3_nomem_nochain "-DOQR_EXP_TRSM_NOLDG -DOQR_EXP_TRSM_NOSTG -DOQR_EXP_TRSM_NOCHAIN" & ;;
  pf8) build k3_pf8 "-DOQR_EXP_TRSM_PF=8" & ;;
  pf16) build k3_pf16 "-DOQR_EXP_TRSM_PF=16" & ;;
  pf8l1) build k3_pf8l1 "-DOQR_EXP_TRSM_PF=8 -DOQR_EXP_TRSM_PFL1" & ;;
  pf4l1) build k3_pf4l1 "-DOQR_EXP_TRSM_PF=4 -DOQR_EXP_TRSM_PFL1" & ;;
  pd3) build k3_pd3 "-DOQR_EXP_TRSM_PD=3" & ;;
  pd6) build k3_pd6 "-DOQR_EXP_TRSM_PD=6" & ;;
esac
done
wait
