#!/bin/bash
# registers / spills per kernel instantiation of one .cu file (sm_100a)
f=${1:-paper_1401_5171_b200/csrc/oqr_gram.cu}
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v -c -o /dev/null "$f" 2>&1 \
 | awk '/Compiling entry function/{match($0,/_Z[A-Za-z0-9_]+/); name=substr($0,RSTART,RLENGTH)} /spill stores/{sp=$5" "$6" "$7} /Used [0-9]+ registers/{match($0,/Used [0-9]+ registers/); print name, substr($0,RSTART,RLENGTH), "spill:", sp}'
