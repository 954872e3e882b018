#!/bin/bash
cd "$(dirname "$0")/../.."
{
for rep in 1 2; do
for lib in "" tools/exp/liboqr_ptr.so; do
echo "== k3 alone ${lib:-product}"; for mn in "40000 200" "100000 200" "100000 100" "100000 232" "100000 48" "4000 50"; do OQR_LIB=$lib python tools/prof_k3.py $mn 3; done
done; done
for lib in "" tools/exp/liboqr_ptr.so; do OQR_LIB=$lib python tools/exp/k3_hash.py; OQR_LIB=$lib python tools/time_steps.py T 20; done
} > gpurun_out/s4_ptr.txt 2>&1
