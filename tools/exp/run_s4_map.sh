#!/bin/bash
cd "$(dirname "$0")/../.."
{
for lib in "" tools/exp/liboqr_map1.so tools/exp/liboqr_map2.so; do
echo "== k3 alone ${lib:-product}"; for mn in "40000 200" "100000 200" "100000 100" "4000 50" "20000 100"; do OQR_LIB=$lib python tools/prof_k3.py $mn 3; done
OQR_LIB=$lib python tools/exp/k3_hash.py
echo "== steps ${lib:-product}"; for c in T 1 4; do OQR_LIB=$lib python tools/time_steps.py $c 20; done
done
} > gpurun_out/s4_map.txt 2>&1
