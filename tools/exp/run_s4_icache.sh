#!/bin/bash
cd "$(dirname "$0")/../.."
{
for rep in 1 2; do
for lib in tools/exp/liboqr_cur.so ""; do
echo "== k3 alone ${lib:-new}"; for mn in "40000 200" "100000 200" "100000 100" "100000 232" "4000 50"; do OQR_LIB=$lib python tools/prof_k3.py $mn 3; done
done; done
for lib in tools/exp/liboqr_cur.so ""; do
OQR_LIB=$lib python tools/exp/ovl_hash.py > gpurun_out/s4_hash_$( [ -n "$lib" ] && echo cur || echo new ).txt 2>&1
echo "== steps ${lib:-new}"; for c in T 1 2; do OQR_LIB=$lib python tools/time_steps.py $c 20; done
done
cmp gpurun_out/s4_hash_cur.txt gpurun_out/s4_hash_new.txt && echo HASHES EQUAL
} > gpurun_out/s4_icache.txt 2>&1
