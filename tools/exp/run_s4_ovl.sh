#!/bin/bash
# session 4: overlapped K2 -> K3 pair: bitwise A/B against the serial build, then step timings
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
{
echo "== hash noovl"; OQR_LIB=tools/exp/liboqr_noovl.so timeout 300 python tools/exp/ovl_hash.py > gpurun_out/s4_hash_noovl.txt 2>&1; tail -2 gpurun_out/s4_hash_noovl.txt
echo "== hash ovl"; timeout 300 python tools/exp/ovl_hash.py > gpurun_out/s4_hash_ovl.txt 2>&1; tail -2 gpurun_out/s4_hash_ovl.txt
echo "== hash ovl_pf8"; OQR_LIB=tools/exp/liboqr_ovl_pf8.so timeout 300 python tools/exp/ovl_hash.py > gpurun_out/s4_hash_ovl_pf8.txt 2>&1; tail -2 gpurun_out/s4_hash_ovl_pf8.txt
cmp gpurun_out/s4_hash_noovl.txt gpurun_out/s4_hash_ovl.txt && echo "HASHES EQUAL (ovl)"
cmp gpurun_out/s4_hash_noovl.txt gpurun_out/s4_hash_ovl_pf8.txt && echo "HASHES EQUAL (ovl_pf8)"
for c in T 1; do
for lib in tools/exp/liboqr_noovl.so "" tools/exp/liboqr_ovl_pf8.so; do
echo "== steps ${lib:-product} $c"; OQR_LIB=$lib timeout 300 python tools/time_steps.py $c 10
done; done
} > gpurun_out/s4_ovl.txt 2>&1
{
for lib in tools/exp/liboqr_noovl.so "" tools/exp/liboqr_ovl_pf8.so; do
echo "== k3 alone ${lib:-product}"; for mn in "40000 200" "100000 200" "100000 100" "4000 50"; do OQR_LIB=$lib python tools/prof_k3.py $mn 3; done
done
} >> gpurun_out/s4_ovl.txt 2>&1
