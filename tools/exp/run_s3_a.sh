#!/bin/bash
# session 3: K3 branch-free selects (A/B vs the HEAD build) and the K2 per-warp phase trace
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
{
echo "== k3 hash base"; OQR_LIB=tools/exp/liboqr_base.so python tools/exp/k3_hash.py
echo "== k3 hash new"; python tools/exp/k3_hash.py
for rep in 1 2; do
for c in T 3 1; do
echo "== steps base $c"; OQR_LIB=tools/exp/liboqr_base.so python tools/time_steps.py $c 10
echo "== steps new $c"; python tools/time_steps.py $c 10
done; done
echo "== k2 trace2"; OQR_LIB=tools/exp/liboqr_k2trace2.so python tools/exp/k2_trace2.py 200
} > gpurun_out/s3_a.txt 2>&1
