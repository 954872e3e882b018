#!/bin/bash
# session 3: K2 trailing loop + deferred sqrt (A/B vs the HEAD build, bitwise R), K2 per-warp trace
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
{
echo "== k2 hash base"; OQR_LIB=tools/exp/liboqr_base.so python tools/exp/k2_hash.py
echo "== k2 hash new"; python tools/exp/k2_hash.py
echo "== k3 hash new"; python tools/exp/k3_hash.py
for c in T 1 4; do
echo "== steps base $c"; OQR_LIB=tools/exp/liboqr_base.so python tools/time_steps.py $c 10
echo "== steps new $c"; python tools/time_steps.py $c 10
done
echo "== k2 trace2"; K2_TRACE_RAW=gpurun_out/s3_k2trace2c_raw.npy OQR_LIB=tools/exp/liboqr_k2trace2.so python tools/exp/k2_trace2.py 200
} > gpurun_out/s3_c.txt 2>&1
