#!/bin/bash
# session 4: ncu source-level stall samples of K3 (product and the no-memory/no-batch diagnostic build)
cd "$(dirname "$0")/../.."
for lib in product nomem_nobatch; do
  L=""; [ "$lib" != product ] && L=tools/exp/liboqr_k3_$lib.so
  OQR_LIB=$L python tools/prof_k3.py 400000 200 3 > gpurun_out/s4_plain_k3_$lib.log 2>&1 && \
  OQR_LIB=$L ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:trsm_dmma -s 3 -c 1 -f -o /tmp/k3_$lib \
      python tools/prof_k3.py 400000 200 3 > gpurun_out/s4_ncu_k3_$lib.log 2>&1
  ncu -i /tmp/k3_$lib.ncu-rep --page source --csv --print-source sass > gpurun_out/s4_k3_${lib}_source.csv 2>/dev/null
  python tools/ncu_source_summary.py gpurun_out/s4_k3_${lib}_source.csv 40 > gpurun_out/s4_k3_${lib}_source_summary.txt 2>&1
done
