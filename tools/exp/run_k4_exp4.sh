python -m pytest tests/test_gpu_tridiag.py tests/test_gpu_parity.py -x -q -k "bitwise or packed_upper or euclid" 2>&1 | tail -2
for lib in "" tools/exp/liboqr_k4_c8_w16.so tools/exp/liboqr_k4_c10_w8.so tools/exp/liboqr_k4_c6_w16.so tools/exp/liboqr_k4_nodmma.so; do
  echo "== lib ${lib:-product}"
  for n in 100 160 200 240; do
    for mode in fused packed euclid; do
      OQR_LIB=$lib python tools/prof_k4t.py 100000 $n 3 $mode 2>&1 | tail -1
    done
  done
done
