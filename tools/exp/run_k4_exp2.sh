for lib in "" tools/exp/liboqr_k4_nocons.so tools/exp/liboqr_k4_nocons_s2.so tools/exp/liboqr_k4_s2.so tools/exp/liboqr_k4_s4.so; do
  echo "== lib ${lib:-product}"
  for n in 100 200; do
    for mode in fused packed euclid euclid_packed; do
      OQR_LIB=$lib python tools/prof_k4t.py 100000 $n 3 $mode
    done
  done
done
