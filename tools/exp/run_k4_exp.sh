# K4 family experiment sweep + ncu captures (round 2, session 2); results in gpurun_out/k4_exp.txt
python -m pytest tests/test_gpu_tridiag.py tests/test_gpu_parity.py -x -q -k "bitwise or packed_upper or euclid" 2>&1 | tail -3
for lib in "" tools/exp/liboqr_k4_p96_w16.so tools/exp/liboqr_k4_p96_w10.so tools/exp/liboqr_k4_p64_w12.so tools/exp/liboqr_k4_p64_w16.so tools/exp/liboqr_k4_nodmma.so; do
  echo "== lib ${lib:-product}"
  for n in 100 200 240; do
    for mode in fused packed euclid; do
      OQR_LIB=$lib python tools/prof_k4t.py 100000 $n 3 $mode
    done
  done
done
for mode in fused; do
  ncu --set full --clock-control none --import-source on -k regex:gram_upper -s 3 -c 1 -f -o /tmp/k4_$mode python tools/prof_k4t.py 100000 200 3 $mode > /dev/null 2>&1
  python tools/ncu_kernel_summary.py /tmp/k4_$mode.ncu-rep gpurun_out/k4_${mode}_summary.txt "K4 $mode m=100000 n=200"
done
