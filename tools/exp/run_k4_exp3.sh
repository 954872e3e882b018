python -m pytest tests/test_gpu_tridiag.py tests/test_gpu_parity.py -x -q -k "bitwise or packed_upper or euclid" 2>&1 | tail -2
for n in 40 100 160 200 240; do
  for mode in fused packed euclid euclid_packed; do
    python tools/prof_k4t.py 100000 $n 3 $mode
  done
done
python tools/time_steps.py T 5
python tools/time_steps.py 3 5
