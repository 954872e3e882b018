python -m pytest tests/test_gpu_tridiag.py tests/test_gpu_parity.py -x -q -k "tridiag or bitwise or packed_upper" 2>&1 | tail -1
for n in 8 40 100 144 160 200 208 240; do python tools/prof_k4t.py 100000 $n 3 fused 2>&1 | tail -1; done
python tools/time_steps.py T 5
