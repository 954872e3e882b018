set -x
python -m pytest tests/test_gpu_tridiag.py tests/test_gpu_parity.py -x -q -k "bitwise or packed_upper or euclid or tridiag or prequr" 2>&1 | tail -15
for n in 40 100 160 200 240; do python tools/prof_k4t.py 100000 $n 3; python tools/prof_k4t.py 100000 $n 3 packed; done
python tools/time_steps.py T 5
python tools/time_steps.py 3 5
