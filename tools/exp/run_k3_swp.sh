python -m pytest tests/test_gpu_parity.py -x -q -k "t4 or t2 or normal" 2>&1 | tail -1
for lib in "" tools/exp/liboqr_k3_noswp.so; do
  echo "== lib ${lib:-product}"
  OQR_LIB=$lib python tools/exp/k3_hash.py
  for mn in "40000 200" "100000 200" "4000 50" "10000 100" "100000 100" "40000 240"; do OQR_LIB=$lib python tools/prof_k3.py $mn 3; done
done
python tools/time_steps.py T 5
