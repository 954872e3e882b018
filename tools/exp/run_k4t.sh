for n in 40 100 160 200 240; do
  python tools/prof_k4t.py 100000 $n >> gpurun_out/r2_k4t_sweep.txt 2>&1
  python tools/prof_k4t.py 100000 $n 3 packed >> gpurun_out/r2_k4t_sweep.txt 2>&1
done
