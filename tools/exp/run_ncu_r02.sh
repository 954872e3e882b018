# round-2 ncu evidence (each command already exited 0 without ncu in the same call, directly before)
set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_k1.py 40000 200 2 > gpurun_out/ncu_plain_k1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram_fused -s 1 -c 1 -o gpurun_out/k1_c3 \
    python tools/prof_k1.py 40000 200 2 > gpurun_out/ncu_k1.log 2>&1
python tools/time_hhqr.py 40000 200 > gpurun_out/ncu_plain_k6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hhqr -s 1 -c 1 -o gpurun_out/k6_c3 \
    python tools/time_hhqr.py 40000 200 > gpurun_out/ncu_k6.log 2>&1
python tools/prof_k4t.py 100000 200 3 > gpurun_out/ncu_plain_k4t.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram_tridiag -s 2 -c 1 -o gpurun_out/k4t_T \
    python tools/prof_k4t.py 100000 200 3 > gpurun_out/ncu_k4t.log 2>&1
