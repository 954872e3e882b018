# round-2 session-2 bench lines + ncu evidence (each ncu command exited 0 without ncu first)
set -x
python bench.py > gpurun_out/s2_bench_c3_normal.json 2> gpurun_out/s2_bench_c3_normal.err
python bench.py --tridiag > gpurun_out/s2_bench_tridiag_normal.json 2> gpurun_out/s2_bench_tridiag_normal.err
python bench.py --variant prequr --no-cpu-baseline > gpurun_out/s2_bench_c3_prequr.json 2> gpurun_out/s2_bench_c3_prequr.err
python tools/prof_k3.py 100000 200 3 > gpurun_out/s2_plain_k3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:trsm_dmma -s 3 -c 1 -f -o /tmp/k3_T \
    python tools/prof_k3.py 100000 200 3 > gpurun_out/s2_ncu_k3.log 2>&1
python tools/ncu_kernel_summary.py /tmp/k3_T.ncu-rep gpurun_out/s2_k3_T_summary.txt "K3 trsm_dmma_kernel<25> m=100000 n=200: python tools/prof_k3.py 100000 200 3"
python tools/prof_k4t.py 100000 200 3 > gpurun_out/s2_plain_k4t.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram_upper -s 3 -c 1 -f -o /tmp/k4t_T \
    python tools/prof_k4t.py 100000 200 3 > gpurun_out/s2_ncu_k4t.log 2>&1
python tools/ncu_kernel_summary.py /tmp/k4t_T.ncu-rep gpurun_out/s2_k4t_T_summary.txt "K4t gram_upper_kernel<25, TRI> m=100000 n=200: python tools/prof_k4t.py 100000 200 3"
python bench.py --tridiag --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s2_plain_tri.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_launches_tridiag.csv \
    python bench.py --tridiag --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s2_ncu_tri.log 2>&1
