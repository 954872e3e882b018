#!/bin/bash
# session 4 final: GPU suite, smoke, bench lines, step timings, ncu launch lists and the K3 summary
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4f_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/s4f_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4f_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/s4f_bench_c3_normal.json 2> gpurun_out/s4f_bench_c3_normal.err
timeout 600 python bench.py --tridiag > gpurun_out/s4f_bench_tridiag_normal.json 2> gpurun_out/s4f_bench_tridiag_normal.err
timeout 600 python bench.py --variant prequr --no-cpu-baseline > gpurun_out/s4f_bench_c3_prequr.json 2> gpurun_out/s4f_bench_c3_prequr.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s4f_bench_reference.json 2> gpurun_out/s4f_bench_reference.err
for c in T 3 1 4 2; do timeout 300 python tools/time_steps.py $c 10; done > gpurun_out/s4f_steps.txt 2>&1
timeout 300 python bench.py --tridiag --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4f_plain_tri.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4f_launches_tridiag.csv \
    python bench.py --tridiag --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4f_ncu_tri.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4f_plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s4f_launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4f_ncu_c3.log 2>&1
timeout 300 python tools/prof_k3.py 100000 200 3 > gpurun_out/s4f_plain_k3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsm_dmma -s 3 -c 1 -f -o /tmp/k3_T \
    python tools/prof_k3.py 100000 200 3 > gpurun_out/s4f_ncu_k3.log 2>&1
python tools/ncu_kernel_summary.py /tmp/k3_T.ncu-rep gpurun_out/s4f_k3_T_summary.txt "K3 trsm_dmma_kernel<25> m=100000 n=200: python tools/prof_k3.py 100000 200 3"
