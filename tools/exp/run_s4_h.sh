#!/bin/bash
# session 4 closing run (2): K3 running pointers A/B over n, then suite, smoke, bench lines, steps, K3 ncu summary
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
{
for lib in tools/exp/liboqr_noptr.so ""; do
echo "== k3 alone ${lib:-product}"; for n in 224 216 208 192 176 160 144 136 128 120 104 96 64; do OQR_LIB=$lib python tools/prof_k3.py 100000 $n 3; done
done
} > gpurun_out/s4h_ptr_sweep.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4h_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/s4h_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4h_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/s4h_bench_c3_normal.json 2> gpurun_out/s4h_bench_c3_normal.err
timeout 600 python bench.py --tridiag > gpurun_out/s4h_bench_tridiag_normal.json 2> gpurun_out/s4h_bench_tridiag_normal.err
for c in T 3 1 4 2; do timeout 300 python tools/time_steps.py $c 10; done > gpurun_out/s4h_steps.txt 2>&1
timeout 300 python tools/prof_k3.py 100000 200 3 > gpurun_out/s4h_plain_k3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsm_dmma -s 3 -c 1 -f -o /tmp/k3_T \
    python tools/prof_k3.py 100000 200 3 > gpurun_out/s4h_ncu_k3.log 2>&1
python tools/ncu_kernel_summary.py /tmp/k3_T.ncu-rep gpurun_out/s4h_k3_T_summary.txt "K3 trsm_dmma_kernel<25> m=100000 n=200: python tools/prof_k3.py 100000 200 3"
