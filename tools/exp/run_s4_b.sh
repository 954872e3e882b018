#!/bin/bash
# session 4: full GPU suite + smoke + bench lines with the overlapped K2 -> K3 pair and K3's L2 prefetch
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4b_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/s4b_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4b_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/s4b_bench_c3_normal.json 2> gpurun_out/s4b_bench_c3_normal.err
timeout 600 python bench.py --tridiag > gpurun_out/s4b_bench_tridiag_normal.json 2> gpurun_out/s4b_bench_tridiag_normal.err
for c in T 3 1 4 2; do timeout 300 python tools/time_steps.py $c 10; done > gpurun_out/s4b_steps.txt 2>&1
