#!/bin/bash
# session 4 closing run (3): run-on abort path -- suite, smoke, bench lines, steps
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4i_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/s4i_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4i_smoke.txt 2>&1
timeout 300 python tools/exp/ovl_hash.py > gpurun_out/s4i_hash.txt 2>&1
timeout 600 python bench.py > gpurun_out/s4i_bench_c3_normal.json 2> gpurun_out/s4i_bench_c3_normal.err
timeout 600 python bench.py --tridiag > gpurun_out/s4i_bench_tridiag_normal.json 2> gpurun_out/s4i_bench_tridiag_normal.err
for c in T 3 1; do timeout 300 python tools/time_steps.py $c 10; done > gpurun_out/s4i_steps.txt 2>&1
