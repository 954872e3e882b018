#!/bin/bash
# session 4: state check after the container re-creation (suite, smoke, bench lines, steps)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/s4_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/s4_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.txt 2>&1
python bench.py > gpurun_out/s4_bench_c3_normal.json 2> gpurun_out/s4_bench_c3_normal.err
python bench.py --tridiag > gpurun_out/s4_bench_tridiag_normal.json 2> gpurun_out/s4_bench_tridiag_normal.err
for c in T 3 1 4 2; do python tools/time_steps.py $c 10; done > gpurun_out/s4_steps.txt 2>&1
