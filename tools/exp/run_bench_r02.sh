set -x
python bench.py > gpurun_out/r02_bench_c3_normal.json 2> gpurun_out/r02_bench_c3_normal.err
python bench.py --variant prequr_hh --no-cpu-baseline > gpurun_out/r02_bench_c3_prequr_hh.json 2> gpurun_out/r02_bench_c3_prequr_hh.err
python bench.py --variant normal2 --no-cpu-baseline > gpurun_out/r02_bench_c3_normal2.json 2> gpurun_out/r02_bench_c3_normal2.err
python bench.py --tridiag > gpurun_out/r02_bench_tridiag_normal.json 2> gpurun_out/r02_bench_tridiag_normal.err
python bench.py --sym --no-cpu-baseline > gpurun_out/r02_bench_c3_normal_sym.json 2> gpurun_out/r02_bench_c3_normal_sym.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
for v in normal normal2 prequr prequr_hh; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --sharded --variant $v --no-cpu-baseline --steps 5 > gpurun_out/r02_bench_sharded_$v.json 2> gpurun_out/r02_bench_sharded_$v.err
done
