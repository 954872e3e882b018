python tools/time_potrf.py 200 20 > gpurun_out/s2_plain_k2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:potrf -s 3 -c 1 -f -o /tmp/k2 python tools/time_potrf.py 200 5 > /dev/null 2>&1
python tools/ncu_kernel_summary.py /tmp/k2.ncu-rep gpurun_out/s2_k2_summary.txt "K2 potrf_kernel n=200: python tools/time_potrf.py 200"
python tools/ncu_sass_dump.py /tmp/k2.ncu-rep gpurun_out/s2_k2_sass.txt
python tools/prof_k3.py 100000 200 3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:trsm_dmma -s 3 -c 1 -f -o /tmp/k3 python tools/prof_k3.py 100000 200 3 > /dev/null 2>&1
python tools/ncu_sass_dump.py /tmp/k3.ncu-rep gpurun_out/s2_k3_sass.txt
cat gpurun_out/s2_plain_k2.log
