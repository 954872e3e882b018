for mode in euclid fused; do
  ncu --set full --clock-control none --import-source on -k regex:gram_upper -s 3 -c 1 -f -o /tmp/k4_$mode python tools/prof_k4t.py 100000 200 3 $mode > /dev/null 2>&1
  python tools/ncu_kernel_summary.py /tmp/k4_$mode.ncu-rep gpurun_out/k4_${mode}_summary.txt "K4 $mode m=100000 n=200 (predicated DMMA)"
  python tools/ncu_sass_dump.py /tmp/k4_$mode.ncu-rep gpurun_out/k4_${mode}_sass.txt
done
