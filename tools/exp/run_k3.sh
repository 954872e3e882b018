for s in "40000 200" "100000 200" "20000 100" "10000 100" "4000 50" "2000 240"; do
  echo -n "NOPANEL " >> gpurun_out/r2_k3_exp3.txt; OQR_LIB=tools/exp/liboqr_K3NOPANEL.so python tools/prof_k3.py $s >> gpurun_out/r2_k3_exp3.txt 2>&1
  echo -n "PANEL " >> gpurun_out/r2_k3_exp3.txt; python tools/prof_k3.py $s >> gpurun_out/r2_k3_exp3.txt 2>&1
done
