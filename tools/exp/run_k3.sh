for s in "40000 200" "100000 200" "20000 100" "4000 50"; do
  echo -n "SERIAL " >> gpurun_out/r2_k3_exp2.txt; OQR_LIB=tools/exp/liboqr_K3SERIAL.so python tools/prof_k3.py $s >> gpurun_out/r2_k3_exp2.txt 2>&1
  echo -n "PIPELINED " >> gpurun_out/r2_k3_exp2.txt; python tools/prof_k3.py $s >> gpurun_out/r2_k3_exp2.txt 2>&1
done
