K2_TRACE_RAW=gpurun_out/s3_k2trace2_raw.npy OQR_LIB=tools/exp/liboqr_k2trace2.so python tools/exp/k2_trace2.py 200 > gpurun_out/s3_k2trace2.txt 2>&1
