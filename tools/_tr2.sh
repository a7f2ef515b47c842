E=$PWD/paper_2501_08582_b200/_native/exp
LORS_B200_LIB=$E/trace/liblors_b200.so python tools/trace_k1.py 8192 11008 4096 64 sp24 > gpurun_out/trace_sp.log 2>&1
LORS_B200_LIB=$E/trace/liblors_b200.so python tools/trace_k1.py 8192 11008 4096 64 > gpurun_out/trace_dense64.log 2>&1
cat gpurun_out/trace_sp.log; echo ====; cat gpurun_out/trace_dense64.log
