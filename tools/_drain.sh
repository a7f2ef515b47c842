E=$PWD/paper_2501_08582_b200/_native/exp
timeout 1200 python -m pytest tests/test_weff_identity.py tests/test_shape_sweep.py tests/test_gpu_parity.py tests/test_fullsize_parity.py -q -m gpu -x > gpurun_out/drain_tests.log 2>&1; tail -n 1 gpurun_out/drain_tests.log
LORS_B200_LIB=$E/trace/liblors_b200.so timeout 300 python tools/trace_k1.py 2>&1 | grep -E "tile [1-5]"
for i in 1 2; do
  for v in prev new; do
    if [ $v = new ]; then timeout 300 python tools/ab_gemm.py >> gpurun_out/abdrain.log 2>&1; else LORS_B200_LIB=$E/$v/liblors_b200.so timeout 300 python tools/ab_gemm.py >> gpurun_out/abdrain.log 2>&1; fi
  done
done
python tools/ab_table.py gpurun_out/abdrain.log
