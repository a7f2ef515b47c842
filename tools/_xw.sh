E=$PWD/paper_2501_08582_b200/_native/exp
LORS_B200_LIB=$E/xw16/liblors_b200.so timeout 1200 python -m pytest tests/test_weff_identity.py tests/test_shape_sweep.py tests/test_gpu_parity.py tests/test_fullsize_parity.py -q -m gpu -x > gpurun_out/xw_tests.log 2>&1; tail -n 1 gpurun_out/xw_tests.log
for i in 1 2; do
  for v in prev xw16; do
    LORS_B200_LIB=$E/$v/liblors_b200.so timeout 300 python tools/ab_gemm.py >> gpurun_out/abxw.log 2>&1
  done
done
python tools/ab_table.py gpurun_out/abxw.log
