E=$PWD/paper_2501_08582_b200/_native/exp
python -m pytest tests/test_weff_identity.py tests/test_gpu_parity.py -q -m gpu > gpurun_out/id3.log 2>&1
for i in 1 2 3; do
  python tools/ab_gemm.py cfg3 >> gpurun_out/ab3.log 2>&1
  LORS_B200_LIB=$E/oldweff/liblors_b200.so python tools/ab_gemm.py cfg3 >> gpurun_out/ab3.log 2>&1
  LORS_B200_LIB=$E/pow2only/liblors_b200.so python tools/ab_gemm.py cfg3 >> gpurun_out/ab3.log 2>&1
done
tail -n 2 gpurun_out/id3.log
