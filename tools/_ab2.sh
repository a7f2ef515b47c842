E=$PWD/paper_2501_08582_b200/_native/exp
python -m pytest tests/test_weff_identity.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/id2.log 2>&1
for i in 1 2; do
  python tools/ab_gemm.py >> gpurun_out/ab2.log 2>&1
  LORS_B200_LIB=$E/oldweff/liblors_b200.so python tools/ab_gemm.py >> gpurun_out/ab2.log 2>&1
done
tail -n 2 gpurun_out/id2.log
