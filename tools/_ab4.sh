E=$PWD/paper_2501_08582_b200/_native/exp
python -m pytest tests/test_weff_identity.py tests/test_gpu_parity.py tests/test_determinism.py -q -m gpu > gpurun_out/id4.log 2>&1
for i in 1 2; do
  python tools/ab_gemm.py >> gpurun_out/ab4.log 2>&1
  LORS_B200_LIB=$E/oldweff/liblors_b200.so python tools/ab_gemm.py >> gpurun_out/ab4.log 2>&1
done
python tools/prof_fwd_pair.py > gpurun_out/pfp.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tc_lors_gemm -c 4 -o gpurun_out/prof_fwdpair python tools/prof_fwd_pair.py > gpurun_out/ncu_fwdpair.log 2>&1
tail -n 2 gpurun_out/id4.log
