E=$PWD/paper_2501_08582_b200/_native/exp
timeout 1200 python -m pytest tests/test_weff_identity.py tests/test_shape_sweep.py tests/test_fullsize_parity.py -q -m gpu -x -k "sparse or sweep or cfg4" > gpurun_out/sp5_tests.log 2>&1; tail -n 1 gpurun_out/sp5_tests.log
LORS_B200_LIB=$E/trace/liblors_b200.so timeout 300 python tools/trace_k1.py 8192 11008 4096 64 sp24 2>&1 | grep -E "issuer iteration|transform period|xf |main completion|issuer wready|CTA0 warp"
for i in 1 2; do
  for v in prev new; do
    if [ $v = new ]; then timeout 300 python tools/ab_gemm.py >> gpurun_out/absp5.log 2>&1; else LORS_B200_LIB=$E/$v/liblors_b200.so timeout 300 python tools/ab_gemm.py >> gpurun_out/absp5.log 2>&1; fi
  done
done
python tools/ab_table.py gpurun_out/absp5.log
