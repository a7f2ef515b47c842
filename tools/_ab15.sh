E=$PWD/paper_2501_08582_b200/_native/exp
timeout 600 python -m pytest tests/test_weff_identity.py -q -m gpu -x > gpurun_out/w2_id.log 2>&1; tail -n 1 gpurun_out/w2_id.log
for i in 1 2; do
  for v in default la2f; do
    if [ $v = default ]; then python tools/ab_gemm.py "cfg" >> gpurun_out/ab15.log 2>&1; else LORS_B200_LIB=$E/$v/liblors_b200.so timeout 300 python tools/ab_gemm.py "cfg" >> gpurun_out/ab15.log 2>&1; fi
  done
done
python tools/ab_table.py gpurun_out/ab15.log
