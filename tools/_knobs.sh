E=$PWD/paper_2501_08582_b200/_native/exp
for i in 1 2; do
  for v in default gt4 gt16 nw3; do
    if [ $v = default ]; then timeout 300 python tools/ab_gemm.py >> gpurun_out/abkn.log 2>&1; else LORS_B200_LIB=$E/$v/liblors_b200.so timeout 300 python tools/ab_gemm.py >> gpurun_out/abkn.log 2>&1; fi
  done
done
python tools/ab_table.py gpurun_out/abkn.log
