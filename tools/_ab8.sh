E=$PWD/paper_2501_08582_b200/_native/exp
for i in 1 2; do
  for v in default non2 norec; do
    if [ $v = default ]; then AB_CLOCKS=1 python tools/ab_gemm.py "cfg3" >> gpurun_out/ab8.log 2>&1; else AB_CLOCKS=1 LORS_B200_LIB=$E/$v/liblors_b200.so python tools/ab_gemm.py "cfg3" >> gpurun_out/ab8.log 2>&1; fi
  done
done
python tools/ab_table.py gpurun_out/ab8.log
