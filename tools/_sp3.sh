E=$PWD/paper_2501_08582_b200/_native/exp
LORS_B200_LIB=$E/trnw3na4/liblors_b200.so timeout 300 python tools/trace_k1.py 8192 11008 4096 64 sp24 2>&1 | grep -E "issuer iteration|transform period|xf |main completion|issuer wready" 
for i in 1 2; do
  for v in new nw3na4; do
    if [ $v = new ]; then timeout 300 python tools/ab_gemm.py "cfg2" >> gpurun_out/absp3.log 2>&1; else LORS_B200_LIB=$E/$v/liblors_b200.so timeout 300 python tools/ab_gemm.py "cfg2" >> gpurun_out/absp3.log 2>&1; fi
  done
done
python tools/ab_table.py gpurun_out/absp3.log
