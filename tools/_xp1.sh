E=$PWD/paper_2501_08582_b200/_native/exp
LORS_B200_LIB=$E/trnoxf/liblors_b200.so timeout 300 python tools/trace_k1.py 8192 11008 4096 64 sp24 2>&1 | grep -E "issuer iteration|transform period|xf |issuer passed"
for v in noxf; do LORS_B200_LIB=$E/$v/liblors_b200.so timeout 300 python tools/ab_gemm.py cfg2 >> gpurun_out/abxp1.log 2>&1; done
timeout 300 python tools/ab_gemm.py cfg2 >> gpurun_out/abxp1.log 2>&1
python tools/ab_table.py gpurun_out/abxp1.log
