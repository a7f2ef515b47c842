E=$PWD/paper_2501_08582_b200/_native/exp
for i in 1 2; do
  for v in default notmem halftmem; do
    if [ $v = default ]; then python tools/ab_gemm.py "cfg" >> gpurun_out/ab6.log 2>&1; else LORS_B200_LIB=$E/$v/liblors_b200.so python tools/ab_gemm.py "cfg" >> gpurun_out/ab6.log 2>&1; fi
  done
done
cat gpurun_out/ab6.log
