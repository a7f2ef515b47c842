E=$PWD/paper_2501_08582_b200/_native/exp
timeout 600 python -m pytest tests/test_weff_identity.py -q -m gpu -x > gpurun_out/n4_id.log 2>&1; tail -n 1 gpurun_out/n4_id.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/n4_par.log 2>&1; tail -n 1 gpurun_out/n4_par.log
for i in 1 2; do
  timeout 300 python tools/ab_gemm.py "cfg" >> gpurun_out/ab7.log 2>&1
  LORS_B200_LIB=$E/nact3/liblors_b200.so timeout 300 python tools/ab_gemm.py "cfg" >> gpurun_out/ab7.log 2>&1
done
python tools/ab_table.py gpurun_out/ab7.log
