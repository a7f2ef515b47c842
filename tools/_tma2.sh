E=$PWD/paper_2501_08582_b200/_native/exp
B=tools/tma_bw/l2_bw
for cfg in "2048 4096 128 8 1 8 1 1" "2048 4096 128 8 1 8 1 2" "2048 4096 128 8 1 8 1 4" "2048 4096 128 8 1 8 1 8" "2048 4096 128 8 2 8 1 4" "2048 4096 256 4 1 8 1 4" "8192 4096 128 8 1 2 1 4"; do
  $B $cfg >> gpurun_out/l2bw2.log 2>&1
done
cat gpurun_out/l2bw2.log
LORS_B200_LIB=$E/act2/liblors_b200.so timeout 300 python -m pytest tests/test_weff_identity.py -q -m gpu -x -k "forward or sparse" > gpurun_out/act2_id.log 2>&1; tail -n 1 gpurun_out/act2_id.log
for i in 1 2; do
  timeout 300 python tools/ab_gemm.py cfg >> gpurun_out/ab5.log 2>&1
  LORS_B200_LIB=$E/act2/liblors_b200.so timeout 300 python tools/ab_gemm.py cfg >> gpurun_out/ab5.log 2>&1
done
python tools/prof_dx_fwd.py > gpurun_out/pdf.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tc_lors_gemm -s 1 -c 3 -o gpurun_out/prof_dxfwd python tools/prof_dx_fwd.py > gpurun_out/ncu_dxfwd.log 2>&1
