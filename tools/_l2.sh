B=tools/tma_bw/l2_bw
for cfg in "2048 4096 128 4 1 8 1" "2048 4096 128 8 1 8 1" "2048 4096 128 4 2 8 1" "2048 4096 128 8 1 8 0" "2048 4096 256 4 1 8 1" "2048 4096 64 8 1 8 1" "512 4096 128 8 1 32 1" "512 4096 128 8 1 32 0" "8192 4096 128 8 1 2 1"; do
  $B $cfg >> gpurun_out/l2bw.log 2>&1
done
python tools/prof_dominant.py > gpurun_out/pd.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tc_lors_gemm -s 2 -c 1 -o gpurun_out/prof_dominant python tools/prof_dominant.py > gpurun_out/ncu_dom.log 2>&1
cat gpurun_out/l2bw.log
