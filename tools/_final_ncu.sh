# final-HEAD captures: the bench line's dominant kernel (--set full) and one graph-replayed cfg3 step's launch list
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_lors_gemm -s 2 -c 1 \
  -o gpurun_out/ncu_r02_final_dominant python tools/prof_dominant.py > gpurun_out/ncu_dom.log 2>&1; tail -n 2 gpurun_out/ncu_dom.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_lors_gemm -s 2 -c 1 \
  -o gpurun_out/ncu_r02_final_dx python tools/prof_dx_fwd.py > gpurun_out/ncu_dx.log 2>&1; tail -n 2 gpurun_out/ncu_dx.log
timeout 900 ncu --nvtx --nvtx-include "step" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r02_final_step.csv python tools/step_nvtx.py llama2-7b graph > gpurun_out/ncu_step.log 2>&1; tail -n 2 gpurun_out/ncu_step.log
