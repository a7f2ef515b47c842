python tools/prof_dominant.py > gpurun_out/pd2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tc_lors_gemm -s 2 -c 1 -o gpurun_out/prof_dominant2 python tools/prof_dominant.py > gpurun_out/ncu_dom2.log 2>&1
python tools/step_nvtx.py > gpurun_out/sn.log 2>&1 && ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python tools/step_nvtx.py > gpurun_out/ncu_step.log 2>&1
tail -n 3 gpurun_out/ncu_step.log; wc -l gpurun_out/launches_r02.csv
