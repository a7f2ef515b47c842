# HEAD record: the default bench line, the reference arm, and one graph-replayed cfg3 step's launch list
timeout 900 python bench.py > gpurun_out/f3_cfg3.json 2> gpurun_out/f3_cfg3.err; tail -c 400 gpurun_out/f3_cfg3.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f3_ref.json 2>/dev/null; tail -c 150 gpurun_out/f3_ref.json
timeout 600 python tools/step_nvtx.py llama2-7b graph > gpurun_out/f3_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "step" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r02_end_step.csv python tools/step_nvtx.py llama2-7b graph > gpurun_out/f3_ncu.log 2>&1; tail -n 2 gpurun_out/f3_ncu.log
