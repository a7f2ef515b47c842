timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/gpu_all4.log 2>&1; tail -n 2 gpurun_out/gpu_all4.log
timeout 900 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; python -c "
import json; d=json.loads(open('gpurun_out/bench4.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['layer_cfg2']['tokens_per_s'], d['layer_cfg2']['step_breakdown_ms'], d['clocks'])"
