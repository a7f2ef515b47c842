timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/gpu_all3.log 2>&1; tail -n 2 gpurun_out/gpu_all3.log
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; python -c "
import json; d=json.loads(open('gpurun_out/bench3.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['layer_cfg2']['tokens_per_s'], d['layer_cfg2']['step_breakdown_ms'], d['clocks'])"
for c in cfg4 cfg5; do timeout 1200 python bench.py --config $c --compare --no-cpu --no-layer --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 300 gpurun_out/bench_$c.json; done
timeout 1200 python bench.py --config cfg3 --compare --no-cpu --no-layer --steps 10 --warmup 3 > gpurun_out/bench_cfg3c.json 2> gpurun_out/bench_cfg3c.err
timeout 1200 python bench.py --config cfg4 --sparse24 --no-cpu --no-layer --steps 10 --warmup 3 > gpurun_out/bench_cfg4sp.json 2> gpurun_out/bench_cfg4sp.err
