# validation after the trainer's no-tail-split default: GPU suite, smoke, default bench twice
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/v3_gpu_tests.log 2>&1; tail -n 2 gpurun_out/v3_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do
timeout 900 python bench.py --no-cpu --no-layer > gpurun_out/v3_cfg3.$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/v3_cfg3.$i.json').read().strip().splitlines()[-1]); print('cfg3', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], d['peak_hbm_gb'])"
done
