# end-of-round record at HEAD: smoke, the default bench line, and the other BASELINE configs
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/f2_cfg3.json 2> gpurun_out/f2_cfg3.err; tail -c 300 gpurun_out/f2_cfg3.json
for c in cfg4 cfg5; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-layer --compare > gpurun_out/f2_$c.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/f2_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), round(d['e2e']['value']), d['memory'], d['clocks']['sm_mhz'])"
done
timeout 600 python bench.py --config cfg4 --sparse24 --steps 10 --warmup 3 --no-cpu --no-layer > gpurun_out/f2_cfg4_sp.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/f2_cfg4_sp.json').read().strip().splitlines()[-1]); print('cfg4 sparse24', round(d['value']), d['peak_hbm_gb'])"
timeout 600 python bench.py --config cfg2 --steps 20 --warmup 5 > gpurun_out/f2_cfg2.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/f2_cfg2.json').read().strip().splitlines()[-1]); print('cfg2', round(d['value']), d['ms_per_step'], d.get('step_breakdown_ms'))"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f2_ref.json 2>/dev/null; tail -c 200 gpurun_out/f2_ref.json
