# cfg4 / cfg5 steps with and without the tail split, alternating
for c in cfg4 cfg5; do
for i in 1 2 3; do
for v in default notail; do
if [ $v = notail ]; then export LORS_NO_TAIL_SPLIT=1; else unset LORS_NO_TAIL_SPLIT; fi
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-layer > gpurun_out/t45_$c.$v.$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/t45_$c.$v.$i.json').read().strip().splitlines()[-1]); print('$c $v', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
done
done
