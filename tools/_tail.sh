# cfg3 step with and without the tail split of the persistent walk, alternating
for i in 1 2 3 4; do
for v in default notail; do
if [ $v = notail ]; then export LORS_NO_TAIL_SPLIT=1; else unset LORS_NO_TAIL_SPLIT; fi
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-layer > gpurun_out/tail_$v.$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/tail_$v.$i.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
done
