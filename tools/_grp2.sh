# grouped forward on / off at cfg3 and cfg4 (trainer default: no tail split), alternating
for c in cfg3 cfg4; do
for i in 1 2 3; do
for g in 1 0; do
LORS_GROUP_FWD=$g timeout 600 python bench.py --config $c --steps 15 --warmup 4 --no-cpu --no-layer > gpurun_out/g2_$c.$g.$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g2_$c.$g.$i.json').read().strip().splitlines()[-1]); print('$c group_fwd=$g', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
done
done
