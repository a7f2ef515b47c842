# cfg3 step: rank-r overlap knobs under the power cap (default / LORS_BWD_OVERLAP=0 / LORS_GROUP_SIDE=1), rotating
for i in 1 2 3; do
for v in default ovl0 side1; do
unset LORS_BWD_OVERLAP LORS_GROUP_SIDE
[ $v = ovl0 ] && export LORS_BWD_OVERLAP=0
[ $v = side1 ] && export LORS_GROUP_SIDE=1
timeout 600 python bench.py --steps 15 --warmup 4 --no-cpu --no-layer > gpurun_out/ovl_$v.$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ovl_$v.$i.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
done
