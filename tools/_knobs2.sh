# cfg3 step: fused Q + dA pass vs separate kernels (LORS_NO_QDA_PASS), and no grouped node (LORS_GROUP=0), rotating
for i in 1 2 3; do
for v in default noqda nogroup; do
unset LORS_NO_QDA_PASS LORS_GROUP
[ $v = noqda ] && export LORS_NO_QDA_PASS=1
[ $v = nogroup ] && export LORS_GROUP=0
timeout 600 python bench.py --steps 15 --warmup 4 --no-cpu --no-layer > gpurun_out/kn_$v.$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/kn_$v.$i.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
done
