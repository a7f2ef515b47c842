# grouped forward: full GPU suite, then the cfg3 bench with and without it, alternating
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/grp_gpu_tests.log 2>&1; tail -n 2 gpurun_out/grp_gpu_tests.log
for i in 1 2; do
for g in 1 0; do
LORS_GROUP_FWD=$g timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-layer > gpurun_out/grp_$g.$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/grp_$g.$i.json').read().strip().splitlines()[-1]); print('group_fwd=$g', round(d['value']), round(d['e2e']['value']), round(d['peak_hbm_gb'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
LORS_GROUP_FWD=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-layer --compare > gpurun_out/grp_cmp.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/grp_cmp.json').read().strip().splitlines()[-1]); print('compare', round(d['value']), d['memory'], d['comparators_tokens_per_s'])"
