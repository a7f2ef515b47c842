for v in 64 32 64 32; do
LORS_SPLIT_MIN_KSTEPS=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-layer > gpurun_out/split_$v.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/split_$v.json').read().strip().splitlines()[-1]); print('min_ksteps $v', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
done
