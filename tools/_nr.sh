for v in 0 1 0 1; do
XP_NO_RANKR=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-layer > gpurun_out/nr_$v.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/nr_$v.json').read().strip().splitlines()[-1]); print('no_rankr=$v', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
done
