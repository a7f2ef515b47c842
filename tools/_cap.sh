E=$PWD/paper_2501_08582_b200/_native/exp
for c in 74 68 62 74 68 62; do
XP_DX_CLUSTERS=$c LORS_B200_LIB=$E/cap/liblors_b200.so timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-layer > gpurun_out/cap_$c.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/cap_$c.json').read().strip().splitlines()[-1]); print('dx clusters $c', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
done
