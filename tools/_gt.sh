# cfg3 step: raster group of 8 token tiles (default) vs 11 (= all of cfg3's token tiles: W read once), alternating
E=$PWD/paper_2501_08582_b200/_native/exp
for i in 1 2 3 4; do
for v in default gt11; do
if [ $v = gt11 ]; then export LORS_B200_LIB=$E/gt11/liblors_b200.so; else unset LORS_B200_LIB; fi
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-layer > gpurun_out/gt_$v.$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/gt_$v.$i.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], round(d['roofline']['ms_per_launch']*1e3,1))"
done
done
