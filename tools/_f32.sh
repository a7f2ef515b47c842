E=$PWD/paper_2501_08582_b200/_native/exp
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_weff_identity.py tests/test_shape_sweep.py tests/test_decoder.py -q -m gpu -x > gpurun_out/f32_tests.log 2>&1; tail -n 1 gpurun_out/f32_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for v in prev new; do
  if [ $v = new ]; then unset LORS_B200_LIB; else export LORS_B200_LIB=$E/prev/liblors_b200.so; fi
  timeout 600 python bench.py --config cfg1 --no-cpu --steps 5 --warmup 3 > gpurun_out/f32_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/f32_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], json.dumps(d.get('step_breakdown_ms') or d.get('config'))[:300]); print(json.dumps(d['roofline'])[:400])"
done
