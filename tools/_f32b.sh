timeout 1200 python -m pytest tests/test_determinism.py tests/test_gpu_parity.py tests/test_loss_curve.py -q -m gpu -x > gpurun_out/f32b_tests.log 2>&1; tail -n 1 gpurun_out/f32b_tests.log
timeout 600 python bench.py --config cfg1 --no-cpu --steps 5 --warmup 3 > gpurun_out/f32b.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/f32b.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d.get('step_breakdown_ms'))[:300])"
