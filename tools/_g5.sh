timeout 1200 python -m pytest tests/test_decoder.py tests/test_loss_curve.py -q -m gpu -x > gpurun_out/g5_tests.log 2>&1; tail -n 1 gpurun_out/g5_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-layer > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err
python -c "import json; d=json.loads(open('gpurun_out/g5_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d['gpu_launches'])"
