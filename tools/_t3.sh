timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_fullsize_parity.py -q -m gpu -x -k fp32 -s 2>&1 | grep -E "fp32|passed|failed|Error" | head -12
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_determinism.py tests/test_loss_curve.py -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --config cfg1 --no-cpu --steps 5 --warmup 3 > gpurun_out/t3.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/t3.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d.get('step_breakdown_ms'))[:300])"
