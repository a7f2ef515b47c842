timeout 600 python -m pytest tests/test_fullsize_parity.py tests/test_determinism.py -q -m gpu -x -k "fp32 or determin" 2>&1 | tail -2
bash tools/_s4.sh
timeout 600 python bench.py --config cfg1 --no-cpu --steps 5 --warmup 3 > gpurun_out/t3.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/t3.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d.get('step_breakdown_ms'))[:300])"
