timeout 1200 python -m pytest tests/test_decoder.py tests/test_loss_curve.py tests/test_determinism.py tests/test_module_api.py tests/test_collective.py -q -m gpu -x > gpurun_out/g1_tests.log 2>&1; tail -n 3 gpurun_out/g1_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-layer > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; tail -c 1500 gpurun_out/g1_bench.json
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-layer --no-graph > gpurun_out/g1_bench_ng.json 2>> gpurun_out/g1_bench.err
python - <<'P'
import json
for f in ("gpurun_out/g1_bench.json", "gpurun_out/g1_bench_ng.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], d["e2e"]["value"], d["gpu_launches"], d["peak_hbm_gb"], d["clocks"]["sm_mhz"], d["path"]["cuda_graph"])
P
