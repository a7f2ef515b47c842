timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/full7_tests.log 2>&1; tail -n 2 gpurun_out/full7_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full7_smoke.log 2>&1; tail -n 1 gpurun_out/full7_smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg3_r02f.json 2> gpurun_out/bench_cfg3_r02f.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02f.json 2>> gpurun_out/bench_cfg3_r02f.err
python - <<'P'
import json
for f in ("cfg3_r02f", "ref_r02f"):
    d = json.loads(open(f"gpurun_out/bench_{f}.json").read().strip().splitlines()[-1])
    print(f, d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), d.get("peak_hbm_gb"), (d.get("clocks") or {}).get("sm_mhz"), (d.get("roofline") or {}).get("frac"), d.get("gpu_launches"), (d.get("layer_cfg2") or {}).get("tokens_per_s"))
P
