timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/full6_tests.log 2>&1; tail -n 2 gpurun_out/full6_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full6_smoke.log 2>&1; tail -n 2 gpurun_out/full6_smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg3_r02d.json 2> gpurun_out/bench_cfg3_r02d.err; tail -c 300 gpurun_out/bench_cfg3_r02d.json
timeout 900 python bench.py --config cfg4 --no-cpu --no-layer --sparse24 > gpurun_out/bench_cfg4_sp_r02d.json 2>> gpurun_out/bench_r02d.err
timeout 900 python bench.py --config cfg4 --no-cpu --no-layer > gpurun_out/bench_cfg4_r02d.json 2>> gpurun_out/bench_r02d.err
timeout 900 python bench.py --config cfg5 --no-cpu --no-layer > gpurun_out/bench_cfg5_r02d.json 2>> gpurun_out/bench_r02d.err
python - <<'P'
import json
for f in ("cfg3_r02d", "cfg4_r02d", "cfg4_sp_r02d", "cfg5_r02d"):
    try:
        d = json.loads(open(f"gpurun_out/bench_{f}.json").read().strip().splitlines()[-1])
        print(f, round(d.get("value")), d.get("ms_per_step"), round((d.get("e2e") or {}).get("value")), d.get("peak_hbm_gb"), (d.get("clocks") or {}).get("sm_mhz"), (d.get("step_roofline") or {}).get("frac_of_spec_roofline"), d["roofline"]["frac"], d.get("gpu_launches"))
    except Exception as e:
        print(f, "ERR", e)
P
