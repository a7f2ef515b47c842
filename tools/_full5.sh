timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/full5_tests.log 2>&1; tail -n 3 gpurun_out/full5_tests.log
timeout 900 python bench.py > gpurun_out/bench_cfg3_r02c.json 2> gpurun_out/bench_cfg3_r02c.err; tail -c 400 gpurun_out/bench_cfg3_r02c.json
timeout 900 python bench.py --config cfg4 --no-cpu --no-layer > gpurun_out/bench_cfg4_r02c.json 2>> gpurun_out/bench_r02c.err
timeout 900 python bench.py --config cfg4 --no-cpu --no-layer --sparse24 > gpurun_out/bench_cfg4_sp_r02c.json 2>> gpurun_out/bench_r02c.err
timeout 900 python bench.py --config cfg5 --no-cpu --no-layer > gpurun_out/bench_cfg5_r02c.json 2>> gpurun_out/bench_r02c.err
timeout 900 python bench.py --config cfg2 --no-cpu > gpurun_out/bench_cfg2_r02c.json 2>> gpurun_out/bench_r02c.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02c.json 2>> gpurun_out/bench_r02c.err
python - <<'P'
import json
for f in ("cfg3_r02c", "cfg4_r02c", "cfg4_sp_r02c", "cfg5_r02c", "cfg2_r02c", "ref_r02c"):
    try:
        d = json.loads(open(f"gpurun_out/bench_{f}.json").read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("unit"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), d.get("peak_hbm_gb"), (d.get("clocks") or {}).get("sm_mhz"), (d.get("step_roofline") or {}).get("frac_of_spec_roofline"))
    except Exception as e:
        print(f, "ERR", e)
P
