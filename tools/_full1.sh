timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/gpu_all.log 2>&1; tail -n 3 gpurun_out/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json
timeout 300 python tools/sanitize_small.py > gpurun_out/san_plain.log 2>&1 && timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_memcheck.log 2>&1; tail -n 5 gpurun_out/san_memcheck.log
