timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final_gpu_tests.log 2>&1; tail -n 2 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_cfg3_final.json 2> gpurun_out/bench_cfg3_final.err; tail -c 600 gpurun_out/bench_cfg3_final.json
timeout 600 python bench.py --config cfg1 --steps 10 --warmup 3 > gpurun_out/bench_cfg1_final.json 2>/dev/null; tail -c 300 gpurun_out/bench_cfg1_final.json
