timeout 600 python -m pytest tests/test_weff_identity.py -q -m gpu -x > gpurun_out/sp_id.log 2>&1
tail -n 3 gpurun_out/sp_id.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -q -m gpu -x -k "sparse or 24 or golden or cfg2" > gpurun_out/sp_par.log 2>&1
tail -n 3 gpurun_out/sp_par.log
timeout 300 python tools/ab_gemm.py cfg > gpurun_out/sp_ab.log 2>&1
cat gpurun_out/sp_ab.log
