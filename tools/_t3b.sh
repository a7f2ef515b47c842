bash tools/_t3.sh
timeout 600 python -m pytest tests/test_determinism.py tests/test_shape_sweep.py -q -m gpu -x 2>&1 | tail -2
