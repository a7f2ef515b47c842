#!/bin/bash
# build an experiment variant of the library ($1 = extra nvcc flag) and time cfg2
python -c "
import sys; sys.path.insert(0, '.')
from paper_2501_08582_b200 import build as B
B.build(force=True, extra_flags=['$1'])
" && timeout 200 python tools/time_cfg2.py 2>&1 | head -2
