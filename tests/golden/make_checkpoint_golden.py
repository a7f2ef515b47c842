"""Golden checkpoint written by the REFERENCE's own writer (run in the build
container, where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_checkpoint_golden.py

Writes tests/golden/ref_model.lors: a two-layer pruned model (24x16 per-row 50%
magnitude, 16x24 2:4) with a bias on layer 0, saved by lors.checkpoint.save_checkpoint.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from lors.checkpoint import save_checkpoint  # noqa: E402
from lors.matrix import DenseMatrix  # noqa: E402
from lors.prune import prune_magnitude, prune_two_four  # noqa: E402

rng = np.random.default_rng(20250115)
w0 = prune_magnitude(DenseMatrix(rng.normal(0, 0.02, size=(24, 16))), 0.5).values
w1 = prune_two_four(DenseMatrix(rng.normal(0, 0.02, size=(16, 24)))).values
b0 = DenseMatrix(rng.normal(0, 0.1, size=(24, 1)))
save_checkpoint(os.path.join(HERE, "ref_model.lors"),
                {"layers.0.weight": w0, "layers.0.bias": b0, "layers.1.weight": w1})
print("wrote", os.path.join(HERE, "ref_model.lors"))
