"""Generate the 200-step loss-curve fixture by running the REFERENCE trainer.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_loss_curve.py

north_star's third parity criterion: "a 200-step loss curve stays within 1% of
the reference's".  The reference has no transformer; its own training task is
the pruning-recovery teacher-student regression of train.py:379-425
(`run_recovery`): a dense 3-layer ReLU teacher, a 50%-pruned student whose
LoRS adapters are initialised by gradient-SVD (initialization.py:171-232) and
trained with the bias-corrected adaptive optimizer (train.py:139-154) on
batches drawn by the reference's counter-based Rng (train.py:271-276).

Everything the GPU test needs travels in the fixture: the dense weights, the
training set, the per-step batch indices, the adapters right after
initialisation, the reference loss per step and the final adapters.  Inputs,
targets and weights are rounded to float32 BEFORE the reference runs, so the
float64 reference and the fp32/bf16 GPU runs see the same numbers.

Rank 8 = the input manifold's dimension (latent_dim 8).  With run_recovery's
default rank 16 the gradient-SVD init has 8 degenerate (zero singular value)
directions in layer 1; the adaptive optimizer turns their rounding-level
gradients into full-size steps of random sign, and a 1e-7 relative
perturbation of the init moves the float64 reference's own curve by ~3%
(measured with the oracle), so a 1% bar is not a meaningful test there.  At
rank 8 the same perturbation moves it by ~2e-8 and bf16 rounding of the
inputs alone by ~3e-3.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

SEED = 3
WIDTH, DEPTH, RANK, PRUNE = 64, 3, 8, 0.5
STEPS, BATCH, LR, N_TRAIN, LATENT = 200, 32, 3e-4, 1024, 8


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    from lors import train
    from lors.initialization import InitSpec
    from lors.matrix import DenseMatrix, Rng

    def f32(m):
        return DenseMatrix(np.asarray(m.data, dtype=np.float32).astype(np.float64))

    dims = (WIDTH,) * (DEPTH + 1)
    weights = [f32(w) for w in train.random_dense_weights(SEED, dims)]
    teacher = train.model_from_weights(weights, variant="lors", rank=1, prune_ratio=0.0)
    data = train.make_teacher_data(teacher, seed=SEED + 1000, n=N_TRAIN, latent_dim=LATENT, latent_seed=SEED)
    x = f32(data.inputs)
    t = f32(teacher.predict(x))
    data = train.Dataset(inputs=x, targets=t, loss="regression")

    def student():
        return train.model_from_weights(weights, variant="lors", rank=RANK, alpha=2.0, prune_ratio=PRUNE)

    cfg = dict(batch_size=BATCH, lr=LR, optimizer="adaptive", variant="lors",
               init=InitSpec(strategy="gradient_svd"), seed=SEED)
    # adapters right after gradient-SVD init (finetune with 0 steps applies the init only)
    init_model, _ = train.finetune(student(), data, train.TrainConfig(steps=0, **cfg))
    model, trace = train.finetune(student(), data, train.TrainConfig(steps=STEPS, **cfg))

    rng = Rng(SEED)                                   # train.py:271-274: same draws as finetune
    idx = np.stack([rng.integers(BATCH, data.size) for _ in range(STEPS)])

    out = {
        "x": x.data.T.astype(np.float32),             # torch layout [N, C]
        "t": t.data.T.astype(np.float32),
        "idx": idx.astype(np.int64),
        "loss": np.array([row[1] for row in trace.rows]),
        "meta": np.array([WIDTH, DEPTH, RANK, STEPS, BATCH, N_TRAIN], dtype=np.int64),
        "lr": np.array(LR), "alpha": np.array(2.0), "prune": np.array(PRUNE),
    }
    for i, layer in enumerate(init_model.layers):
        out[f"w{i}"] = weights[i].data.astype(np.float32)          # dense (the test prunes it)
        out[f"base{i}"] = layer.base.values.data.astype(np.float32)  # the reference's pruned base
        out[f"a0_{i}"] = layer.adapter.a.data
        out[f"b0_{i}"] = layer.adapter.b.data
    for i, layer in enumerate(model.layers):
        out[f"a_{i}"] = layer.adapter.a.data
        out[f"b_{i}"] = layer.adapter.b.data
    path = os.path.join(HERE, "loss_curve.npz")
    np.savez_compressed(path, **out)
    ls = out["loss"]
    print(f"wrote {path}: loss {ls[0]:.6g} -> {ls[-1]:.6g} over {STEPS} steps "
          f"({os.path.getsize(path) / 1e6:.2f} MB); finite={bool(np.all(np.isfinite(ls)))}; "
          f"max|a| {max(float(np.abs(out[f'a_{i}']).max()) for i in range(DEPTH)):.3g}")
    assert math.isfinite(ls[-1])


if __name__ == "__main__":
    main()
