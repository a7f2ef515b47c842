"""On-disk formats: the reference checkpoint read / written
bit-compatibly (golden file written by the reference's own writer,
tests/golden/make_checkpoint_golden.py), its validation errors, pruned-model
import into LoRS layers and merged-model export (GPU)."""

import json
import os
import struct

import numpy as np
import pytest
import torch

from paper_2501_08582_b200 import checkpoint as ck
from paper_2501_08582_b200.errors import CheckpointFormatError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_model.lors")


def test_reads_reference_file_and_rewrites_identical_bytes(tmp_path):
    t = ck.load_checkpoint(GOLDEN)
    assert sorted(t) == ["layers.0.bias", "layers.0.weight", "layers.1.weight"]
    assert t["layers.0.weight"].shape == (24, 16) and t["layers.0.bias"].shape == (24, 1)
    assert ck.model_weight_names(t) == ["layers.0.weight", "layers.1.weight"]
    # the pruning survived the round trip: 50% magnitude, 2:4 along the input axis
    assert (t["layers.0.weight"] != 0).sum() == 24 * 16 // 2
    assert ((t["layers.1.weight"].reshape(16, 6, 4) != 0).sum(-1) <= 2).all()
    out = tmp_path / "again.lors"
    ck.save_checkpoint(out, dict(t))
    assert out.read_bytes() == open(GOLDEN, "rb").read()


def test_torch_and_1d_inputs_round_trip(tmp_path):
    w = torch.randn(5, 7, dtype=torch.float64)
    b = torch.randn(5, dtype=torch.float64)
    p = tmp_path / "m.lors"
    ck.save_checkpoint(p, {"layers.0.weight": w, "layers.0.bias": b})
    t = ck.load_checkpoint(p)
    assert np.array_equal(t["layers.0.weight"], w.numpy())
    assert t["layers.0.bias"].shape == (5, 1) and np.array_equal(t["layers.0.bias"][:, 0], b.numpy())


def _write_raw(path, manifest, payload=b"", magic=b"LORS", version=1):
    m = json.dumps(manifest).encode()
    with open(path, "wb") as fh:
        fh.write(struct.pack("<4sIQ", magic, version, len(m)) + m + payload)


@pytest.mark.parametrize("case", ["magic", "version", "truncated", "not_list", "missing", "dtype", "shape",
                                  "extent", "duplicate", "overlap", "empty"])
def test_validation_errors(tmp_path, case):
    p = tmp_path / "bad.lors"
    ok = {"name": "a", "shape": [1, 2], "dtype": "f64", "offset": 0}
    pay = np.zeros(4).tobytes()
    if case == "magic":
        _write_raw(p, [ok], pay, magic=b"NOPE")
    elif case == "version":
        _write_raw(p, [ok], pay, version=2)
    elif case == "truncated":
        p.write_bytes(b"LORS")
    elif case == "not_list":
        _write_raw(p, {"a": 1}, pay)
    elif case == "missing":
        _write_raw(p, [{"name": "a", "shape": [1, 2]}], pay)
    elif case == "dtype":
        _write_raw(p, [dict(ok, dtype="f32")], pay)
    elif case == "shape":
        _write_raw(p, [dict(ok, shape=[0, 2])], pay)
    elif case == "extent":
        _write_raw(p, [dict(ok, shape=[3, 2])], pay)
    elif case == "duplicate":
        _write_raw(p, [ok, dict(ok, offset=16)], pay)
    elif case == "overlap":
        _write_raw(p, [ok, dict(ok, name="b", offset=8)], pay)
    if case == "empty":
        with pytest.raises(CheckpointFormatError):
            ck.save_checkpoint(p, {})
        return
    with pytest.raises(CheckpointFormatError):
        ck.load_checkpoint(p)


def test_model_weight_names_contiguity():
    with pytest.raises(CheckpointFormatError):
        ck.model_weight_names({"layers.0.weight": 1, "layers.2.weight": 2})
    with pytest.raises(CheckpointFormatError):
        ck.model_weight_names({"calib": 1})


@pytest.mark.gpu
def test_import_pruned_and_export_merged(tmp_path):
    from oracle import lors_oracle as orc
    layers = ck.load_pruned_layers(GOLDEN, rank=4, dtype=torch.float32)
    ref = ck.load_checkpoint(GOLDEN)
    assert len(layers) == 2 and layers[0].bias is not None and layers[1].bias is None
    g = torch.Generator(device="cuda").manual_seed(5)
    for ly in layers:                              # adapters as after some training
        with torch.no_grad():
            ly.a.copy_(torch.randn(ly.a.shape, generator=g, device="cuda") * 0.05)
            ly.b.copy_(torch.randn(ly.b.shape, generator=g, device="cuda") * 0.5)
    p = tmp_path / "merged.lors"
    ck.save_merged(layers, p)
    merged = ck.load_checkpoint(p)
    for i, ly in enumerate(layers):
        w = ref[f"layers.{i}.weight"]
        want = orc.merge(w, ly.a.detach().double().cpu().numpy(), ly.b.detach().double().cpu().numpy(),
                         ly.alpha, w != 0)
        got = merged[f"layers.{i}.weight"]
        assert np.all(got[w == 0].view(np.int64) == 0)            # bit-exact +0 outside the mask
        assert np.abs(got - want).max() <= 1e-5 * max(1.0, np.abs(want).max())
    assert np.allclose(merged["layers.0.bias"], ref["layers.0.bias"])
