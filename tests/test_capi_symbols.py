"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/lors_b200.h declares, and the ctypes structs match the C layout
(checked by compiling a probe against the header with gcc).  No GPU calls."""

import ctypes as ct
import os
import re
import subprocess

import pytest

from paper_2501_08582_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lors_b200.h")
HEADERS = [os.path.join(ROOT, "include", h) for h in sorted(os.listdir(os.path.join(ROOT, "include"))) if h.endswith(".h")]


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIB_PATH):
        from paper_2501_08582_b200 import build
        build.build()
    return N.load()


def _declared_functions(headers=None):
    names = set()
    for h in headers or HEADERS:
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(lors_[a-z_0-9]+)\s*\(", src, flags=re.M))
    return sorted(names)


def test_header_declares_expected_symbols():
    assert _declared_functions([HEADER]) == sorted(N.EXPORTED_SYMBOLS)
    assert _declared_functions() == sorted(N.EXPORTED_SYMBOLS + N.DECODER_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (lors_[a-z_0-9]+)$", out, flags=re.M))
    missing = set(_declared_functions()) - exported
    assert not missing, missing
    for name in _declared_functions():
        assert getattr(lib, name) is not None


def test_abi_version_and_no_device(lib):
    assert lib.lors_abi_version() == 1
    import torch
    if not torch.cuda.is_available():
        assert lib.lors_device_check() == N.LORS_ERR_DEVICE
        assert b"sm_100" in lib.lors_last_error()


PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "lors_b200.h"
#define F(s, m) printf(#s "." #m " %zu\n", offsetof(s, m));
int main(void) {
  printf("lors_fwd_args %zu\n", sizeof(lors_fwd_args));
  printf("lors_bwd_args %zu\n", sizeof(lors_bwd_args));
  F(lors_fwd_args, L) F(lors_fwd_args, dtype) F(lors_fwd_args, flags) F(lors_fwd_args, alpha)
  F(lors_fwd_args, x) F(lors_fwd_args, mask_bits) F(lors_fwd_args, meta24) F(lors_fwd_args, bias)
  F(lors_fwd_args, p) F(lors_fwd_args, workspace_bytes)
  F(lors_bwd_args, grad_mode) F(lors_bwd_args, alpha) F(lors_bwd_args, x) F(lors_bwd_args, dy)
  F(lors_bwd_args, p) F(lors_bwd_args, dx) F(lors_bwd_args, dbias) F(lors_bwd_args, workspace_bytes)
  return 0;
}
"""


def test_ctypes_structs_match_c_layout(tmp_path):
    src = tmp_path / "probe.c"
    exe = tmp_path / "probe"
    src.write_text(PROBE)
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = dict(line.rsplit(" ", 1) for line in lines if line)
    assert int(got["lors_fwd_args"]) == ct.sizeof(N.FwdArgs)
    assert int(got["lors_bwd_args"]) == ct.sizeof(N.BwdArgs)
    for key, val in got.items():
        if "." in key:
            sname, field = key.split(".")
            cls = N.FwdArgs if sname == "lors_fwd_args" else N.BwdArgs
            assert getattr(cls, field).offset == int(val), key


def test_status_mapping():
    from paper_2501_08582_b200.errors import ArgumentError, DeviceError, ShapeError
    N.load()
    with pytest.raises(ShapeError):
        N.check(N.LORS_ERR_SHAPE)
    with pytest.raises(ArgumentError):
        N.check(N.LORS_ERR_ARGUMENT)
    with pytest.raises(DeviceError):
        N.check(N.LORS_ERR_CUDA)
    N.check(N.LORS_OK)


def test_c_side_validation_without_gpu(lib):
    """Argument errors are reported before any device work (rank/alpha rules of AdapterPair)."""
    a = N.FwdArgs()
    a.L, a.R, a.C, a.r = 8, 4, 4, 5   # r > min(R, C)
    a.dtype, a.alpha = N.DTYPE_F32, 2.0
    assert lib.lors_fwd(ct.byref(a), None) == N.LORS_ERR_ARGUMENT
    a.r, a.alpha = 2, 0.0
    assert lib.lors_fwd(ct.byref(a), None) == N.LORS_ERR_ARGUMENT
    a.alpha, a.R = 2.0, 0
    assert lib.lors_fwd(ct.byref(a), None) == N.LORS_ERR_SHAPE


def test_bwd_flag_validation_without_gpu(lib):
    """DX_ONLY (dX alone, no workspace) and NO_DX are exclusive; DX_ONLY needs no dA/dB."""
    b = N.BwdArgs()
    b.L, b.R, b.C, b.r = 8, 16, 16, 4
    b.dtype, b.alpha, b.grad_mode = N.DTYPE_BF16, 2.0, N.GRAD_STE
    b.flags = N.FLAG_DX_ONLY | N.FLAG_NO_DX
    b.w = b.a = b.b = b.x = b.dy = b.dx = ct.c_void_p(16)
    assert lib.lors_bwd(ct.byref(b), None) == N.LORS_ERR_ARGUMENT
    b.flags = N.FLAG_DX_ONLY
    assert lib.lors_bwd_workspace(ct.byref(b)) == 0
    b.flags = 0
    assert lib.lors_bwd_workspace(ct.byref(b)) > 0
    assert lib.lors_bwd(ct.byref(b), None) == N.LORS_ERR_ARGUMENT      # dA / dB missing without DX_ONLY
