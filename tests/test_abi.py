"""The C-ABI boundary: the library loads here (no GPU needed), exports every
symbol include/curvkit_b200.h declares, and reproduces the reference's
contract errors, which are raised before any device work."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1905_05559_b200 import _lib, curv
from paper_1905_05559_b200.errors import ContractError, ShapeError


def header_symbols():
    syms = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        txt = open(os.path.join(ROOT, "include", h)).read()
        syms |= set(re.findall(r"\b(curvkit_[a-z0-9_]+)\s*\(", txt))
    return syms


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(_lib.SIGNATURES) == syms


def test_version_and_param_count_on_host():
    assert b"sm_100a" in _lib.load().curvkit_version()
    assert curv.param_count(curv.ModelSpec([64, 32])) == 2080          # paper Out [9]
    assert curv.param_count(curv.ModelSpec([3, 5, 2])) == 32
    assert curv.param_count(curv.ModelSpec([784, 32, 10])) == 25450


def test_flatten_unflatten_roundtrip():
    spec = curv.ModelSpec([3, 5, 2])
    p = np.arange(32, dtype=float)
    w, b = curv.unflatten_params(spec, p)
    assert w[0].shape == (5, 3) and b[1].shape == (2,)
    assert np.array_equal(curv.flatten_params(w, b), p)
    assert curv.weight_block_offset(spec, 1) == 20 and curv.bias_block_offset(spec, 1) == 30
    assert np.array_equal(curv.flatten_params([[[1, 2], [3, 4]]], [[5, 6]]), [1, 2, 3, 4, 5, 6])


def _raw_model(widths, act=2, mode=0):
    w = (C.c_int64 * len(widths))(*widths)
    m = _lib.Model(len(widths), w, act, mode)
    m._k = w
    return m


def test_contract_errors_through_the_abi():
    lib = _lib.load()
    out = C.c_int64()
    assert lib.curvkit_param_count(C.byref(_raw_model([4])), C.byref(out)) == 2
    assert b"at least an input and an output layer" in lib.curvkit_last_error()
    assert lib.curvkit_param_count(C.byref(_raw_model([4, 0, 2])), C.byref(out)) == 2
    assert b"layer widths must be >= 1" in lib.curvkit_last_error()
    assert lib.curvkit_param_count(C.byref(_raw_model([4, 3], 0, 1)), C.byref(out)) == 2
    assert b"raw_mean_output requires an output width of 1" in lib.curvkit_last_error()


def test_host_api_contract_errors():
    spec = curv.ModelSpec([3, 2])
    p = np.zeros(8)
    x = np.zeros((7, 3))
    y = np.zeros((7, 2)); y[:, 0] = 1
    with pytest.raises(ContractError, match="not divisible by batch size 2"):
        curv.assemble_opg(spec, p, curv.Batch(x, y), curv.CurvatureConfig(batch_size_g=2))
    with pytest.raises(ContractError, match="refusing to drop the remainder"):
        curv.assemble_hessian(spec, p, curv.Batch(x, y), curv.CurvatureConfig(batch_size_h=2))
    big = curv.ModelSpec([100, 50])
    with pytest.raises(ContractError, match="exceeds the dense memory cap"):
        curv.assemble_hessian(big, np.zeros(5050), curv.Batch(np.zeros((2, 100)), np.eye(50)[:2]),
                              curv.CurvatureConfig(batch_size_h=2))
    ybad = y.copy(); ybad[3] = [0.5, 0.5]
    with pytest.raises(ContractError, match="target row 3 is not one-hot"):
        curv.assemble_opg(spec, p, curv.Batch(x, ybad), curv.CurvatureConfig(batch_size_g=7))
    with pytest.raises(ShapeError):
        curv.hvp(spec, p, curv.Batch(x, y), np.zeros(5))
    with pytest.raises(ContractError, match="HvpOperator: dataset size 7"):
        curv.HvpOperator(spec, p, curv.Batch(x, y), 2)
    with pytest.raises(ContractError, match="unknown precision"):
        curv.assemble_opg(spec, p, curv.Batch(x, y), precision="bf16")
