"""The C-ABI library loads, exports every symbol include/vsp_b200.h declares, and its
host-side validation mirrors the reference's exception types (no GPU needed)."""
import os
import re

import pytest

import paper_2010_09410_b200 as vsp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "vsp_b200.h")).read()
    return sorted(set(re.findall(r"\b(vsp_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol():
    L = vsp.lib()
    names = declared_symbols()
    assert len(names) >= 15
    for s in names:
        assert hasattr(L, s), f"{s} declared in vsp_b200.h but not exported"


def test_params_by_name():
    p = vsp.ParameterSet("tfhe-80")
    assert (p.n, p.N1, p.l1, p.Bg1Bits, p.N2, p.l2, p.Bg2Bits) == (500, 1024, 2, 10, 2048, 4, 9)
    assert (p.ksBaseBits, p.ksLen, p.pksBaseBits, p.pksLen, p.fft) == (2, 8, 3, 10, 1)
    d = vsp.ParameterSet("test-det")
    assert d.deterministic and d.n == 16 and d.N1 == 64
    assert vsp.ParameterSet("tfhe-80", 630).n == 630
    with pytest.raises(ValueError):
        vsp.ParameterSet("nope")


def test_engine_fails_loudly_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(RuntimeError):
        vsp.Engine("test-det")


def test_gate_kind_ids_names_ints_and_arrays():
    """GateKind ids (ops.hpp:183-194) from names, ints or an int array (the array path
    does no per-gate Python work); unknown names raise like homGate."""
    import numpy as np
    ids = vsp.Engine._kind_ids(["AND", "MUX", "XOR", 5])
    assert ids.dtype == np.int32 and list(ids) == [0, 2, 9, 5]
    arr = np.array([3, 9, 9, 3], np.int64)
    out = vsp.Engine._kind_ids(arr)
    assert out.dtype == np.int32 and out.flags["C_CONTIGUOUS"] and list(out) == [3, 9, 9, 3]
    with pytest.raises(ValueError):
        vsp.Engine._kind_ids(["NAND", "XAND"])
