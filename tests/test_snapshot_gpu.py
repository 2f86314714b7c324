"""Snapshot / resume (HVPS, snapshot.cpp:13-176) of the device-resident runner:
byte-identical to the reference's snapshotSave on the same state, loadable in both
directions, and run(k); save; load; run(k') == run(k + k')."""
import ctypes

import numpy as np
import pytest

import paper_2010_09410_b200 as vsp
from oracle import pyoracle
from oracle.pyoracle import CpuTfhe
from paper_2010_09410_b200 import netlist as N
from tests.helpers import oracle_keys
from tests.test_netlist_gpu import RefEval, words_to_image

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not pyoracle.available("ref"), reason="reference not built")]

SEED = 515253


@pytest.fixture(scope="module")
def setup():
    r = CpuTfhe("ref", "test-det", seed=SEED)
    r.keygen(True)
    e = vsp.Engine("test-det")
    e.upload_keys(oracle_keys("test-det", SEED, True))
    nl = N.synthetic_netlist(seed=3, scale=0.03, levels=6, dffs=40, ram=(3, 4))
    nl.name = "snapshot_probe"
    return r, e, nl


def _prime(r, ev, rev, nl):
    rng = np.random.default_rng(7)
    v, w = 3, 4
    ram = r.encrypt_ram(words_to_image([int(x) for x in rng.integers(0, 16, 8)], v, w), v, w)
    luts = r.encrypt_rom(rng.integers(0, 256, 512).astype(np.uint8))
    init = np.stack([r.encrypt(int(b)) for b in rng.integers(0, 2, ev.n_dffs)])
    ins = [r.encrypt(int(rng.integers(0, 2))) for _ in nl.inputs[0].bits]
    for x in (ev, rev):
        x.set_ram(ram, v, w)
        x.set_rom(luts, 512)
        for i, ct in enumerate(ins):
            x.set_input("in", i, ct)
    ev.set_dff_state_raw(init)
    assert rev.L.ref_eval_set_dff(rev.h, init.ctypes.data_as(ctypes.c_void_p),
                                  ctypes.c_uint32(r.n)) == 0
    return ins


def _ref_snapshot(rev):
    n = ctypes.c_size_t()
    assert rev.L.ref_eval_snapshot_save(rev.h, None, 0, ctypes.byref(n)) == 0
    buf = np.zeros(n.value, np.uint8)
    assert rev.L.ref_eval_snapshot_save(rev.h, buf.ctypes.data_as(ctypes.c_void_p), buf.size,
                                        ctypes.byref(n)) == 0
    return buf.tobytes()


def test_snapshot_bytes_match_reference_and_resume(setup):
    r, e, nl = setup
    text = N.netlist_to_json(nl)
    ev = N.Evaluator(nl, e)
    rev = RefEval(r, text)
    ins = _prime(r, ev, rev, nl)
    ev.run(2)
    rev.run(2)
    mine = ev.snapshot_save()
    theirs = _ref_snapshot(rev)
    assert mine == theirs, "HVPS bytes differ from the reference's snapshotSave"
    assert N.snapshot_peek(mine) == {"backend": "tfhe", "param": "test-det",
                                     "netlist": "snapshot_probe"}
    # resume here from the reference's bytes, and in the reference from ours
    ev2 = N.Evaluator(nl, e)
    ev2.snapshot_load(theirs)
    assert ev2.cycle == 2
    h = rev.L.ref_eval_snapshot_load(r.h, text.encode(), mine, len(mine), 4)
    assert h, rev.L.ref_last_error()
    for i, ct in enumerate(ins):
        ev2.set_input("in", i, ct)
    ev.run(2)  # continuous: 4 cycles
    ev2.run(2)  # resumed: 2 + 2
    assert np.array_equal(ev.dff_state(), ev2.dff_state())
    assert np.array_equal(ev.ram(), ev2.ram())
    assert ev.snapshot_save() == ev2.snapshot_save()


def test_snapshot_rejections(setup):
    r, e, nl = setup
    ev = N.Evaluator(nl, e)
    good = ev.snapshot_save()
    with pytest.raises(RuntimeError, match="bad snapshot magic"):
        ev.snapshot_load(b"XXXX" + good[4:])
    with pytest.raises(RuntimeError, match="parameter set"):
        ev.snapshot_load(good, param_name="tfhe-80")
    with pytest.raises(RuntimeError, match="truncated"):
        ev.snapshot_load(good[:len(good) // 2])
    other = N.synthetic_netlist(seed=4, scale=0.03, levels=6, dffs=40, ram=(3, 4))
    other.name = "snapshot_probe"
    with pytest.raises(RuntimeError, match="snapshot was taken on netlist"):
        N.Evaluator(other, e).snapshot_load(good)
