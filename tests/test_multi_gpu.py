"""The multi-GPU level path on one GPU: a one-rank NCCL communicator (VSP_NCCL_SINGLE=1)
drives the sharded code path of vsp_hom_gate_level_dev -- the per-rank slice, the
ncclAllGather of the slice outputs on the engine stream and the copy-out -- which must
give exactly the single-GPU result.  (NCCL refuses two ranks on one device, so the
world > 1 exchange is covered by construction plus the gloo tests in test_multi_cpu.py.)
"""
import os

import numpy as np
import pytest

import paper_2010_09410_b200 as vsp
from oracle.pyoracle import GATE_KINDS
from tests.helpers import TRUTH, oracle_keys

pytestmark = pytest.mark.gpu


def test_sharded_level_path_with_one_rank_nccl_equals_plain_call(monkeypatch):
    import torch
    p = vsp.ParameterSet("tfhe-80")
    keys = oracle_keys("tfhe-80", 20200729, False)
    plain = vsp.Engine("tfhe-80")
    plain.upload_keys(keys)
    sharded = vsp.Engine("tfhe-80")
    sharded.upload_keys(keys)
    monkeypatch.setenv("VSP_NCCL_SINGLE", "1")
    sharded.attach_comm(vsp.nccl_unique_id(), 0, 1)

    rng = np.random.default_rng(5)
    G = 1500  # whole wave + remainder on the gate path
    kid = rng.integers(0, len(GATE_KINDS), G).astype(np.int32)
    bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    ins = vsp.encrypt(p, keys["lv0"], bits.reshape(-1), 17).reshape(G, 3, p.n + 1)
    d_in = torch.from_numpy(ins.view(np.int32)).cuda()
    outs = []
    for e in (plain, sharded):
        d_out = torch.empty((G, p.n + 1), dtype=torch.int32, device="cuda")
        e.hom_gate_level_dev(kid, d_in.data_ptr(), d_out.data_ptr(), G)
        torch.cuda.synchronize()
        outs.append(d_out.cpu().numpy().view(np.uint32))
    assert np.array_equal(outs[0], outs[1])
    dec = vsp.decrypt(keys["lv0"], outs[1])
    want = np.array([TRUTH[GATE_KINDS[k]](*(int(x) for x in b)) for k, b in zip(kid, bits)])
    assert np.array_equal(dec, want)
