"""World-2 run of the ENGINE's C++ sharded path (multi.cuh), not a Python mirror: two
processes on the one GPU of the box, each with its own engine context, exchanging through
vsp_attach_exchange with a torch.distributed all-gather over gloo.  Everything the NCCL
path does except the transport runs: task-balanced level slices, the padded all-gather and
repack, RAM bit-block sharding with the read-out all-gather, and the RAM gather for the
getter.  Results must equal a single-rank engine bit for bit."""
import os
import pickle
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _entry(rank, world, port, job, outdir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        res = job(rank, world, dist)
        with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump(res, f)
    finally:
        dist.destroy_process_group()


def _allgather(dist, world):
    def ag(b: bytes):
        box = [None] * world
        dist.all_gather_object(box, b)
        return box
    return ag


def _level_job(rank, world, dist):
    """A mixed level (MUX-heavy front, NOTs, all kinds): sharded == single rank."""
    import paper_2010_09410_b200 as vsp
    import torch
    p = vsp.ParameterSet("tfhe-80")
    k = vsp.keygen(p, 2024, False)
    rng = np.random.default_rng(5)
    G = 1001
    kinds = np.array([2] * 300 + list(rng.integers(0, 10, G - 300)), np.int32)
    ins = vsp.encrypt(p, k["lv0"], rng.integers(0, 2, G * 3).astype(np.uint8), 6)
    ins = ins.reshape(G, 3, p.n + 1)
    single = vsp.Engine(p)
    single.upload_keys(k)
    want = single.hom_gate_batch(kinds, ins)
    e = vsp.Engine(p)
    e.upload_keys(k)
    e.attach_exchange(rank, world, _allgather(dist, world))
    d_in = torch.from_numpy(ins.view(np.int32)).cuda()
    d_out = torch.zeros((G, p.n + 1), dtype=torch.int32, device="cuda")
    e.hom_gate_level_dev(kinds, d_in.data_ptr(), d_out.data_ptr(), G)
    torch.cuda.synchronize()
    got = d_out.cpu().numpy().view(np.uint32)
    lo, hi, per = vsp.level_partition(G, world, rank, kinds)
    return {"equal": bool(np.array_equal(got, want)), "slice": (lo, hi, per)}


def _runner_job(rank, world, dist):
    """A netlist with a ROM port and a RAM port (w = 4: two bit-blocks per rank) at
    test-det, 3 cycles: DFF state, outputs and the gathered RAM image == single rank."""
    import paper_2010_09410_b200 as vsp
    from paper_2010_09410_b200 import netlist as N
    p = vsp.ParameterSet("test-det")
    k = vsp.keygen(p, 515253, True)
    nl = N.synthetic_netlist(seed=3, scale=0.03, levels=6, dffs=40, ram=(3, 4))
    rng = np.random.default_rng(1)
    v, w = 3, 4
    ram = vsp.encrypt_ram(p, k, rng.integers(0, 256, (w << v) // 8).astype(np.uint8), v, w, 2)
    luts = vsp.encrypt_rom(p, k, rng.integers(0, 256, 512).astype(np.uint8), 3)
    dff0 = vsp.encrypt(p, k["lv0"], rng.integers(0, 2, 40).astype(np.uint8), 4)
    ins = vsp.encrypt(p, k["lv0"], rng.integers(0, 2, len(nl.inputs[0].bits)).astype(np.uint8), 5)
    outs = []
    for sharded in (False, True):
        e = vsp.Engine(p)
        e.upload_keys(k)
        if sharded:
            e.attach_exchange(rank, world, _allgather(dist, world))
        ev = N.Evaluator(nl, e)
        ev.set_ram(ram, v, w)
        ev.set_rom(luts, 512)
        ev.set_dff_state_raw(dff0)
        for i, ct in enumerate(ins):
            ev.set_input("in", i, ct)
        trace = []
        for _ in range(3):
            ev.run(1)
            trace.append((ev.dff_state(), np.stack([ev.output("out", j) for j in range(16)])))
        outs.append((trace, ev.ram()))
        ev.close()
        e.close()
    (t0, r0), (t1, r1) = outs
    same = all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) for a, b in zip(t0, t1))
    return {"equal": bool(same and np.array_equal(r0, r1))}


@pytest.mark.parametrize("job", [_level_job, _runner_job], ids=["level", "runner_with_ram"])
def test_engine_sharded_path_world2_equals_single_rank(job, tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_entry, args=(world, _free_port(), job, str(tmp_path)), nprocs=world, join=True)
    res = [pickle.load(open(tmp_path / f"r{r}.pkl", "rb")) for r in range(world)]
    assert all(r["equal"] for r in res), res
    if job is _level_job:  # task-balanced: rank 0 takes the 300 MUX gates' share
        (lo0, hi0, _), (lo1, hi1, _) = res[0]["slice"], res[1]["slice"]
        assert lo0 == 0 and hi0 == lo1 and hi1 == 1001 and hi0 < 500
