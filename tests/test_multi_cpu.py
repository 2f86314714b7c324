"""Multi-GPU host logic on CPU (world_size 2, gloo): the runner's level partition, the
sharded level schedule (slice + all-gather) against the single-rank evaluator, and the
NCCL unique-id distribution used by Engine.connect."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2010_09410_b200 as vsp
from paper_2010_09410_b200 import netlist as N


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world=2):
    port = _free_port()
    mp.spawn(_entry, args=(fn, world, port), nprocs=world, join=True)


def _entry(rank, fn, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_level_partition_covers_each_gate_once(world):
    for G in [0, 1, 2, 7, 114, 4096, 4097]:
        seen = []
        per0 = None
        for r in range(world):
            lo, hi, per = vsp.level_partition(G, world, r)
            per0 = per if per0 is None else per0
            assert per == per0 == -(-G // world)
            assert 0 <= hi - lo <= per
            if hi > lo and G % world == 0:
                assert lo == r * per  # equal slices: rank r's slice is slot r * per
            seen.extend(range(lo, hi))
        assert seen == list(range(G))
    with pytest.raises(ValueError):
        vsp.level_partition(4, world, world)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_level_partition_balances_blind_rotation_tasks(world):
    """Slices hold equal numbers of blind-rotation tasks (MUX = 2, NOT = 0): every slice
    is within one MUX of T / world, and together they cover each gate once."""
    rng = np.random.default_rng(world)
    for G in [5, 300, 4097]:
        kinds = [vsp.GATE_KINDS[int(x)] for x in rng.integers(0, 10, G)]
        if G == 300:
            kinds = ["MUX"] * 150 + ["AND"] * 150  # heavy front: gate-count slices would skew
        cost = [2 if k == "MUX" else 0 if k == "NOT" else 1 for k in kinds]
        T = sum(cost)
        seen = []
        for r in range(world):
            lo, hi, per = vsp.level_partition(G, world, r, kinds)
            assert hi - lo <= per
            assert abs(sum(cost[lo:hi]) - T / world) <= 2
            seen.extend(range(lo, hi))
        assert seen == list(range(G))


def _setup(ev, nl, seed):
    rng = np.random.default_rng(seed)
    for p in nl.inputs:
        for i in range(len(p.bits)):
            ev.set_input(p.name, i, int(rng.integers(0, 2)))
    for i in ev.dff:
        ev.dff[i] = int(rng.integers(0, 2))
    ev.rom = list(rng.integers(0, 256, 512))
    ev.ram = (8, 16, [int(x) for x in rng.integers(0, 1 << 16, 256)])


def _sharded_equals_single(rank, world):
    nl = N.synthetic_netlist(seed=5, levels=12, scale=0.25)
    ref = N.PlainEvaluator(nl)
    sh = N.ShardedPlainEvaluator(nl)
    _setup(ref, nl, 9)
    _setup(sh, nl, 9)
    ref.run(3)
    sh.run(3)
    assert sh.dff == ref.dff
    assert sh.values == ref.values
    m = sh.owned_ram_bits()  # each rank keeps only its own bit-blocks of the RAM current
    assert [x & m for x in sh.ram[2]] == [x & m for x in ref.ram[2]]
    n_gates = sum(1 for c in nl.cells if c.kind in N.GATES)
    total = [None] * world
    dist.all_gather_object(total, sh.gate_evals)
    assert sum(total) == 3 * n_gates  # every gate evaluated exactly once per cycle
    assert max(total) - min(total) <= 3 * sh.dag["depth"]  # balanced slices


def test_sharded_level_schedule_matches_single_rank_gloo():
    _spawn(_sharded_equals_single)


def _uid_broadcast(rank, world):
    box = [vsp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    assert isinstance(box[0], bytes) and len(box[0]) == 128
    got = [None] * world
    dist.all_gather_object(got, box[0])
    assert all(g == got[0] for g in got)


def test_nccl_unique_id_distribution_gloo():
    try:
        vsp.nccl_unique_id()
    except RuntimeError as e:  # no NCCL on this host
        pytest.skip(str(e))
    _spawn(_uid_broadcast)
