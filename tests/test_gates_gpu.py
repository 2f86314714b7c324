"""GPU parity of the batched gate-bootstrapping path (blind rotation, sample extract,
identity key switch) against the CPU oracle and the reference's golden vectors.

Bar: bit-exact ciphertexts (integer torus words) on identical keys and inputs.
"""
import numpy as np
import pytest

import paper_2010_09410_b200 as vsp
from oracle.pyoracle import GATE_KINDS
from tests.helpers import TRUTH, golden, oracle, oracle_keys, random_gate_batch

pytestmark = pytest.mark.gpu


def engine(params, seed, with_cb=False, n_override=0):
    e = vsp.Engine(params, n_override=n_override)
    e.upload_keys(oracle_keys(params, seed, with_cb, n_override))
    return e


@pytest.fixture(scope="module")
def det():
    return engine("test-det", 515253, True), oracle("test-det", 515253, True)


@pytest.fixture(scope="module")
def prod():
    return engine("tfhe-80", 20200729), oracle("tfhe-80", 20200729, False)


def test_golden_testdet(det):
    e, _ = det
    g = golden("testdet_seed515253.npz")
    out = e.hom_gate_batch(list(g["kinds"]), g["ins"])
    assert np.array_equal(out, g["outs"])


def test_golden_tfhe80(prod):
    e, _ = prod
    g = golden("tfhe80_seed20200729.npz")
    out = e.hom_gate_batch(list(g["kinds"]), g["ins"])
    assert np.array_equal(out, g["outs"])
    assert np.array_equal(e.bootstrap_to_trlwe(g["br_in"]), g["br_out"])


def test_golden_n630():
    e = engine("tfhe-80", 630, n_override=630)
    g = golden("tfhe80n630_seed630.npz")
    assert np.array_equal(e.hom_gate_batch(list(g["kinds"]), g["ins"]), g["outs"])


@pytest.mark.parametrize("kind", GATE_KINDS)
def test_truth_tables_testdet_exhaustive(det, kind):
    e, o = det
    ar = vsp.GATE_ARITY[kind]
    combos = [(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)]
    ins = np.zeros((len(combos), 3, o.n + 1), np.uint32)
    for i, bits in enumerate(combos):
        for j in range(3):
            ins[i, j] = o.encrypt(bits[j])
    out = e.hom_gate_batch([kind] * len(combos), ins)
    for i, bits in enumerate(combos):
        ref = o.hom_gate(kind, list(ins[i][:ar]))
        assert np.array_equal(out[i], ref)
        assert o.decrypt(out[i]) == TRUTH[kind](*bits)


def test_random_mixed_batch_tfhe80_bit_exact(prod):
    e, o = prod
    rng = np.random.default_rng(11)
    kinds, bits, ins = random_gate_batch(o, rng, 37)   # ragged: not a multiple of 8 warps
    out = e.hom_gate_batch(kinds, ins)
    ref = o.hom_gate_batch(np.array([GATE_KINDS.index(k) for k in kinds]), ins, threads=8)
    assert np.array_equal(out, ref)
    for g, k in enumerate(kinds):
        assert o.decrypt(out[g]) == TRUTH[k](*bits[g])


def test_nand_xor_4096_decrypt_and_sample_bit_exact(prod):
    """BASELINE config-1 shape at full size: every output decrypts to the truth table;
    a strided sample is bit-exact against the oracle."""
    e, o = prod
    rng = np.random.default_rng(3)
    G = 4096
    kinds = [("NAND", "XOR")[int(x)] for x in rng.integers(0, 2, G)]
    bits = rng.integers(0, 2, size=(G, 2)).astype(np.uint8)
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    ins = np.zeros((G, 3, p.n + 1), np.uint32)
    ins[:, :2] = vsp.encrypt(p, k["lv0"], bits.reshape(-1), 1234).reshape(G, 2, p.n + 1)
    out = e.hom_gate_batch(kinds, ins)
    dec = vsp.decrypt(k["lv0"], out)
    want = np.array([TRUTH[kk](int(a), int(b), 0) for kk, (a, b) in zip(kinds, bits)])
    assert np.array_equal(dec, want)
    idx = np.arange(0, G, 293)
    ref = o.hom_gate_batch(np.array([GATE_KINDS.index(kinds[i]) for i in idx]), ins[idx],
                           threads=8)
    assert np.array_equal(out[idx], ref)


def test_identity_key_switch_and_gate_bootstrap(prod):
    e, o = prod
    rng = np.random.default_rng(7)
    x = np.stack([o.encrypt(int(b)) for b in rng.integers(0, 2, 5)])
    gb = e.gate_bootstrap(x)
    for i in range(len(x)):
        assert np.array_equal(gb[i], o.gate_bootstrap(x[i]))
    tr = e.bootstrap_to_trlwe(x)
    lvl1 = np.stack([o.sample_extract(t, 0) for t in tr])
    ks = e.identity_key_switch(lvl1)
    for i in range(len(x)):
        assert np.array_equal(ks[i], o.identity_key_switch(lvl1[i]))


def test_noise_inflated_to_0p9_mu_still_decodes(prod):
    """test_tfhe.cpp:462-472 on the GPU path."""
    e, o = prod
    rng = np.random.default_rng(8)
    xs, ms = [], []
    for i in range(64):
        m = int(rng.integers(0, 2))
        c = o.encrypt(m)
        c[-1] = np.uint32((int(c[-1]) + (int(0.9 * vsp.MU32) * (1 if i & 1 else -1))) % 2**32)
        xs.append(c)
        ms.append(m)
    out = e.gate_bootstrap(np.stack(xs))
    assert [o.decrypt(c) for c in out] == ms


def test_edge_cases_and_errors(det):
    e, o = det
    empty = e.hom_gate_batch([], np.zeros((0, 3, o.n + 1), np.uint32))
    assert empty.shape == (0, o.n + 1)
    one = e.hom_gate("NOT", [o.encrypt(1)])
    assert o.decrypt(one) == 0
    twice = e.hom_gate("NOT", [one])
    assert o.decrypt(twice) == 1
    with pytest.raises(ValueError):
        e.hom_gate("AND", [o.encrypt(1)])
    with pytest.raises(ValueError):
        e.hom_gate_batch([11], np.zeros((1, 3, o.n + 1), np.uint32))


def test_counters_match_reference_semantics(det):
    e, o = det
    e.counters_reset()
    o.counters_reset()
    x = [o.encrypt(1), o.encrypt(0), o.encrypt(1)]
    ins = np.zeros((3, 3, o.n + 1), np.uint32)
    for i in range(3):
        ins[i] = np.stack(x)
    e.hom_gate_batch(["MUX", "NAND", "NOT"], ins)
    o.hom_gate("MUX", x)
    o.hom_gate("NAND", x[:2])
    o.hom_gate("NOT", x[:1])
    c = e.counters()
    oc = o.counters()
    assert (c["cmux"], c["blindRotate"], c["identityKeySwitch"]) == (oc[0], oc[1], oc[2])


def test_pipelined_host_batch_equals_single_device_call(prod):
    """vsp_hom_gate_batch cuts a large host batch into blind-rotation waves with the
    uploads/downloads overlapped on a copy stream; the result must equal one device-side
    call of the same batch (all ten kinds, MUX = 2 tasks, NOT = 0), and decrypt right."""
    import torch
    e, o = prod
    rng = np.random.default_rng(21)
    G = 3001
    kinds = [GATE_KINDS[int(x)] for x in rng.integers(0, len(GATE_KINDS), G)]
    bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    ins = vsp.encrypt(p, k["lv0"], bits.reshape(-1), 99).reshape(G, 3, p.n + 1)
    out = e.hom_gate_batch(kinds, ins)
    d_in = torch.from_numpy(ins.view(np.int32)).cuda()
    d_out = torch.empty((G, p.n + 1), dtype=torch.int32, device="cuda")
    e.hom_gate_batch_dev(kinds, d_in.data_ptr(), d_out.data_ptr(), G)
    torch.cuda.synchronize()
    assert np.array_equal(out, d_out.cpu().numpy().view(np.uint32))
    dec = vsp.decrypt(k["lv0"], out)
    want = np.array([TRUTH[kk](*(int(x) for x in b)) for kk, b in zip(kinds, bits)])
    assert np.array_equal(dec, want)


# (tasks) -> launch plan the engine must pick on a 148-SM B200 (vsp_br_plan, cost model)
WAVE_PLANS = {
    1: {"lat": True, "full": 0, "w_rem": 0, "rem_kernel": "none"},        # latency kernel
    150: {"lat": True, "full": 0, "w_rem": 0, "rem_kernel": "none"},      # 150 CTAs
    2368: {"lat": False, "full": 2368, "w_rem": 0, "rem_kernel": "none"},  # two whole waves
    2400: {"lat": False, "full": 2368, "w_rem": 0, "rem_kernel": "br_lat"},  # + 32 on br_lat
    2995: {"lat": False, "full": 2368, "w_rem": 5, "rem_kernel": "br1024"},  # + W=5 wave
    300: {"lat": False, "full": 0, "w_rem": 3, "rem_kernel": "br1024p"},  # two warps/task
}


@pytest.mark.parametrize("G", sorted(WAVE_PLANS))
def test_wave_boundaries_host_and_device_paths(prod, G):
    """Launch-policy boundaries (the plan is asserted, so the test covers what it names):
    latency kernel (1 and 150 tasks), exactly two whole W=8 waves, one W=6 launch, and two
    whole waves + a remainder (key switch forked under the remainder, host pipeline with an
    early download).  Host-pipelined and device calls agree and every output decrypts
    right."""
    import torch
    e, o = prod
    if e.sms == 148:
        assert e.br_plan(G) == WAVE_PLANS[G]
    rng = np.random.default_rng(G)
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    kid = rng.choice([GATE_KINDS.index("NAND"), GATE_KINDS.index("XOR")], G).astype(np.int32)
    bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    ins = vsp.encrypt(p, k["lv0"], bits.reshape(-1), 5 + G).reshape(G, 3, p.n + 1)
    out = e.hom_gate_batch(kid, ins)
    d_in = torch.from_numpy(ins.view(np.int32)).cuda()
    d_out = torch.empty((G, p.n + 1), dtype=torch.int32, device="cuda")
    e.hom_gate_batch_dev(kid, d_in.data_ptr(), d_out.data_ptr(), G)
    torch.cuda.synchronize()
    assert np.array_equal(out, d_out.cpu().numpy().view(np.uint32))
    want = np.array([TRUTH[GATE_KINDS[kk]](*(int(x) for x in b)) for kk, b in zip(kid, bits)])
    assert np.array_equal(vsp.decrypt(k["lv0"], out), want)


def test_mux_straddling_wave_boundaries_host_pipeline(prod):
    """Advisor finding r01: the host pipeline preps the gates of each whole wave before it
    launches; a MUX whose two tasks straddle a wave boundary (tasks 1183/1184 and 2367/2368
    after one leading AND) must be prepped before the first wave that reads it.  [AND] +
    1600 MUX = 3,201 tasks: two whole W=8 waves + a remainder.  Host-pipelined call ==
    device call == oracle on the straddling gates; every output decrypts right."""
    import torch
    e, o = prod
    G = 1601
    kid = np.array([GATE_KINDS.index("AND")] + [GATE_KINDS.index("MUX")] * 1600, np.int32)
    if e.sms == 148:
        # the 833-task remainder: one W=6 wave (7.72 ms) beats two W=3 two-warp waves (8.62)
        assert e.br_plan(3201) == {"lat": False, "full": 2368, "w_rem": 6, "rem_kernel": "br1024"}
    rng = np.random.default_rng(1601)
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    ins = vsp.encrypt(p, k["lv0"], bits.reshape(-1), 1601).reshape(G, 3, p.n + 1)
    out = e.hom_gate_batch(kid, ins)
    d_in = torch.from_numpy(ins.view(np.int32)).cuda()
    d_out = torch.empty((G, p.n + 1), dtype=torch.int32, device="cuda")
    e.hom_gate_batch_dev(kid, d_in.data_ptr(), d_out.data_ptr(), G)
    torch.cuda.synchronize()
    assert np.array_equal(out, d_out.cpu().numpy().view(np.uint32))
    want = np.array([TRUTH[GATE_KINDS[kk]](*(int(x) for x in b)) for kk, b in zip(kid, bits)])
    assert np.array_equal(vsp.decrypt(k["lv0"], out), want)
    straddle = np.array([0, 591, 592, 1183, 1184, 1600])  # MUX i owns tasks 2i+1, 2i+2
    ref = o.hom_gate_batch(kid[straddle], ins[straddle], threads=8)
    assert np.array_equal(out[straddle], ref)


def test_not_only_and_mux_heavy_batches_tfhe80(prod):
    """Batches without any blind rotation (all NOT: the host pipeline uploads and negates
    only) and MUX-heavy batches (two tasks per gate across the wave boundary)."""
    e, o = prod
    rng = np.random.default_rng(33)
    x = np.zeros((40, 3, o.n + 1), np.uint32)
    bits = rng.integers(0, 2, 40)
    for i, b in enumerate(bits):
        x[i, 0] = o.encrypt(int(b))
    out = e.hom_gate_batch(["NOT"] * 40, x)
    assert [o.decrypt(c) for c in out] == [1 - int(b) for b in bits]
    G = 700  # 1,400 blind-rotation tasks: one whole W=8 wave + 216 on the latency kernel
    if e.sms == 148:
        assert e.br_plan(2 * G) == {"lat": False, "full": 1184, "w_rem": 0, "rem_kernel": "br_lat"}
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    mb = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    ins = vsp.encrypt(p, k["lv0"], mb.reshape(-1), 44).reshape(G, 3, p.n + 1)
    out = e.hom_gate_batch(["MUX"] * G, ins)
    want = np.array([TRUTH["MUX"](*(int(v) for v in b)) for b in mb])
    assert np.array_equal(vsp.decrypt(k["lv0"], out), want)


def test_back_to_back_calls_on_different_streams(prod):
    """Two device calls on two streams without a host sync in between: the second waits for
    the first (the context's scratch buffers are shared), both results are right."""
    import torch
    e, o = prod
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    rng = np.random.default_rng(77)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    jobs = []
    for G in (1500, 300):
        kid = rng.integers(0, len(GATE_KINDS), G).astype(np.int32)
        bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
        ins = vsp.encrypt(p, k["lv0"], bits.reshape(-1), G).reshape(G, 3, p.n + 1)
        d_in = torch.from_numpy(ins.view(np.int32)).cuda()
        d_out = torch.empty((G, p.n + 1), dtype=torch.int32, device="cuda")
        want = np.array([TRUTH[GATE_KINDS[kk]](*(int(x) for x in b)) for kk, b in zip(kid, bits)])
        jobs.append((kid, d_in, d_out, G, want))
    torch.cuda.synchronize()
    for s, (kid, d_in, d_out, G, _) in zip(streams, jobs):  # no host sync in between
        e.hom_gate_batch_dev(kid, d_in.data_ptr(), d_out.data_ptr(), G, s.cuda_stream)
    outs = [j[2] for j in jobs]
    wants = [j[4] for j in jobs]
    torch.cuda.synchronize()
    for d_out, want in zip(outs, wants):
        assert np.array_equal(vsp.decrypt(k["lv0"], d_out.cpu().numpy().view(np.uint32)), want)


@pytest.mark.parametrize("G", [1, 2, 77, 141, 148])
def test_two_tasks_per_sm_latency_kernel_equals_one(prod, G):
    """br_lat2_kernel (two narrow-level tasks per SM, chunked key ring) gives the same
    words as br_lat_kernel on ragged narrow levels (odd task counts shadow the last task),
    all gate kinds; sampled against the oracle."""
    e, o = prod
    rng = np.random.default_rng(500 + G)
    kid = rng.integers(0, len(GATE_KINDS), G).astype(np.int32)
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    ins = vsp.encrypt(p, k["lv0"], bits.reshape(-1), 600 + G).reshape(G, 3, p.n + 1)
    tasks = int(sum(2 if x == 2 else 0 if x == 5 else 1 for x in kid))
    if e.sms == 148 and tasks:
        assert e.br_plan(tasks)["lat"]
    one = e.hom_gate_batch(kid, ins)
    e.set_option("lat_tasks", 2)
    try:
        two = e.hom_gate_batch(kid, ins)
    finally:
        e.set_option("lat_tasks", 1)
    assert np.array_equal(one, two)
    idx = np.arange(0, G, max(1, G // 5))
    assert np.array_equal(two[idx], o.hom_gate_batch(kid[idx], ins[idx], threads=8))


@pytest.mark.parametrize("G", [64, 141, 1500])
def test_int8_gemm_key_switch_equals_tensor_free(prod, G):
    """The key switch as an INT8 tensor-core GEMM (one-hot digit selectors x the key in
    signed-byte planes, iks_gemm.cuh) gives the same words as iks_b2_kernel and the oracle:
    identity key switches, and whole gate batches (MUX sums, NOT) with and without it."""
    e, o = prod
    rng = np.random.default_rng(900 + G)
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    kid = rng.integers(0, len(GATE_KINDS), G).astype(np.int32)
    bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    ins = vsp.encrypt(p, k["lv0"], bits.reshape(-1), 901 + G).reshape(G, 3, p.n + 1)
    e.set_option("iks_gemm", 1)
    with_gemm = e.hom_gate_batch(kid, ins)
    e.set_option("iks_gemm", 0)
    try:
        without = e.hom_gate_batch(kid, ins)
    finally:
        e.set_option("iks_gemm", 1)
    assert np.array_equal(with_gemm, without)
    idx = np.arange(0, G, max(1, G // 6))
    assert np.array_equal(with_gemm[idx], o.hom_gate_batch(kid[idx], ins[idx], threads=8))
    lvl1 = np.stack([o.sample_extract(t, 0) for t in e.bootstrap_to_trlwe(ins[:G, 0])])
    ks = e.identity_key_switch(lvl1)
    for i in range(0, G, max(1, G // 4)):
        assert np.array_equal(ks[i], o.identity_key_switch(lvl1[i]))


@pytest.mark.parametrize("G", [70, 1200])
def test_int8_gemm_split_k_equals_unsplit(prod, G):
    """Split-K key-switch GEMM (K_ = 24,576 cut into strided batches whose int32 partial
    products the epilogue sums mod 2^32): every split factor gives the same words,
    including a non-power-of-two split and the automatic choice."""
    e, _ = prod
    rng = np.random.default_rng(950 + G)
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    kid = rng.integers(0, len(GATE_KINDS), G).astype(np.int32)
    bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    ins = vsp.encrypt(p, k["lv0"], bits.reshape(-1), 951 + G).reshape(G, 3, p.n + 1)
    outs = []
    try:
        for s in (1, 3, 4, 8, 0):
            e.set_option("iks_split", s)
            outs.append(e.hom_gate_batch(kid, ins))
    finally:
        e.set_option("iks_split", 0)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    with pytest.raises(ValueError):
        e.set_option("iks_split", 5)  # 24,576 / 5 is not an integer


@pytest.mark.parametrize("G", [300, 4096])
def test_two_warps_per_task_partial_wave_equals_one(prod, G):
    """br1024p_kernel (partial waves with two warps per task: a single W=3 launch for 300
    tasks, the 544-task W=4 remainder of 4,096) gives the same words as br1024_kernel."""
    e, o = prod
    rng = np.random.default_rng(1200 + G)
    k = oracle_keys("tfhe-80", 20200729, False)
    p = vsp.ParameterSet("tfhe-80")
    kid = rng.choice([GATE_KINDS.index("NAND"), GATE_KINDS.index("XOR")], G).astype(np.int32)
    bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    ins = vsp.encrypt(p, k["lv0"], bits.reshape(-1), 1201 + G).reshape(G, 3, p.n + 1)
    if e.sms == 148:
        assert e.br_plan(G)["rem_kernel"] == "br1024p"
    two = e.hom_gate_batch(kid, ins)
    e.set_option("br_pair", 0)
    try:
        one = e.hom_gate_batch(kid, ins)
    finally:
        e.set_option("br_pair", 1)
    assert np.array_equal(one, two)
    want = np.array([TRUTH[GATE_KINDS[kk]](*(int(x) for x in b)) for kk, b in zip(kid, bits)])
    assert np.array_equal(vsp.decrypt(k["lv0"], two), want)
