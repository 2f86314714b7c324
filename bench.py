#!/usr/bin/env python
"""Benchmark of the VSP hot path on B200 (north_star: bootstrapped gates/s at 1/2/4/8 GPUs
and per-clock-cycle latency).

Headline (BASELINE.json configs[0]): one batch of G=4096 independent random NAND/XOR gates
per GPU bootstrapped at the paper's TFHE parameters with n=630 (tfhe-80 copy with n=630,
N=1024, l=2, Bg=2^10).  One "step" = one pass of the hot path over the batch (linear
combination -> blind rotation -> sample extract -> identity key switch).  The same JSON
line carries two sub-objects measured in the same run:
  "memory": configs[1], one ROM read (512 B) + one RAM cycle (512 B), s/access;
  "cycle":  configs[2], one clock cycle of the seeded synthetic Ruby-shaped netlist, s/cycle
            (no processor netlist exists in the reference).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                    [--config gates|memory|cycle] [--headline-only]

--gpus N > 1 without torchrun: the script relaunches itself under torch.distributed.run
(one rank per GPU, 127.0.0.1).  Under torchrun WORLD_SIZE must equal --gpus.
Multi-GPU: one netlist level of G x N gates; each rank bootstraps its slice and the engine
all-gathers the level's outputs over NCCL (weak scaling); value = all gates / max-over-
ranks device time.

Prints ONE JSON line (rank 0).  `value` is device-timed with CUDA events with inputs
resident in HBM and L2 flushed between steps; `e2e` is the same metric through the C-ABI
host entry point (vsp_hom_gate_batch) with pinned host buffers and the H2D/D2H copies
inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "bootstrapped_gates_per_sec"
UNIT = "gates/s"
# Algorithmic work per external product and per level-1 bootstrap:
# F_EP = (2l+2)*5*M*log2(M) + 2l*2*8*M with M = 512, l = 2.
F_EP = (2 * 2 + 2) * 5 * 512 * 9 + 2 * 2 * 2 * 8 * 512
# level-2 external product (circuit bootstrap): M = 1024, l2 = 4
F_EP2 = (2 * 4 + 2) * 5 * 1024 * 10 + 2 * 4 * 2 * 8 * 1024
KERNEL_TIMERS = ("br1024", "br_lat", "iks", "gate_prep", "cmux_chain", "br2", "pks")


def work_roofline(counters: dict, n: int, seconds: float, peak: float) -> dict:
    """FFT-compute roofline of a memory access / clock cycle from the op counters: every
    level-1 blind rotation is n external products, every CMUX one, every circuit bootstrap
    l1 = 2 level-2 blind rotations of n level-2 external products."""
    flops = (counters["blindRotate"] * n * F_EP + counters["cmux"] * F_EP +
             counters["circuitBootstrap"] * 2 * n * F_EP2)
    achieved = flops / seconds / 1e12
    return {"bound": "fp64", "achieved": round(achieved, 3), "peak": round(peak, 3),
            "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "flops": int(flops),
            "t_roof_s": round(flops / (peak * 1e12), 5),
            "flops_rule": "blindRotate*n*F_EP + cmux*F_EP + circuitBootstrap*2*n*F_EP2, "
                          "F_EP = 171008, F_EP2 = 643072",
            "note": "the narrow levels are latency-bound (n dependent external products per "
                    "level), so a cycle cannot reach the throughput roofline"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gates", type=int, default=4096)
    ap.add_argument("--n", type=int, default=630, help="LWE dimension (630 = BASELINE config)")
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="gates per CPU-baseline sample (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--config", default="gates", choices=["gates", "memory", "cycle"],
                    help="gates: BASELINE configs[0] (default, headline, with the memory and "
                         "cycle sub-objects); memory: configs[1] alone; cycle: configs[2] alone")
    ap.add_argument("--headline-only", action="store_true",
                    help="gates line without the memory / cycle sub-objects")
    ap.add_argument("--levels", type=int, default=32, help="cycle config: logic depth")
    ap.add_argument("--sub-steps", type=int, default=0,
                    help="timed steps of the memory / cycle sub-objects (0 = --steps)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "gloo"],
                    help="multi-GPU exchange: NCCL over NVLink (default) or the engine's "
                         "host-callback exchange over gloo (flow check on a 1-GPU box; "
                         "timings are not a scaling result)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn_ranks(n: int) -> int:
    """--gpus N outside torchrun: relaunch this script as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1 and pass its output through."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


class Ctx:
    """Per-process state shared by the three measurements (device, ranks, keys)."""

    def __init__(self, args, world, rank, local):
        import torch
        self.args, self.world, self.rank, self.local = args, world, rank, local
        # one GPU per rank; on a box with fewer GPUs than ranks (--exchange gloo smoke runs)
        # ranks share devices round robin
        self.local = local = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        self.dist = None
        self.gloo = args.exchange == "gloo"
        if world > 1:
            import torch.distributed as dist
            if self.gloo:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            self.dist = dist
        self.dev = f"cuda:{local}"
        self._peak = None
        self._cb = None

    def peak(self) -> float:
        import paper_2010_09410_b200 as vsp
        if self._peak is None:
            self._peak = vsp.fp64_peak_tflops(self.local)
        return self._peak

    def connect(self, eng):
        """Attach an engine to the ranks: NCCL over NVLink (default), or the host-callback
        exchange over gloo (--exchange gloo: exercises the multi-rank flow on any box)."""
        if self.world == 1:
            return
        if self.gloo:
            dist = self.dist

            def ag(b: bytes):
                box = [None] * self.world
                dist.all_gather_object(box, b)
                return box
            eng.attach_exchange(self.rank, self.world, ag)
        else:
            eng.connect()

    def max_over_ranks(self, x: float) -> float:
        if not self.dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if self.gloo else self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def cb_keys(self, p):
        """tfhe-80 n=630 keys with circuit-bootstrapping material for the memory / cycle
        measurements (client keygen with the b = a*s products on this GPU)."""
        import paper_2010_09410_b200 as vsp
        if self._cb is None:
            t0 = time.perf_counter()
            self._cb = vsp.keygen(p, 99, True, device=self.local)
            self.cb_keygen_s = time.perf_counter() - t0
        return self._cb


def make_workload(vsp, p, G, seed):
    rng = np.random.default_rng(seed)
    keys = vsp.keygen(p, seed, False)
    kinds = [("NAND", "XOR")[int(x)] for x in rng.integers(0, 2, G)]
    bits = rng.integers(0, 2, size=(G, 2)).astype(np.uint8)
    ins = np.zeros((G, 3, p.n + 1), np.uint32)
    ins[:, :2] = vsp.encrypt(p, keys["lv0"], bits.reshape(-1), seed + 1).reshape(G, 2, p.n + 1)
    truth = np.where(np.array(kinds) == "NAND", 1 - (bits[:, 0] & bits[:, 1]),
                     bits[:, 0] ^ bits[:, 1]).astype(np.uint8)
    return keys, kinds, ins, truth


STOCK = "the reference's own Release build (-O3 -DNDEBUG, native ISA level)"
PARITY = "the reference built for bit-exact parity (-O2 -ffp-contract=off, portable ISA)"


def cpu_reference_rate(kind, n, keys, kinds, ins, sample, threads):
    """Time the reference's own homGate batch (parallelFor over host threads) on a bounded
    sample of the workload; returns gates/s."""
    from oracle.pyoracle import CpuTfhe, GATE_KINDS
    r = CpuTfhe(kind, "tfhe-80", n_override=n, seed=1)
    r.import_keys(keys)
    kid = np.array([GATE_KINDS.index(k) for k in kinds[:sample]], np.int32)
    r.hom_gate_batch(kid[:threads], ins[:threads], threads=threads)  # warm caches/plans
    t0 = time.perf_counter()
    r.hom_gate_batch(kid, ins[:sample], threads=threads)
    dt = time.perf_counter() - t0
    return sample / dt, dt


def ref_kind(stock: bool = True):
    from oracle.pyoracle import available
    if stock and available("ref_stock"):
        return "ref_stock"
    return "ref" if available("ref") else "orc"


def traffic_from_profiles():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        try:
            return json.load(open(path)).get("br1024_bytes_per_launch")
        except Exception:
            return None
    return None


# --------------------------------------------------------------------------------------
# configs[0]: gates/s (headline)

def measure_gates(cx: Ctx) -> dict | None:
    """One step = one netlist level of G x world independent gates, sharded across the
    ranks by the engine (vsp_hom_gate_level_dev: each GPU bootstraps its slice, then one
    NCCL all-gather over NVLink leaves every output on every GPU).  N = 1 is the same call
    with no exchange."""
    import torch
    import paper_2010_09410_b200 as vsp
    args, world, rank, local = cx.args, cx.world, cx.rank, cx.local
    p = vsp.ParameterSet("tfhe-80", n_override=args.n)
    G = args.gates
    GA = G * world
    # identical keys and level on every rank (keys are replicated)
    keys, kinds, ins, truth = make_workload(vsp, p, GA, 1000)
    eng = vsp.Engine(p, device=local)
    eng.upload_keys(keys)
    cx.connect(eng)

    d_in = torch.from_numpy(ins.view(np.int32)).to(cx.dev)
    d_out = torch.empty((GA, p.n + 1), dtype=torch.int32, device=cx.dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=cx.dev)
    stream = torch.cuda.current_stream()
    kid = np.array([vsp.GATE_KINDS.index(k) for k in kinds], np.int32)  # GateKind ids

    def step():
        eng.hom_gate_level_dev(kid, d_in.data_ptr(), d_out.data_ptr(), GA, stream.cuda_stream)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    out = d_out.cpu().numpy().view(np.uint32)
    correct = bool(np.array_equal(vsp.decrypt(keys["lv0"], out), truth))

    # ---- device-timed region: inputs resident, L2 flushed between steps ----
    eng.profile_reset()
    eng.profile_enable(True)
    launches0 = eng.kernel_launches()
    cx.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    evs = []
    for _ in range(args.steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    cx.barrier()
    clk = clocks.stop()
    launches = eng.kernel_launches() - launches0
    eng.profile_enable(False)
    ms = sum(a.elapsed_time(b) for a, b in evs)
    br_ms, br_n = eng.profile_read("br1024")
    iks_ms, _ = eng.profile_read("iks")
    prep_ms, _ = eng.profile_read("gate_prep")
    ms_max = cx.max_over_ranks(ms)
    value = GA * args.steps / (ms_max / 1e3)

    # ---- end to end: host level in, host level out, through the engine API ----
    e2e = None
    if not args.no_e2e:
        lo, hi, _ = vsp.level_partition(GA, world, rank)
        if world == 1:
            h_in = torch.from_numpy(ins.view(np.int32)).pin_memory()
            h_in_np = h_in.numpy().view(np.uint32)
            h_out = torch.empty((GA, p.n + 1), dtype=torch.int32).pin_memory()
            h_out_np = h_out.numpy().view(np.uint32)
            res = eng.hom_gate_batch(kid, h_in_np, out=h_out_np)  # warm
            t0 = time.perf_counter()
            for _ in range(args.steps):
                res = eng.hom_gate_batch(kid, h_in_np, out=h_out_np)
            dt = time.perf_counter() - t0
            e2e_ok = bool(np.array_equal(vsp.decrypt(keys["lv0"], res), truth))
            h2d, d2h, api = int(ins.nbytes), int(res.nbytes), \
                "vsp_hom_gate_batch (C ABI, pinned host buffers)"
        else:
            # each rank uploads its slice, the engine shards + all-gathers, every rank
            # reads the whole level back (pinned host buffers, copies inside the timing)
            h_in = torch.from_numpy(ins[lo:hi].view(np.int32)).pin_memory()
            h_out = torch.empty((GA, p.n + 1), dtype=torch.int32).pin_memory()

            def e2e_step():
                d_in[lo:hi].copy_(h_in, non_blocking=True)
                step()
                h_out.copy_(d_out, non_blocking=True)
                torch.cuda.synchronize()

            e2e_step()
            cx.barrier()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                e2e_step()
            dt = time.perf_counter() - t0
            h2d, d2h, api = int(ins.nbytes), int(world * h_out.numel() * 4), \
                "vsp_hom_gate_level_dev (C ABI, NCCL all-gather) + pinned H2D/D2H per rank"
        dt = cx.max_over_ranks(dt)
        e2e = {"value": round(GA * args.steps / dt, 1), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "api": api}
        if world == 1:
            e2e["outputs_decrypt_correct"] = e2e_ok

    if rank != 0:
        eng.close()
        return None

    peak = cx.peak()
    avg_br = br_ms / max(br_n, 1)
    flops = G * p.n * F_EP
    achieved = flops / (avg_br * 1e-3) / 1e12
    roofline = {"bound": "fp64", "kernel": "br1024_kernel (blind rotation)",
                "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4), "traffic": traffic_from_profiles(),
                "peak_source": "measured live: vsp_fp64_peak_probe (DFMA loop) on this GPU",
                "flops_per_launch": flops,
                "flops_rule": "G * n * F_EP, F_EP = (2l+2)*5*M*log2 M + 2l*2*8*M = 171008"}
    # the kernel's other ceiling: shared-memory wavefronts (1 per SM-cycle), 2,080 per
    # external product of one task by design
    sm_clk = float((clk or {}).get("sm_max_mhz") or 1965.0) * 1e6
    import torch as _t
    props = _t.cuda.get_device_properties(local)
    wf_rate = 2080.0 * G * p.n / (avg_br * 1e-3)
    wf_peak = props.multi_processor_count * sm_clk
    roofline["secondary"] = {"bound": "smem", "achieved": round(wf_rate / 1e9, 2),
                             "peak": round(wf_peak / 1e9, 2), "unit": "Gwavefronts/s",
                             "frac": round(wf_rate / wf_peak, 4),
                             "rule": "2,080 shared-memory wavefronts per external product "
                                     "(algorithmic count)"}
    share = {"br1024_ms_per_step": round(br_ms / args.steps, 3),
             "iks_ms_per_step": round(iks_ms / args.steps, 3),
             "gate_prep_ms_per_step": round(prep_ms / args.steps, 3)}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        sample = args.cpu_sample or min(G, max(64 * threads, 512))
        kind = ref_kind(stock=True)
        rate, dt = cpu_reference_rate(kind, args.n, keys, kinds, ins, sample, threads)
        cpu = {"value": round(rate, 2), "unit": UNIT, "cores": threads,
               "kind": "reference" if kind.startswith("ref") else "port",
               "build": STOCK if kind == "ref_stock" else PARITY,
               "sample": f"{sample} of the {G} gates (same keys/ciphertexts), homGate via the "
                         f"reference's parallelFor on {threads} threads, {dt:.1f} s wall"}
        if kind == "ref_stock":
            rate2, dt2 = cpu_reference_rate("ref", args.n, keys, kinds, ins, sample, threads)
            cpu["parity_build"] = {"value": round(rate2, 2), "unit": UNIT, "build": PARITY,
                                   "sample": f"same {sample} gates, {dt2:.1f} s wall"}

    eng.close()
    return {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32+f64",
        "data": "synthetic (seeded client keygen + encryption of uniform random bits)",
        "config": {"workload": f"one level of {GA} random NAND/XOR gates ({G} per GPU), "
                               f"tfhe-80 with n={p.n} (BASELINE.json configs[0])",
                   "gates_per_gpu": G, "n": p.n, "N": p.N1, "l": p.l1, "Bg_bits": p.Bg1Bits,
                   "ks": f"2^{p.ksBaseBits} x {p.ksLen}", "l2": "flushed (512 MiB write) "
                   "between timed steps",
                   "parallelism": (f"level sharded over {world} GPU(s), outputs all-gathered "
                                   + ("through the engine's host-callback exchange over gloo "
                                      "(flow check; ranks may share a GPU)" if cx.gloo else
                                      "over NCCL")) if world > 1 else "1 GPU"},
        "outputs_decrypt_correct": correct,
        "gpu_launches": int(launches),
        "e2e": e2e,
        "roofline": roofline,
        "breakdown": share,
        "cpu_baseline": cpu,
        "clocks": clk,
    }


# --------------------------------------------------------------------------------------
# configs[1]: ROM read + RAM cycle, s/access

def words_to_image(words, v, w):
    img = np.zeros((w << v) // 8, np.uint8)
    for A, x in enumerate(words):
        for j in range(w):
            if (x >> j) & 1:
                b = A * w + j
                img[b // 8] |= 1 << (b % 8)
    return img


def measure_memory(cx: Ctx, steps: int) -> dict | None:
    """BASELINE configs[1]: encrypted ROM read (512 B) + RAM read/write (512 B) with an
    encrypted address; one step = one access of both ports (vsp_mem_ports_dev: the address
    circuit bootstraps of both ports batched, RAM image resident in HBM)."""
    import torch
    import paper_2010_09410_b200 as vsp
    args, world, rank, local = cx.args, cx.world, cx.rank, cx.local
    p = vsp.ParameterSet("tfhe-80", n_override=args.n)
    keys = cx.cb_keys(p)
    rng = np.random.default_rng(77)
    eng = vsp.Engine(p, device=local)
    eng.upload_keys(keys)
    cx.connect(eng)
    v, w = 8, 16
    words = [int(x) for x in rng.integers(0, 1 << w, 1 << v)]
    ram = vsp.encrypt_ram(p, keys, words_to_image(words, v, w), v, w, 5)
    rom_img = rng.integers(0, 256, 512).astype(np.uint8)
    luts = vsp.encrypt_rom(p, keys, rom_img, 6)
    A, blk = int(rng.integers(0, 1 << v)), int(rng.integers(0, 128))
    X = int(rng.integers(0, 1 << w))
    addr = vsp.encrypt(p, keys["lv0"], [(A >> i) & 1 for i in range(v)], 7)
    wflag = vsp.encrypt(p, keys["lv0"], [1], 8)[0]
    wdata = vsp.encrypt(p, keys["lv0"], [(X >> i) & 1 for i in range(w)], 9)
    raddr = vsp.encrypt(p, keys["lv0"], [(blk >> i) & 1 for i in range(7)], 10)
    t32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(cx.dev)
    d_ram, d_addr, d_wf, d_wd = t32(ram), t32(addr), t32(wflag), t32(wdata)
    d_ro = torch.empty((w, p.n + 1), dtype=torch.int32, device=cx.dev)
    d_luts, d_raddr = t32(luts), t32(raddr)
    d_rout = torch.empty((32, p.n + 1), dtype=torch.int32, device=cx.dev)
    stream = torch.cuda.current_stream()

    def access():
        eng.mem_ports_dev(d_luts.data_ptr(), luts.shape[0], 512, d_raddr.data_ptr(), 7,
                          d_rout.data_ptr(), d_ram.data_ptr(), v, w, d_addr.data_ptr(),
                          d_wf.data_ptr(), d_wd.data_ptr(), d_ro.data_ptr(), stream.cuda_stream)

    # first access checked against the plain model (and the reference below)
    access()
    torch.cuda.synchronize()
    ro0 = d_ro.cpu().numpy().view(np.uint32).copy()
    rout0 = d_rout.cpu().numpy().view(np.uint32).copy()
    dec = lambda c: sum(int(b) << i for i, b in enumerate(vsp.decrypt(keys["lv0"], c)))
    correct = dec(ro0) == words[A] and \
        dec(rout0) == int.from_bytes(bytes(rom_img[4 * blk:4 * blk + 4]), "little")
    for _ in range(max(args.warmup - 1, 0)):
        access()
    torch.cuda.synchronize()
    eng.profile_reset()
    eng.counters_reset()
    eng.profile_enable(True)
    launches0 = eng.kernel_launches()
    cx.barrier()
    clocks = ClockSampler(local).start()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        access()
    b.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = eng.kernel_launches() - launches0
    eng.profile_enable(False)
    kernels = {}
    for k in KERNEL_TIMERS:
        ms, cnt = eng.profile_read(k)
        if cnt:
            kernels[k] = round(ms / steps, 3)
    val = cx.max_over_ranks(a.elapsed_time(b) / 1e3 / steps)
    cpa = {k: v_ // max(steps, 1) for k, v_ in eng.counters().items()}
    # e2e: the host API (vsp_ram_cycle + vsp_rom_read), RAM image H2D + D2H every access
    e2e = None
    if not args.no_e2e and world == 1:
        # pinned host buffers (torch's allocator; numpy views, no copies): the RAM image
        # goes in and comes back every access
        def pinned(x):
            return torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).pin_memory().numpy().view(np.uint32)
        ram_h = pinned(ram)
        luts_h, raddr_h = pinned(luts), pinned(raddr)
        addr_h, wflag_h, wdata_h = pinned(addr), pinned(wflag), pinned(wdata)
        eng.mem_ports(luts_h, 512, raddr_h, ram_h, v, w, addr_h, wflag_h, wdata_h)
        t0 = time.perf_counter()
        for _ in range(steps):
            rom_h, ro_h, ram_h = eng.mem_ports(luts_h, 512, raddr_h, ram_h, v, w, addr_h, wflag_h,
                                               wdata_h)
        dt = (time.perf_counter() - t0) / steps
        e2e = {"value": round(dt, 5), "unit": "s/access",
               "h2d_bytes_per_step": int(ram.nbytes + luts.nbytes + (v + w + 1 + 7) * (p.n + 1) * 4),
               "d2h_bytes_per_step": int(ram.nbytes + (w + 32) * (p.n + 1) * 4),
               "api": "vsp_mem_ports host call (romRead + ramCycle, batched address bootstraps; "
                      "pinned host buffers; the 32 MiB encrypted RAM image in and out every "
                      "access, as the reference's EncryptedRam round trip)"}
        e2e["outputs_decrypt_correct"] = bool(
            dec(rom_h) == int.from_bytes(bytes(rom_img[4 * blk:4 * blk + 4]), "little"))
    if rank != 0:
        eng.close()
        return None
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        from oracle.pyoracle import CpuTfhe
        kind = ref_kind(stock=True)
        r = CpuTfhe(kind, "tfhe-80", n_override=args.n, seed=1)
        r.import_keys(keys)
        th = os.cpu_count() or 1
        t0 = time.perf_counter()
        ro_r, _ = r.ram_cycle(ram, v, w, addr, wflag, wdata, threads=th)
        t1 = time.perf_counter()
        rout_r = r.rom_read(luts, 512, raddr, threads=th)
        t2 = time.perf_counter()
        same = bool(np.array_equal(vsp.decrypt(keys["lv0"], ro_r), vsp.decrypt(keys["lv0"], ro0))
                    and np.array_equal(vsp.decrypt(keys["lv0"], rout_r),
                                       vsp.decrypt(keys["lv0"], rout0)))
        cpu = {"value": round(t2 - t0, 3), "unit": "s/access", "cores": th, "kind": "reference",
               "build": STOCK if kind == "ref_stock" else PARITY,
               "sample": f"one ramCycle (v=8,w=16) {t1 - t0:.2f}s + one romRead(512B) "
                         f"{t2 - t1:.2f}s via the reference with {th} threads, same keys "
                         "and ciphertexts",
               "decrypted_outputs_equal_ours": same}
    eng.close()
    return {
        "metric": "cmux_memory_seconds_per_access", "value": round(val, 5), "unit": "s/access",
        "n_gpus": world, "steps": steps, "warmup": args.warmup, "higher_is_better": False,
        "config": {"workload": "BASELINE configs[1]: ROM read 512 B (7 addr bits) + RAM cycle "
                               "v=8 w=16 (512 B), encrypted address, tfhe-80 n=%d" % p.n,
                   "ram": "device-resident (HBM) across accesses",
                   "parallelism": "RAM bit-blocks sharded over the ranks" if world > 1
                   else "1 GPU"},
        "timing": "CUDA events around `steps` back-to-back vsp_mem_ports_dev calls (ROM read + "
                  "RAM cycle, batched address bootstraps), max over ranks",
        "outputs_decrypt_correct": bool(correct),
        "gpu_launches": int(launches),
        "kernel_ms_per_access": kernels,
        "counters_per_access": cpa,
        "roofline": work_roofline(cpa, p.n, val, cx.peak()),
        "e2e": e2e, "cpu_baseline": cpu, "clocks": clk,
        "keygen_s": round(getattr(cx, "cb_keygen_s", 0.0), 2)}


# --------------------------------------------------------------------------------------
# configs[2]: one clock cycle of the synthetic Ruby-shaped netlist, s/cycle

def measure_cycle(cx: Ctx, steps: int) -> dict | None:
    """BASELINE configs[2]: seconds per clock cycle of a seeded synthetic Ruby-shaped
    pipelined-processor netlist (gate mix of PAPER.md:1376-1385, one ROM + one RAM port).
    The first cycle is checked against the reference's own Evaluator<TfheBackend> run from
    the same state (decrypted DFF state and outputs)."""
    import torch
    import paper_2010_09410_b200 as vsp
    from paper_2010_09410_b200 import netlist as N
    args, world, rank, local = cx.args, cx.world, cx.rank, cx.local
    p = vsp.ParameterSet("tfhe-80", n_override=args.n)
    keys = cx.cb_keys(p)
    rng = np.random.default_rng(99)
    eng = vsp.Engine(p, device=local)
    eng.upload_keys(keys)
    cx.connect(eng)  # every level's gates sharded across the ranks + all-gathered
    nl = N.synthetic_netlist(seed=1, levels=args.levels)
    ev = N.Evaluator(nl, eng)
    v, w = 8, 16
    ram = vsp.encrypt_ram(p, keys, rng.integers(0, 256, (w << v) // 8).astype(np.uint8), v, w, 3)
    luts = vsp.encrypt_rom(p, keys, rng.integers(0, 256, 512).astype(np.uint8), 4)
    dff0 = vsp.encrypt(p, keys["lv0"], rng.integers(0, 2, ev.n_dffs), 5)
    ins = vsp.encrypt(p, keys["lv0"], rng.integers(0, 2, len(nl.inputs[0].bits)), 6)
    ev.set_ram(ram, v, w)
    ev.set_rom(luts, 512)
    ev.set_dff_state_raw(dff0)
    for i, ct in enumerate(ins):
        ev.set_input("in", i, ct)
    ev.run(1)
    dff1 = ev.dff_state()
    outs1 = np.stack([ev.output("out", j) for j in range(len(nl.outputs[0].bits))])
    # warm-up: the first cycles run eagerly, then the runner captures the cycle as a CUDA
    # graph (one GPU) and replays it
    ev.run(max(args.warmup - 1, 2))
    eng.synchronize()
    eng.counters_reset()
    launches0 = eng.kernel_launches()
    cx.barrier()
    clocks = ClockSampler(local).start()
    stats = []
    ev.run(steps, N.RunOptions(stats=stats))
    eng.synchronize()
    clk = clocks.stop()
    launches = eng.kernel_launches() - launches0
    secs = cx.max_over_ranks(float(np.mean([s.seconds for s in stats])))
    cpc = {k: v_ // max(steps, 1) for k, v_ in eng.counters().items()}  # timed cycles only
    # per-kernel breakdown from separate cycles with CUDA-event timing around every launch
    # (profiling runs the cycle eagerly, not as the graph; not part of the timed value)
    prof_steps = min(steps, 3)
    eng.profile_reset()
    eng.profile_enable(True)
    ev.run(prof_steps)
    eng.synchronize()
    eng.profile_enable(False)
    kernels = {k: round(eng.profile_read(k)[0] / prof_steps, 3) for k in KERNEL_TIMERS}
    # e2e through the Evaluator API: every cycle sets the 8 input TLWEs from host memory
    # and reads the 16 output TLWEs back
    e2e = None
    if not args.no_e2e:
        nin, nout = len(nl.inputs[0].bits), len(nl.outputs[0].bits)
        cx.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            for i in range(nin):
                ev.set_input("in", i, ins[i])
            ev.run(1)
            for j in range(nout):
                ev.output("out", j)
        dt = cx.max_over_ranks((time.perf_counter() - t0) / steps)
        e2e = {"value": round(dt, 5), "unit": "s/cycle",
               "h2d_bytes_per_step": nin * (p.n + 1) * 4, "d2h_bytes_per_step": nout * (p.n + 1) * 4,
               "api": "Evaluator.set_input + run(1) + output (vsp_netlist_* C ABI)"}
    if rank != 0:
        ev.close()
        eng.close()
        return None
    st = N.netlist_stats(nl)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cycle_cpu_baseline(p, keys, nl, ram, v, w, luts, dff0, ins, dff1, outs1)
    ev.close()
    eng.close()
    return {
        "metric": "seconds_per_clock_cycle", "value": round(secs, 5),
        "unit": "s/cycle", "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "higher_is_better": False,
        "config": {"workload": "BASELINE configs[2] proxy: synthetic Ruby-shaped netlist "
                               "(no processor netlist exists in the reference)",
                   "gates": sum(st["count_by_kind"][k] for k in N.GATES),
                   "dffs": st["dff_count"], "depth": st["depth"], "gmax": st["gmax"],
                   "rom": "512 B, 7 addr bits", "ram": "v=8 w=16", "n": p.n,
                   "parallelism": f"levels sharded over {world} GPUs" if world > 1 else "1 GPU"},
        "gpu_launches": int(launches),
        "counters_per_cycle": cpc,
        "roofline": work_roofline(cpc, p.n, secs, cx.peak()),
        "kernel_ms_per_cycle": kernels, "e2e": e2e, "cpu_baseline": cpu, "clocks": clk,
        "timing": "CUDA events around each device-resident cycle, replayed as a CUDA graph on "
                  "one GPU (mean, max over ranks); kernel_ms_per_cycle from 3 separate "
                  "event-timed eager cycles"}


def cycle_cpu_baseline(p, keys, nl, ram, v, w, luts, dff0, ins, dff1, outs1):
    """One cycle of the reference's own Evaluator<TfheBackend> (oracle/_ref, patched
    engine.hpp) on the same netlist, keys and state, on all host cores; its decrypted DFF
    state and outputs must equal the engine's first cycle."""
    import ctypes
    import paper_2010_09410_b200 as vsp
    from oracle.pyoracle import CpuTfhe
    from paper_2010_09410_b200 import netlist as N
    kind = ref_kind(stock=True)
    if not kind.startswith("ref"):
        return None
    th = os.cpu_count() or 1
    r = CpuTfhe(kind, "tfhe-80", n_override=p.n, seed=1)
    r.import_keys(keys)
    L = r.L
    h = ctypes.c_void_p(L.ref_eval_new(r.h, N.netlist_to_json(nl).encode(), th))
    vp = ctypes.c_void_p
    ram = np.ascontiguousarray(ram)
    luts = np.ascontiguousarray(luts)
    dff0 = np.ascontiguousarray(dff0)
    L.ref_eval_set_ram(h, v, w, ram.ctypes.data_as(vp), p.N1)
    L.ref_eval_set_rom(h, 512, luts.ctypes.data_as(vp), luts.shape[0], p.N1)
    L.ref_eval_set_dff(h, dff0.ctypes.data_as(vp), ctypes.c_uint32(p.n))
    for i, ct in enumerate(ins):
        L.ref_eval_set_input(h, b"in", i, np.ascontiguousarray(ct).ctypes.data, p.n)
    t0 = time.perf_counter()
    rc = L.ref_eval_run(h, 1, th, 0, None)
    dt = time.perf_counter() - t0
    same = None
    if rc == 0:
        dref = np.zeros_like(dff1)
        L.ref_eval_get_dff(h, dref.ctypes.data_as(vp), ctypes.c_uint32(p.n))
        oref = np.zeros_like(outs1)
        for j in range(outs1.shape[0]):
            o = np.zeros(p.n + 1, np.uint32)
            L.ref_eval_output(h, b"out", j, o.ctypes.data)
            oref[j] = o
        dec = lambda x: vsp.decrypt(keys["lv0"], x)
        same = bool(np.array_equal(dec(dref), dec(dff1)) and np.array_equal(dec(oref), dec(outs1)))
    L.ref_eval_free(h)
    if rc:
        return None
    return {"value": round(dt, 3), "unit": "s/cycle", "cores": th, "kind": "reference",
            "build": STOCK if kind == "ref_stock" else PARITY,
            "sample": f"one cycle of hvp::netlist::Evaluator<TfheBackend> (reference, "
                      f"{th} workers) on the same netlist, keys and state",
            "decrypted_dff_and_outputs_equal_ours": same}


# --------------------------------------------------------------------------------------
# reference arm

def run_reference(args, world, rank, local):
    """The reference's own CPU implementation of the path (oracle/_ref built from the
    reference sources with its stock Release flags) on the host cores, same metric/config,
    bounded samples."""
    if rank != 0:
        return
    from oracle.pyoracle import CpuTfhe, GATE_KINDS, available
    if not available("ref"):
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libhvpref.so not built (needs /root/reference at build)"}))
        return
    kind = ref_kind(stock=True)
    threads = os.cpu_count() or 1
    sample = args.cpu_sample or max(16 * threads, 128)
    r = CpuTfhe(kind, "tfhe-80", n_override=args.n, seed=1000)
    r.keygen(False)  # the reference's own BootstrappingKey::generate
    rng = np.random.default_rng(1000)
    kinds = np.array([GATE_KINDS.index(("NAND", "XOR")[int(x)]) for x in
                      rng.integers(0, 2, sample)], np.int32)
    ins = np.zeros((sample, 3, r.n + 1), np.uint32)
    for g in range(sample):
        ins[g, 0] = r.encrypt(int(rng.integers(0, 2)))
        ins[g, 1] = r.encrypt(int(rng.integers(0, 2)))
    for _ in range(args.warmup):
        r.hom_gate_batch(kinds[:threads], ins[:threads], threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r.hom_gate_batch(kinds, ins, threads=threads)
        times.append(time.perf_counter() - t0)
    value = sample * args.steps / sum(times)
    build = STOCK if kind == "ref_stock" else PARITY
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(times) / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32+f64",
        "data": "synthetic (reference keygen + encryption of uniform random bits)",
        "config": {"workload": f"{args.gates} random NAND/XOR gates, tfhe-80 with n={args.n} "
                               "(BASELINE.json configs[0]); each step times a bounded sample",
                   "gates_per_step_sample": sample, "n": args.n, "build": build},
        "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": threads,
                         "kind": "reference", "build": build,
                         "sample": f"{sample} gates per step, homGate via parallelFor"},
        "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world, rank, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, world, rank, local)
        return
    cx = Ctx(args, world, rank, local)
    sub = args.sub_steps or args.steps
    if args.config == "memory":
        line = measure_memory(cx, args.steps)
    elif args.config == "cycle":
        line = measure_cycle(cx, args.steps)
    else:
        line = measure_gates(cx)
        if not args.headline_only:
            mem = measure_memory(cx, sub)
            cyc = measure_cycle(cx, sub)
            if line is not None:
                line["memory"] = mem
                line["cycle"] = cyc
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if cx.dist:
        cx.dist.destroy_process_group()


if __name__ == "__main__":
    main()
