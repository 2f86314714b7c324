/*
 * vsp_b200.h — C ABI of the B200-native VSP hot-path engine (libvsp_b200.so).
 *
 * Drop-in boundary for the reference's gate-evaluation / CMUX-memory / netlist-runner
 * path (hvp, /root/reference/proj).  The reference exposes C++ only;
 * every entry point below names the reference interface it replaces (file:line).
 * Plain pointers and sizes only.  All functions return 0 on success and a nonzero
 * status otherwise; vsp_last_error() gives the message.  Status codes mirror the
 * reference's exception types so the C++/Python facades rethrow the same kind:
 *   VSP_EINVAL  std::invalid_argument   (arity, geometry, parameters)
 *   VSP_ERANGE  std::out_of_range       (sample-extract index)
 *   VSP_ERUNTIME std::runtime_error     (missing key material, CUDA failure, ...)
 *
 * Flat layouts (little-endian u32 torus words, identical to the reference vectors):
 *   TLWE  level 0 : (n+1)  u32   a[0..n) then b          (ciphertext.hpp:14-28)
 *   TLWE  level 1 : (N1+1) u32
 *   TRLWE         : 2*N1 u32     a[0..N1) then b[0..N1)  (ciphertext.hpp:34-53)
 *   TRGSW         : 2*l1 TRLWE rows                      (ciphertext.hpp:60-64)
 *   bk1           : n x TRGSW                            (BootstrappingKey::bk1Raw, ops.hpp:98)
 *   bk2           : n x 2*l2 x 2 x N2 u64                (BootstrappingKey::bk2Raw, ops.hpp:102)
 *   ksk           : N1 x ksLen x (2^ksBaseBits-1) x (n+1) u32     (KeySwitchKey, ops.hpp:18-29)
 *   pks           : (N2+1) x pksLen x (2^pksBaseBits-1) x 2*N1 u32 (PrivKeySwitchKey, ops.hpp:32-42)
 *   RAM           : w*2^v TRLWE cells, cells[j*2^v + A]  (EncryptedRam, mem.hpp:32-46)
 *   ROM           : 2^highBits TRLWE LUTs                (EncryptedRom, mem.hpp:48-61)
 * Gate kinds use hvp::tfhe::GateKind order (ops.hpp:183-194):
 *   0 AND, 1 ANDNOT, 2 MUX, 3 NAND, 4 NOR, 5 NOT, 6 OR, 7 ORNOT, 8 XNOR, 9 XOR.
 */
#ifndef VSP_B200_H
#define VSP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VSP_OK 0
#define VSP_EINVAL 1
#define VSP_ERANGE 2
#define VSP_ERUNTIME 3

typedef struct vsp_ctx vsp_ctx;

/* hvp::tfhe::ParameterSet (params.hpp:23-66), integer fields. */
typedef struct vsp_params {
    uint32_t n, N1, l1, Bg1Bits, N2, l2, Bg2Bits, ksBaseBits, ksLen, pksBaseBits, pksLen;
    int32_t fft; /* MulBackend: 1 = Fft, 0 = Exact */
} vsp_params;

/* ParameterSet::byName (params.cpp:88-95) + ParameterSet::validate (params.cpp:17-29).
 * n_override > 0 replaces n (BASELINE's n=630 copy of tfhe-80). */
int vsp_params_by_name(const char* name, uint32_t n_override, vsp_params* out);

const char* vsp_last_error(void);

/* Engine context on one CUDA device.  Replaces the implicit global state of the
 * reference (thread-local FFT plans fft.cpp:79-85, scratch ops.cpp:20-33). */
vsp_ctx* vsp_create(const vsp_params* params, int device);
void vsp_destroy(vsp_ctx* ctx);

/* BootstrappingKey::fromParts + prepareAll (ops.cpp:387-415): upload raw key
 * material once and transform it on the device.  bk2/pks may be NULL when
 * has_cb == 0 (key without circuit-bootstrapping material, ops.cpp:417-423); has_cb == 2
 * uploads bk2 without the private key-switching tables (level-2 blind rotation only). */
int vsp_upload_keys(vsp_ctx* ctx, const uint32_t* bk1, const uint32_t* ksk,
                    const uint64_t* bk2, const uint32_t* pks_negs, const uint32_t* pks_id,
                    int has_cb);

/* deserializeBootstrappingKey (serialize.cpp:209-230) + upload: the reference's "HVP1"
 * key file (tag 2) as produced by serializeBootstrappingKey, checked against the
 * context's parameters (VSP_ERUNTIME with the reference's messages on mismatch). */
int vsp_upload_keys_hvp1(vsp_ctx* ctx, const uint8_t* bytes, size_t len);

/* HVP1 ciphertext containers (serialize.cpp:240-245, mem.cpp:340-403): TLWE (tag 3),
 * TRLWE (4), RAM (6), ROM (7) flattened to the layouts above.  out == NULL returns the
 * size in *words; meta = {tag, count, v, w, depthBytes}. */
int vsp_read_hvp1(vsp_ctx* ctx, const uint8_t* bytes, size_t len, uint32_t* out, size_t cap,
                  size_t* words, uint32_t meta[5]);

/* homGate (ops.cpp:839-896) over a batch of independent gates, host buffers.
 * kinds[G]; in[G x 3 x (n+1)] (unused operand slots ignored; MUX = {sel, a, b});
 * out[G x (n+1)].  Equivalent to G calls of homGate. */
int vsp_hom_gate_batch(vsp_ctx* ctx, const int32_t* kinds, const uint32_t* in,
                       uint32_t* out, size_t G);

/* Same with device-resident ciphertexts, enqueued on `stream` (a cudaStream_t; 0 is
 * the legacy default stream); kinds stay in host memory.  Asynchronous. */
int vsp_hom_gate_batch_dev(vsp_ctx* ctx, const int32_t* kinds, const uint32_t* d_in,
                           uint32_t* d_out, size_t G, void* stream);

/* bootstrapToTrlwe (ops.cpp:750-757) for G level-0 TLWEs -> G TRLWEs (host). */
int vsp_bootstrap_to_trlwe_batch(vsp_ctx* ctx, const uint32_t* in, uint32_t* out, size_t G);

/* gateBootstrap (ops.cpp:759-762) batch (host). */
int vsp_gate_bootstrap_batch(vsp_ctx* ctx, const uint32_t* in, uint32_t* out, size_t G);

/* identityKeySwitch (ops.cpp:651-679): G level-1 TLWEs -> G level-0 TLWEs (host). */
int vsp_identity_key_switch_batch(vsp_ctx* ctx, const uint32_t* in, uint32_t* out, size_t G);

/* ---- circuit bootstrapping and CMUX memory (host buffers) ---------------------- */

/* circuitBootstrap (ops.cpp:914-935): C level-0 TLWEs -> C TRGSWs (level 1).
 * Requires a key uploaded with has_cb = 1 (otherwise VSP_ERUNTIME, ops.cpp:417-423). */
int vsp_circuit_bootstrap_batch(vsp_ctx* ctx, const uint32_t* in, uint32_t* out, size_t C);

/* cmux (ops.cpp:606-626, convenience form that prepares the selector per call):
 * out[g] = c0[g] + ExtProd(c1[g] - c0[g], sel[g]); sel: G raw TRGSWs. */
int vsp_cmux_batch(vsp_ctx* ctx, const uint32_t* sel, const uint32_t* c1, const uint32_t* c0,
                   uint32_t* out, size_t G);

/* homMuxNoSeIks (ops.cpp:898-909): G x (sel, a, b) level-0 TLWEs -> G TRLWEs. */
int vsp_hom_mux_no_se_iks_batch(vsp_ctx* ctx, const uint32_t* sel, const uint32_t* a,
                                const uint32_t* b, uint32_t* out, size_t G);

/* mem::ramCycle (mem.cpp:122-135): read-before-write single-port cycle.
 * ram: w*2^v TRLWE cells, updated in place; addr: v TLWEs (LSB first); wflag: 1 TLWE;
 * wdata: w TLWEs; readout: w TLWEs (the pre-write word). */
int vsp_ram_cycle(vsp_ctx* ctx, uint32_t v, uint32_t w, uint32_t* ram, const uint32_t* addr,
                  const uint32_t* wflag, const uint32_t* wdata, uint32_t* readout);

/* addressToTrgsw + prepareAddress + mem::romRead (engine.cpp:133-143, mem.cpp:137-177):
 * luts: nluts TRLWEs of an EncryptedRom of depth_bytes; addr: vrom TLWEs; out: 32 TLWEs. */
int vsp_rom_read(vsp_ctx* ctx, uint32_t depth_bytes, const uint32_t* luts, uint32_t nluts,
                 const uint32_t* addr, uint32_t vrom, uint32_t* out);

/* The units of a RAM cycle and the ROM read on given address selectors (RamAddress: one
 * raw TRGSW per address bit, LSB first, e.g. circuit-bootstrapped or client-encrypted);
 * each prepares the selectors like prepareAddress (mem.cpp:21-36).
 *   vsp_ram_read_unit    mem::ramReadUnit   (mem.cpp:49-72):  out = w TRLWEs
 *   vsp_ram_control_unit mem::ramControlUnit (mem.cpp:74-90): read = w TRLWEs ->
 *                        readout (w TLWEs), controlled (w TRLWEs)
 *   vsp_ram_write_unit   mem::ramWriteUnit  (mem.cpp:92-120): ram updated in place
 *   vsp_rom_read_sel     mem::romRead       (mem.cpp:137-177): 32 TLWEs */
int vsp_ram_read_unit(vsp_ctx* ctx, uint32_t v, uint32_t w, const uint32_t* ram,
                      const uint32_t* sel, uint32_t* out);
int vsp_ram_control_unit(vsp_ctx* ctx, uint32_t w, const uint32_t* read, const uint32_t* wflag,
                         const uint32_t* wdata, uint32_t* readout, uint32_t* controlled);
int vsp_ram_write_unit(vsp_ctx* ctx, uint32_t v, uint32_t w, uint32_t* ram, const uint32_t* sel,
                       const uint32_t* controlled);
int vsp_rom_read_sel(vsp_ctx* ctx, uint32_t depth_bytes, const uint32_t* luts, uint32_t nluts,
                     const uint32_t* sel, uint32_t vrom, uint32_t* out);

/* Device-resident ramCycle / romRead (same arguments as device pointers, asynchronous on
 * `stream`, a cudaStream_t): the RAM image stays in HBM across cycles, as in the netlist
 * runner.  Replace the same reference calls (mem.cpp:122-135, :137-177). */
int vsp_ram_cycle_dev(vsp_ctx* ctx, uint32_t v, uint32_t w, uint32_t* d_ram,
                      const uint32_t* d_addr, const uint32_t* d_wflag, const uint32_t* d_wdata,
                      uint32_t* d_readout, void* stream);
int vsp_rom_read_dev(vsp_ctx* ctx, uint32_t depth_bytes, const uint32_t* d_luts, uint32_t nluts,
                     const uint32_t* d_addr, uint32_t vrom, uint32_t* d_out, void* stream);

/* One access of a ROM port and a RAM port together, as the processor issues them each
 * cycle (the netlist runner's path for two ports in one level, Evaluator::evaluateCycle
 * engine.hpp:263-351 with engine.cpp:133-148): both ports' address circuit bootstraps run
 * as one batch, then romRead and ramCycle proceed; results equal the separate calls. */
int vsp_mem_ports_dev(vsp_ctx* ctx, uint32_t depth_bytes, const uint32_t* d_luts, uint32_t nluts,
                      const uint32_t* d_rom_addr, uint32_t vrom, uint32_t* d_rom_out,
                      uint32_t v, uint32_t w, uint32_t* d_ram, const uint32_t* d_ram_addr,
                      const uint32_t* d_wflag, const uint32_t* d_wdata, uint32_t* d_readout,
                      void* stream);

/* The same access with HOST buffers (the drop-in form of one memory stage: romRead +
 * ramCycle, mem.cpp:122-177, engine.cpp:133-148): luts (nluts x 2 N1) and both ports'
 * ciphertexts in, rom_out (32 x (n+1)) and readout (w x (n+1)) out, and the RAM image
 * (w 2^v x 2 N1) in AND out, updated in place like the reference's EncryptedRam&.  Pinned
 * host buffers (cudaHostAlloc / cudaHostRegister) make the copies run at link speed. */
int vsp_mem_ports(vsp_ctx* ctx, uint32_t depth_bytes, const uint32_t* luts, uint32_t nluts,
                  const uint32_t* rom_addr, uint32_t vrom, uint32_t* rom_out, uint32_t v,
                  uint32_t w, uint32_t* ram, const uint32_t* ram_addr, const uint32_t* wflag,
                  const uint32_t* wdata, uint32_t* readout);

/* blindRotate<uint64_t> (ops.cpp:713-742) with test vector (0, h[t]/2 ...): T level-0
 * TLWEs -> T level-2 TRLWE accumulators (2 x N2 u64).  Exposed for parity tests of the
 * circuit-bootstrapping inner loop. */
int vsp_blind_rotate_lvl2_batch(vsp_ctx* ctx, const uint32_t* in, const uint64_t* h,
                                uint64_t* out, size_t T);

/* ---- netlist runner (hvp::netlist::Evaluator<TfheBackend>, engine.hpp:107-405) ------
 * The netlist is uploaded as flat arrays (Netlist, netlist.hpp:44-63): cell kinds in
 * hvp::netlist::CellKind order (0..9 gates as GateKind, 10 DFF, 11 ROM, 12 RAM,
 * 13 CONST0, 14 CONST1), cell ids, CSR lists of input / output nets per cell (pin order
 * of netlist.hpp:38-43), and the nets driven by module input ports.  The DAG is built
 * and levelled exactly as buildDag (netlist.cpp:348-432); each cycle evaluates it one
 * ASAP level per batched launch and then latches the DFFs (engine.hpp:263-351).  Value
 * table, DFF state, ROM and RAM stay device-resident. */
typedef struct vsp_netlist vsp_netlist;

vsp_netlist* vsp_netlist_create(vsp_ctx* ctx, int32_t net_count, int32_t cells,
                                const int32_t* kinds, const int32_t* ids, const int32_t* in_off,
                                const int32_t* in_nets, const int32_t* out_off,
                                const int32_t* out_nets, const int32_t* input_nets,
                                int32_t n_inputs);
void vsp_netlist_destroy(vsp_netlist* nl);
/* out6: dag nodes, dffs, gMax, depth, rom cell, ram cell; levels[dag node] optional. */
int vsp_netlist_info(vsp_netlist* nl, int32_t* out6, int32_t* levels);
/* The level each DAG node is EVALUATED in (same order as vsp_netlist_info's levels): the
 * ASAP level, except gates with slack moved one level later out of a level that holds
 * more blind-rotation tasks than the device has SMs (a 149-task level would cost two
 * latency waves).  Results are unchanged: every gate still runs after all its producers
 * and before all its consumers.  No reference counterpart (scheduling only). */
int vsp_netlist_launch_levels(vsp_netlist* nl, int32_t* levels);
/* The same schedule without a device (host only): validates the flat netlist like
 * vsp_netlist_create and returns, per DAG node, the ASAP level (buildDag, netlist.cpp:348-432)
 * and the launch level for a device with `sms` SMs, plus the depth. */
int vsp_netlist_schedule(int32_t net_count, int32_t cells, const int32_t* kinds, const int32_t* ids,
                         const int32_t* in_off, const int32_t* in_nets, const int32_t* out_off,
                         const int32_t* out_nets, const int32_t* input_nets, int32_t n_inputs,
                         int32_t sms, int32_t* asap_levels, int32_t* launch_levels,
                         int32_t* depth);
/* Evaluator::setInput (engine.hpp:160-163) by index into input_nets. */
int vsp_netlist_set_input(vsp_netlist* nl, int32_t input_index, const uint32_t* tlwe);
/* Evaluator::output (engine.hpp:165-176) for any net. */
int vsp_netlist_get_net(vsp_netlist* nl, int32_t net, uint32_t* tlwe);
/* dffState / setDffStateRaw (engine.hpp:185-194); either pointer may be NULL. */
int vsp_netlist_dff(vsp_netlist* nl, uint32_t* get, const uint32_t* set);
/* setRom / setRam / ram (engine.hpp:204-221). */
int vsp_netlist_set_rom(vsp_netlist* nl, uint32_t depth_bytes, const uint32_t* luts,
                        uint32_t nluts);
int vsp_netlist_ram(vsp_netlist* nl, uint32_t v, uint32_t w, uint32_t* get, const uint32_t* set);
/* Evaluator::run (engine.hpp:238-247); stats: 4 doubles per cycle (evaluated cells,
 * gMax, depth, seconds) or NULL. */
int vsp_netlist_run(vsp_netlist* nl, uint64_t cycles, double* stats);
uint64_t vsp_netlist_cycle(vsp_netlist* nl);
/* Geometry (v, w) of the bound RAM image (Evaluator::ram().enc.geom). */
int vsp_netlist_ram_geometry(vsp_netlist* nl, uint32_t* v, uint32_t* w);
/* Netlist::name (netlist.hpp:58), recorded in snapshots. */
int vsp_netlist_set_name(vsp_netlist* nl, const char* name);
/* snapshotSave / snapshotLoad / snapshotPeek (snapshot.hpp:17-33, snapshot.cpp:84-176):
 * the reference's "HVPS" byte format, so snapshots move between this runner and
 * hvp::netlist::Evaluator<TfheBackend> in both directions.  param_name is the parameter
 * set's name (ParameterSet::name) written/checked in the header.  save: out == NULL
 * returns the size in *len.  load errors are VSP_ERUNTIME with the reference's text
 * (magic, version, backend, parameter set, netlist name/hash, truncated input). */
int vsp_netlist_snapshot_save(vsp_netlist* nl, const char* param_name, uint8_t* out,
                              size_t cap, size_t* len);
int vsp_netlist_snapshot_load(vsp_netlist* nl, const char* param_name, const uint8_t* in,
                              size_t len);
int vsp_snapshot_peek(const uint8_t* in, size_t len, char* backend, char* param,
                      char* netlist, size_t cap);
int vsp_netlist_set_cycle(vsp_netlist* nl, uint64_t cycle);

/* ---- multi-GPU --------------------------------------------------------
 * One process per GPU.  Rank 0 creates an NCCL unique id, the host distributes it (e.g.
 * torch.distributed broadcast), every rank attaches its context.  Afterwards the
 * netlist runner shards each level's gates across the ranks (contiguous slices of equal
 * blind-rotation task count) and all-gathers the output TLWEs over NVLink; keys stay
 * replicated.  A RAM port is sharded by bit-block: rank r owns blocks
 * [r w/world, (r+1) w/world) (read trees, control bits, write bars) and the read-out TLWEs
 * are all-gathered; ramCycle / mem_ports on device buffers then update only the owned
 * blocks of the RAM image (the host ramCycle, the runner's RAM getter and snapshots
 * gather the whole image).  Circuit bootstraps and the ROM run redundantly on every rank.
 * The reference has no distributed path (parallelFor on host threads only). */
int vsp_nccl_unique_id(uint8_t out[128]);
int vsp_attach_comm(vsp_ctx* ctx, const uint8_t id[128], int rank, int world);
/* Host-callback exchange instead of NCCL (e.g. torch.distributed over gloo / TCP, or the
 * tests' two processes on one GPU): allgather(send, recv, bytes, user) must fill
 * recv[r * bytes ...] with rank r's `bytes` for every rank r (host buffers) and return 0.
 * The engine stages its slice in pinned host memory around each call. */
int vsp_attach_exchange(vsp_ctx* ctx, int rank, int world,
                        int (*allgather)(const void* send, void* recv, size_t bytes, void* user),
                        void* user);
/* The slice [lo, hi) of a G-gate level owned by `rank`: slices hold equal numbers of
 * blind-rotation TASKS (MUX = 2, NOT = 0, others 1); per = the largest slice (the
 * all-gather's per-rank count).  kinds == NULL: all gates one task each. */
int vsp_level_partition(size_t G, int world, int rank, size_t* lo, size_t* hi, size_t* per);
int vsp_level_partition_kinds(const int32_t* kinds, size_t G, int world, int rank, size_t* lo,
                              size_t* hi, size_t* per);
/* homGate over one whole level, sharded across the attached ranks: every rank passes
 * all G gates' inputs (device) and receives all G outputs (device) on `stream`. */
int vsp_hom_gate_level_dev(vsp_ctx* ctx, const int32_t* kinds, const uint32_t* d_in,
                           uint32_t* d_out, size_t G, void* stream);

/* OpCounters (counters.hpp:11-28): cmux, blindRotate, identityKeySwitch,
 * privateKeySwitch, circuitBootstrap — counted per batched operation exactly as
 * the reference increments them per call. */
int vsp_counters(vsp_ctx* ctx, uint64_t out[5]);
int vsp_counters_reset(vsp_ctx* ctx);

/* Number of engine kernel launches issued so far (evidence for bench.py). */
uint64_t vsp_kernel_launches(vsp_ctx* ctx);

int vsp_synchronize(vsp_ctx* ctx);

/* Optional per-kernel CUDA-event timing on the launching stream (bench.py's live
 * roofline): enable, then read the accumulated time/count of a kernel by name
 * ("br1024", "br_exact", "iks", "gate_prep", ...). */
int vsp_profile_enable(vsp_ctx* ctx, int on);
int vsp_profile_read(vsp_ctx* ctx, const char* name, double* total_ms, uint64_t* count);
int vsp_profile_reset(vsp_ctx* ctx);

/* Launch plan the engine picks for a level-1 blind rotation of `tasks` tasks (FFT path;
 * test-det runs the exact kernel): out = {narrow-level latency kernel (1/0), tasks in
 * whole 8-task-per-SM waves, tasks per SM of the remainder / single launch (0 = none),
 * its kernel (0 none, 1 br1024, 2 br1024p two warps per task, 3 br_lat)}.  Lets the tests
 * assert which wave boundaries a batch really crosses.  No reference counterpart. */
int vsp_br_plan(vsp_ctx* ctx, size_t tasks, int32_t out[4]);
/* Streaming multiprocessors of the context's device (sizes every launch plan). */
int vsp_sm_count(vsp_ctx* ctx);
/* Engine tuning options (no reference counterpart; results are bit-identical either way):
 *   "lat_tasks" 1|2: blind-rotation tasks per SM of narrow levels (br_lat / br_lat2);
 *   "ram_overlap" 0|1: the netlist runner's deferred RAM write unit;
 *   "iks_gemm" 0|1: identity key switching as an INT8 tensor-core GEMM (default 1);
 *   "br_pair" 0|1: partial blind-rotation waves with two warps per task (default 1);
 *   "iks_split" k: split-K factor of the key-switch GEMM, k divides 24,576 into multiples
 *      of 16 (0 = automatic: 4 up to 512 key switches, else 2);
 *   "backfill" 0|1: the netlist runner's write-bar backfill (default 1);
 *   "graph" 0|1: the runner replays each clock cycle as a CUDA graph (one GPU, captured
 *      after one eager cycle, recaptured when buffers, options, keys or the ROM / RAM
 *      geometry change; default 1). */
int vsp_set_option(vsp_ctx* ctx, const char* name, int64_t value);
/* Reads an option back, or the statistic "bars_backfilled" (write-bar blind rotations the
 * runner has run inside narrow levels since the context was created). */
int vsp_get_option(vsp_ctx* ctx, const char* name, int64_t* value);

/* Measured dense FP64 FMA throughput of `device` in TFLOP/s (the denominator of the
 * blind-rotation roofline; MEASURED_PEAKS.json carries no FP64 figure). */
int vsp_fp64_peak_probe(int device, double* tflops);

/* ---- client side (Alice): key generation / encryption / decryption -------------
 * Not on the evaluation hot path; provided so the engine can be driven without the
 * reference.  Same CSPRNG stream and draw order as the reference client code. */

const char* vsp_client_last_error(void);

/* genSecretKey + BootstrappingKey::generate (ops.cpp:264-385) from
 * Csprng::fromSeed(seed) (rng.cpp:81-91).  bk2/pks_* only written when with_cb. */
int vsp_client_keygen(const vsp_params* params, uint64_t seed, int with_cb, uint32_t* lv0,
                      uint32_t* lv1, uint32_t* lv2, uint32_t* bk1, uint32_t* ksk,
                      uint64_t* bk2, uint32_t* pks_negs, uint32_t* pks_id);

/* Same keys, bit for bit, with the b = a*s products of every TRLWE-of-zero encryption
 * (bk1, bk2 and the 2 x 143,430 private key-switching rows: ~3e11 torus adds at tfhe-80)
 * computed on CUDA device `device`; the CSPRNG draws stay on the host in reference order.
 * (client key generation, ops.cpp:264-385.) */
int vsp_client_keygen_dev(const vsp_params* params, uint64_t seed, int with_cb, int device,
                          uint32_t* lv0, uint32_t* lv1, uint32_t* lv2, uint32_t* bk1,
                          uint32_t* ksk, uint64_t* bk2, uint32_t* pks_negs, uint32_t* pks_id);

/* tlweEncrypt (ops.cpp:428-440) of count bits, one CSPRNG stream from seed. */
int vsp_client_tlwe_encrypt(const vsp_params* params, const uint32_t* lv0, uint64_t seed,
                            const uint8_t* bits, size_t count, uint32_t* out);

/* trlweEncrypt (ops.cpp:458-468) of count N1-bit polynomials (alpha1 noise): the cells
 * of encryptRam / LUTs of encryptRom (mem.cpp:202-263).  out: count x 2*N1. */
int vsp_client_trlwe_encrypt(const vsp_params* params, const uint32_t* lv1, uint64_t seed,
                             const uint8_t* bits, size_t count, uint32_t* out);

/* trlwePhaseAt (ops.cpp:494-505) of coefficient k for count TRLWEs. */
int vsp_client_trlwe_phase_at(const uint32_t* lv1, uint32_t N, const uint32_t* ct, size_t count,
                              uint32_t k, uint32_t* phases);

/* tlwePhase / tlweDecrypt (ops.cpp:442-456); bits and/or phases may be NULL. */
int vsp_client_tlwe_decrypt(const uint32_t* key, uint32_t dim, const uint32_t* ct,
                            size_t count, uint8_t* bits, uint32_t* phases);

#ifdef __cplusplus
}
#endif
#endif
