// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (hvp, /root/reference/proj),
// compiled from the reference sources where they lie by oracle/Makefile into
// oracle/_ref/libhvpref.so.  Python tests, __graft_entry__.smoke() and bench.py's
// `--impl reference` / cpu_baseline legs load it through ctypes to (a) generate
// key material and golden vectors with the reference's own code and (b) time the
// reference CPU path on the host cores.  No reference source is copied here: this
// file only calls the public API declared in proj/include/hvp/**.
//
// Flat layouts (shared with include/vsp_b200.h):
//   TLWE   : (dim+1) u32, a[0..dim) then b
//   TRLWE  : 2N u32, a[0..N) then b[0..N)
//   TRGSW  : 2l rows x TRLWE  (row-major, reference row order ciphertext.hpp:57-64)
//   bk1    : n x TRGSW                    (BootstrappingKey::bk1Raw, ops.hpp:98)
//   bk2    : n x 2l2 x 2 x N2 u64          (BootstrappingKey::bk2Raw, ops.hpp:102)
//   ksk    : KeySwitchKey::data           (ops.hpp:18-29)
//   pks    : PrivKeySwitchKey::data       (ops.hpp:32-42)
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "hvp/common/parallel.hpp"
#include "hvp/mem/mem.hpp"
#include "hvp/netlist/engine.hpp"
#include "hvp/netlist/netlist.hpp"
#include "hvp/netlist/snapshot.hpp"
#include "hvp/tfhe/counters.hpp"
#include "hvp/tfhe/ops.hpp"
#include "hvp/tfhe/serialize.hpp"

using namespace hvp;
using namespace hvp::tfhe;

namespace {

thread_local std::string g_err;

struct RefCtx {
    ParameterSet params;
    Csprng rng = Csprng::fromSeed(0);
    SecretKey sk;
    std::optional<BootstrappingKey> bk;
};

template <class F>
int guard(F&& f)
{
    try {
        f();
        return 0;
    }
    catch (const std::invalid_argument& e) {
        g_err = std::string("invalid_argument: ") + e.what();
        return 1;
    }
    catch (const std::out_of_range& e) {
        g_err = std::string("out_of_range: ") + e.what();
        return 2;
    }
    catch (const std::exception& e) {
        g_err = std::string("runtime_error: ") + e.what();
        return 3;
    }
}

Tlwe toTlwe(const uint32_t* p, uint32_t dim, uint8_t level)
{
    Tlwe c;
    c.level = level;
    c.a.assign(p, p + dim);
    c.b = p[dim];
    return c;
}

void fromTlwe(const Tlwe& c, uint32_t* out)
{
    std::copy(c.a.begin(), c.a.end(), out);
    out[c.a.size()] = c.b;
}

Trlwe toTrlwe(const uint32_t* p, uint32_t N)
{
    Trlwe c;
    c.level = 1;
    c.a.assign(p, p + N);
    c.b.assign(p + N, p + 2 * N);
    return c;
}

void fromTrlwe(const Trlwe& c, uint32_t* out)
{
    const size_t N = c.a.size();
    std::copy(c.a.begin(), c.a.end(), out);
    std::copy(c.b.begin(), c.b.end(), out + N);
}

Trgsw toTrgsw(const uint32_t* p, uint32_t N, uint32_t l)
{
    Trgsw g;
    g.level = 1;
    for (uint32_t r = 0; r < 2 * l; r++)
        g.rows.push_back(toTrlwe(p + size_t{r} * 2 * N, N));
    return g;
}

void fromTrgsw(const Trgsw& g, uint32_t* out)
{
    const size_t N = g.rows.at(0).a.size();
    for (size_t r = 0; r < g.rows.size(); r++)
        fromTrlwe(g.rows[r], out + r * 2 * N);
}

}  // namespace

extern "C" {

const char* ref_last_error()
{
    return g_err.c_str();
}

// param_name: "tfhe-80" | "test-det"; n_override > 0 replaces n (the BASELINE
// n=630 variant of tfhe-80).  The secret key is drawn immediately from the
// seeded CSPRNG exactly as the reference fixture does (test_tfhe.cpp:35-39).
void* ref_ctx_new(const char* param_name, uint32_t n_override, uint64_t seed)
{
    RefCtx* c = nullptr;
    int rc = guard([&] {
        auto ctx = std::make_unique<RefCtx>();
        ctx->params = ParameterSet::byName(param_name);
        if (n_override > 0)
            ctx->params.n = n_override;
        ctx->params.validate();
        ctx->rng = Csprng::fromSeed(seed);
        ctx->sk = genSecretKey(ctx->params, ctx->rng);
        c = ctx.release();
    });
    return rc == 0 ? c : nullptr;
}

void ref_ctx_free(void* h)
{
    delete static_cast<RefCtx*>(h);
}

// out: n, N1, l1, Bg1Bits, N2, l2, Bg2Bits, ksBaseBits, ksLen, pksBaseBits,
// pksLen, mul(0 exact / 1 fft), hasBk, hasCb
void ref_params(void* h, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    const ParameterSet& p = c->params;
    uint32_t v[] = {p.n,          p.N1,        p.l1,    p.Bg1Bits, p.N2,
                    p.l2,         p.Bg2Bits,   p.ksBaseBits, p.ksLen,
                    p.pksBaseBits, p.pksLen,
                    p.mul == MulBackend::Fft ? 1u : 0u,
                    c->bk ? 1u : 0u,
                    c->bk && c->bk->hasCircuitBootstrapping() ? 1u : 0u};
    std::memcpy(out, v, sizeof(v));
}

int ref_keygen(void* h, int with_cb)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        c->bk.emplace(BootstrappingKey::generate(c->sk, c->rng, with_cb != 0));
    });
}

int ref_export_sk(void* h, uint32_t* lv0, uint32_t* lv1, uint32_t* lv2)
{
    auto* c = static_cast<RefCtx*>(h);
    std::copy(c->sk.lv0.begin(), c->sk.lv0.end(), lv0);
    std::copy(c->sk.lv1.begin(), c->sk.lv1.end(), lv1);
    std::copy(c->sk.lv2.begin(), c->sk.lv2.end(), lv2);
    return 0;
}

int ref_import_sk(void* h, const uint32_t* lv0, const uint32_t* lv1,
                  const uint32_t* lv2)
{
    auto* c = static_cast<RefCtx*>(h);
    const ParameterSet& p = c->params;
    c->sk.lv0.assign(lv0, lv0 + p.n);
    c->sk.lv1.assign(lv1, lv1 + p.N1);
    c->sk.lv2.assign(lv2, lv2 + p.N2);
    return 0;
}

int ref_export_bk1(void* h, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const auto& raw = c->bk.value().bk1Raw();
        const size_t per = size_t{2} * c->params.l1 * 2 * c->params.N1;
        for (size_t i = 0; i < raw.size(); i++)
            fromTrgsw(raw[i], out + i * per);
    });
}

int ref_export_bk2(void* h, uint64_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const auto& raw = c->bk.value().bk2Raw();
        size_t pos = 0;
        for (const auto& g : raw)
            for (const auto& row : g.rows) {
                std::copy(row.a.begin(), row.a.end(), out + pos);
                pos += row.a.size();
                std::copy(row.b.begin(), row.b.end(), out + pos);
                pos += row.b.size();
            }
    });
}

size_t ref_ksk_words(void* h)
{
    auto* c = static_cast<RefCtx*>(h);
    return c->bk ? c->bk->ksk().data.size() : 0;
}

int ref_export_ksk(void* h, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const auto& d = c->bk.value().ksk().data;
        std::copy(d.begin(), d.end(), out);
    });
}

size_t ref_pks_words(void* h)
{
    auto* c = static_cast<RefCtx*>(h);
    return c->bk && c->bk->hasCircuitBootstrapping() ? c->bk->pksId().data.size()
                                                     : 0;
}

// which: 0 = pksNegS, 1 = pksId
int ref_export_pks(void* h, int which, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const auto& k = which == 0 ? c->bk.value().pksNegS() : c->bk.value().pksId();
        std::copy(k.data.begin(), k.data.end(), out);
    });
}

// Rebuild the BootstrappingKey from raw arrays (BootstrappingKey::fromParts,
// ops.cpp:387-402).  bk2/pks may be null when has_cb == 0.
int ref_import_bk(void* h, const uint32_t* bk1, const uint64_t* bk2,
                  const uint32_t* ksk, const uint32_t* pks_negs,
                  const uint32_t* pks_id, int has_cb)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const ParameterSet& p = c->params;
        std::vector<Trgsw> b1;
        const size_t per1 = size_t{2} * p.l1 * 2 * p.N1;
        for (uint32_t i = 0; i < p.n; i++)
            b1.push_back(toTrgsw(bk1 + i * per1, p.N1, p.l1));
        std::vector<TrgswLvl2> b2;
        if (has_cb) {
            const size_t per2 = size_t{2} * p.l2 * 2 * p.N2;
            for (uint32_t i = 0; i < p.n; i++) {
                TrgswLvl2 g;
                g.level = 2;
                for (uint32_t r = 0; r < 2 * p.l2; r++) {
                    TrlweLvl2 row;
                    row.level = 2;
                    const uint64_t* q = bk2 + i * per2 + size_t{r} * 2 * p.N2;
                    row.a.assign(q, q + p.N2);
                    row.b.assign(q + p.N2, q + 2 * p.N2);
                    g.rows.push_back(std::move(row));
                }
                b2.push_back(std::move(g));
            }
        }
        KeySwitchKey k;
        k.N1 = p.N1;
        k.t = p.ksLen;
        k.baseBits = p.ksBaseBits;
        k.n = p.n;
        k.data.assign(ksk, ksk + size_t{p.N1} * p.ksLen *
                                     ((size_t{1} << p.ksBaseBits) - 1) * (p.n + 1));
        PrivKeySwitchKey pn, pi;
        if (has_cb) {
            for (PrivKeySwitchKey* q : {&pn, &pi}) {
                q->N2 = p.N2;
                q->t = p.pksLen;
                q->baseBits = p.pksBaseBits;
                q->N1 = p.N1;
            }
            const size_t words = (size_t{p.N2} + 1) * p.pksLen *
                                 ((size_t{1} << p.pksBaseBits) - 1) * 2 * p.N1;
            pn.data.assign(pks_negs, pks_negs + words);
            pi.data.assign(pks_id, pks_id + words);
        }
        c->bk.emplace(BootstrappingKey::fromParts(p, std::move(b1), std::move(b2),
                                                  std::move(k), std::move(pn),
                                                  std::move(pi), has_cb != 0));
    });
}

// --- encryption / decryption (client side, ops.cpp:428-515) ---------------

// Encrypts with the context CSPRNG and alpha0 noise (tlweEncrypt, ops.cpp:428).
int ref_tlwe_encrypt(void* h, int m, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        NoiseSampler ns(c->rng, c->params.alpha0);
        fromTlwe(tlweEncrypt(m != 0, c->sk, ns), out);
    });
}

uint32_t ref_tlwe_phase(void* h, const uint32_t* ct, int level)
{
    auto* c = static_cast<RefCtx*>(h);
    const uint32_t dim = level == 0 ? c->params.n : c->params.N1;
    return tlwePhase(toTlwe(ct, dim, static_cast<uint8_t>(level)), c->sk);
}

int ref_trlwe_encrypt(void* h, const uint32_t* bits, double alpha, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        NoiseSampler ns(c->rng, alpha);
        std::vector<uint32_t> m(bits, bits + c->params.N1);
        fromTrlwe(trlweEncrypt(m, c->sk, ns), out);
    });
}

uint32_t ref_trlwe_phase_at(void* h, const uint32_t* ct, uint32_t k)
{
    auto* c = static_cast<RefCtx*>(h);
    return trlwePhaseAt(toTrlwe(ct, c->params.N1), k, c->sk);
}

int ref_trgsw_encrypt(void* h, int m, double alpha, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        NoiseSampler ns(c->rng, alpha);
        fromTrgsw(trgswEncrypt(m != 0, c->sk, ns), out);
    });
}

// --- evaluation (the hot path, ops.cpp:553-947) ---------------------------

int ref_hom_gate(void* h, int kind, const uint32_t* in, int nin, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        std::vector<Tlwe> v;
        for (int i = 0; i < nin; i++)
            v.push_back(toTlwe(in + size_t{i} * (c->params.n + 1), c->params.n, 0));
        fromTlwe(homGate(static_cast<GateKind>(kind), v, c->bk.value()), out);
    });
}

// in: G x 3 x (n+1) (unused operand slots ignored); out: G x (n+1).
// Parallelised with the reference's own parallelFor (parallel.cpp:15-44).
int ref_hom_gate_batch(void* h, const int* kinds, const uint32_t* in,
                       uint32_t* out, size_t G, unsigned threads)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const uint32_t n = c->params.n;
        const BootstrappingKey& bk = c->bk.value();
        parallelFor(threads, G, [&](size_t g) {
            const GateKind k = static_cast<GateKind>(kinds[g]);
            std::vector<Tlwe> v;
            for (int i = 0; i < gateArity(k); i++)
                v.push_back(toTlwe(in + (g * 3 + i) * (n + 1), n, 0));
            fromTlwe(homGate(k, v, bk), out + g * (n + 1));
        });
    });
}

int ref_gate_bootstrap(void* h, const uint32_t* in, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        fromTlwe(gateBootstrap(toTlwe(in, c->params.n, 0), c->bk.value()), out);
    });
}

int ref_bootstrap_to_trlwe(void* h, const uint32_t* in, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        fromTrlwe(bootstrapToTrlwe(toTlwe(in, c->params.n, 0), c->bk.value()), out);
    });
}

int ref_identity_key_switch(void* h, const uint32_t* in, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        fromTlwe(identityKeySwitch(toTlwe(in, c->params.N1, 1), c->bk.value()), out);
    });
}

int ref_sample_extract(void* h, const uint32_t* trlwe, uint32_t k, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] { fromTlwe(sampleExtract(toTrlwe(trlwe, c->params.N1), k), out); });
}

int ref_cmux(void* h, const uint32_t* sel, const uint32_t* c1, const uint32_t* c0,
             uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const ParameterSet& p = c->params;
        fromTrlwe(cmux(toTrgsw(sel, p.N1, p.l1), toTrlwe(c1, p.N1), toTrlwe(c0, p.N1), p),
                  out);
    });
}

int ref_hom_mux_no_se_iks(void* h, const uint32_t* sel, const uint32_t* a,
                          const uint32_t* b, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const uint32_t n = c->params.n;
        fromTrlwe(homMuxNoSeIks(toTlwe(sel, n, 0), toTlwe(a, n, 0), toTlwe(b, n, 0),
                                c->bk.value()),
                  out);
    });
}

int ref_circuit_bootstrap(void* h, const uint32_t* in, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        fromTrgsw(circuitBootstrap(toTlwe(in, c->params.n, 0), c->bk.value()), out);
    });
}

// which: 0 = pksNegS, 1 = pksId.  in: (N2+1) u64 level-2 TLWE.
int ref_private_key_switch(void* h, const uint64_t* in, int which, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        TlweLvl2 t;
        t.level = 2;
        t.a.assign(in, in + c->params.N2);
        t.b = in[c->params.N2];
        const auto& bk = c->bk.value();
        fromTrlwe(privateKeySwitch(t, which == 0 ? bk.pksNegS() : bk.pksId()), out);
    });
}

int ref_trgsw_not(void* h, const uint32_t* in, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const ParameterSet& p = c->params;
        fromTrgsw(trgswNot(toTrgsw(in, p.N1, p.l1), p), out);
    });
}

// --- CMUX memory (mem.cpp) ------------------------------------------------

// ram: w*2^v TRLWE cells (cells[j*2^v + A], mem.hpp:32-46), flat.
int ref_ram_cycle(void* h, uint32_t v, uint32_t w, uint32_t* ram,
                  const uint32_t* addr, const uint32_t* wflag, const uint32_t* wdata,
                  uint32_t* readout, unsigned threads)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const ParameterSet& p = c->params;
        const uint32_t n = p.n;
        mem::EncryptedRam r;
        r.geom.v = v;
        r.geom.w = w;
        const size_t cells = size_t{w} << v;
        for (size_t i = 0; i < cells; i++)
            r.cells.push_back(toTrlwe(ram + i * 2 * p.N1, p.N1));
        std::vector<Tlwe> a, d;
        for (uint32_t i = 0; i < v; i++)
            a.push_back(toTlwe(addr + size_t{i} * (n + 1), n, 0));
        for (uint32_t i = 0; i < w; i++)
            d.push_back(toTlwe(wdata + size_t{i} * (n + 1), n, 0));
        mem::RamCycleOut o =
            mem::ramCycle(r, a, toTlwe(wflag, n, 0), d, c->bk.value(), threads);
        for (uint32_t i = 0; i < w; i++)
            fromTlwe(o.readOut[i], readout + size_t{i} * (n + 1));
        for (size_t i = 0; i < cells; i++)
            fromTrlwe(o.ram.cells[i], ram + i * 2 * p.N1);
    });
}

// rom: luts as produced by encryptRom (mem.cpp:236-263); addr: vrom TLWEs.
// Runs addressToTrgsw + prepareAddress + romRead exactly like
// TfheBackend::romRead (engine.cpp:133-143).
int ref_rom_read(void* h, uint32_t depth_bytes, const uint32_t* luts, uint32_t nluts,
                 const uint32_t* addr, uint32_t vrom, uint32_t* out, unsigned threads)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const ParameterSet& p = c->params;
        mem::EncryptedRom rom;
        rom.depthBytes = depth_bytes;
        for (uint32_t t = 0; t < nluts; t++)
            rom.luts.push_back(toTrlwe(luts + size_t{t} * 2 * p.N1, p.N1));
        std::vector<Tlwe> a;
        for (uint32_t i = 0; i < vrom; i++)
            a.push_back(toTlwe(addr + size_t{i} * (p.n + 1), p.n, 0));
        const auto& bk = c->bk.value();
        mem::RamAddress sel = mem::addressToTrgsw(a, bk, threads);
        auto res = mem::romRead(rom, mem::prepareAddress(sel, p), bk, threads);
        for (size_t k = 0; k < res.size(); k++)
            fromTlwe(res[k], out + k * (p.n + 1));
    });
}

// The units of ramCycle / romRead on given selectors (RamAddress: v raw TRGSWs, LSB
// first), each through prepareAddress (mem.cpp:21-36) -- mem.hpp:75-124.
namespace {
mem::EncryptedRam toRam(const uint32_t* ram, uint32_t v, uint32_t w, uint32_t N)
{
    mem::EncryptedRam r;
    r.geom.v = v;
    r.geom.w = w;
    const size_t cells = size_t{w} << v;
    for (size_t i = 0; i < cells; i++)
        r.cells.push_back(toTrlwe(ram + i * 2 * N, N));
    return r;
}

mem::RamAddress toAddr(const uint32_t* sel, uint32_t v, uint32_t N, uint32_t l)
{
    mem::RamAddress a;
    for (uint32_t d = 0; d < v; d++)
        a.bits.push_back(toTrgsw(sel + size_t{d} * 2 * l * 2 * N, N, l));
    return a;
}
}  // namespace

int ref_ram_read_unit(void* h, uint32_t v, uint32_t w, const uint32_t* ram, const uint32_t* sel,
                      uint32_t* out, unsigned threads)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const ParameterSet& p = c->params;
        auto res = mem::ramReadUnit(toRam(ram, v, w, p.N1),
                                    mem::prepareAddress(toAddr(sel, v, p.N1, p.l1), p), threads);
        for (size_t j = 0; j < res.size(); j++)
            fromTrlwe(res[j], out + j * 2 * p.N1);
    });
}

int ref_ram_control_unit(void* h, uint32_t w, const uint32_t* read, const uint32_t* wflag,
                         const uint32_t* wdata, uint32_t* readout, uint32_t* controlled,
                         unsigned threads)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const ParameterSet& p = c->params;
        std::vector<Trlwe> rd;
        std::vector<Tlwe> d;
        for (uint32_t j = 0; j < w; j++) {
            rd.push_back(toTrlwe(read + size_t{j} * 2 * p.N1, p.N1));
            d.push_back(toTlwe(wdata + size_t{j} * (p.n + 1), p.n, 0));
        }
        mem::ControlOut o = mem::ramControlUnit(rd, toTlwe(wflag, p.n, 0), d, c->bk.value(),
                                                threads);
        for (uint32_t j = 0; j < w; j++) {
            fromTlwe(o.readOut[j], readout + size_t{j} * (p.n + 1));
            fromTrlwe(o.controlled[j], controlled + size_t{j} * 2 * p.N1);
        }
    });
}

int ref_ram_write_unit(void* h, uint32_t v, uint32_t w, uint32_t* ram, const uint32_t* sel,
                       const uint32_t* controlled, unsigned threads)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const ParameterSet& p = c->params;
        std::vector<Trlwe> ctl;
        for (uint32_t j = 0; j < w; j++)
            ctl.push_back(toTrlwe(controlled + size_t{j} * 2 * p.N1, p.N1));
        mem::EncryptedRam r =
            mem::ramWriteUnit(toRam(ram, v, w, p.N1),
                              mem::prepareAddress(toAddr(sel, v, p.N1, p.l1), p), ctl,
                              c->bk.value(), threads);
        for (size_t i = 0; i < r.cells.size(); i++)
            fromTrlwe(r.cells[i], ram + i * 2 * p.N1);
    });
}

int ref_rom_read_sel(void* h, uint32_t depth_bytes, const uint32_t* luts, uint32_t nluts,
                     const uint32_t* sel, uint32_t vrom, uint32_t* out, unsigned threads)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        const ParameterSet& p = c->params;
        mem::EncryptedRom rom;
        rom.depthBytes = depth_bytes;
        for (uint32_t t = 0; t < nluts; t++)
            rom.luts.push_back(toTrlwe(luts + size_t{t} * 2 * p.N1, p.N1));
        auto res = mem::romRead(rom, mem::prepareAddress(toAddr(sel, vrom, p.N1, p.l1), p),
                                c->bk.value(), threads);
        for (size_t k = 0; k < res.size(); k++)
            fromTlwe(res[k], out + k * (p.n + 1));
    });
}

// Trivial (sk == nullptr) or secret-key encryption of a RAM/ROM image.
int ref_encrypt_ram(void* h, const uint8_t* image, uint32_t v, uint32_t w,
                    int trivial, uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        mem::MemoryGeometry g{v, w};
        NoiseSampler ns(c->rng, c->params.alpha1);
        auto r = mem::encryptRam(std::span<const uint8_t>(image, g.imageBytes()), g,
                                 c->params, trivial ? nullptr : &c->sk,
                                 trivial ? nullptr : &ns);
        for (size_t i = 0; i < r.cells.size(); i++)
            fromTrlwe(r.cells[i], out + i * 2 * c->params.N1);
    });
}

int ref_decrypt_ram(void* h, const uint32_t* ram, uint32_t v, uint32_t w,
                    uint8_t* image)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        mem::EncryptedRam r;
        r.geom = {v, w};
        for (size_t i = 0; i < r.geom.bits(); i++)
            r.cells.push_back(toTrlwe(ram + i * 2 * c->params.N1, c->params.N1));
        auto img = mem::decryptRam(r, c->sk);
        std::copy(img.begin(), img.end(), image);
    });
}

uint32_t ref_rom_luts(void* h, uint32_t depth_bytes)
{
    auto* c = static_cast<RefCtx*>(h);
    const uint32_t blocks = depth_bytes / 4;
    const uint32_t vrom = static_cast<uint32_t>(std::countr_zero(blocks));
    const uint32_t lowBits = std::min(
        vrom, static_cast<uint32_t>(std::countr_zero(c->params.N1 / 32)));
    return 1u << (vrom - lowBits);
}

int ref_encrypt_rom(void* h, const uint8_t* image, uint32_t depth_bytes, int trivial,
                    uint32_t* out)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        NoiseSampler ns(c->rng, c->params.alpha1);
        auto r = mem::encryptRom(std::span<const uint8_t>(image, depth_bytes), c->params,
                                 trivial ? nullptr : &c->sk, trivial ? nullptr : &ns);
        for (size_t t = 0; t < r.luts.size(); t++)
            fromTrlwe(r.luts[t], out + t * 2 * c->params.N1);
    });
}

// counters: cmux, blindRotate, identityKeySwitch, privateKeySwitch, circuitBootstrap
void ref_counters(uint64_t* out)
{
    auto& k = opCounters();
    out[0] = k.cmux.load();
    out[1] = k.blindRotate.load();
    out[2] = k.identityKeySwitch.load();
    out[3] = k.privateKeySwitch.load();
    out[4] = k.circuitBootstrap.load();
}

void ref_counters_reset()
{
    opCounters().reset();
}

unsigned ref_hardware_threads()
{
    return hardwareThreads();
}

// --- netlist runner (engine.hpp, built with the two-member fix) ------------

struct RefEval {
    std::unique_ptr<netlist::Evaluator<netlist::TfheBackend>> ev;
};

void* ref_eval_new(void* h, const char* json, unsigned threads)
{
    auto* c = static_cast<RefCtx*>(h);
    RefEval* out = nullptr;
    int rc = guard([&] {
        netlist::Netlist nl = netlist::parseNetlist(json);
        netlist::TfheBackend be;
        be.bk = &c->bk.value();
        be.threads = threads;
        auto e = std::make_unique<RefEval>();
        e->ev = std::make_unique<netlist::Evaluator<netlist::TfheBackend>>(nl, be);
        out = e.release();
    });
    return rc == 0 ? out : nullptr;
}

void ref_eval_free(void* e)
{
    delete static_cast<RefEval*>(e);
}

int ref_eval_set_input(void* e, const char* port, size_t idx, const uint32_t* ct,
                       uint32_t n)
{
    auto* r = static_cast<RefEval*>(e);
    return guard([&] { r->ev->setInput(port, idx, toTlwe(ct, n, 0)); });
}

int ref_eval_output(void* e, const char* port, size_t idx, uint32_t* ct)
{
    auto* r = static_cast<RefEval*>(e);
    return guard([&] { fromTlwe(r->ev->output(port, idx), ct); });
}

int ref_eval_set_ram(void* e, uint32_t v, uint32_t w, const uint32_t* ram, uint32_t N)
{
    auto* r = static_cast<RefEval*>(e);
    return guard([&] {
        netlist::TfheBackend::Ram ram_;
        ram_.enc.geom = {v, w};
        for (size_t i = 0; i < ram_.enc.geom.bits(); i++)
            ram_.enc.cells.push_back(toTrlwe(ram + i * 2 * N, N));
        r->ev->setRam(std::move(ram_));
    });
}

int ref_eval_get_ram(void* e, uint32_t* ram)
{
    auto* r = static_cast<RefEval*>(e);
    return guard([&] {
        const auto& cells = r->ev->ram().enc.cells;
        for (size_t i = 0; i < cells.size(); i++)
            fromTrlwe(cells[i], ram + i * 2 * cells[i].a.size());
    });
}

int ref_eval_set_rom(void* e, uint32_t depth_bytes, const uint32_t* luts, uint32_t nluts,
                     uint32_t N)
{
    auto* r = static_cast<RefEval*>(e);
    return guard([&] {
        netlist::TfheBackend::Rom rom;
        rom.enc.depthBytes = depth_bytes;
        for (uint32_t t = 0; t < nluts; t++)
            rom.enc.luts.push_back(toTrlwe(luts + size_t{t} * 2 * N, N));
        r->ev->setRom(std::move(rom));
    });
}

size_t ref_eval_dff_count(void* e)
{
    return static_cast<RefEval*>(e)->ev->dffState().size();
}

int ref_eval_get_dff(void* e, uint32_t* out, uint32_t n)
{
    auto* r = static_cast<RefEval*>(e);
    return guard([&] {
        const auto& s = r->ev->dffState();
        for (size_t i = 0; i < s.size(); i++)
            fromTlwe(s[i], out + i * (n + 1));
    });
}

int ref_eval_set_dff(void* e, const uint32_t* in, uint32_t n)
{
    auto* r = static_cast<RefEval*>(e);
    return guard([&] {
        std::vector<Tlwe> s;
        for (size_t i = 0; i < r->ev->dffState().size(); i++)
            s.push_back(toTlwe(in + i * (n + 1), n, 0));
        r->ev->setDffStateRaw(std::move(s));
    });
}

// stats_out (optional): per cycle [evaluatedTotal, gMax, depth, wallSeconds*1e6]
int ref_eval_run(void* e, uint64_t cycles, unsigned workers, uint64_t shuffle_seed,
                 double* stats_out)
{
    auto* r = static_cast<RefEval*>(e);
    return guard([&] {
        std::vector<netlist::CycleStats> st;
        netlist::RunOptions o;
        o.workers = workers;
        o.shuffleSeed = shuffle_seed;
        o.stats = &st;
        r->ev->run(cycles, o);
        if (stats_out)
            for (size_t i = 0; i < st.size(); i++) {
                stats_out[4 * i + 0] = static_cast<double>(st[i].evaluatedTotal());
                stats_out[4 * i + 1] = st[i].gMax;
                stats_out[4 * i + 2] = st[i].depth;
                stats_out[4 * i + 3] = st[i].wallSeconds * 1e6;
            }
    });
}

// HVP1 containers written by the reference (serialize.cpp:190-245, mem.cpp:354-396).
static int put_bytes(const std::vector<uint8_t>& b, uint8_t* out, size_t cap, size_t* len)
{
    *len = b.size();
    if (out) {
        if (cap < b.size())
            throw std::invalid_argument("buffer too small");
        std::memcpy(out, b.data(), b.size());
    }
    return 0;
}

int ref_serialize_bk(void* h, uint8_t* out, size_t cap, size_t* len)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] { put_bytes(serializeBootstrappingKey(c->bk.value()), out, cap, len); });
}

int ref_serialize_tlwe(void* h, const uint32_t* ct, uint8_t* out, size_t cap, size_t* len)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        put_bytes(serializeTlwe(toTlwe(ct, c->params.n, 0), c->params), out, cap, len);
    });
}

int ref_serialize_ram(void* h, uint32_t v, uint32_t w, const uint32_t* ram, uint8_t* out,
                      size_t cap, size_t* len)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        mem::EncryptedRam r;
        r.geom = {v, w};
        for (size_t i = 0; i < r.geom.bits(); i++)
            r.cells.push_back(toTrlwe(ram + i * 2 * c->params.N1, c->params.N1));
        put_bytes(mem::serializeRam(r, c->params), out, cap, len);
    });
}

int ref_serialize_rom(void* h, uint32_t depth, const uint32_t* luts, uint32_t nluts, uint8_t* out,
                      size_t cap, size_t* len)
{
    auto* c = static_cast<RefCtx*>(h);
    return guard([&] {
        mem::EncryptedRom r;
        r.depthBytes = depth;
        for (uint32_t t = 0; t < nluts; t++)
            r.luts.push_back(toTrlwe(luts + size_t{t} * 2 * c->params.N1, c->params.N1));
        put_bytes(mem::serializeRom(r, c->params), out, cap, len);
    });
}

// snapshotSave / snapshotLoad (snapshot.cpp:84-158) of the reference evaluator.
int ref_eval_snapshot_save(void* e, uint8_t* out, size_t cap, size_t* len)
{
    auto* r = static_cast<RefEval*>(e);
    return guard([&] {
        const std::vector<uint8_t> b = netlist::snapshotSave(*r->ev);
        *len = b.size();
        if (out) {
            if (cap < b.size())
                throw std::invalid_argument("buffer too small");
            std::memcpy(out, b.data(), b.size());
        }
    });
}

void* ref_eval_snapshot_load(void* h, const char* json, const uint8_t* in, size_t len,
                             unsigned threads)
{
    auto* c = static_cast<RefCtx*>(h);
    RefEval* out = nullptr;
    int rc = guard([&] {
        netlist::Netlist nl = netlist::parseNetlist(json);
        netlist::TfheBackend be;
        be.bk = &c->bk.value();
        be.threads = threads;
        auto e = std::make_unique<RefEval>();
        e->ev = std::make_unique<netlist::Evaluator<netlist::TfheBackend>>(
            netlist::snapshotLoad(nl, be, std::vector<uint8_t>(in, in + len)));
        out = e.release();
    });
    return rc == 0 ? out : nullptr;
}

// DAG analysis (buildDag, netlist.cpp:348-432): levels per DAG node, in
// Netlist::cells order for non-DFF cells; returns node count.
int ref_netlist_levels(const char* json, int* level_out, int* cell_out, int* gmax,
                       int* depth, size_t* nodes)
{
    return guard([&] {
        netlist::Netlist nl = netlist::parseNetlist(json);
        netlist::Dag d = netlist::buildDag(nl);
        for (size_t i = 0; i < d.dagCells.size(); i++) {
            if (level_out)
                level_out[i] = d.level[i];
            if (cell_out)
                cell_out[i] = d.dagCells[i];
        }
        *gmax = d.gMax;
        *depth = d.depth;
        *nodes = d.dagCells.size();
    });
}

}  // extern "C"
