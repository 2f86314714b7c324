/*
 * vsp_b200.hpp — C++20 host facade over the C ABI (vsp_b200.h).
 *
 * Keeps the reference's C++ surface for the hot path (hvp, /root/reference/proj):
 * the same namespaces (tfhe / mem / netlist), function names, argument meaning and
 * exception types, so a caller of hvp::tfhe::homGate, hvp::mem::ramCycle or
 * hvp::netlist::Evaluator<TfheBackend> switches by changing the namespace and
 * constructing a device-resident BootstrappingKey.
 *
 *   reference                                   here
 *   hvp::tfhe::homGate        (ops.hpp:212-213)  vsp::tfhe::homGate / homGateBatch
 *   hvp::tfhe::gateBootstrap  (ops.hpp:178)  vsp::tfhe::gateBootstrap
 *   hvp::tfhe::bootstrapToTrlwe (ops.hpp:181) vsp::tfhe::bootstrapToTrlwe
 *   hvp::tfhe::identityKeySwitch (ops.hpp:164) vsp::tfhe::identityKeySwitch
 *   hvp::tfhe::cmux           (ops.hpp:154-158)  vsp::tfhe::cmux (raw TRGSW selector)
 *   hvp::tfhe::homMuxNoSeIks  (ops.hpp:215-216)  vsp::tfhe::homMuxNoSeIks
 *   hvp::tfhe::circuitBootstrap (ops.hpp:218) vsp::tfhe::circuitBootstrap
 *   hvp::mem::ramCycle        (mem.hpp:113-117)  vsp::mem::ramCycle
 *   hvp::mem::romRead         (mem.hpp:121-124)  vsp::mem::romRead (takes the TLWE address
 *                                                bits; addressToTrgsw + prepareAddress run
 *                                                on the device, engine.cpp:133-143)
 *   hvp::netlist::TfheBackend (engine.hpp:73-98) vsp::netlist::GpuBackend (same concept)
 *   hvp::netlist::Evaluator::run (engine.hpp:238-247)  vsp::netlist::Runner (level-batched)
 *
 * Ciphertexts are flat std::vector<uint32_t> in the reference's word order
 * (TLWE: a[0..n) then b; TRLWE: a[0..N) then b[0..N); TRGSW: 2l TRLWE rows).
 * Errors: VSP_EINVAL -> std::invalid_argument, VSP_ERANGE -> std::out_of_range,
 * VSP_ERUNTIME -> std::runtime_error (the reference's exception types).
 * Header-only; link with -lvsp_b200.
 */
#ifndef VSP_B200_HPP
#define VSP_B200_HPP

#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "vsp_b200.h"

namespace vsp {
namespace detail {

inline void raise(int rc, const char* msg)
{
    const std::string m = msg ? msg : "";
    if (rc == VSP_EINVAL)
        throw std::invalid_argument(m);
    if (rc == VSP_ERANGE)
        throw std::out_of_range(m);
    throw std::runtime_error(m);
}

inline void check(int rc)
{
    if (rc != VSP_OK)
        raise(rc, vsp_last_error());
}

inline void check_client(int rc)
{
    if (rc != VSP_OK)
        raise(rc, vsp_client_last_error());
}

inline std::vector<uint32_t> flatten(std::span<const std::vector<uint32_t>> v, size_t words, const char* what)
{
    std::vector<uint32_t> flat(v.size() * words);
    for (size_t i = 0; i < v.size(); i++) {
        if (v[i].size() != words)
            throw std::invalid_argument(std::string(what) + ": ciphertext dimension mismatch");
        std::copy(v[i].begin(), v[i].end(), flat.begin() + i * words);
    }
    return flat;
}
inline std::vector<std::vector<uint32_t>> split(const std::vector<uint32_t>& flat, size_t words)
{
    std::vector<std::vector<uint32_t>> out(words ? flat.size() / words : 0);
    for (size_t i = 0; i < out.size(); i++)
        out[i].assign(flat.begin() + i * words, flat.begin() + (i + 1) * words);
    return out;
}
}  // namespace detail

namespace tfhe {

// hvp::tfhe::GateKind (ops.hpp:183-194), same order and values.
enum class GateKind : int32_t { And, AndNot, Mux, Nand, Nor, Not, Or, OrNot, Xnor, Xor };

inline constexpr uint32_t kMu32 = 1u << 29;  // params.hpp:12

using Tlwe = std::vector<uint32_t>;   // TlweSample<uint32_t> (ciphertext.hpp:14-28), flat
using Trlwe = std::vector<uint32_t>;  // TrlweSample<uint32_t> (ciphertext.hpp:34-53), flat
using Trgsw = std::vector<uint32_t>;  // TrgswSample<uint32_t> (ciphertext.hpp:60-64), flat

// hvp::tfhe::ParameterSet (params.hpp:23-66); byName (params.cpp:88-95) + validate.
struct ParameterSet {
    vsp_params raw{};
    std::string name;

    static ParameterSet byName(const std::string& name, uint32_t nOverride = 0)
    {
        ParameterSet p;
        detail::check(vsp_params_by_name(name.c_str(), nOverride, &p.raw));
        p.name = name;
        return p;
    }
    size_t tlweWords(int level = 0) const { return (level == 0 ? raw.n : raw.N1) + 1; }
    size_t trlweWords() const { return 2 * (size_t)raw.N1; }
    size_t trgswWords() const { return 2 * (size_t)raw.l1 * trlweWords(); }
    size_t kskWords() const
    {
        return (size_t)raw.N1 * raw.ksLen * ((1u << raw.ksBaseBits) - 1) * (raw.n + 1);
    }
    size_t pksWords() const
    {
        return ((size_t)raw.N2 + 1) * raw.pksLen * ((1u << raw.pksBaseBits) - 1) * 2 * raw.N1;
    }
};

// Client-side key material (Alice): genSecretKey + BootstrappingKey::generate
// (ops.cpp:264-385) in the reference's raw layouts.  Not on the evaluation path.
struct KeyMaterial {
    ParameterSet params;
    std::vector<uint32_t> lv0, lv1, lv2, bk1, ksk, pksNegS, pksId;
    std::vector<uint64_t> bk2;
    int withCb = 0;  // 0: none, 1: bk2 + PKS tables, 2: bk2 only

    static KeyMaterial generate(const ParameterSet& p, uint64_t seed, int withCb)
    {
        KeyMaterial k;
        k.params = p;
        k.withCb = withCb;
        const auto& r = p.raw;
        k.lv0.resize(r.n);
        k.lv1.resize(r.N1);
        k.lv2.resize(r.N2);
        k.bk1.resize((size_t)r.n * 2 * r.l1 * 2 * r.N1);
        k.ksk.resize(p.kskWords());
        if (withCb)
            k.bk2.resize((size_t)r.n * 2 * r.l2 * 2 * r.N2);
        if (withCb == 1) {
            k.pksNegS.resize(p.pksWords());
            k.pksId.resize(p.pksWords());
        }
        detail::check_client(vsp_client_keygen(
            &p.raw, seed, withCb, k.lv0.data(), k.lv1.data(), k.lv2.data(), k.bk1.data(),
            k.ksk.data(), withCb ? k.bk2.data() : nullptr,
            withCb == 1 ? k.pksNegS.data() : nullptr, withCb == 1 ? k.pksId.data() : nullptr));
        return k;
    }
};

// tlweEncrypt (ops.cpp:428-440) of `bits`, one CSPRNG stream from `seed`.
inline std::vector<Tlwe> tlweEncrypt(const ParameterSet& p, const std::vector<uint32_t>& lv0,
                                     std::span<const uint8_t> bits, uint64_t seed)
{
    std::vector<uint32_t> flat(bits.size() * p.tlweWords());
    detail::check_client(vsp_client_tlwe_encrypt(&p.raw, lv0.data(), seed, bits.data(),
                                                 bits.size(), flat.data()));
    std::vector<Tlwe> out(bits.size());
    for (size_t i = 0; i < bits.size(); i++)
        out[i].assign(flat.begin() + i * p.tlweWords(), flat.begin() + (i + 1) * p.tlweWords());
    return out;
}

// tlweDecrypt (ops.cpp:452-456) under `key` (level-0 or level-1 secret key).
inline bool tlweDecrypt(const Tlwe& c, const std::vector<uint32_t>& key)
{
    uint8_t bit = 0;
    detail::check_client(
        vsp_client_tlwe_decrypt(key.data(), (uint32_t)key.size(), c.data(), 1, &bit, nullptr));
    return bit != 0;
}

// tlweTrivial (ops.cpp:212-217): a = 0, b = +-mu.
inline Tlwe tlweTrivial(bool b, const ParameterSet& p)
{
    Tlwe t(p.tlweWords(), 0u);
    t.back() = b ? kMu32 : 0u - kMu32;
    return t;
}

// The evaluation key bundle, resident on one GPU (BootstrappingKey::fromParts +
// prepareAll, ops.cpp:387-415, with the FFT preparation done on the device).  Owns the
// engine context; move-only, like the reference's key which is shared read-only.
class BootstrappingKey {
public:
    BootstrappingKey(const KeyMaterial& k, int device = 0) : params_(k.params)
    {
        ctx_ = vsp_create(&params_.raw, device);
        if (!ctx_)
            detail::raise(VSP_ERUNTIME, vsp_last_error());
        try {
            detail::check(vsp_upload_keys(
                ctx_, k.bk1.data(), k.ksk.data(), k.withCb ? k.bk2.data() : nullptr,
                k.withCb == 1 ? k.pksNegS.data() : nullptr,
                k.withCb == 1 ? k.pksId.data() : nullptr, k.withCb));
        }
        catch (...) {
            vsp_destroy(ctx_);
            throw;
        }
    }
    BootstrappingKey(const BootstrappingKey&) = delete;
    BootstrappingKey& operator=(const BootstrappingKey&) = delete;
    BootstrappingKey(BootstrappingKey&& o) noexcept
        : params_(std::move(o.params_)), ctx_(std::exchange(o.ctx_, nullptr))
    {
    }
    ~BootstrappingKey()
    {
        if (ctx_)
            vsp_destroy(ctx_);
    }
    const ParameterSet& params() const { return params_; }
    vsp_ctx* ctx() const { return ctx_; }

private:
    ParameterSet params_;
    vsp_ctx* ctx_ = nullptr;
};


// homGate over a batch of independent gates: ONE batched launch sequence for the whole
// batch (the netlist runner's per-level call).  ins[g] holds the gate's operands in pin
// order (MUX: {s, a, b}; NOT: {a}).  Equivalent to G calls of homGate.
inline std::vector<Tlwe> homGateBatch(std::span<const GateKind> kinds,
                                      std::span<const std::vector<Tlwe>> ins,
                                      const BootstrappingKey& bk)
{
    if (kinds.size() != ins.size())
        throw std::invalid_argument("homGateBatch: kinds/inputs size mismatch");
    const size_t w = bk.params().tlweWords();
    std::vector<uint32_t> in(kinds.size() * 3 * w, 0u), out(kinds.size() * w);
    for (size_t g = 0; g < kinds.size(); g++) {
        if (ins[g].size() > 3)
            throw std::invalid_argument("homGate: wrong number of inputs");
        for (size_t k = 0; k < ins[g].size(); k++) {
            if (ins[g][k].size() != w)
                throw std::invalid_argument("homGate: ciphertext dimension mismatch");
            std::copy(ins[g][k].begin(), ins[g][k].end(), in.begin() + (g * 3 + k) * w);
        }
        const GateKind kd = kinds[g];
        const size_t need = kd == GateKind::Not ? 1 : kd == GateKind::Mux ? 3 : 2;
        if (ins[g].size() != need)  // ops.cpp:844-846
            throw std::invalid_argument("homGate: wrong number of inputs");
    }
    detail::check(vsp_hom_gate_batch(bk.ctx(), reinterpret_cast<const int32_t*>(kinds.data()),
                                     in.data(), out.data(), kinds.size()));
    return detail::split(out, w);
}

// homGate (ops.cpp:839-896).
inline Tlwe homGate(GateKind kind, std::span<const Tlwe> in, const BootstrappingKey& bk)
{
    const std::vector<Tlwe> one(in.begin(), in.end());
    return homGateBatch(std::span<const GateKind>(&kind, 1),
                        std::span<const std::vector<Tlwe>>(&one, 1), bk)[0];
}

// gateBootstrap (ops.cpp:759-762), batched.
inline std::vector<Tlwe> gateBootstrap(std::span<const Tlwe> in, const BootstrappingKey& bk)
{
    const size_t w = bk.params().tlweWords();
    auto flat = detail::flatten(in, w, "gateBootstrap");
    std::vector<uint32_t> out(in.size() * w);
    detail::check(vsp_gate_bootstrap_batch(bk.ctx(), flat.data(), out.data(), in.size()));
    return detail::split(out, w);
}

// bootstrapToTrlwe (ops.cpp:750-757), batched.
inline std::vector<Trlwe> bootstrapToTrlwe(std::span<const Tlwe> in, const BootstrappingKey& bk)
{
    const auto& p = bk.params();
    auto flat = detail::flatten(in, p.tlweWords(), "bootstrapToTrlwe");
    std::vector<uint32_t> out(in.size() * p.trlweWords());
    detail::check(vsp_bootstrap_to_trlwe_batch(bk.ctx(), flat.data(), out.data(), in.size()));
    return detail::split(out, p.trlweWords());
}

// identityKeySwitch (ops.cpp:651-679): level-1 TLWEs (N1+1 words) -> level 0, batched.
inline std::vector<Tlwe> identityKeySwitch(std::span<const Tlwe> in, const BootstrappingKey& bk)
{
    const auto& p = bk.params();
    auto flat = detail::flatten(in, p.tlweWords(1), "identityKeySwitch");
    std::vector<uint32_t> out(in.size() * p.tlweWords());
    detail::check(vsp_identity_key_switch_batch(bk.ctx(), flat.data(), out.data(), in.size()));
    return detail::split(out, p.tlweWords());
}

// circuitBootstrap (ops.cpp:914-935), batched: level-0 TLWEs -> raw TRGSWs.
inline std::vector<Trgsw> circuitBootstrap(std::span<const Tlwe> in, const BootstrappingKey& bk)
{
    const auto& p = bk.params();
    auto flat = detail::flatten(in, p.tlweWords(), "circuitBootstrap");
    std::vector<uint32_t> out(in.size() * p.trgswWords());
    detail::check(vsp_circuit_bootstrap_batch(bk.ctx(), flat.data(), out.data(), in.size()));
    return detail::split(out, p.trgswWords());
}

// cmux (ops.cpp:606-626): c0 + ExtProd(c1 - c0, sel).
inline Trlwe cmux(const Trgsw& sel, const Trlwe& c1, const Trlwe& c0, const BootstrappingKey& bk)
{
    const auto& p = bk.params();
    if (sel.size() != p.trgswWords() || c1.size() != p.trlweWords() || c0.size() != p.trlweWords())
        throw std::invalid_argument("cmux: dimension mismatch");
    Trlwe out(p.trlweWords());
    detail::check(vsp_cmux_batch(bk.ctx(), sel.data(), c1.data(), c0.data(), out.data(), 1));
    return out;
}

// homMuxNoSeIks (ops.cpp:898-909).
inline Trlwe homMuxNoSeIks(const Tlwe& sel, const Tlwe& a, const Tlwe& b,
                           const BootstrappingKey& bk)
{
    const auto& p = bk.params();
    if (sel.size() != p.tlweWords() || a.size() != p.tlweWords() || b.size() != p.tlweWords())
        throw std::invalid_argument("homMuxNoSeIks: dimension mismatch");
    Trlwe out(p.trlweWords());
    detail::check(
        vsp_hom_mux_no_se_iks_batch(bk.ctx(), sel.data(), a.data(), b.data(), out.data(), 1));
    return out;
}

// OpCounters (counters.hpp:11-28).
struct OpCounters {
    uint64_t cmux = 0, blindRotate = 0, identityKeySwitch = 0, privateKeySwitch = 0,
             circuitBootstrap = 0;
};
inline OpCounters counters(const BootstrappingKey& bk)
{
    uint64_t c[5];
    detail::check(vsp_counters(bk.ctx(), c));
    return {c[0], c[1], c[2], c[3], c[4]};
}
inline void resetCounters(const BootstrappingKey& bk) { detail::check(vsp_counters_reset(bk.ctx())); }

}  // namespace tfhe

namespace mem {

// hvp::mem::MemoryGeometry / EncryptedRam / EncryptedRom / RamCycleOut (mem.hpp:14-61,107-110).
struct MemoryGeometry {
    uint32_t v = 8;
    uint32_t w = 16;
    uint32_t words() const { return 1u << v; }
    size_t bits() const { return size_t{w} << v; }
    size_t imageBytes() const { return bits() / 8; }
};
struct EncryptedRam {
    MemoryGeometry geom;
    std::vector<tfhe::Trlwe> cells;  // cells[j * 2^v + A]
};
struct EncryptedRom {
    uint32_t depthBytes = 0;
    std::vector<tfhe::Trlwe> luts;
};
struct RamCycleOut {
    std::vector<tfhe::Tlwe> readOut;
    EncryptedRam ram;
};

// ramCycle (mem.cpp:122-135).  `threads` is accepted for signature compatibility; the
// parallelism is the GPU grid.
inline RamCycleOut ramCycle(const EncryptedRam& ram, std::span<const tfhe::Tlwe> addrBits,
                            const tfhe::Tlwe& writeFlag, std::span<const tfhe::Tlwe> writeData,
                            const tfhe::BootstrappingKey& bk, unsigned threads = 1)
{
    (void)threads;
    const auto& p = bk.params();
    const size_t tw = p.tlweWords(), rw = p.trlweWords();
    if (addrBits.size() != ram.geom.v || writeData.size() != ram.geom.w ||
        ram.cells.size() != ram.geom.bits() || writeFlag.size() != tw)
        throw std::invalid_argument("ramCycle: geometry mismatch");  // mem.cpp:126-127
    auto cells = detail::flatten(ram.cells, rw, "ramCycle");
    auto addr = detail::flatten(addrBits, tw, "ramCycle");
    auto wdata = detail::flatten(writeData, tw, "ramCycle");
    std::vector<uint32_t> rd(ram.geom.w * tw);
    detail::check(vsp_ram_cycle(bk.ctx(), ram.geom.v, ram.geom.w, cells.data(), addr.data(),
                                writeFlag.data(), wdata.data(), rd.data()));
    RamCycleOut out;
    out.readOut = detail::split(rd, tw);
    out.ram.geom = ram.geom;
    out.ram.cells = detail::split(cells, rw);
    return out;
}

// addressToTrgsw + prepareAddress + romRead (engine.cpp:133-143, mem.cpp:137-177):
// the 32-bit block at the encrypted block address (LSB-first TLWE bits).
inline std::vector<tfhe::Tlwe> romRead(const EncryptedRom& rom, std::span<const tfhe::Tlwe> addrBits,
                                       const tfhe::BootstrappingKey& bk, unsigned threads = 1)
{
    (void)threads;
    const auto& p = bk.params();
    auto luts = detail::flatten(rom.luts, p.trlweWords(), "romRead");
    auto addr = detail::flatten(addrBits, p.tlweWords(), "romRead");
    std::vector<uint32_t> out(32 * p.tlweWords());
    detail::check(vsp_rom_read(bk.ctx(), rom.depthBytes, luts.data(), (uint32_t)rom.luts.size(),
                               addr.data(), (uint32_t)addrBits.size(), out.data()));
    return detail::split(out, p.tlweWords());
}

}  // namespace mem

namespace netlist {

// hvp::netlist::CellKind (netlist.hpp:12-28), same order.
enum class CellKind : int32_t {
    And, AndNot, Mux, Nand, Nor, Not, Or, OrNot, Xnor, Xor, Dff, RomPort, RamPort, Const0, Const1
};

// The reference Backend concept (engine.hpp:48-98) on the GPU engine.  Satisfies what
// hvp::netlist::Evaluator<B> requires (Bit, Rom, Ram, tag, constant, gate, romRead,
// ramCycle); `gate` accepts any cell-kind enum with the reference's numbering, so the
// reference's own Evaluator template can be instantiated on it.  Per-cell calls are
// batches of one: use Runner for level-batched throughput.
struct GpuBackend {
    using Bit = tfhe::Tlwe;
    struct Rom {
        mem::EncryptedRom enc;
    };
    struct Ram {
        mem::EncryptedRam enc;
    };
    static constexpr const char* tag = "tfhe";

    const tfhe::BootstrappingKey* bk = nullptr;
    unsigned threads = 1;

    Bit constant(bool b) const { return tfhe::tlweTrivial(b, bk->params()); }

    template <class Kind>
    Bit gate(Kind kind, std::span<const Bit* const> in) const  // engine.cpp:113-121
    {
        std::vector<tfhe::Tlwe> ops;
        ops.reserve(in.size());
        for (const Bit* b : in)
            ops.push_back(*b);
        return tfhe::homGate(static_cast<tfhe::GateKind>(static_cast<int32_t>(kind)), ops, *bk);
    }
    std::vector<Bit> romRead(const Rom& rom, std::span<const Bit* const> addr) const
    {
        std::vector<tfhe::Tlwe> a;
        for (const Bit* b : addr)
            a.push_back(*b);
        return mem::romRead(rom.enc, a, *bk, threads);
    }
    std::vector<Bit> ramCycle(Ram& ram, std::span<const Bit* const> addr, const Bit& wflag,
                              std::span<const Bit* const> wdata) const  // engine.cpp:145-148
    {
        std::vector<tfhe::Tlwe> a, d;
        for (const Bit* b : addr)
            a.push_back(*b);
        for (const Bit* b : wdata)
            d.push_back(*b);
        auto r = mem::ramCycle(ram.enc, a, wflag, d, *bk, threads);
        ram.enc = std::move(r.ram);
        return std::move(r.readOut);
    }
};

// CycleStats / RunOptions (engine.hpp:22-43).  The runner is level-synchronous, so
// `workers` and `shuffleSeed` have no effect on it (results never depended on them).
struct CycleStats {
    uint64_t evaluated = 0;
    int gMax = 0;
    int depth = 0;
    double wallSeconds = 0.0;  // device time of the cycle
};
struct RunOptions {
    unsigned workers = 1;
    uint64_t shuffleSeed = 0;
    std::vector<CycleStats>* stats = nullptr;
};

// The level-batched runner with hvp::netlist::Evaluator's surface (engine.hpp:107-247):
// one batched launch sequence per ASAP level; value table, DFFs, RAM and ROM stay in HBM.
class Runner {
public:
    // Flat form of hvp::netlist::Netlist (netlist.hpp:44-63): cell kinds and ids, CSR lists
    // of input/output nets in the reference pin order, and the nets of every module input.
    Runner(const tfhe::BootstrappingKey& bk, int32_t netCount, std::span<const int32_t> kinds,
           std::span<const int32_t> ids, std::span<const int32_t> inOff,
           std::span<const int32_t> inNets, std::span<const int32_t> outOff,
           std::span<const int32_t> outNets, std::span<const int32_t> inputNets)
        : bk_(&bk), inputNets_(inputNets.begin(), inputNets.end())
    {
        h_ = vsp_netlist_create(bk.ctx(), netCount, (int32_t)kinds.size(), kinds.data(),
                                ids.data(), inOff.data(), inNets.data(), outOff.data(),
                                outNets.data(), inputNets.data(), (int32_t)inputNets.size());
        if (!h_)
            detail::raise(VSP_ERUNTIME, vsp_last_error());
        int32_t info[6];
        detail::check(vsp_netlist_info(h_, info, nullptr));
        dagNodes_ = info[0];
        dffs_ = info[1];
        gMax_ = info[2];
        depth_ = info[3];
    }

    // From any netlist type shaped like hvp::netlist::Netlist (cells[].kind/id/inputs/
    // outputs, inputs[].bits, netCount), e.g. the reference's own parseNetlist result.
    template <class NetlistT>
    static Runner fromNetlist(const tfhe::BootstrappingKey& bk, const NetlistT& nl)
    {
        std::vector<int32_t> kinds, ids, inOff{0}, inNets, outOff{0}, outNets, inputNets;
        for (const auto& c : nl.cells) {
            kinds.push_back(static_cast<int32_t>(c.kind));
            ids.push_back(c.id);
            inNets.insert(inNets.end(), c.inputs.begin(), c.inputs.end());
            outNets.insert(outNets.end(), c.outputs.begin(), c.outputs.end());
            inOff.push_back((int32_t)inNets.size());
            outOff.push_back((int32_t)outNets.size());
        }
        for (const auto& port : nl.inputs)
            inputNets.insert(inputNets.end(), port.bits.begin(), port.bits.end());
        Runner r(bk, nl.netCount, kinds, ids, inOff, inNets, outOff, outNets, inputNets);
        r.setName(nl.name);
        return r;
    }

    Runner(const Runner&) = delete;
    Runner& operator=(const Runner&) = delete;
    Runner(Runner&& o) noexcept
        : bk_(o.bk_), h_(std::exchange(o.h_, nullptr)), inputNets_(std::move(o.inputNets_)),
          dagNodes_(o.dagNodes_), dffs_(o.dffs_), gMax_(o.gMax_), depth_(o.depth_)
    {
    }
    ~Runner()
    {
        if (h_)
            vsp_netlist_destroy(h_);
    }

    int gMax() const { return gMax_; }
    int depth() const { return depth_; }
    int dffCount() const { return dffs_; }
    uint64_t cycle() const { return vsp_netlist_cycle(h_); }
    void setCycle(uint64_t c) { detail::check(vsp_netlist_set_cycle(h_, c)); }

    // setInput by index into the concatenated input-port bits (engine.hpp:160-163).
    void setInput(size_t inputIndex, const tfhe::Tlwe& v)
    {
        check_tlwe(v);
        detail::check(vsp_netlist_set_input(h_, (int32_t)inputIndex, v.data()));
    }
    // Value of any net (Evaluator::output semantics, engine.hpp:165-176).
    tfhe::Tlwe net(int32_t net) const
    {
        tfhe::Tlwe v(bk_->params().tlweWords());
        detail::check(vsp_netlist_get_net(h_, net, v.data()));
        return v;
    }
    std::vector<tfhe::Tlwe> dffState() const
    {
        const size_t w = bk_->params().tlweWords();
        std::vector<uint32_t> flat(dffs_ * w);
        detail::check(vsp_netlist_dff(h_, flat.data(), nullptr));
        return detail::split(flat, w);
    }
    void setDffStateRaw(const std::vector<tfhe::Tlwe>& state)
    {
        if ((int)state.size() != dffs_)
            throw std::runtime_error("DFF state size mismatch");  // engine.hpp:188-189
        auto flat = detail::flatten(state, bk_->params().tlweWords(), "setDffStateRaw");
        detail::check(vsp_netlist_dff(h_, nullptr, flat.data()));
    }
    void setRom(const mem::EncryptedRom& rom)
    {
        auto flat = detail::flatten(rom.luts, bk_->params().trlweWords(), "setRom");
        detail::check(vsp_netlist_set_rom(h_, rom.depthBytes, flat.data(), (uint32_t)rom.luts.size()));
    }
    void setRam(const mem::EncryptedRam& ram)
    {
        auto flat = detail::flatten(ram.cells, bk_->params().trlweWords(), "setRam");
        detail::check(vsp_netlist_ram(h_, ram.geom.v, ram.geom.w, nullptr, flat.data()));
        geom_ = ram.geom;
    }
    mem::EncryptedRam ram() const
    {
        std::vector<uint32_t> flat(geom_.bits() * bk_->params().trlweWords());
        detail::check(vsp_netlist_ram(h_, geom_.v, geom_.w, flat.data(), nullptr));
        return {geom_, detail::split(flat, bk_->params().trlweWords())};
    }

    // snapshotSave / snapshotLoad (snapshot.hpp:17-29): the reference's HVPS bytes,
    // interchangeable with hvp::netlist::Evaluator<TfheBackend> snapshots.
    void setName(const std::string& name) { detail::check(vsp_netlist_set_name(h_, name.c_str())); }
    std::vector<uint8_t> snapshotSave() const
    {
        size_t n = 0;
        detail::check(vsp_netlist_snapshot_save(h_, bk_->params().name.c_str(), nullptr, 0, &n));
        std::vector<uint8_t> b(n);
        detail::check(vsp_netlist_snapshot_save(h_, bk_->params().name.c_str(), b.data(), n, &n));
        return b;
    }
    void snapshotLoad(const std::vector<uint8_t>& bytes)
    {
        detail::check(vsp_netlist_snapshot_load(h_, bk_->params().name.c_str(), bytes.data(),
                                                bytes.size()));
        uint32_t v = 0, w = 0;
        if (vsp_netlist_ram_geometry(h_, &v, &w) == VSP_OK)
            geom_ = {v, w};
    }

    // Evaluator::run (engine.hpp:238-247).
    void run(uint64_t cycles, const RunOptions& opt = {})
    {
        std::vector<double> st(4 * cycles);
        detail::check(vsp_netlist_run(h_, cycles, st.data()));
        if (opt.stats)
            for (uint64_t i = 0; i < cycles; i++)
                opt.stats->push_back({(uint64_t)st[4 * i], (int)st[4 * i + 1],
                                      (int)st[4 * i + 2], st[4 * i + 3]});
    }

private:
    void check_tlwe(const tfhe::Tlwe& v) const
    {
        if (v.size() != bk_->params().tlweWords())
            throw std::invalid_argument("netlist: ciphertext dimension mismatch");
    }
    const tfhe::BootstrappingKey* bk_;
    vsp_netlist* h_ = nullptr;
    std::vector<int32_t> inputNets_;
    int dagNodes_ = 0, dffs_ = 0, gMax_ = 0, depth_ = 0;
    mem::MemoryGeometry geom_{};
};

}  // namespace netlist
}  // namespace vsp

#endif
