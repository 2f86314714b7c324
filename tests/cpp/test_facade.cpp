// GPU test of the C++ host facade (include/vsp_b200.hpp) through the C ABI.
// Built by tests/cpp/Makefile; run by tests/test_cpp_gpu.py.  Exit code 0 = pass.
//
// Mirrors the reference's own tests for the path:
//   truth tables of all 10 gates (test_tfhe.cpp:509-575), half adder (:577-599),
//   arity errors (ops.cpp:844-846), ramCycle read-before-write against a plaintext RAM
//   (test_mem.cpp:30-43, 256-344), and the Evaluator surface (engine.hpp:107-247).
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>
#include <vector>

#include "vsp_b200.hpp"

using namespace vsp;
using tfhe::GateKind;
using tfhe::Tlwe;

static int g_fail = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            g_fail++;                                                            \
        }                                                                        \
    } while (0)

static bool plain(GateKind k, int a, int b, int c)
{
    switch (k) {
    case GateKind::And: return a & b;
    case GateKind::AndNot: return a & !b;
    case GateKind::Mux: return a ? b : c;  // {s, a, b}: s ? a : b
    case GateKind::Nand: return !(a & b);
    case GateKind::Nor: return !(a | b);
    case GateKind::Not: return !a;
    case GateKind::Or: return a | b;
    case GateKind::OrNot: return a | !b;
    case GateKind::Xnor: return !(a ^ b);
    case GateKind::Xor: return a ^ b;
    }
    return false;
}

static void gates(const tfhe::KeyMaterial& km, const tfhe::BootstrappingKey& bk)
{
    const auto& p = km.params;
    std::vector<GateKind> kinds;
    std::vector<std::vector<Tlwe>> ins;
    std::vector<int> expect;
    uint64_t seed = 100;
    for (int k = 0; k < 10; k++)
        for (int m = 0; m < 8; m++) {
            const GateKind kind = static_cast<GateKind>(k);
            const int ar = kind == GateKind::Not ? 1 : kind == GateKind::Mux ? 3 : 2;
            if (m >= (1 << ar))
                continue;
            std::vector<uint8_t> bits(ar);
            for (int i = 0; i < ar; i++)
                bits[i] = (m >> i) & 1;
            ins.push_back(tfhe::tlweEncrypt(p, km.lv0, bits, seed++));
            kinds.push_back(kind);
            expect.push_back(plain(kind, bits[0], ar > 1 ? bits[1] : 0, ar > 2 ? bits[2] : 0));
        }
    auto out = tfhe::homGateBatch(kinds, ins, bk);
    CHECK(out.size() == kinds.size());
    for (size_t g = 0; g < out.size(); g++) {
        CHECK(tfhe::tlweDecrypt(out[g], km.lv0) == (expect[g] != 0));
        // one gate through homGate == the same gate inside the batch, word for word
        if (g % 7 == 0)
            CHECK(tfhe::homGate(kinds[g], ins[g], bk) == out[g]);
    }
    // arity errors keep the reference's exception type (ops.cpp:844-846)
    bool threw = false;
    try {
        tfhe::homGate(GateKind::Nand, std::vector<Tlwe>(1, ins[0][0]), bk);
    }
    catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    // NOT o NOT is the identity, byte for byte (test_tfhe.cpp:557-568)
    auto n1 = tfhe::homGate(GateKind::Not, std::vector<Tlwe>{ins[0][0]}, bk);
    auto n2 = tfhe::homGate(GateKind::Not, std::vector<Tlwe>{n1}, bk);
    CHECK(n2 == ins[0][0]);
    std::printf("gates %s: %zu gates ok\n", p.name.c_str(), out.size());
}

static void ram(const tfhe::KeyMaterial& km, const tfhe::BootstrappingKey& bk)
{
    const auto& p = km.params;
    const uint32_t v = 2, w = 2;
    std::mt19937 rng(7);
    std::vector<uint8_t> words(1u << v);
    mem::EncryptedRam ram;
    ram.geom = {v, w};
    ram.cells.resize(ram.geom.bits());
    for (auto& x : words)
        x = rng() & ((1u << w) - 1);
    // encryptRam (mem.cpp:202-222): cell j*2^v + A carries bit j of word A at coefficient 0
    for (uint32_t j = 0; j < w; j++)
        for (uint32_t A = 0; A < (1u << v); A++) {
            std::vector<uint8_t> poly(p.raw.N1, 0);
            poly[0] = (words[A] >> j) & 1;
            tfhe::Trlwe c(p.trlweWords());
            if (vsp_client_trlwe_encrypt(&p.raw, km.lv1.data(), 1000 + j * 16 + A, poly.data(), 1,
                                         c.data()) != 0)
                throw std::runtime_error(vsp_client_last_error());
            ram.cells[j * (1u << v) + A] = c;
        }
    for (int cyc = 0; cyc < 6; cyc++) {
        const uint32_t addr = rng() & ((1u << v) - 1), wflag = rng() & 1,
                       wdata = rng() & ((1u << w) - 1);
        std::vector<uint8_t> ab(v), db(w), fb{(uint8_t)wflag};
        for (uint32_t i = 0; i < v; i++)
            ab[i] = (addr >> i) & 1;
        for (uint32_t j = 0; j < w; j++)
            db[j] = (wdata >> j) & 1;
        auto ea = tfhe::tlweEncrypt(p, km.lv0, ab, 50 + cyc);
        auto ed = tfhe::tlweEncrypt(p, km.lv0, db, 60 + cyc);
        auto ef = tfhe::tlweEncrypt(p, km.lv0, fb, 70 + cyc)[0];
        auto r = mem::ramCycle(ram, ea, ef, ed, bk);
        uint32_t got = 0;
        for (uint32_t j = 0; j < w; j++)
            got |= (uint32_t)tfhe::tlweDecrypt(r.readOut[j], km.lv0) << j;
        CHECK(got == words[addr]);  // read-before-write (test_mem.cpp:330-344)
        if (wflag)
            words[addr] = (uint8_t)wdata;
        ram = std::move(r.ram);
    }
    auto c = tfhe::counters(bk);
    CHECK(c.circuitBootstrap > 0 && c.cmux > 0);
    std::printf("ramCycle %s: 6 cycles ok (cmux %llu, cb %llu)\n", p.name.c_str(),
                (unsigned long long)c.cmux, (unsigned long long)c.circuitBootstrap);
}

static void runner(const tfhe::KeyMaterial& km, const tfhe::BootstrappingKey& bk)
{
    // half adder (nets 0,1 -> S 5, C 6) + a toggling DFF (q 7, d 8 = NOT q)
    using K = netlist::CellKind;
    std::vector<int32_t> kinds{(int32_t)K::Nand, (int32_t)K::Nand, (int32_t)K::Nand,
                               (int32_t)K::Nand, (int32_t)K::Not,  (int32_t)K::Dff,
                               (int32_t)K::Not};
    std::vector<int32_t> ids{1, 2, 3, 4, 5, 6, 7};
    std::vector<int32_t> inOff{0, 2, 4, 6, 8, 9, 10, 11}, inNets{0, 1, 0, 2, 2, 1, 3, 4, 2, 8, 7};
    std::vector<int32_t> outOff{0, 1, 2, 3, 4, 5, 6, 7}, outNets{2, 3, 4, 5, 6, 7, 8};
    std::vector<int32_t> inputNets{0, 1};
    netlist::Runner r(bk, 9, kinds, ids, inOff, inNets, outOff, outNets, inputNets);
    CHECK(r.depth() == 3 && r.dffCount() == 1);
    const auto& p = km.params;
    int q = 0;
    for (int m = 0; m < 4; m++) {
        std::vector<uint8_t> bits{(uint8_t)(m & 1), (uint8_t)(m >> 1)};
        auto e = tfhe::tlweEncrypt(p, km.lv0, bits, 300 + m);
        r.setInput(0, e[0]);
        r.setInput(1, e[1]);
        std::vector<netlist::CycleStats> st;
        r.run(1, {1, 0, &st});
        CHECK(st.size() == 1 && st[0].depth == 3);
        CHECK(tfhe::tlweDecrypt(r.net(5), km.lv0) == (((m & 1) ^ (m >> 1)) != 0));
        CHECK(tfhe::tlweDecrypt(r.net(6), km.lv0) == (((m & 1) & (m >> 1)) != 0));
        q ^= 1;
        CHECK(tfhe::tlweDecrypt(r.dffState()[0], km.lv0) == (q != 0));
    }
    CHECK(r.cycle() == 4);
    std::printf("runner %s: half adder + DFF over 4 cycles ok\n", p.name.c_str());
}

int main()
{
    try {
        auto det = tfhe::KeyMaterial::generate(tfhe::ParameterSet::byName("test-det"), 515253, 1);
        tfhe::BootstrappingKey bkd(det, 0);
        gates(det, bkd);
        ram(det, bkd);
        runner(det, bkd);
        auto prod = tfhe::KeyMaterial::generate(tfhe::ParameterSet::byName("tfhe-80", 630), 630, 0);
        tfhe::BootstrappingKey bkp(prod, 0);
        gates(prod, bkp);
        runner(prod, bkp);
    }
    catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 2;
    }
    if (g_fail) {
        std::fprintf(stderr, "%d checks failed\n", g_fail);
        return 1;
    }
    std::printf("test_facade OK\n");
    return 0;
}
