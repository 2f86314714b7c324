// TEST ONLY — the drop-in proof for the netlist-runner boundary.
//
// Instantiates the REFERENCE's own hvp::netlist::Evaluator template (engine.hpp:107-405,
// compiled from /root/reference with the two-member fix, oracle/Makefile) on two
// backends over the same keys, netlist and ciphertexts:
//   Evaluator<hvp::netlist::TfheBackend>   the reference CPU backend (engine.cpp:113-148)
//   Evaluator<vsp::netlist::GpuBackend>    this engine, through include/vsp_b200.hpp
// and requires every output, DFF state and RAM cell to be identical word for word after
// several cycles.  Also checks vsp::netlist::Runner (the level-batched runner) against
// the same reference run.  Built by tests/cpp/Makefile only where /root/reference exists;
// run by tests/test_cpp_gpu.py.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "hvp/mem/mem.hpp"
#include "hvp/netlist/engine.hpp"
#include "hvp/netlist/netlist.hpp"
#include "hvp/netlist/snapshot.hpp"
#include "hvp/tfhe/ops.hpp"
#include "vsp_b200.hpp"

static int g_fail = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            g_fail++;                                                            \
        }                                                                        \
    } while (0)

static std::vector<uint32_t> flat(const hvp::tfhe::Tlwe& t)
{
    std::vector<uint32_t> v(t.a);
    v.push_back(t.b);
    return v;
}
static std::vector<uint32_t> flat(const hvp::tfhe::Trlwe& t)
{
    std::vector<uint32_t> v(t.a);
    v.insert(v.end(), t.b.begin(), t.b.end());
    return v;
}

// Ripple-carry accumulator: 4-bit register R (DFFs) += input X every cycle, with a 2x2
// RAM port addressed by R[1:0], written with R[1:0] when X[0] is set.  Gates of every
// kind that a pipelined processor netlist uses (AND/XOR/OR/MUX/NOT/NAND/...).
static std::string netlist_json()
{
    std::string cells;
    int id = 1;
    auto cell = [&](const std::string& kind, const std::string& pins) {
        if (!cells.empty())
            cells += ",";
        cells += "{\"id\":" + std::to_string(id++) + ",\"kind\":\"" + kind + "\",\"pins\":{" +
                 pins + "}}";
    };
    auto p2 = [](int a, int b, int y) {
        return "\"a\":" + std::to_string(a) + ",\"b\":" + std::to_string(b) +
               ",\"y\":" + std::to_string(y);
    };
    // nets: X 0..3, R(q) 4..7, sum 8..11, carries 12..15, scratch from 16
    int net = 16;
    int carry = -1;
    for (int i = 0; i < 4; i++) {
        const int x = i, r = 4 + i, s = 8 + i;
        if (carry < 0) {
            cell("XOR", p2(x, r, s));
            carry = 12;
            cell("AND", p2(x, r, carry));
        }
        else {
            const int t = net++;
            cell("XOR", p2(x, r, t));
            cell("XNOR", p2(t, carry, net));  // s = NOT XNOR = XOR
            cell("NOT", "\"a\":" + std::to_string(net) + ",\"y\":" + std::to_string(s));
            net++;
            const int g = net++, pr = net++;
            cell("AND", p2(x, r, g));
            cell("NAND", p2(t, carry, pr));  // ~(t & c)
            const int c2 = 12 + i;
            cell("ORNOT", p2(g, pr, c2));  // g | ~~(t&c)
            carry = c2;
        }
    }
    for (int i = 0; i < 4; i++)
        cell("DFF", "\"d\":" + std::to_string(8 + i) + ",\"q\":" + std::to_string(4 + i));
    // RAM v=2, w=2: addr = R[1:0], wdata = {R[0] MUX, R[1] ANDNOT}, wflag = X[0]
    const int w0 = net++, w1 = net++, rd0 = net++, rd1 = net++;
    cell("MUX", "\"s\":0,\"a\":4,\"b\":5,\"y\":" + std::to_string(w0));
    cell("ANDNOT", p2(5, 1, w1));
    cell("RAM", "\"addr\":[4,5],\"wdata\":[" + std::to_string(w0) + "," + std::to_string(w1) +
                    "],\"wflag\":0,\"rdata\":[" + std::to_string(rd0) + "," +
                    std::to_string(rd1) + "]");
    const int o = net++;
    cell("NOR", p2(rd0, rd1, o));
    cell("OR", p2(rd0, 15, net++));
    return "{\"name\":\"acc4\",\"ports\":{\"in\":[{\"name\":\"X\",\"bits\":[0,1,2,3]}],"
           "\"out\":[{\"name\":\"S\",\"bits\":[8,9,10,11]},{\"name\":\"R\",\"bits\":[" +
           std::to_string(rd0) + "," + std::to_string(rd1) + "," + std::to_string(o) +
           "]}]},\"cells\":[" + cells + "]}";
}

int main()
{
    using namespace hvp;
    try {
        const uint64_t seed = 515253;
        // the reference's key generation and ours, from the same seed (identical keys,
        // tests/test_client.py)
        tfhe::ParameterSet P = tfhe::ParameterSet::byName("test-det");
        tfhe::Csprng rng = tfhe::Csprng::fromSeed(seed);
        tfhe::SecretKey sk = tfhe::genSecretKey(P, rng);
        tfhe::BootstrappingKey refBk = tfhe::BootstrappingKey::generate(sk, rng, true);
        auto km = vsp::tfhe::KeyMaterial::generate(vsp::tfhe::ParameterSet::byName("test-det"),
                                                   seed, 1);
        CHECK(km.lv0 == sk.lv0);
        vsp::tfhe::BootstrappingKey gpuBk(km, 0);

        const netlist::Netlist nl = netlist::parseNetlist(netlist_json());
        netlist::TfheBackend rb;
        rb.bk = &refBk;
        rb.threads = 4;
        vsp::netlist::GpuBackend gb;
        gb.bk = &gpuBk;
        netlist::Evaluator<netlist::TfheBackend> ref(nl, rb);
        netlist::Evaluator<vsp::netlist::GpuBackend> gpu(nl, gb);
        auto runner = vsp::netlist::Runner::fromNetlist(gpuBk, nl);

        // same encrypted RAM image for all three
        mem::MemoryGeometry geom{2, 2};
        const std::vector<uint8_t> image{0xB4};
        tfhe::NoiseSampler ns(rng, P.alpha0);
        mem::EncryptedRam eram = mem::encryptRam(image, geom, *sk.params, &sk, &ns);
        vsp::mem::EncryptedRam vram;
        vram.geom = {2, 2};
        for (const auto& c : eram.cells)
            vram.cells.push_back(flat(c));
        ref.setRam({eram});
        gpu.setRam({{vram}});
        runner.setRam(vram);

        std::mt19937 mt(3);
        for (int cyc = 0; cyc < 4; cyc++) {
            for (int i = 0; i < 4; i++) {
                const bool bit = mt() & 1;
                tfhe::Tlwe x = tfhe::tlweEncrypt(bit, sk, ns);
                ref.setInput("X", i, x);
                gpu.setInput("X", i, flat(x));
                runner.setInput(i, flat(x));
            }
            ref.run(1);
            gpu.run(1);
            runner.run(1);
            for (int i = 0; i < 4; i++) {
                CHECK(flat(ref.output("S", i)) == gpu.output("S", i));
                CHECK(flat(ref.output("S", i)) == runner.net(nl.outputs[0].bits[i]));
            }
            for (int i = 0; i < 3; i++) {
                CHECK(flat(ref.output("R", i)) == gpu.output("R", i));
                CHECK(flat(ref.output("R", i)) == runner.net(nl.outputs[1].bits[i]));
            }
            const auto rs = ref.dffState();
            const auto gs = gpu.dffState();
            const auto us = runner.dffState();
            CHECK(rs.size() == gs.size() && rs.size() == us.size());
            for (size_t i = 0; i < rs.size() && i < gs.size() && i < us.size(); i++) {
                CHECK(flat(rs[i]) == gs[i]);
                CHECK(flat(rs[i]) == us[i]);
            }
        }
        // HVPS snapshots are interchangeable: the runner's bytes == the reference's
        const std::vector<uint8_t> refSnap = netlist::snapshotSave(ref);
        CHECK(runner.snapshotSave() == refSnap);
        auto resumed = vsp::netlist::Runner::fromNetlist(gpuBk, nl);
        resumed.snapshotLoad(refSnap);
        CHECK(resumed.cycle() == 4 && resumed.dffState() == runner.dffState());
        const auto& rc = ref.ram().enc.cells;
        const auto& gc = gpu.ram().enc.cells;
        const auto uc = runner.ram().cells;
        for (size_t i = 0; i < rc.size(); i++) {
            CHECK(flat(rc[i]) == gc[i]);
            CHECK(flat(rc[i]) == uc[i]);
        }
        std::printf("Evaluator<TfheBackend> == Evaluator<vsp::GpuBackend> == vsp::Runner over "
                    "4 cycles (%zu cells, %zu RAM cells)\n", nl.cells.size(), rc.size());
    }
    catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 2;
    }
    if (g_fail) {
        std::fprintf(stderr, "%d checks failed\n", g_fail);
        return 1;
    }
    std::printf("test_dropin_evaluator OK\n");
    return 0;
}
