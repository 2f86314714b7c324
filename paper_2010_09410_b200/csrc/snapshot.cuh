// Snapshot / resume of the device-resident runner state in the reference's "HVPS" file
// format (snapshot.cpp:13-176, snapshot.hpp:10-33), byte-compatible: a snapshot taken
// here loads into hvp::netlist::snapshotLoad and vice versa (tests/test_snapshot_gpu.py).
//
//   "HVPS" u16 version=1 u8 backend(1 = tfhe) str param-name str netlist-name
//   u64 netlistHash (engine.cpp:150-168) u64 cycle
//   u32 #dff, per DFF writeTlwe (serialize.cpp:39-44): u8 level, u32vec a, u32 b
//   u8 hasRam [writeRam (mem.cpp:331-338): u32 v, u32 w, u32 #cells, writeTrlwe each]
//   u8 hasRom [writeRom (mem.cpp:370-376): u32 depthBytes, u32 #luts, writeTrlwe each]
// writeTrlwe (serialize.cpp:55-60): u8 level, u32vec a, u32vec b.  All little-endian
// (BinWriter, binio.hpp:14-68); str = u16 length + bytes.  Included by vsp_capi.cu.
#pragma once

namespace {

struct SnapWriter {
    std::vector<uint8_t> b;
    void u8(uint8_t v) { b.push_back(v); }
    void u16(uint16_t v)
    {
        for (int i = 0; i < 2; i++)
            b.push_back((uint8_t)(v >> (8 * i)));
    }
    void u32(uint32_t v)
    {
        for (int i = 0; i < 4; i++)
            b.push_back((uint8_t)(v >> (8 * i)));
    }
    void u64(uint64_t v)
    {
        for (int i = 0; i < 8; i++)
            b.push_back((uint8_t)(v >> (8 * i)));
    }
    void raw(const void* p, size_t n)
    {
        const uint8_t* q = static_cast<const uint8_t*>(p);
        b.insert(b.end(), q, q + n);
    }
    void str(const std::string& s)
    {
        if (s.size() > 0xFFFF)
            throw std::invalid_argument("string too long to serialize");
        u16((uint16_t)s.size());
        raw(s.data(), s.size());
    }
    void u32vec(const uint32_t* p, size_t n)
    {
        u32((uint32_t)n);
        raw(p, n * 4);  // little-endian host (x86-64 / aarch64)
    }
};

struct SnapReader {
    const uint8_t* p;
    const uint8_t* end;
    void need(size_t n)
    {
        if ((size_t)(end - p) < n)
            throw std::runtime_error("truncated input");  // BinReader::need (binio.hpp)
    }
    uint64_t le(int bytes)
    {
        need(bytes);
        uint64_t v = 0;
        for (int i = 0; i < bytes; i++)
            v |= (uint64_t)p[i] << (8 * i);
        p += bytes;
        return v;
    }
    uint8_t u8() { return (uint8_t)le(1); }
    uint16_t u16() { return (uint16_t)le(2); }
    uint32_t u32() { return (uint32_t)le(4); }
    uint64_t u64() { return le(8); }
    std::string str()
    {
        const uint16_t n = u16();
        need(n);
        std::string s(reinterpret_cast<const char*>(p), n);
        p += n;
        return s;
    }
    void u32vec(uint32_t* dst, size_t expect, const char* what)
    {
        const uint32_t n = u32();
        if (n != expect)
            throw std::runtime_error(std::string("snapshot: ") + what + " dimension mismatch");
        need((size_t)n * 4);
        std::memcpy(dst, p, (size_t)n * 4);
        p += (size_t)n * 4;
    }
};

constexpr char kSnapMagic[4] = {'H', 'V', 'P', 'S'};
constexpr uint16_t kSnapVersion = 1;
constexpr uint8_t kSnapTfhe = 1;

// netlistHash (engine.cpp:150-168): FNV-1a style over the structure.
uint64_t netlist_hash(const vsp_netlist* nl)
{
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) {
        h ^= v;
        h *= 1099511628211ull;
    };
    mix((uint64_t)nl->nets);
    mix((uint64_t)nl->kind.size());
    for (size_t c = 0; c < nl->kind.size(); c++) {
        mix((uint64_t)(int64_t)nl->id[c]);
        mix((uint64_t)nl->kind[c]);
        for (int k = nl->in_off[c]; k < nl->in_off[c + 1]; k++)
            mix((uint64_t)(int64_t)nl->in_nets[k] + 0x9e3779b9);
        for (int k = nl->out_off[c]; k < nl->out_off[c + 1]; k++)
            mix((uint64_t)(int64_t)nl->out_nets[k] + 0x7f4a7c15);
    }
    return h;
}

void snap_trlwe(SnapWriter& w, const uint32_t* t, uint32_t N)
{
    w.u8(1);  // level 1
    w.u32vec(t, N);
    w.u32vec(t + N, N);
}

void read_trlwe(SnapReader& r, uint32_t* t, uint32_t N)
{
    (void)r.u8();
    r.u32vec(t, N, "TRLWE");
    r.u32vec(t + N, N, "TRLWE");
}

// snapshotSave(const Evaluator<TfheBackend>&) (snapshot.cpp:84-101) of the runner state.
std::vector<uint8_t> snapshot_save(vsp_netlist* nl, const std::string& param_name)
{
    vsp_ctx* c = nl->ctx;
    const uint32_t n = c->p.n, N = c->p.N1;
    SnapWriter w;
    w.raw(kSnapMagic, 4);
    w.u16(kSnapVersion);
    w.u8(kSnapTfhe);
    w.str(param_name);
    w.str(nl->name);
    w.u64(netlist_hash(nl));
    w.u64(nl->cycle);
    const size_t nd = nl->dff_cells.size();
    std::vector<uint32_t> dff(nd * (n + 1));
    if (nd)
        VSP_CUDA_CHECK(cudaMemcpy(dff.data(), nl->dff.as<uint32_t>(0), dff.size() * 4,
                                  cudaMemcpyDeviceToHost));
    w.u32((uint32_t)nd);
    for (size_t i = 0; i < nd; i++) {
        w.u8(0);  // level 0
        w.u32vec(&dff[i * (n + 1)], n);
        w.u32(dff[i * (n + 1) + n]);
    }
    w.u8(nl->has_ram ? 1 : 0);
    if (nl->has_ram) {
        const size_t cells = (size_t)nl->ram_w << nl->ram_v;
        std::vector<uint32_t> ram(cells * 2 * N);
        VSP_CUDA_CHECK(cudaMemcpy(ram.data(), nl->ram.as<uint32_t>(0), ram.size() * 4,
                                  cudaMemcpyDeviceToHost));
        w.u32(nl->ram_v);
        w.u32(nl->ram_w);
        w.u32((uint32_t)cells);
        for (size_t i = 0; i < cells; i++)
            snap_trlwe(w, &ram[i * 2 * N], N);
    }
    w.u8(nl->has_rom ? 1 : 0);
    if (nl->has_rom) {
        std::vector<uint32_t> rom((size_t)nl->rom_nluts * 2 * N);
        VSP_CUDA_CHECK(cudaMemcpy(rom.data(), nl->rom.as<uint32_t>(0), rom.size() * 4,
                                  cudaMemcpyDeviceToHost));
        w.u32(nl->rom_depth);
        w.u32(nl->rom_nluts);
        for (uint32_t t = 0; t < nl->rom_nluts; t++)
            snap_trlwe(w, &rom[(size_t)t * 2 * N], N);
    }
    return std::move(w.b);
}

// snapshotLoad(nl, TfheBackend, bytes) (snapshot.cpp:124-158): checks, then restores the
// cycle counter, DFF state, RAM and ROM into the device-resident runner.
void snapshot_load(vsp_netlist* nl, const std::string& param_name, const uint8_t* bytes,
                   size_t len)
{
    vsp_ctx* c = nl->ctx;
    const uint32_t n = c->p.n, N = c->p.N1;
    SnapReader r{bytes, bytes + len};
    r.need(4);
    if (std::memcmp(r.p, kSnapMagic, 4) != 0)
        throw std::runtime_error("bad snapshot magic (expected HVPS)");
    r.p += 4;
    const uint16_t version = r.u16();
    if (version != kSnapVersion)
        throw std::runtime_error("unsupported snapshot version " + std::to_string(version));
    if (r.u8() != kSnapTfhe)
        throw std::runtime_error("snapshot backend is not 'tfhe'");
    const std::string pname = r.str();
    if (pname != param_name)
        throw std::runtime_error("snapshot parameter set '" + pname +
                                 "' does not match key '" + param_name + "'");
    const std::string nname = r.str();
    const uint64_t hash = r.u64();
    if (nname != nl->name || hash != netlist_hash(nl))
        throw std::runtime_error("snapshot was taken on netlist '" + nname + "', not '" +
                                 nl->name + "'");
    const uint64_t cycle = r.u64();
    const uint32_t nd = r.u32();
    if (nd != nl->dff_cells.size())
        throw std::runtime_error("DFF state size mismatch");  // setDffStateRaw
    std::vector<uint32_t> dff((size_t)nd * (n + 1));
    for (uint32_t i = 0; i < nd; i++) {
        (void)r.u8();
        r.u32vec(&dff[(size_t)i * (n + 1)], n, "TLWE");
        dff[(size_t)i * (n + 1) + n] = r.u32();
    }
    std::vector<uint32_t> ram, rom;
    uint32_t v = 0, w = 0, depth = 0, nluts = 0;
    const bool has_ram = r.u8() != 0;
    if (has_ram) {
        if (nl->ram_cell < 0)
            throw std::runtime_error("netlist has no RAM port");
        v = r.u32();
        w = r.u32();
        const uint32_t cells = r.u32();
        if (cells != ((size_t)w << v))
            throw std::runtime_error("corrupt RAM: cell count mismatch");
        ram.resize((size_t)cells * 2 * N);
        for (uint32_t i = 0; i < cells; i++)
            read_trlwe(r, &ram[(size_t)i * 2 * N], N);
    }
    const bool has_rom = r.u8() != 0;
    if (has_rom) {
        if (nl->rom_cell < 0)
            throw std::runtime_error("netlist has no ROM port");
        depth = r.u32();
        nluts = r.u32();
        rom.resize((size_t)nluts * 2 * N);
        for (uint32_t t = 0; t < nluts; t++)
            read_trlwe(r, &rom[(size_t)t * 2 * N], N);
    }
    // all checks passed: commit to the device
    if (nd)
        VSP_CUDA_CHECK(cudaMemcpy(nl->dff.as<uint32_t>(dff.size()), dff.data(), dff.size() * 4,
                                  cudaMemcpyHostToDevice));
    if (has_ram) {
        VSP_CUDA_CHECK(cudaMemcpy(nl->ram.as<uint32_t>(ram.size()), ram.data(), ram.size() * 4,
                                  cudaMemcpyHostToDevice));
        nl->ram_v = v;
        nl->ram_w = w;
        nl->has_ram = true;
    }
    if (has_rom) {
        VSP_CUDA_CHECK(cudaMemcpy(nl->rom.as<uint32_t>(rom.size()), rom.data(), rom.size() * 4,
                                  cudaMemcpyHostToDevice));
        nl->rom_depth = depth;
        nl->rom_nluts = nluts;
        nl->has_rom = true;
    }
    nl->cycle = cycle;
    nl->table_valid = false;
}

}  // namespace
