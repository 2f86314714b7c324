// Readers for the reference's "HVP1" containers (serialize.hpp:15-34, serialize.cpp,
// mem.cpp:331-403): keys and ciphertexts produced by the client tools enter the engine
// without going through the reference library.  Host code; included by vsp_capi.cu after
// snapshot.cuh (reuses SnapReader, the little-endian BinReader equivalent).
//
//   header: "HVP1" u8 tag u16 version=1 str param-name          (writeHeader, :5-11)
//   tag 2 BootstrappingKey (:190-206): u8 hasCb, u32 #bk1, TRGSW each, u32 #bk2,
//          TRGSW-lvl2 each, KeySwitchKey {u32 N1,t,baseBits,n, u32vec}, [2 x PKS
//          {u32 N2,t,baseBits,N1, u32vec}]
//   TRGSW: u8 level, u32 rows, per row u32vec a, u32vec b (lvl2: u64vec)
//   tag 3 TLWE: u8 level, u32vec a, u32 b;  tag 4 TRLWE: u8 level, u32vec a, u32vec b
//   tag 6 RAM: u32 v, u32 w, u32 #cells, TRLWE each;  tag 7 ROM: u32 depth, u32 #luts, TRLWE
#pragma once

namespace {

constexpr char kHvp1Magic[4] = {'H', 'V', 'P', '1'};

struct Hvp1Header {
    uint8_t tag;
    std::string param;
};

Hvp1Header hvp1_header(SnapReader& r)
{
    r.need(4);
    if (std::memcmp(r.p, kHvp1Magic, 4) != 0)
        throw std::runtime_error("bad file magic (expected HVP1)");
    r.p += 4;
    Hvp1Header h;
    h.tag = r.u8();
    const uint16_t version = r.u16();
    if (version != 1)
        throw std::runtime_error("unsupported format version " + std::to_string(version));
    h.param = r.str();
    return h;
}

template <class T>
void hvp1_vec(SnapReader& r, T* dst, size_t expect, const char* what)
{
    const uint32_t n = r.u32();
    if (n != expect)
        throw std::runtime_error(std::string(what) + " does not match parameter set");
    r.need((size_t)n * sizeof(T));
    std::memcpy(dst, r.p, (size_t)n * sizeof(T));
    r.p += (size_t)n * sizeof(T);
}

// deserializeBootstrappingKey (serialize.cpp:209-230) into the flat raw layouts that
// vsp_upload_keys takes; checks every dimension against the context's parameters.
struct Hvp1Keys {
    std::vector<uint32_t> bk1, ksk, pks_negs, pks_id;
    std::vector<uint64_t> bk2;
    int has_cb = 0;
};

Hvp1Keys hvp1_keys(const Params& p, const uint8_t* bytes, size_t len)
{
    SnapReader r{bytes, bytes + len};
    const Hvp1Header h = hvp1_header(r);
    if (h.tag != 2)
        throw std::runtime_error("unexpected file type tag " + std::to_string(h.tag) +
                                 " (expected 2)");
    Hvp1Keys k;
    const bool cb = r.u8() != 0;
    const uint32_t n1 = r.u32();
    if (n1 != p.n)
        throw std::runtime_error("bootstrapping key does not match parameter set");
    const size_t row1 = 2 * (size_t)p.N1, rows1 = 2 * (size_t)p.l1;
    k.bk1.resize((size_t)p.n * rows1 * row1);
    for (uint32_t i = 0; i < p.n; i++) {
        (void)r.u8();
        if (r.u32() != rows1)
            throw std::runtime_error("bootstrapping key does not match parameter set");
        for (size_t q = 0; q < rows1; q++) {
            uint32_t* row = &k.bk1[((size_t)i * rows1 + q) * row1];
            hvp1_vec(r, row, p.N1, "TRGSW row");
            hvp1_vec(r, row + p.N1, p.N1, "TRGSW row");
        }
    }
    const uint32_t n2 = r.u32();
    if (n2) {
        if (n2 != p.n)
            throw std::runtime_error("bootstrapping key does not match parameter set");
        const size_t row2 = 2 * (size_t)p.N2, rows2 = 2 * (size_t)p.l2;
        k.bk2.resize((size_t)p.n * rows2 * row2);
        for (uint32_t i = 0; i < p.n; i++) {
            (void)r.u8();
            if (r.u32() != rows2)
                throw std::runtime_error("bootstrapping key does not match parameter set");
            for (size_t q = 0; q < rows2; q++) {
                uint64_t* row = &k.bk2[((size_t)i * rows2 + q) * row2];
                hvp1_vec(r, row, p.N2, "TRGSW row");
                hvp1_vec(r, row + p.N2, p.N2, "TRGSW row");
            }
        }
    }
    // KeySwitchKey {N1, t, baseBits, n} (serialize.cpp:150-167)
    if (r.u32() != p.N1 || r.u32() != p.ksLen || r.u32() != p.ksBaseBits || r.u32() != p.n)
        throw std::runtime_error("key switching key does not match parameter set");
    const size_t kw = (size_t)p.N1 * p.ksLen * ((1u << p.ksBaseBits) - 1) * (p.n + 1);
    k.ksk.resize(kw);
    hvp1_vec(r, k.ksk.data(), kw, "key switching key");
    if (cb) {
        const size_t pw = ((size_t)p.N2 + 1) * p.pksLen * ((1u << p.pksBaseBits) - 1) * 2 * p.N1;
        for (auto* dst : {&k.pks_negs, &k.pks_id}) {
            if (r.u32() != p.N2 || r.u32() != p.pksLen || r.u32() != p.pksBaseBits ||
                r.u32() != p.N1)
                throw std::runtime_error("private key switching key does not match parameter set");
            dst->resize(pw);
            hvp1_vec(r, dst->data(), pw, "private key switching key");
        }
    }
    k.has_cb = cb ? 1 : (n2 ? 2 : 0);
    return k;
}

// Ciphertext containers (tags 3, 4, 6, 7) flattened to the engine layouts.
// meta: [tag, count, v, w, depthBytes]; out receives count x (TLWE n+1 | TRLWE 2N) words.
std::vector<uint32_t> hvp1_ciphertexts(const Params& p, const uint8_t* bytes, size_t len,
                                       uint32_t meta[5])
{
    SnapReader r{bytes, bytes + len};
    const Hvp1Header h = hvp1_header(r);
    std::vector<uint32_t> out;
    meta[0] = h.tag;
    meta[2] = meta[3] = meta[4] = 0;
    auto trlwe = [&]() {
        const size_t o = out.size();
        out.resize(o + 2 * (size_t)p.N1);
        (void)r.u8();
        hvp1_vec(r, &out[o], p.N1, "TRLWE");
        hvp1_vec(r, &out[o + p.N1], p.N1, "TRLWE");
    };
    if (h.tag == 3) {  // deserializeTlwe (serialize.cpp:240-245): level-0 TLWE
        const uint8_t level = r.u8();
        const uint32_t dim = level == 0 ? p.n : p.N1;
        out.resize(dim + 1);
        hvp1_vec(r, out.data(), dim, "TLWE");
        out[dim] = r.u32();
        meta[1] = 1;
    }
    else if (h.tag == 4) {
        trlwe();
        meta[1] = 1;
    }
    else if (h.tag == 6) {  // readRam (mem.cpp:340-352)
        meta[2] = r.u32();
        meta[3] = r.u32();
        meta[1] = r.u32();
        if (meta[1] != ((size_t)meta[3] << meta[2]))
            throw std::runtime_error("corrupt RAM: cell count mismatch");
        for (uint32_t i = 0; i < meta[1]; i++)
            trlwe();
    }
    else if (h.tag == 7) {  // readRom (mem.cpp:378-387)
        meta[4] = r.u32();
        meta[1] = r.u32();
        for (uint32_t i = 0; i < meta[1]; i++)
            trlwe();
    }
    else {
        throw std::runtime_error("unexpected file type tag " + std::to_string(h.tag));
    }
    return out;
}

}  // namespace
