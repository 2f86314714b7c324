// Client-side TFHE (key generation, encryption, decryption) for the VSP B200 engine.
//
// This is the "Alice" side of VSP (SPEC.md protocol): it produces the key material
// and ciphertexts the engine consumes.  It follows the reference's client code
// (rng.cpp, ops.cpp:212-515) step for step — same ChaCha20 stream, same draw order,
// same libstdc++ normal_distribution — so a given seed yields the same keys as the
// reference's BootstrappingKey::generate when both are built with
// -ffp-contract=off (checked by tests/test_client.py against oracle/_ref).
// polyMulBinary products run on host threads; everything else is the sequential
// CSPRNG stream.  Not on the evaluation hot path.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vsp_b200.h"
#include "client_internal.h"

namespace {

thread_local std::string g_cerr;

constexpr uint32_t kMu32 = 1u << 29;

// ChaCha20 CSPRNG (rng.cpp:16-99, rng.hpp:13-50)
class Csprng {
public:
    using result_type = uint32_t;
    static constexpr result_type min() { return 0; }
    static constexpr result_type max() { return 0xffffffffu; }

    explicit Csprng(uint64_t seed)
    {
        uint64_t s = seed;
        uint32_t key[8];
        for (int i = 0; i < 4; i++) {
            s += 0x9e3779b97f4a7c15ull;
            uint64_t z = s;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            z ^= z >> 31;
            key[2 * i] = (uint32_t)z;
            key[2 * i + 1] = (uint32_t)(z >> 32);
        }
        state_[0] = 0x61707865;
        state_[1] = 0x3320646e;
        state_[2] = 0x79622d32;
        state_[3] = 0x6b206574;
        for (int i = 0; i < 8; i++)
            state_[4 + i] = key[i];
        state_[12] = state_[13] = state_[14] = state_[15] = 0;
        pos_ = 16;
    }

    result_type operator()()
    {
        if (pos_ == 16)
            refill();
        return block_[pos_++];
    }
    uint64_t nextU64()
    {
        uint64_t lo = (*this)();
        uint64_t hi = (*this)();
        return lo | (hi << 32);
    }

private:
    static uint32_t rotl(uint32_t x, int k) { return (x << k) | (x >> (32 - k)); }
    static void qr(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d)
    {
        a += b; d = rotl(d ^ a, 16);
        c += d; b = rotl(b ^ c, 12);
        a += b; d = rotl(d ^ a, 8);
        c += d; b = rotl(b ^ c, 7);
    }
    void refill()
    {
        std::array<uint32_t, 16> x = state_;
        for (int r = 0; r < 10; r++) {
            qr(x[0], x[4], x[8], x[12]);
            qr(x[1], x[5], x[9], x[13]);
            qr(x[2], x[6], x[10], x[14]);
            qr(x[3], x[7], x[11], x[15]);
            qr(x[0], x[5], x[10], x[15]);
            qr(x[1], x[6], x[11], x[12]);
            qr(x[2], x[7], x[8], x[13]);
            qr(x[3], x[4], x[9], x[14]);
        }
        for (int i = 0; i < 16; i++)
            block_[i] = x[i] + state_[i];
        pos_ = 0;
        if (++state_[12] == 0)
            ++state_[13];
    }
    std::array<uint32_t, 16> state_{}, block_{};
    int pos_;
};

uint32_t doubleToTorus32(double d)  // rng.cpp:101-105
{
    return (uint32_t)(int64_t)std::llround((d - std::floor(d)) * 4294967296.0);
}

uint64_t doubleToTorus64(double d)  // rng.cpp:107-115
{
    double frac = d - std::floor(d);
    double hi = std::floor(frac * 4294967296.0);
    double lo = (frac * 4294967296.0 - hi) * 4294967296.0;
    return ((uint64_t)hi << 32) + (uint64_t)(int64_t)std::llround(lo);
}

uint32_t noise32(Csprng& r, double sigma)  // rng.cpp:117-123
{
    if (sigma == 0.0)
        return 0;
    std::normal_distribution<double> g(0.0, sigma);
    return doubleToTorus32(g(r));
}

uint64_t noise64(Csprng& r, double sigma)
{
    if (sigma == 0.0)
        return 0;
    std::normal_distribution<double> g(0.0, sigma);
    return doubleToTorus64(g(r));
}

struct Alphas {
    double a0, a1, a2, pks;
};

Alphas alphas_for(const vsp_params& p)
{
    // tfhe-80 noise (params.cpp:34-50); test-det is noiseless (params.cpp:64-80).
    if (p.fft)
        return {2.44e-5, 3.73e-9, std::pow(2.0, -44), std::pow(2.0, -31)};
    return {0.0, 0.0, 0.0, 0.0};
}

template <class T>
void polyMulBinary(T* out, const T* torus, const uint32_t* bits, size_t N)  // poly.hpp:61-75
{
    std::fill(out, out + N, (T)0);
    for (size_t i = 0; i < N; i++) {
        if (!bits[i])
            continue;
        size_t j = 0;
        for (; j < N - i; j++)
            out[i + j] += torus[j];
        for (; j < N; j++)
            out[i + j - N] -= torus[j];
    }
}

// Deferred TRLWE-of-zero encryptions: the sequential stream draws a and the noise
// e in reference order; b = a*s + e (+ message) is computed afterwards in parallel.
template <class T>
struct ZeroEnc {
    T* a;      // N words
    T* b;      // N words (holds e until finalised)
    size_t N;
};

template <class T>
void draw_zero(Csprng& rng, T* a, T* b, size_t N, double alpha)  // ops.cpp:161-180 (draw part)
{
    for (size_t i = 0; i < N; i++) {
        if constexpr (sizeof(T) == 8)
            a[i] = rng.nextU64();
        else
            a[i] = rng();
    }
    for (size_t i = 0; i < N; i++)
        b[i] = 0;
    if (alpha != 0.0)
        for (size_t i = 0; i < N; i++) {
            if constexpr (sizeof(T) == 8)
                b[i] = noise64(rng, alpha);
            else
                b[i] = noise32(rng, alpha);
        }
}

template <class T>
void finalize_parallel(std::vector<ZeroEnc<T>>& jobs, const uint32_t* key)
{
    unsigned th = std::max(1u, std::thread::hardware_concurrency());
    th = std::min<unsigned>(th, (unsigned)std::max<size_t>(1, jobs.size()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < th; t++)
        pool.emplace_back([&, t] {
            std::vector<T> prod;
            for (size_t k = t; k < jobs.size(); k += th) {
                auto& j = jobs[k];
                prod.resize(j.N);
                polyMulBinary(prod.data(), j.a, key, j.N);
                for (size_t i = 0; i < j.N; i++)
                    j.b[i] += prod[i];
            }
        });
    for (auto& x : pool)
        x.join();
}

template <class F>
int cguard(F&& f)
{
    try {
        f();
        return VSP_OK;
    }
    catch (const std::invalid_argument& e) {
        g_cerr = std::string("invalid_argument: ") + e.what();
        return VSP_EINVAL;
    }
    catch (const std::exception& e) {
        g_cerr = std::string("runtime_error: ") + e.what();
        return VSP_ERUNTIME;
    }
}

}  // namespace

extern "C" {

const char* vsp_client_last_error(void) { return g_cerr.c_str(); }

// genSecretKey + BootstrappingKey::generate (ops.cpp:264-385) from Csprng::fromSeed(seed).
// Output buffers: lv0[n], lv1[N1], lv2[N2], bk1[n*2l1*2*N1], ksk[...]; bk2/pks only
// when with_cb (may be NULL otherwise).  with_cb == 2 draws bk2 but stops before the
// private key-switching tables (identical bk2; used by level-2 unit tests).
int vsp_client_keygen(const vsp_params* pp, uint64_t seed, int with_cb, uint32_t* lv0,
                      uint32_t* lv1, uint32_t* lv2, uint32_t* bk1, uint32_t* ksk, uint64_t* bk2,
                      uint32_t* pks_negs, uint32_t* pks_id)
{
    return cguard([&] {
        vsp_internal::keygen(*pp, seed, with_cb, lv0, lv1, lv2, bk1, ksk, bk2, pks_negs, pks_id,
                             {});
    });
}

}  // extern "C"

// The sequential CSPRNG draws in reference order; every b = a*s product (the TRLWE-of-
// zero encryptions of bk1, bk2 and the private key-switching tables) is deferred to
// `fin` (host threads when empty; the GPU in vsp_client_keygen_dev).
void vsp_internal::keygen(const vsp_params& p, uint64_t seed, int with_cb, uint32_t* lv0,
                          uint32_t* lv1, uint32_t* lv2, uint32_t* bk1, uint32_t* ksk,
                          uint64_t* bk2, uint32_t* pks_negs, uint32_t* pks_id,
                          const Finalizer& fin)
{
    {
        const Alphas al = alphas_for(p);
        Csprng rng(seed);
        for (uint32_t i = 0; i < p.n; i++)
            lv0[i] = rng() & 1;
        for (uint32_t i = 0; i < p.N1; i++)
            lv1[i] = rng() & 1;
        for (uint32_t i = 0; i < p.N2; i++)
            lv2[i] = rng() & 1;
        // bk1 / bk2: trgswEncryptAtLevel (ops.cpp:182-205)
        std::vector<ZeroEnc<uint32_t>> j1;
        const size_t N1 = p.N1, N2 = p.N2;
        for (uint32_t i = 0; i < p.n; i++)
            for (uint32_t r = 0; r < 2 * p.l1; r++) {
                uint32_t* row = bk1 + ((size_t)i * 2 * p.l1 + r) * 2 * N1;
                draw_zero(rng, row, row + N1, N1, al.a1);
                j1.push_back({row, row + N1, N1});
            }
        std::vector<ZeroEnc<uint64_t>> j2;
        if (with_cb)
            for (uint32_t i = 0; i < p.n; i++)
                for (uint32_t r = 0; r < 2 * p.l2; r++) {
                    uint64_t* row = bk2 + ((size_t)i * 2 * p.l2 + r) * 2 * N2;
                    draw_zero(rng, row, row + N2, N2, al.a2);
                    j2.push_back({row, row + N2, N2});
                }
        // key switching key (ops.cpp:283-313)
        {
            const uint32_t perBase = (1u << p.ksBaseBits) - 1;
            size_t pos = 0;
            for (uint32_t i = 0; i < p.N1; i++)
                for (uint32_t j = 0; j < p.ksLen; j++)
                    for (uint32_t u = 0; u < perBase; u++) {
                        const uint32_t msg = (lv1[i] * (u + 1)) << (32 - (j + 1) * p.ksBaseBits);
                        uint32_t b = msg + noise32(rng, al.a0);
                        for (uint32_t k = 0; k < p.n; k++) {
                            const uint32_t a = rng();
                            ksk[pos + k] = a;
                            b += a * lv0[k];
                        }
                        ksk[pos + p.n] = b;
                        pos += p.n + 1;
                    }
        }
        // private key switching keys (ops.cpp:315-351)
        std::vector<ZeroEnc<uint32_t>> jp;
        if (with_cb == 1) {
            const uint32_t perBase = (1u << p.pksBaseBits) - 1;
            for (int which = 0; which < 2; which++) {
                uint32_t* d = which == 0 ? pks_negs : pks_id;
                size_t pos = 0;
                for (uint32_t i = 0; i <= p.N2; i++)
                    for (uint32_t j = 0; j < p.pksLen; j++)
                        for (uint32_t u = 0; u < perBase; u++) {
                            draw_zero(rng, d + pos, d + pos + N1, N1, al.pks);
                            jp.push_back({d + pos, d + pos + N1, N1});
                            pos += 2 * N1;
                        }
            }
        }
        if (fin) {
            // each group is one contiguous array of (a[N], b[N]) pairs
            fin(32, bk1, j1.size(), N1, lv1);
            if (!j2.empty())
                fin(64, bk2, j2.size(), N2, lv2);
            if (!jp.empty()) {
                fin(32, pks_negs, jp.size() / 2, N1, lv1);
                fin(32, pks_id, jp.size() / 2, N1, lv1);
            }
        }
        else {
            finalize_parallel(j1, lv1);
            finalize_parallel(j2, lv2);
            finalize_parallel(jp, lv1);
        }
        // gadget offsets of the TRGSWs of lv0[i] (ops.cpp:197-203)
        for (uint32_t i = 0; i < p.n; i++) {
            if (!lv0[i])
                continue;
            for (uint32_t k = 0; k < p.l1; k++) {
                const uint32_t h = 1u << (32 - (k + 1) * p.Bg1Bits);
                bk1[((size_t)i * 2 * p.l1 + k) * 2 * N1] += h;
                bk1[((size_t)i * 2 * p.l1 + p.l1 + k) * 2 * N1 + N1] += h;
            }
            if (with_cb)
                for (uint32_t k = 0; k < p.l2; k++) {
                    const uint64_t h = 1ull << (64 - (k + 1) * p.Bg2Bits);
                    bk2[((size_t)i * 2 * p.l2 + k) * 2 * N2] += h;
                    bk2[((size_t)i * 2 * p.l2 + p.l2 + k) * 2 * N2 + N2] += h;
                }
        }
        // PKS messages: func * key2[i] * (u+1) / base^(j+1) on b (ops.cpp:332-341)
        if (with_cb == 1) {
            const uint32_t perBase = (1u << p.pksBaseBits) - 1;
            for (int which = 0; which < 2; which++) {
                uint32_t* d = which == 0 ? pks_negs : pks_id;
                size_t pos = 0;
                for (uint32_t i = 0; i <= p.N2; i++) {
                    const uint32_t factor = i < p.N2 ? lv2[i] : (uint32_t)-1;
                    for (uint32_t j = 0; j < p.pksLen; j++)
                        for (uint32_t u = 0; u < perBase; u++) {
                            const uint32_t scale = ((u + 1) * factor)
                                                   << (32 - (j + 1) * p.pksBaseBits);
                            uint32_t* b = d + pos + N1;
                            if (which == 0) {
                                for (uint32_t k = 0; k < N1; k++)
                                    b[k] += (uint32_t)(-(int64_t)lv1[k]) * scale;
                            }
                            else {
                                b[0] += scale;
                            }
                            pos += 2 * N1;
                        }
                }
            }
        }
    }
}

extern "C" {

// tlweEncrypt (ops.cpp:428-440) of count bits with one CSPRNG stream; alpha0 noise.
int vsp_client_tlwe_encrypt(const vsp_params* pp, const uint32_t* lv0, uint64_t seed,
                            const uint8_t* bits, size_t count, uint32_t* out)
{
    return cguard([&] {
        const vsp_params& p = *pp;
        const Alphas al = alphas_for(p);
        Csprng rng(seed);
        for (size_t c = 0; c < count; c++) {
            uint32_t* o = out + c * (p.n + 1);
            uint32_t b = (bits[c] ? kMu32 : 0u - kMu32) + noise32(rng, al.a0);
            for (uint32_t i = 0; i < p.n; i++) {
                o[i] = rng();
                b += o[i] * lv0[i];
            }
            o[p.n] = b;
        }
    });
}

// trlweEncrypt (ops.cpp:458-468) of count bit polynomials (N1 bits each) under lv1 with
// alpha1 noise, one CSPRNG stream; out: count x 2*N1 (a then b).  Used for the RAM/ROM
// images of encryptRam / encryptRom (mem.cpp:202-263).
int vsp_client_trlwe_encrypt(const vsp_params* pp, const uint32_t* lv1, uint64_t seed,
                             const uint8_t* bits, size_t count, uint32_t* out)
{
    return cguard([&] {
        const vsp_params& p = *pp;
        const Alphas al = alphas_for(p);
        const size_t N = p.N1;
        Csprng rng(seed);
        std::vector<ZeroEnc<uint32_t>> jobs;
        jobs.reserve(count);
        for (size_t c = 0; c < count; c++) {
            uint32_t* o = out + c * 2 * N;
            draw_zero(rng, o, o + N, N, al.a1);
            jobs.push_back({o, o + N, N});
        }
        finalize_parallel(jobs, lv1);
        for (size_t c = 0; c < count; c++)
            for (size_t i = 0; i < N; i++)
                out[c * 2 * N + N + i] += bits[c * N + i] ? kMu32 : 0u - kMu32;
    });
}

// trlwePhaseAt (ops.cpp:494-505) of coefficient k for count TRLWEs (N = dim).
int vsp_client_trlwe_phase_at(const uint32_t* lv1, uint32_t N, const uint32_t* ct, size_t count,
                              uint32_t k, uint32_t* phases)
{
    return cguard([&] {
        for (size_t c = 0; c < count; c++) {
            const uint32_t* a = ct + c * 2 * N;
            uint32_t acc = 0;
            for (uint32_t j = 0; j <= k; j++)
                acc += a[k - j] * lv1[j];
            for (uint32_t j = k + 1; j < N; j++)
                acc -= a[k + N - j] * lv1[j];
            phases[c] = a[N + k] - acc;
        }
    });
}

// tlwePhase / tlweDecrypt (ops.cpp:442-456) for count ciphertexts of dimension dim.
int vsp_client_tlwe_decrypt(const uint32_t* key, uint32_t dim, const uint32_t* ct, size_t count,
                            uint8_t* bits, uint32_t* phases)
{
    return cguard([&] {
        for (size_t c = 0; c < count; c++) {
            const uint32_t* x = ct + c * (dim + 1);
            uint32_t ph = x[dim];
            for (uint32_t i = 0; i < dim; i++)
                ph -= x[i] * key[i];
            if (phases)
                phases[c] = ph;
            if (bits)
                bits[c] = (int32_t)ph >= 0 ? 1 : 0;
        }
    });
}

}  // extern "C"
