// Circuit bootstrapping (level 2, N2 = 2048, 64-bit torus) for tfhe-80.
//
// Reference: circuitBootstrap (ops.cpp:914-935) = for i < l1:
//   blindRotate<uint64_t>(ct, bk2, testvec b == h/2) (ops.cpp:713-742) -> sampleExtract(.,0)
//   -> b += h/2 -> privateKeySwitch (ops.cpp:681-708) with pksNegS and pksId.
//
// The reference multiplies level-2 polynomials in double precision after casting the
// 64-bit torus words to double (fft.hpp:64-75), which is only accurate to ~2^30
// (test_tfhe.cpp:142-175).  Here every BK2 word is split exactly into two signed
// 32-bit halves, x = hi * 2^32 + lo, and both halves go through the FFT; each partial
// product is an exact integer below 2^53, so the external product is EXACT mod 2^64
// (the reference's MulBackend::Exact result), at the cost of a second MAC/inverse.
//
// The 1024-point transform (Y^1024 = i) is one split stage into Y^512 = +-sqrt(i)
// followed by two 512-point warp transforms (fft512 ROOT 1 / ROOT 2).
#pragma once

#include <cooperative_groups.h>

#include "fft512.cuh"

namespace vsp {

// s = sqrt(i) = e^{i pi/4}
__device__ __forceinline__ double2 split_fwd(double2 u, double2 v, int branch)
{
    const double c = 0.70710678118654752440;
    const double sx = c * (v.x - v.y), sy = c * (v.x + v.y);  // s * v
    return branch == 0 ? make_double2(u.x + sx, u.y + sy) : make_double2(u.x - sx, u.y - sy);
}

// ---------------------------------------------------------------------------
// BK2 preparation: raw u64 rows [i][r][poly][2048] -> [i][r][q][branch][j][lane]
// double2 with q = poly*2 + half (half 0 = signed low word, 1 = high word), scaled by
// 1/1024.  One warp per (i, r, q, branch).
__global__ void __launch_bounds__(64) prepare_bk2_kernel(const uint64_t* __restrict__ raw,
                                                          const double2* __restrict__ tw2g,
                                                          double2* __restrict__ out, int jobs)
{
    __shared__ double2 tw2[2][kTw2Entries * 32];
    __shared__ double2 xb[2][kFftXbufStride];
    for (int i = threadIdx.x; i < 2 * kTw2Entries * 32; i += blockDim.x)
        tw2[i / (kTw2Entries * 32)][i % (kTw2Entries * 32)] = tw2g[kTw2Entries * 32 + i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int job = blockIdx.x * 2 + warp;
    if (job >= jobs)
        return;
    const int branch = job & 1, q = (job >> 1) & 3, ir = job >> 3;  // ir = i*8 + r
    const int poly = q >> 1, half = q & 1;
    const uint64_t* src = raw + ((size_t)ir * 2 + poly) * 2048;
    auto word = [&](int k) -> double {
        const uint64_t x = src[k];
        const int32_t lo = (int32_t)(uint32_t)x;
        if (half == 0)
            return (double)lo;
        const uint64_t h = (x - (uint64_t)(int64_t)lo) >> 32;
        return (double)(int32_t)(uint32_t)h;
    };
    double2 z[16];
#pragma unroll
    for (int j = 0; j < 16; j++) {
        const int p = lane + 32 * j;
        const double2 u = make_double2(word(p), word(p + 1024));
        const double2 v = make_double2(word(p + 512), word(p + 1536));
        z[j] = split_fwd(u, v, branch);
    }
    if (branch == 0)
        fft512_fwd<1>(z, xb[warp], tw2[0], lane);
    else
        fft512_fwd<2>(z, xb[warp], tw2[1], lane);
    double2* dst = out + (size_t)job * 512;
    const double sc = 1.0 / 1024.0;
#pragma unroll
    for (int j = 0; j < 16; j++)
        dst[j * 32 + lane] = make_double2(z[j].x * sc, z[j].y * sc);
}

// ---------------------------------------------------------------------------
// Level-2 blind rotation, one CTA (8 warps) per task.  Task t rotates the test vector
// (0, h/2 ... h/2) with h = hv[t] by the level-0 TLWE tasks[t % ninputs]; the accumulator
// (2 x 2048 u64) is written to out[t].
constexpr int kRegion = kFftXbufStride;  // double2 per smem region (8704 B)

struct Br2Smem {
    uint64_t acc[2][2048];
    double2 reg[16][kRegion];
    double2 tw2[2][kTw2Entries * 32];
};

__global__ void __launch_bounds__(256, 1)
    br2_kernel(const uint32_t* __restrict__ tasks, int ninputs, const uint64_t* __restrict__ hv,
               const double2* __restrict__ bk2fd, const double2* __restrict__ tw2g,
               uint64_t* __restrict__ out, int n, int bgbits)
{
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Br2Smem& sm = *reinterpret_cast<Br2Smem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t* lwe = tasks + (size_t)(blockIdx.x % ninputs) * (n + 1);
    for (int i = tid; i < 2 * kTw2Entries * 32; i += blockDim.x)
        sm.tw2[i / (kTw2Entries * 32)][i % (kTw2Entries * 32)] = tw2g[kTw2Entries * 32 + i];
    {
        const uint64_t h2 = hv[blockIdx.x] / 2;
        const uint32_t rot = (4096u - mod_switch_2n(lwe[n], 12)) & 4095u;
        for (int q = tid; q < 2048; q += blockDim.x) {
            sm.acc[0][q] = 0;
            uint64_t val;
            if (rot < 2048)
                val = ((uint32_t)q < rot) ? (0ull - h2) : h2;
            else
                val = ((uint32_t)q < rot - 2048) ? h2 : (0ull - h2);
            sm.acc[1][q] = val;
        }
    }
    __syncthreads();
    // decomposePoly<uint64_t> constants (poly.hpp:79-97), l2 = 4
    const uint64_t half = 1ull << (bgbits - 1);
    const uint64_t mask = (1ull << bgbits) - 1;
    uint64_t offset = 0;
    for (int i = 1; i <= 4; i++)
        offset += half << (64 - i * bgbits);

    // a_i is fetched one step ahead (lwe[i + 1] <= lwe[n] is in bounds) so the global
    // load latency hides behind the current external product
    uint32_t a_next = lwe[0];
#pragma unroll 1
    for (int i = 0; i < n; i++) {
        const uint32_t bara = mod_switch_2n(a_next, 12);
        a_next = lwe[i + 1];
        // ---- phase A: row r = warp (poly r/4, digit level r%4), forward transforms
        {
            const int P = warp >> 2, L = warp & 3;
            const uint64_t* src = sm.acc[P];
            const int sh = 64 - (L + 1) * bgbits;
            auto digit = [&](uint32_t q) -> double {
                const uint32_t idx = (q - bara) & 4095u;
                const uint64_t r = idx < 2048 ? src[idx] : 0ull - src[idx - 2048];
                const uint64_t v = r - src[q] + offset;
                return (double)(int32_t)(int64_t)(((v >> sh) & mask) - half);
            };
            double2 z0[16], z1[16];
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const uint32_t p = lane + 32 * j;
                const double2 u = make_double2(digit(p), digit(p + 1024));
                const double2 v = make_double2(digit(p + 512), digit(p + 1536));
                z0[j] = split_fwd(u, v, 0);
                z1[j] = split_fwd(u, v, 1);
            }
            double2* r0 = sm.reg[2 * warp];
            double2* r1 = sm.reg[2 * warp + 1];
            fft512_fwd<1>(z0, r0, sm.tw2[0], lane);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++)
                r0[j * 32 + lane] = z0[j];
            fft512_fwd<2>(z1, r1, sm.tw2[1], lane);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++)
                r1[j * 32 + lane] = z1[j];
        }
        __syncthreads();
        // ---- phase B: MAC over the 8 rows for 4 outputs (a_lo, a_hi, b_lo, b_hi)
        {
            const double2* K = bk2fd + (size_t)i * 8 * 4 * 1024;
#pragma unroll 1
            for (int m = 0; m < 4; m++) {
                const int f = tid + 256 * m;
                const int b = f >> 9, s = f & 511;
                double2 o[4];
#pragma unroll
                for (int q = 0; q < 4; q++)
                    o[q] = make_double2(0.0, 0.0);
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    const double2 d = sm.reg[2 * r + b][s];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const double2 k = __ldg(K + ((size_t)(r * 4 + q)) * 1024 + f);
                        o[q].x = fma(d.x, k.x, fma(-d.y, k.y, o[q].x));
                        o[q].y = fma(d.x, k.y, fma(d.y, k.x, o[q].y));
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; q++)
                    sm.reg[2 * q + b][s] = o[q];
            }
        }
        __syncthreads();
        // ---- phase C: inverse 512-point transforms, warp = (q, branch)
        {
            const int q = warp >> 1, b = warp & 1;
            double2* rg = sm.reg[2 * q + b];
            double2 v[16];
#pragma unroll
            for (int j = 0; j < 16; j++)
                v[j] = rg[j * 32 + lane];
            __syncwarp();
            if (b == 0)
                fft512_inv<1>(v, rg, sm.tw2[0], lane);
            else
                fft512_inv<2>(v, rg, sm.tw2[1], lane);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++)
                rg[lane + 32 * j] = v[j];
        }
        __syncthreads();
        // ---- phase D: inverse split stage, exact rounding, lo/hi recombination
        {
            const double c = 0.70710678118654752440;
#pragma unroll 1
            for (int w = 0; w < 2; w++) {
                const int p = tid + 256 * w;
#pragma unroll
                for (int P = 0; P < 2; P++) {
                    int64_t part[2][4];
#pragma unroll
                    for (int hh = 0; hh < 2; hh++) {
                        const int q = 2 * P + hh;
                        const double2 A = sm.reg[2 * q][p], B = sm.reg[2 * q + 1][p];
                        const double2 u = make_double2(A.x + B.x, A.y + B.y);
                        const double dx = A.x - B.x, dy = A.y - B.y;
                        // (A - B) * conj(s), s = c (1 + i)
                        const double2 v = make_double2(c * (dx + dy), c * (dy - dx));
                        part[hh][0] = __double2ll_rn(u.x);  // coefficient p
                        part[hh][1] = __double2ll_rn(v.x);  // p + 512
                        part[hh][2] = __double2ll_rn(u.y);  // p + 1024
                        part[hh][3] = __double2ll_rn(v.y);  // p + 1536
                    }
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const uint64_t val =
                            (uint64_t)part[0][e] + ((uint64_t)part[1][e] << 32);
                        sm.acc[P][p + 512 * e] += val;
                    }
                }
            }
        }
        __syncthreads();
    }
    uint64_t* dst = out + (size_t)blockIdx.x * 4096;
    for (int q = tid; q < 4096; q += blockDim.x)
        dst[q] = (&sm.acc[0][0])[q];
}

// ---------------------------------------------------------------------------
// Level-2 blind rotation on a CLUSTER of two CTAs per task (thread-block cluster, DSMEM).
// CTA P of the pair owns accumulator polynomial P (0: a, 1: b) of the task:
//   A. its four gadget rows (P, L), L < 4, digits + split + forward transforms, one
//      (row, branch) per warp;
//   B. partial MAC over its own four rows for all four outputs (a_lo, a_hi, b_lo, b_hi):
//      only half of bk2[i] (rows 4P..4P+3, 256 KiB) streams through this SM; the two
//      outputs of the OTHER polynomial go straight into the peer CTA's shared memory
//      (st.shared::cluster, double-buffered by step parity), one cluster barrier per step;
//   C. own outputs = rows 0..3 partial + rows 4..7 partial (the same association on both
//      CTAs), inverse transforms split over warp pairs (fft512_inv_pair);
//   D. inverse split stage, exact rounding, lo/hi recombination into acc[P].
// Same arithmetic per output as br2_kernel up to the association of the row sums, and each
// coefficient rounds back to the same exact integer.
constexpr int kBr2cRegion = kFftXbufStride;

struct Br2cSmem {
    uint64_t acc[2048];                 // this CTA's polynomial
    double2 reg[8][kBr2cRegion];        // (row L, branch b) -> 2L + b; MAC outputs (2k + b)
    double2 part[2][4][512];            // peer's partial outputs, by step parity
    double2 tw2[2][kTw2Entries * 32];
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    br2c_kernel(const uint32_t* __restrict__ tasks, int ninputs, const uint64_t* __restrict__ hv,
                const double2* __restrict__ bk2fd, const double2* __restrict__ tw2g,
                uint64_t* __restrict__ out, int n, int bgbits)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Br2cSmem& sm = *reinterpret_cast<Br2cSmem*>(smem_raw);
    const int P = (int)cluster.block_rank();
    const int task = blockIdx.x >> 1;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t* lwe = tasks + (size_t)(task % ninputs) * (n + 1);
    Br2cSmem* peer = cluster.map_shared_rank(&sm, P ^ 1);
    for (int i = tid; i < 2 * kTw2Entries * 32; i += blockDim.x)
        sm.tw2[i / (kTw2Entries * 32)][i % (kTw2Entries * 32)] = tw2g[kTw2Entries * 32 + i];
    {
        const uint64_t h2 = hv[task] / 2;
        const uint32_t rot = (4096u - mod_switch_2n(lwe[n], 12)) & 4095u;
        for (int q = tid; q < 2048; q += blockDim.x) {
            uint64_t val = 0;
            if (P == 1) {
                if (rot < 2048)
                    val = ((uint32_t)q < rot) ? (0ull - h2) : h2;
                else
                    val = ((uint32_t)q < rot - 2048) ? h2 : (0ull - h2);
            }
            sm.acc[q] = val;
        }
    }
    cluster.sync();  // both CTAs initialised before any remote store
    const uint64_t half = 1ull << (bgbits - 1);
    const uint64_t mask = (1ull << bgbits) - 1;
    uint64_t offset = 0;
    for (int i = 1; i <= 4; i++)
        offset += half << (64 - i * bgbits);

    uint32_t a_next = lwe[0];
#pragma unroll 1
    for (int i = 0; i < n; i++) {
        const uint32_t bara = mod_switch_2n(a_next, 12);
        a_next = lwe[i + 1];
        const int buf = i & 1;
        if (tid == 0 && i + 1 < n) {
            // bring next step's half of bk2 (256 KiB, 4 x 64 KiB) into L2 while this step
            // runs: the MAC's loads then hit L2 instead of HBM (bk2 does not fit in L2)
            const char* nk = reinterpret_cast<const char*>(
                bk2fd + (size_t)(i + 1) * 8 * 4 * 1024 + (size_t)(4 * P) * 4 * 1024);
#pragma unroll
            for (int q = 0; q < 4; q++)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nk + q * 65536),
                             "r"(65536)
                             : "memory");
        }
        // ---- A: warp = (row L, branch b)
        {
            const int L = warp & 3, b = warp >> 2;
            const int sh = 64 - (L + 1) * bgbits;
            auto digit = [&](uint32_t q) -> double {
                const uint32_t idx = (q - bara) & 4095u;
                const uint64_t r = idx < 2048 ? sm.acc[idx] : 0ull - sm.acc[idx - 2048];
                const uint64_t v = r - sm.acc[q] + offset;
                return (double)(int32_t)(int64_t)(((v >> sh) & mask) - half);
            };
            double2 z[16];
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const uint32_t p = lane + 32 * j;
                const double2 u = make_double2(digit(p), digit(p + 1024));
                const double2 v = make_double2(digit(p + 512), digit(p + 1536));
                z[j] = split_fwd(u, v, b);
            }
            double2* rg = sm.reg[2 * L + b];
            if (b == 0)
                fft512_fwd<1>(z, rg, sm.tw2[0], lane);
            else
                fft512_fwd<2>(z, rg, sm.tw2[1], lane);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++)
                rg[j * 32 + lane] = z[j];
        }
        __syncthreads();
        // ---- B: partial MAC over rows 4P..4P+3 for the four outputs.  Bound by the L2
        // latency of the bk2 loads: the loads of the next point are issued before the FMAs
        // of the current one (two register sets of 16 x double2; the compiler barrier at the
        // end of each point keeps ptxas from hoisting more)
        {
            const double2* K = bk2fd + (size_t)i * 8 * 4 * 1024 + (size_t)(4 * P) * 4 * 1024;
            double2 kc[16], kn[16];
            auto load = [&](double2 (&kk)[16], int m) {
                const int f = tid + 256 * m;
#pragma unroll
                for (int u = 0; u < 16; u++)
                    kk[u] = __ldg(K + (size_t)u * 1024 + f);  // u = L * 4 + q
            };
            load(kc, 0);
#pragma unroll
            for (int m = 0; m < 4; m++) {
                if (m < 3)
                    load(kn, m + 1);
                const int f = tid + 256 * m;
                const int b = f >> 9, s = f & 511;
                double2 o[4];
#pragma unroll
                for (int q = 0; q < 4; q++)
                    o[q] = make_double2(0.0, 0.0);
#pragma unroll
                for (int L = 0; L < 4; L++) {
                    const double2 d = sm.reg[2 * L + b][s];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const double2 k = kc[L * 4 + q];
                        o[q].x = fma(d.x, k.x, fma(-d.y, k.y, o[q].x));
                        o[q].y = fma(d.x, k.y, fma(d.y, k.x, o[q].y));
                    }
                }
                // own outputs q = 2P + k stay (in place of this thread's own Z slots), the
                // other polynomial's go to the peer
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    // (static register indices: P selects, it does not index)
                    sm.reg[2 * k + b][s] = P ? o[2 + k] : o[k];
                    peer->part[buf][2 * k + b][s] = P ? o[k] : o[2 + k];
                }
                asm volatile("" ::: "memory");
                if (m < 3) {
#pragma unroll
                    for (int u = 0; u < 16; u++)
                        kc[u] = kn[u];
                }
            }
        }
        cluster.sync();  // partials exchanged (and the peer is done with last step's buffer)
        // ---- C: own outputs, inverse transforms on warp pairs (region g = 2k + b)
        {
            const int g = warp & 3, h = warp >> 2, b = g & 1;
            double2* rg = sm.reg[g];
            const int Lv = 16 * h + (lane & 15), e = lane >> 4;
            double2 u[8];
#pragma unroll
            for (int t = 0; t < 8; t++) {
                const int q = (2 * t + e) * 32 + Lv;
                const double2 mine = rg[q], oth = sm.part[buf][g][q];
                // rows 0..3 first, then rows 4..7, on both CTAs
                u[t] = P == 0 ? make_double2(mine.x + oth.x, mine.y + oth.y)
                              : make_double2(oth.x + mine.x, oth.y + mine.y);
            }
            asm volatile("bar.sync %0, 64;" ::"r"(1 + g) : "memory");  // inputs read
            if (b == 0)
                fft512_inv_pair<1>(u, rg, sm.tw2[0], lane, h, 1 + g);
            else
                fft512_inv_pair<2>(u, rg, sm.tw2[1], lane, h, 1 + g);
            asm volatile("bar.sync %0, 64;" ::"r"(1 + g) : "memory");  // transpose reads done
#pragma unroll
            for (int t = 0; t < 8; t++)
                rg[Lv + 32 * (t + 8 * e)] = u[t];
        }
        __syncthreads();
        // ---- D: inverse split stage, exact rounding, lo/hi recombination into acc[P]
        {
            const double c = 0.70710678118654752440;
#pragma unroll 1
            for (int w = 0; w < 2; w++) {
                const int p = tid + 256 * w;
                int64_t part[2][4];
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    const double2 A = sm.reg[2 * hh][p], B = sm.reg[2 * hh + 1][p];
                    const double2 uu = make_double2(A.x + B.x, A.y + B.y);
                    const double dx = A.x - B.x, dy = A.y - B.y;
                    const double2 vv = make_double2(c * (dx + dy), c * (dy - dx));
                    part[hh][0] = __double2ll_rn(uu.x);  // coefficient p
                    part[hh][1] = __double2ll_rn(vv.x);  // p + 512
                    part[hh][2] = __double2ll_rn(uu.y);  // p + 1024
                    part[hh][3] = __double2ll_rn(vv.y);  // p + 1536
                }
#pragma unroll
                for (int e4 = 0; e4 < 4; e4++)
                    sm.acc[p + 512 * e4] += (uint64_t)part[0][e4] + ((uint64_t)part[1][e4] << 32);
            }
        }
        __syncthreads();
    }
    uint64_t* dst = out + (size_t)task * 4096 + (size_t)P * 2048;
    for (int q = tid; q < 2048; q += blockDim.x)
        dst[q] = sm.acc[q];
}

// ---------------------------------------------------------------------------
// Level-2 blind rotation on a cluster of FOUR CTAs per task.  CTA (P, b) owns accumulator
// polynomial P and branch b of the level-2 split Y^1024 = +-sqrt(i) (the two 512-point
// halves of every transform):
//   A. digits of its polynomial's four rows and their branch-b forward transforms, each
//      split over a warp pair (fft512_fwd_pair);
//   B. partial MAC over its four rows for all four outputs at the branch-b points (a
//      quarter of bk2[i], 128 KiB, per SM); the other polynomial's two outputs go to CTA
//      (1-P, b) through DSMEM;
//   C. own outputs (rows 0..3 first, then 4..7), branch-b inverse transforms on warp pairs;
//      the results also go to the branch partner (P, 1-b);
//   D. both CTAs of polynomial P recombine branches, lo/hi halves and round exactly into
//      identical copies of acc[P].
// Two cluster barriers per step; each exchange buffer is written and read between the
// same pair of barriers, so single buffers suffice.
struct Br2qSmem {
    uint64_t acc[4096];                 // polynomial P (identical on both branch CTAs); EXT:
                                        // its negacyclic extension (acc, -acc)
    double2 reg[4][kBr2cRegion];        // row L (forward), then own outputs k (2 x)
    double2 part[2][512];               // MAC partials from (1-P, b), by output k
    double2 xin[2][512];                // branch 1-b inverse outputs from (P, 1-b)
    double2 tw2[kTw2Entries * 32];      // this branch's root (1 + b)
};

// PROBE: clock64 totals per phase -> probe[cta rank][warp][8] of task 0 (tuning).
// EXT: digits read X^-bara acc at a per-lane base plus immediate offsets from the
// (acc, -acc) extension with one per-lane sign, and convert by the offset-binary DADD
// (EXT = false: the round-1 index wrap / select per coefficient and I2F; A/B only).
template <bool PROBE = false, bool EXT = true>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(256, 1)
    br2q_kernel(const uint32_t* __restrict__ tasks, int ninputs, const uint64_t* __restrict__ hv,
                const double2* __restrict__ bk2fd, const double2* __restrict__ tw2g,
                uint64_t* __restrict__ out, int n, int bgbits,
                unsigned long long* __restrict__ probe = nullptr)
{
    unsigned long long ph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tprev = 0;
    auto mark = [&](int k) {
        if constexpr (PROBE) {
            const long long t = clock64();
            ph[k] += (unsigned long long)(t - tprev);
            tprev = t;
        }
    };
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Br2qSmem& sm = *reinterpret_cast<Br2qSmem*>(smem_raw);
    const int cr = (int)cluster.block_rank();
    const int P = cr >> 1, br = cr & 1;
    const int task = blockIdx.x >> 2;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t* lwe = tasks + (size_t)(task % ninputs) * (n + 1);
    Br2qSmem* mac_peer = cluster.map_shared_rank(&sm, cr ^ 2);  // (1-P, b)
    Br2qSmem* br_peer = cluster.map_shared_rank(&sm, cr ^ 1);   // (P, 1-b)
    for (int i = tid; i < kTw2Entries * 32; i += blockDim.x)
        sm.tw2[i] = tw2g[(1 + br) * kTw2Entries * 32 + i];
    {
        const uint64_t h2 = hv[task] / 2;
        const uint32_t rot = (4096u - mod_switch_2n(lwe[n], 12)) & 4095u;
        for (int q = tid; q < 2048; q += blockDim.x) {
            uint64_t val = 0;
            if (P == 1) {
                if (rot < 2048)
                    val = ((uint32_t)q < rot) ? (0ull - h2) : h2;
                else
                    val = ((uint32_t)q < rot - 2048) ? h2 : (0ull - h2);
            }
            sm.acc[q] = val;
            if constexpr (EXT)
                sm.acc[2048 + q] = 0ull - val;
        }
    }
    cluster.sync();
    const uint64_t half = 1ull << (bgbits - 1);
    const uint64_t mask = (1ull << bgbits) - 1;
    uint64_t offset = 0;
    for (int i = 1; i <= 4; i++)
        offset += half << (64 - i * bgbits);

    uint32_t a_next = lwe[0];
    if constexpr (PROBE)
        tprev = clock64();
#pragma unroll 1
    for (int i = 0; i < n; i++) {
        const uint32_t bara = mod_switch_2n(a_next, 12);
        a_next = lwe[i + 1];
        if (tid < 16 && i + 1 < n) {
            // next step's quarter of bk2 (16 segments of 8 KiB: row u, this CTA's polynomial
            // half and branch) into L2 while this step runs, as br2c_kernel does
            const double2* nk = bk2fd + (size_t)(i + 1) * 8 * 4 * 1024 + (size_t)(4 * P) * 4 * 1024 +
                                (size_t)br * 512 + (size_t)tid * 1024;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nk), "r"(8192) : "memory");
        }
        // ---- A: row L on the warp pair (L, L + 4), branch br
        {
            const int L = warp & 3, h = warp >> 2;
            const int Lv = 16 * h + (lane & 15), e = lane >> 4;
            const int sh = 64 - (L + 1) * bgbits;
            auto digit = [&](uint32_t q) -> double {
                const uint32_t idx = (q - bara) & 4095u;
                const uint64_t r = idx < 2048 ? sm.acc[idx] : 0ull - sm.acc[idx - 2048];
                const uint64_t v = r - sm.acc[q] + offset;
                return (double)(int32_t)(int64_t)(((v >> sh) & mask) - half);
            };
            // EXT: coefficient q = Lv + 256 e + o of X^-bara acc is (-1)^sg srcr[o]
            const uint32_t lk = (uint32_t)(Lv + 256 * e) - bara;
            const uint64_t* srcr = sm.acc + (lk & 2047u);
            const uint64_t* srcl = sm.acc + Lv + 256 * e;
            const uint32_t sg = (lk >> 11) & 1u;
            const uint64_t sgm = 0ull - (uint64_t)sg, off2 = offset + sg;
            const double obc = 4503599627370496.0 + (double)half;  // 2^52 + half
            auto digit_ext = [&](int o) -> double {
                const uint64_t v = (srcr[o] ^ sgm) - srcl[o] + off2;
                return __hiloint2double(0x43300000, (int)(uint32_t)((v >> sh) & mask)) - obc;
            };
            double2 z[8];
#pragma unroll
            for (int t = 0; t < 8; t++) {
                if constexpr (EXT) {
                    const double2 u = make_double2(digit_ext(32 * t), digit_ext(32 * t + 1024));
                    const double2 v = make_double2(digit_ext(32 * t + 512), digit_ext(32 * t + 1536));
                    z[t] = split_fwd(u, v, br);
                }
                else {
                    const uint32_t p = (uint32_t)(Lv + 32 * (t + 8 * e));
                    const double2 u = make_double2(digit(p), digit(p + 1024));
                    const double2 v = make_double2(digit(p + 512), digit(p + 1536));
                    z[t] = split_fwd(u, v, br);
                }
            }
            mark(8);  // digits + split (probe slot 8); the forward transform is slot 0
            double2* rg = sm.reg[L];
            if (br == 0)
                fft512_fwd_pair<1>(z, rg, sm.tw2, lane, h, 1 + L);
            else
                fft512_fwd_pair<2>(z, rg, sm.tw2, lane, h, 1 + L);
            asm volatile("bar.sync %0, 64;" ::"r"(1 + L) : "memory");  // transpose reads done
#pragma unroll
            for (int t = 0; t < 8; t++)
                rg[(2 * t + e) * 32 + Lv] = z[t];
        }
        mark(0);
        __syncthreads();
        mark(1);
        // ---- B: partial MAC at this branch's 512 points, 2 per thread
        {
            const double2* K = bk2fd + (size_t)i * 8 * 4 * 1024 + (size_t)(4 * P) * 4 * 1024 +
                               (size_t)br * 512;
            double2 kc[16], kn[16];
            auto load = [&](double2 (&kk)[16], int m) {
                const int s = tid + 256 * m;
#pragma unroll
                for (int u = 0; u < 16; u++)
                    kk[u] = __ldg(K + (size_t)u * 1024 + s);  // u = L * 4 + q
            };
            load(kc, 0);
#pragma unroll
            for (int m = 0; m < 2; m++) {
                if (m < 1)
                    load(kn, m + 1);
                const int s = tid + 256 * m;
                double2 o[4];
#pragma unroll
                for (int q = 0; q < 4; q++)
                    o[q] = make_double2(0.0, 0.0);
#pragma unroll
                for (int L = 0; L < 4; L++) {
                    const double2 d = sm.reg[L][s];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const double2 k = kc[L * 4 + q];
                        o[q].x = fma(d.x, k.x, fma(-d.y, k.y, o[q].x));
                        o[q].y = fma(d.x, k.y, fma(d.y, k.x, o[q].y));
                    }
                }
                // own outputs in place of this thread's own row slots (only it reads them)
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    sm.reg[k][s] = P ? o[2 + k] : o[k];
                    mac_peer->part[k][s] = P ? o[k] : o[2 + k];
                }
                asm volatile("" ::: "memory");
                if (m < 1) {
#pragma unroll
                    for (int u = 0; u < 16; u++)
                        kc[u] = kn[u];
                }
            }
        }
        mark(2);
        cluster.sync();  // partials exchanged
        mark(3);
        // ---- C: own outputs k = 0, 1 (lo, hi) on warp pairs (k, k + 4); warps 2, 3, 6, 7
        // idle here
        {
            const int k = warp & 3, h = warp >> 2;
            if (k < 2) {
                double2* rg = sm.reg[k];
                const int Lv = 16 * h + (lane & 15), e = lane >> 4;
                double2 u[8];
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    const int q = (2 * t + e) * 32 + Lv;
                    const double2 mine = rg[q], oth = sm.part[k][q];
                    u[t] = P == 0 ? make_double2(mine.x + oth.x, mine.y + oth.y)
                                  : make_double2(oth.x + mine.x, oth.y + mine.y);
                }
                asm volatile("bar.sync %0, 64;" ::"r"(5 + k) : "memory");  // inputs read
                if (br == 0)
                    fft512_inv_pair<1>(u, rg, sm.tw2, lane, h, 5 + k);
                else
                    fft512_inv_pair<2>(u, rg, sm.tw2, lane, h, 5 + k);
                asm volatile("bar.sync %0, 64;" ::"r"(5 + k) : "memory");  // transpose reads done
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    const int pos = Lv + 32 * (t + 8 * e);
                    rg[pos] = u[t];
                    br_peer->xin[k][pos] = u[t];
                }
            }
        }
        mark(4);
        cluster.sync();  // both branches' inverse outputs in place
        mark(5);
        // ---- D: inverse split stage, exact rounding, lo/hi recombination into acc[P]
        {
            const double c = 0.70710678118654752440;
#pragma unroll 1
            for (int w = 0; w < 2; w++) {
                const int p = tid + 256 * w;
                int64_t part[2][4];
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    const double2 mine = sm.reg[hh][p], oth = sm.xin[hh][p];
                    const double2 A = br == 0 ? mine : oth, B = br == 0 ? oth : mine;
                    const double2 uu = make_double2(A.x + B.x, A.y + B.y);
                    const double dx = A.x - B.x, dy = A.y - B.y;
                    const double2 vv = make_double2(c * (dx + dy), c * (dy - dx));
                    part[hh][0] = __double2ll_rn(uu.x);  // coefficient p
                    part[hh][1] = __double2ll_rn(vv.x);  // p + 512
                    part[hh][2] = __double2ll_rn(uu.y);  // p + 1024
                    part[hh][3] = __double2ll_rn(vv.y);  // p + 1536
                }
#pragma unroll
                for (int e4 = 0; e4 < 4; e4++) {
                    const uint64_t nv = sm.acc[p + 512 * e4] + (uint64_t)part[0][e4] +
                                        ((uint64_t)part[1][e4] << 32);
                    sm.acc[p + 512 * e4] = nv;
                    if constexpr (EXT)
                        sm.acc[2048 + p + 512 * e4] = 0ull - nv;
                }
            }
        }
        mark(6);
        __syncthreads();
        mark(7);
    }
    if constexpr (PROBE) {
        if (lane == 0 && task == 0)
            for (int k = 0; k < 10; k++)
                probe[((size_t)cr * 8 + warp) * 10 + k] = ph[k];
    }
    if (br == 0) {
        uint64_t* dst = out + (size_t)task * 4096 + (size_t)P * 2048;
        for (int q = tid; q < 2048; q += blockDim.x)
            dst[q] = sm.acc[q];
    }
}

// ---------------------------------------------------------------------------
// Batched private key switch (ops.cpp:681-708), fused with sampleExtract(acc2, 0)
// and b += h/2 (ops.cpp:928-930).  Input task g: level-2 accumulator acc2[g]
// (a[2048], b[2048] u64); out_rows[g] receives -sum_{i,j} table[i][j][d-1] for
// table 0 (pksNegS) into row rowA[g] and table 1 (pksId) into row rowB[g] of the
// destination (each row 2*N1 u32, pre-zeroed).
// Grid: (islices, N1*2 / 512, 2 tables); CTA: 256 threads x 2 coordinates x GT tasks.
// Streaming private key switch (same result as pks_kernel, all tasks of the batch in one
// CTA): for every (i, j) the CTA reads the 2^b - 1 candidate rows of the table once,
// coalesced, at its 512 coordinates (two per thread), and each task adds the row its digit
// selects -- the digit is the same for every thread of the CTA, so the selection is an
// indexed read of the thread's own shared-memory column (row 0 = zeros: digit 0 adds
// nothing).  The tables (2 x 1.175 GB) stream from HBM once instead of being gathered as
// 8-byte rows per task (pks_kernel, latency-bound at ~63% of the copy bandwidth).  Each
// thread stages its own candidates with cp.async kPksRing steps ahead (no barrier: a thread
// reads only what it copied); a task's digits of one i sit in a register for its t steps.
// Grid (islices, 2 N1 / 512, 2 tables); TM >= T2 tasks (the others read digit 0).
constexpr int kPksRing = 4;
template <int TM>
__global__ void __launch_bounds__(256) pks_stream_kernel(
    const uint64_t* __restrict__ acc2, const uint64_t* __restrict__ hv, int T2,
    const uint32_t* __restrict__ pks_negs, const uint32_t* __restrict__ pks_id,
    uint32_t* __restrict__ dst, const int* __restrict__ rowA, const int* __restrict__ rowB,
    int N2, int N1, int basebits, int t, int islice)
{
    constexpr int kMaxBase = 7;  // 2^b - 1 for b <= 3 (tfhe-80: b = 3)
    extern __shared__ uint32_t pks_sm[];
    uint32_t* pk = pks_sm;                                             // [islice][TM]
    uint2* ring = reinterpret_cast<uint2*>(pks_sm + (size_t)islice * TM);  // [R][8][256]
    const int i0 = blockIdx.x * islice;
    const int i1 = min(N2 + 1, i0 + islice);
    const int table = blockIdx.z;
    const uint32_t* tab = table == 0 ? pks_negs : pks_id;
    const int nb = basebits * t;
    const uint64_t offset = nb >= 64 ? 0ull : 1ull << (64 - (1 + nb));
    const int perBase = (1 << basebits) - 1;
    const uint32_t dmask = (1u << basebits) - 1;
    const int tid = threadIdx.x;
    const int k = (blockIdx.y * 256 + tid) * 2;
    const bool kvalid = k < 2 * N1;
    const int kk = kvalid ? k : 0;
    for (int x = tid; x < (i1 - i0) * TM; x += blockDim.x) {
        const int ii = x / TM, g = x % TM;
        uint32_t w = 0;
        if (g < T2) {
            const int i = i0 + ii;
            const uint64_t* A = acc2 + (size_t)g * 2 * N2;
            uint64_t val;
            if (i < N2)
                val = (i == 0) ? A[0] : 0ull - A[N2 - i];
            else
                val = A[N2] + hv[g] / 2;
            w = (uint32_t)((val + offset) >> (64 - nb));
        }
        pk[x] = w;
    }
    for (int q = 0; q < kPksRing; q++)
        ring[(q * (kMaxBase + 1)) * 256 + tid] = make_uint2(0, 0);  // digit 0 of every slot
    __syncthreads();
    uint32_t acc[TM][2];
#pragma unroll
    for (int g = 0; g < TM; g++)
        acc[g][0] = acc[g][1] = 0;
    const int steps = (i1 - i0) * t;
    // candidate row d of step s = (i, j): tab[((i t + j) perBase + d - 1) 2 N1 + k]
    auto issue = [&](int s) {
        if (s < steps) {
            const uint32_t* r = tab + ((size_t)(i0 * t + s) * perBase) * 2 * N1 + kk;
            uint2* slot = ring + (size_t)((s % kPksRing) * (kMaxBase + 1) + 1) * 256 + tid;
#pragma unroll
            for (int d = 0; d < kMaxBase; d++)
                if (d < perBase)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(slot + d * 256)),
                                 "l"(r + (size_t)d * 2 * N1)
                                 : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int s = 0; s < kPksRing - 1; s++)
        issue(s);
    int s = 0;
#pragma unroll 1
    for (int ii = 0; ii < i1 - i0; ii++) {
        uint32_t pkr[TM];
#pragma unroll
        for (int g = 0; g < TM; g++)
            pkr[g] = pk[ii * TM + g];
#pragma unroll 1
        for (int j = 0; j < t; j++, s++) {
            issue(s + kPksRing - 1);
            asm volatile("cp.async.wait_group %0;" ::"n"(kPksRing - 1) : "memory");
            const int sh = nb - (j + 1) * basebits;
            const uint2* slot = ring + (size_t)((s % kPksRing) * (kMaxBase + 1)) * 256 + tid;
#pragma unroll
            for (int g = 0; g < TM; g++) {
                const uint32_t d = (pkr[g] >> sh) & dmask;  // same for every thread
                const uint2 v = slot[d * 256];
                acc[g][0] += v.x;
                acc[g][1] += v.y;
            }
        }
    }
    if (!kvalid)
        return;
#pragma unroll
    for (int g = 0; g < TM; g++) {
        if (g >= T2)
            break;
        const int r = table == 0 ? rowA[g] : rowB[g];
        uint32_t* o = dst + (size_t)r * 2 * N1 + k;
        if (acc[g][0])
            atomicAdd(o, 0u - acc[g][0]);
        if (acc[g][1])
            atomicAdd(o + 1, 0u - acc[g][1]);
    }
}

template <int GT>
__global__ void __launch_bounds__(256) pks_kernel(const uint64_t* __restrict__ acc2,
                                                  const uint64_t* __restrict__ hv, int T2,
                                                  const uint32_t* __restrict__ pks_negs,
                                                  const uint32_t* __restrict__ pks_id,
                                                  uint32_t* __restrict__ dst,
                                                  const int* __restrict__ rowA,
                                                  const int* __restrict__ rowB, int N2, int N1,
                                                  int basebits, int t)
{
    extern __shared__ uint32_t pk[];  // [islice][GT]: top (basebits*t) bits of v
    const int islice = (N2 + 1 + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * islice;
    const int i1 = min(N2 + 1, i0 + islice);
    const int table = blockIdx.z;
    const uint32_t* tab = table == 0 ? pks_negs : pks_id;
    const int nb = basebits * t;  // digits kept (30 for tfhe-80)
    const uint64_t offset = nb >= 64 ? 0ull : 1ull << (64 - (1 + nb));
    const int perBase = (1 << basebits) - 1;
    const uint32_t dmask = (1u << basebits) - 1;
    for (int g0 = 0; g0 < T2; g0 += GT) {
        const int ng = min(GT, T2 - g0);
        __syncthreads();
        for (int x = threadIdx.x; x < (i1 - i0) * GT; x += blockDim.x) {
            const int ii = x / GT, g = x % GT;
            uint32_t w = 0;
            if (g < ng) {
                const int i = i0 + ii;
                const uint64_t* A = acc2 + (size_t)(g0 + g) * 2 * N2;
                uint64_t val;
                if (i < N2)
                    val = (i == 0) ? A[0] : 0ull - A[N2 - i];
                else
                    val = A[N2] + hv[g0 + g] / 2;
                const uint64_t v = val + offset;
                w = (uint32_t)(v >> (64 - nb));
            }
            pk[x] = w;
        }
        __syncthreads();
        const int k = (blockIdx.y * 256 + threadIdx.x) * 2;
        const bool kvalid = k < 2 * N1;
        uint32_t acc[GT][2];
#pragma unroll
        for (int g = 0; g < GT; g++)
            acc[g][0] = acc[g][1] = 0;
        for (int i = i0; i < i1; i++) {
            for (int j = 0; j < t; j++) {
                const uint32_t* base = tab + ((size_t)i * t + j) * perBase * 2 * N1 + (kvalid ? k : 0);
                // every gate's row load is issued unconditionally (digit 0 and padding
                // gates read row 0 and are masked) so all GT gathers are in flight at once:
                // the kernel is bound by the latency of these 8-byte-per-lane row gathers
#pragma unroll
                for (int g = 0; g < GT; g++) {
                    const uint32_t d = (pk[(i - i0) * GT + g] >> (nb - (j + 1) * basebits)) & dmask;
                    const uint32_t m = d ? 0xffffffffu : 0u;
                    const uint2 r = __ldg(reinterpret_cast<const uint2*>(
                        base + (size_t)(d ? d - 1 : 0) * 2 * N1));
                    acc[g][0] += r.x & m;
                    acc[g][1] += r.y & m;
                }
            }
        }
#pragma unroll
        for (int g = 0; g < GT; g++) {
            if (g >= ng)
                break;
            if (!kvalid)
                break;
            const int row = table == 0 ? rowA[g0 + g] : rowB[g0 + g];
            uint32_t* o = dst + (size_t)row * 2 * N1 + k;
            if (acc[g][0])
                atomicAdd(o, 0u - acc[g][0]);
            if (acc[g][1])
                atomicAdd(o + 1, 0u - acc[g][1]);
        }
    }
}

}  // namespace vsp
