// Gate-bootstrapping kernels (level 1, N1 = 1024, FFT path) plus the batched
// identity key switch and the gate linear-combination / finalize kernels.
//
// Reference path replaced (ops.cpp): homGate (839-896) -> linComb (774-806) ->
// gateBootstrap (759-762) -> bootstrapToTrlwe (750-757) -> blindRotate (713-742)
// -> externalProduct (553-599) -> sampleExtract (628-643) -> identityKeySwitch (651-679).
#pragma once

#include "fft512.cuh"


namespace vsp {

// Gate kinds in hvp::tfhe::GateKind order (ops.hpp:183-194).
enum GateKindDev : int {
    kAnd = 0, kAndNot, kMux, kNand, kNor, kNot, kOr, kOrNot, kXnor, kXor
};

// ---------------------------------------------------------------------------
// Bootstrapping-key preparation: raw TRGSW rows (u32, signed interpretation as in
// FftPlan::forward, fft.hpp:64-75) -> transformed rows in the kernel's slot layout
// [row][poly][j][lane] (double2), pre-scaled by 1/512 so the inverse needs no scale.
// One warp per polynomial.  (prepareTrgsw, ops.cpp:520-546.)
__global__ void __launch_bounds__(128) prepare_poly1024_kernel(
    const uint32_t* __restrict__ raw, const double2* __restrict__ tw2g,
    double2* __restrict__ out, int npolys)
{
    __shared__ double2 tw2[kTw2Entries * 32];
    __shared__ double2 xb[4][kFftXbufStride];
    for (int i = threadIdx.x; i < kTw2Entries * 32; i += blockDim.x)
        tw2[i] = tw2g[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = blockIdx.x * 4 + warp;
    if (q >= npolys)
        return;
    const uint32_t* src = raw + (size_t)q * 1024;
    double2 z[16];
#pragma unroll
    for (int j = 0; j < 16; j++) {
        z[j].x = (double)(int32_t)src[lane + 32 * j];
        z[j].y = (double)(int32_t)src[lane + 32 * j + 512];
    }
    fft512_fwd(z, xb[warp], tw2, lane);
    double2* dst = out + (size_t)(q >> 1) * 1024 + (q & 1) * 512;
    const double s = 1.0 / 512.0;
#pragma unroll
    for (int j = 0; j < 16; j++)
        dst[j * 32 + lane] = make_double2(z[j].x * s, z[j].y * s);
}

// ---------------------------------------------------------------------------
// Batched blind rotation, one warp per task (bootstrapToTrlwe: test vector
// a = 0, b = mu everywhere).  All warps of a CTA walk the same bootstrapping key
// bk[i] row by row; each 16 KiB row (both output polynomials) is staged once per
// CTA through a ring of S shared-memory slots by the bulk-copy (TMA) engine and
// consumed by every warp.  The last warp to release a slot refills it.
//
// Output: the full TRLWE accumulator (a[1024], b[1024]) per task.
template <int WARPS, int S>
struct Br1024Smem {
    double2 ring[S][1024];
    double2 tw2[kTw2Entries * 32];
    double2 xbuf[WARPS][kFftXbufStride];
    uint32_t acc[WARPS][2048];
    uint32_t dig[WARPS][16 * 32];  // level-1 digits, packed 2 x 16-bit offset binary
    uint64_t full[S];
    uint32_t cnt[S];
    uint64_t tfull[3];  // TM variant: chunk copied into TMEM slot (tcgen05.commit)
    uint32_t tcnt[3];   // TM variant: warps done with a TMEM slot
    uint32_t tstart[3]; // TM variant: warps that started a chunk (the first refills smem)
    uint32_t taddr;     // TM variant: TMEM base (512 columns: three 128-column slots)
    uint32_t go;        // OFS variant: the upper warp half may start
};

// TM: the bootstrapping-key rows reach the warps through TENSOR MEMORY instead of shared-
// memory loads: each 16 KiB chunk, staged in smem by the bulk-copy engine (S = 3 slots), is
// copied once per CTA into one of three 128-column TMEM slots by tcgen05.cp (multicast to
// the four warp quadrants; every warp needs the same per-lane data) and each warp reads its
// lane's 32 values with tcgen05.ld -- the key no longer crosses the shared-memory read
// port once per warp.  Chunk c lives in smem slot and TMEM slot c % 3: the first warp to
// start chunk c (its copy is complete) bulk-loads chunk c + 3 into the smem slot, the last
// warp to finish it copies chunk c + 3 into the TMEM slot.
// OFS: the upper half of the warps starts half a step (two key chunks) after the lower
// half, so the two warps sharing a scheduler (w, w + WARPS/2) run out of phase: one in its
// FP64-bound butterflies while the other is in its shared-memory-bound transposes / key
// reads.  Needs S >= 3 ring slots for the lead.
template <int WARPS, int S, int BG, bool TM = false, bool OFS = false>
__global__ void __launch_bounds__(WARPS * 32, 1)
    br1024_kernel(const uint32_t* __restrict__ tasks, const double2* __restrict__ bkfd,
                  const double2* __restrict__ tw2g, uint32_t* __restrict__ out, int T, int n)
{
    static_assert(!TM || S == 3, "TM uses a three-slot smem ring");
    static_assert(!OFS || (S >= 3 && !TM), "OFS needs >= 3 slots");
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<Br1024Smem<WARPS, S>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int task = blockIdx.x * WARPS + warp;
    const bool active = task < T;
    if (!active)
        task = T - 1;  // inactive warps shadow a real task to keep the slot protocol
    const uint32_t* lwe = tasks + (size_t)task * (n + 1);
    const int nchunks = 4 * n;

    for (int i = threadIdx.x; i < kTw2Entries * 32; i += blockDim.x)
        sm.tw2[i] = tw2g[i];
    if (threadIdx.x == 0) {
        sm.go = 0;
        for (int s = 0; s < S; s++) {
            mbar_init(&sm.full[s], 1);
            sm.cnt[s] = 0;
        }
        if constexpr (TM) {
            for (int s = 0; s < 3; s++) {
                mbar_init(&sm.tfull[s], 1);
                sm.tcnt[s] = 0;
                sm.tstart[s] = 0;
            }
        }
    }
    if constexpr (TM) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             smem_u32(&sm.taddr))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        tmem_fence_before();
    }
    __syncthreads();
    if constexpr (TM)
        tmem_fence_after();
    // TM: copy chunk cn (smem slot cn % 3) into TMEM slot cn % 3, completion on tfull
    auto issue_cp = [&](int cn) {
        const int s3 = cn % 3;
        mbar_wait(&sm.full[s3], (uint32_t)((cn / 3) & 1));
        const uint32_t tb = sm.taddr + (uint32_t)(s3 * 128);
#pragma unroll 1
        for (int q = 0; q < 32; q++)  // row q = (poly, j): 32 lanes x 16 bytes
            tmem_cp_32x128b_x4(tb + (uint32_t)(q * 4), &sm.ring[s3][q * 32]);
        tmem_commit(&sm.tfull[s3]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < S && s < nchunks; s++) {
            mbar_arrive_expect_tx(&sm.full[s], 16384);
            bulk_g2s(sm.ring[s], bkfd + (size_t)s * 1024, 16384, &sm.full[s]);
        }
        if constexpr (TM) {
            for (int cn = 0; cn < 3 && cn < nchunks; cn++)
                issue_cp(cn);
        }
    }

    // acc = X^{-round(2N b)} * (0, mu...mu)  (blindRotate init, ops.cpp:727-730)
    uint32_t* acc = sm.acc[warp];
    {
        const uint32_t rot = (2048u - mod_switch_2n(lwe[n], 11)) & 2047u;
        for (int q = lane; q < 1024; q += 32) {
            acc[q] = 0;
            uint32_t val;
            if (rot < 1024)
                val = ((uint32_t)q < rot) ? (0u - kMu32) : kMu32;
            else
                val = ((uint32_t)q < rot - 1024) ? kMu32 : (0u - kMu32);
            acc[1024 + q] = val;
        }
    }
    __syncwarp();

    // decomposePoly constants (poly.hpp:79-97), l = 2: no final rounding bit.
    constexpr uint32_t kHalf = 1u << (BG - 1);
    constexpr uint32_t kMask = (1u << BG) - 1;
    constexpr uint32_t kOffset = (kHalf << (32 - BG)) + (kHalf << (32 - 2 * BG));
    double2* xbuf = sm.xbuf[warp];

    double2 accA[16], accB[16];

    // Slot release: the last warp to finish with chunk c refills its slot with c + S.
    auto release = [&](int c) {
        if constexpr (TM) {
            tmem_fence_before();
            __syncwarp();
            if (lane == 0) {
                const int s3 = c % 3;
                const uint32_t old = atomicAdd(&sm.tcnt[s3], 1u);
                if (old == WARPS - 1) {
                    sm.tcnt[s3] = 0;
                    tmem_fence_after();
                    if (c + 3 < nchunks)
                        issue_cp(c + 3);  // TMEM slot free; waits for the bulk load of c + 3
                }
            }
            return;
        }
        __syncwarp();
        if (lane == 0) {
            const int s = c % S;
            const uint32_t old = atomicAdd(&sm.cnt[s], 1u);
            if (old == WARPS - 1) {
                sm.cnt[s] = 0;
                const int cn = c + S;
                if (cn < nchunks) {
                    fence_proxy_async();
                    mbar_arrive_expect_tx(&sm.full[s], 16384);
                    bulk_g2s(sm.ring[s], bkfd + (size_t)cn * 1024, 16384, &sm.full[s]);
                }
            }
        }
    };
    // diff = (X^bara - 1) * acc_P (polyMulByXkMinusOne, poly.hpp:51-57) computed once per
    // polynomial; of its two digit levels (decomposePoly, poly.hpp:79-97) level 0 goes
    // straight into the transform registers z and level 1 is parked in smem as packed
    // 16-bit offset-binary pairs (coefficients p, p+512) for the second transform.
    // lane + 32 j is recomputed from an opaque base every step so the compiler does not
    // hoist 32 loop-invariant indices into (spilled) registers.
    auto digits = [&](int P, uint32_t bara, double2 (&z)[16]) {
        const uint32_t* src = acc + P * 1024;
        const uint32_t lo = (uint32_t)lane + (uint32_t)opaque_zero();
        const uint32_t lk = lo - bara;
        const uint32_t* srcl = src + lo;
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const uint32_t v0 = rot_coef1024(src, lk + 32 * j) - srcl[32 * j] + kOffset;
            const uint32_t v1 = rot_coef1024(src, lk + 32 * j + 512) - srcl[32 * j + 512] + kOffset;
            // digits parked in 16-bit offset binary (digit + 2^15) for ob_to_double
            const uint32_t d0 = (v0 >> (32 - BG)) + (32768u - kHalf);
            const uint32_t d1 = (v1 >> (32 - BG)) + (32768u - kHalf);
            const uint32_t e0 = ((v0 >> (32 - 2 * BG)) & kMask) + (32768u - kHalf);
            const uint32_t e1 = ((v1 >> (32 - 2 * BG)) & kMask) + (32768u - kHalf);
            z[j].x = ob_to_double<15>(d0);
            z[j].y = ob_to_double<15>(d1);
            sm.dig[warp][j * 32 + lane] = e0 | (e1 << 16);
        }
    };
    auto load_digits1 = [&](double2 (&z)[16]) {
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const uint32_t w = sm.dig[warp][j * 32 + lane];
            z[j].x = ob_to_double<15>(w & 0xffffu);
            z[j].y = ob_to_double<15>(w >> 16);
        }
    };

    if constexpr (OFS) {
        if (warp >= WARPS / 2) {
            if (lane == 0)
                while (*reinterpret_cast<volatile uint32_t*>(&sm.go) == 0)
                    __nanosleep(64);
            __syncwarp();
        }
    }
#pragma unroll 1
    for (int i = 0; i < n; i++) {
        const uint32_t bara = mod_switch_2n(lwe[i], 11);
        const int c0 = i * 4;
#pragma unroll
        for (int j = 0; j < 16; j++) {
            accA[j] = make_double2(0.0, 0.0);
            accB[j] = make_double2(0.0, 0.0);
        }
#pragma unroll 1
        for (int P = 0; P < 2; P++) {
            double2 z[16];
            digits(P, bara, z);
#pragma unroll 1
            for (int lvl = 0; lvl < 2; lvl++) {
                if (lvl)
                    load_digits1(z);
                fft512_fwd(z, xbuf, sm.tw2, lane);
                const int c = c0 + P * 2 + lvl;
                if constexpr (TM) {
                    const int s3 = c % 3;
                    mbar_wait(&sm.tfull[s3], (uint32_t)((c / 3) & 1));
                    tmem_fence_after();
                    if (lane == 0 && c + 3 < nchunks) {
                        // the first warp to start chunk c refills its smem slot with c + 3
                        // (chunk c's copy into TMEM has completed)
                        const uint32_t st = atomicAdd(&sm.tstart[s3], 1u);
                        if (st == 0) {
                            fence_proxy_async();
                            mbar_arrive_expect_tx(&sm.full[s3], 16384);
                            bulk_g2s(sm.ring[s3], bkfd + (size_t)(c + 3) * 1024, 16384,
                                     &sm.full[s3]);
                        }
                        if (st == WARPS - 1)
                            atomicExch(&sm.tstart[s3], 0u);
                    }
                    const uint32_t tb = sm.taddr + ((uint32_t)(32 * (warp & 3)) << 16) +
                                        (uint32_t)(s3 * 128);
#pragma unroll
                    for (int jb = 0; jb < 16; jb += 4) {
                        uint32_t ra[16], rb[16];
                        tmem_ld_x16(tb + (uint32_t)(jb * 4), ra);         // poly a, j..j+3
                        tmem_ld_x16(tb + (uint32_t)((16 + jb) * 4), rb);  // poly b
                        tmem_wait_ld();
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const int j = jb + u;
                            const double2 ba = make_double2(
                                __hiloint2double((int)ra[4 * u + 1], (int)ra[4 * u]),
                                __hiloint2double((int)ra[4 * u + 3], (int)ra[4 * u + 2]));
                            const double2 bb = make_double2(
                                __hiloint2double((int)rb[4 * u + 1], (int)rb[4 * u]),
                                __hiloint2double((int)rb[4 * u + 3], (int)rb[4 * u + 2]));
                            accA[j].x = fma(z[j].x, ba.x, fma(-z[j].y, ba.y, accA[j].x));
                            accA[j].y = fma(z[j].x, ba.y, fma(z[j].y, ba.x, accA[j].y));
                            accB[j].x = fma(z[j].x, bb.x, fma(-z[j].y, bb.y, accB[j].x));
                            accB[j].y = fma(z[j].x, bb.y, fma(z[j].y, bb.x, accB[j].y));
                        }
                    }
                }
                else {
                    const int s = c % S;
                    mbar_wait(&sm.full[s], (uint32_t)((c / S) & 1));
                    const double2* bk = sm.ring[s];
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        const double2 ba = bk[j * 32 + lane];
                        const double2 bb = bk[512 + j * 32 + lane];
                        accA[j].x = fma(z[j].x, ba.x, fma(-z[j].y, ba.y, accA[j].x));
                        accA[j].y = fma(z[j].x, ba.y, fma(z[j].y, ba.x, accA[j].y));
                        accB[j].x = fma(z[j].x, bb.x, fma(-z[j].y, bb.y, accB[j].x));
                        accB[j].y = fma(z[j].x, bb.y, fma(z[j].y, bb.x, accB[j].y));
                    }
                }
                release(c);
                if constexpr (OFS) {
                    if (c == 1 && warp == 0 && lane == 0)
                        atomicExch(&sm.go, 1u);  // lower half is two chunks ahead
                }
            }
        }
        // inverse transforms, round (llrint, fft.hpp:47-50) and accumulate
        fft512_inv2(accA, accB, xbuf, sm.tw2, lane);
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int p = lane + 32 * j;
            acc[p] += (uint32_t)__double2ll_rn(accA[j].x);
            acc[p + 512] += (uint32_t)__double2ll_rn(accA[j].y);
        }
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int p = lane + 32 * j;
            acc[1024 + p] += (uint32_t)__double2ll_rn(accB[j].x);
            acc[1024 + p + 512] += (uint32_t)__double2ll_rn(accB[j].y);
        }
        __syncwarp();
    }
    if (active) {
        uint4* dst = reinterpret_cast<uint4*>(out + (size_t)task * 2048);
        const uint4* s4 = reinterpret_cast<const uint4*>(acc);
        for (int q = lane; q < 512; q += 32)
            dst[q] = s4[q];
    }
    if constexpr (TM) {
        tmem_fence_before();
        __syncthreads();
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(sm.taddr)
                         : "memory");
    }
}

// ---------------------------------------------------------------------------
// br1024p_kernel: the throughput kernel with TWO warps per task, for partial waves (the
// remainder of a split batch, mid-size batches).  A wave of W <= 4 tasks per SM leaves a
// single warp per scheduler and runs at the latency of one task's 630-step chain; here
// warp P of a task owns accumulator polynomial P: its digits (both levels), its two
// forward transforms, the MAC of its two rows into both outputs, then the partners swap
// the partial sums of each other's output through shared memory, and each warp inverts,
// rounds and accumulates its own polynomial -- the next step's digits of polynomial P only
// read polynomial P, so the pair needs no other synchronisation.  The four key rows of a
// step sit in four 16 KiB slots (chunk 4 i + 2P + lvl in slot 2P + lvl, used by the TASKS
// warps of parity P; the last of them refills it).
template <int TASKS>
struct BrPairSmem {
    double2 ring[4][1024];
    double2 tw2[kTw2Entries * 32];
    double2 xbuf[2 * TASKS][kFftXbufStride];  // transposes, then the partial-sum exchange
    uint32_t acc[TASKS][2048];
    uint32_t dig[2 * TASKS][16 * 32];
    uint64_t full[4];
    uint32_t cnt[4];
};

template <int TASKS, int BG>
__global__ void __launch_bounds__(64 * TASKS, 1)
    br1024p_kernel(const uint32_t* __restrict__ tasks, const double2* __restrict__ bkfd,
                   const double2* __restrict__ tw2g, uint32_t* __restrict__ out, int T, int n)
{
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<BrPairSmem<TASKS>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tl = warp >> 1, P = warp & 1;
    int task = blockIdx.x * TASKS + tl;
    const bool active = task < T;
    if (!active)
        task = T - 1;  // shadow a real task to keep the slot protocol
    const uint32_t* lwe = tasks + (size_t)task * (n + 1);
    const int nchunks = 4 * n;

    for (int i = threadIdx.x; i < kTw2Entries * 32; i += blockDim.x)
        sm.tw2[i] = tw2g[i];
    if (threadIdx.x == 0) {
        for (int s = 0; s < 4; s++) {
            mbar_init(&sm.full[s], 1);
            sm.cnt[s] = 0;
        }
    }
    uint32_t* acc = sm.acc[tl];
    {
        // acc = X^{-round(2N b)} * (0, mu...mu); warp P writes polynomial P
        const uint32_t rot = (2048u - mod_switch_2n(lwe[n], 11)) & 2047u;
        for (int q = lane; q < 1024; q += 32) {
            uint32_t val = 0;
            if (P == 1) {
                if (rot < 1024)
                    val = ((uint32_t)q < rot) ? (0u - kMu32) : kMu32;
                else
                    val = ((uint32_t)q < rot - 1024) ? kMu32 : (0u - kMu32);
            }
            acc[P * 1024 + q] = val;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < 4 && s < nchunks; s++) {
            mbar_arrive_expect_tx(&sm.full[s], 16384);
            bulk_g2s(sm.ring[s], bkfd + (size_t)s * 1024, 16384, &sm.full[s]);
        }
    }

    constexpr uint32_t kHalf = 1u << (BG - 1);
    constexpr uint32_t kMask = (1u << BG) - 1;
    constexpr uint32_t kOffset = (kHalf << (32 - BG)) + (kHalf << (32 - 2 * BG));
    double2* xbuf = sm.xbuf[warp];
    const double2* xpeer = sm.xbuf[warp ^ 1];
    const uint32_t* src = acc + P * 1024;
    double2 accOwn[16], accOth[16];

    auto release = [&](int c) {
        __syncwarp();
        if (lane == 0) {
            const int s = c & 3;
            const uint32_t old = atomicAdd(&sm.cnt[s], 1u);
            if (old == TASKS - 1) {
                sm.cnt[s] = 0;
                const int cn = c + 4;
                if (cn < nchunks) {
                    fence_proxy_async();
                    mbar_arrive_expect_tx(&sm.full[s], 16384);
                    bulk_g2s(sm.ring[s], bkfd + (size_t)cn * 1024, 16384, &sm.full[s]);
                }
            }
        }
    };

#pragma unroll 1
    for (int i = 0; i < n; i++) {
        const uint32_t bara = mod_switch_2n(lwe[i], 11);
#pragma unroll
        for (int j = 0; j < 16; j++) {
            accOwn[j] = make_double2(0.0, 0.0);
            accOth[j] = make_double2(0.0, 0.0);
        }
        double2 z[16];
        {
            // (X^bara - 1) acc_P; level-0 digits to z, level-1 parked (see br1024_kernel)
            const uint32_t lo = (uint32_t)lane + (uint32_t)opaque_zero();
            const uint32_t lk = lo - bara;
            const uint32_t* srcl = src + lo;
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const uint32_t v0 = rot_coef1024(src, lk + 32 * j) - srcl[32 * j] + kOffset;
                const uint32_t v1 = rot_coef1024(src, lk + 32 * j + 512) - srcl[32 * j + 512] + kOffset;
                const uint32_t d0 = (v0 >> (32 - BG)) + (32768u - kHalf);
                const uint32_t d1 = (v1 >> (32 - BG)) + (32768u - kHalf);
                const uint32_t e0 = ((v0 >> (32 - 2 * BG)) & kMask) + (32768u - kHalf);
                const uint32_t e1 = ((v1 >> (32 - 2 * BG)) & kMask) + (32768u - kHalf);
                z[j].x = ob_to_double<15>(d0);
                z[j].y = ob_to_double<15>(d1);
                sm.dig[warp][j * 32 + lane] = e0 | (e1 << 16);
            }
        }
#pragma unroll 1
        for (int lvl = 0; lvl < 2; lvl++) {
            if (lvl) {
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    const uint32_t w = sm.dig[warp][j * 32 + lane];
                    z[j].x = ob_to_double<15>(w & 0xffffu);
                    z[j].y = ob_to_double<15>(w >> 16);
                }
            }
            fft512_fwd(z, xbuf, sm.tw2, lane);
            const int c = 4 * i + 2 * P + lvl;
            mbar_wait(&sm.full[c & 3], (uint32_t)(i & 1));
            const double2* bo = sm.ring[c & 3] + P * 512;
            const double2* bt = sm.ring[c & 3] + (1 - P) * 512;
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const double2 ba = bo[j * 32 + lane];
                const double2 bb = bt[j * 32 + lane];
                accOwn[j].x = fma(z[j].x, ba.x, fma(-z[j].y, ba.y, accOwn[j].x));
                accOwn[j].y = fma(z[j].x, ba.y, fma(z[j].y, ba.x, accOwn[j].y));
                accOth[j].x = fma(z[j].x, bb.x, fma(-z[j].y, bb.y, accOth[j].x));
                accOth[j].y = fma(z[j].x, bb.y, fma(z[j].y, bb.x, accOth[j].y));
            }
            release(c);
        }
        // swap the partial sums of the partner's output, then invert my own output
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            xbuf[j * 32 + lane] = accOth[j];
        bar_group(1 + tl, 64);
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const double2 q = xpeer[j * 32 + lane];
            accOwn[j].x += q.x;
            accOwn[j].y += q.y;
        }
        bar_group(1 + tl, 64);  // the partner has read my buffer before I transpose in it
        fft512_inv(accOwn, xbuf, sm.tw2, lane);
        uint32_t* dst = acc + P * 1024;
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int p = lane + 32 * j;
            dst[p] += (uint32_t)__double2ll_rn(accOwn[j].x);
            dst[p + 512] += (uint32_t)__double2ll_rn(accOwn[j].y);
        }
        __syncwarp();
    }
    __syncthreads();
    if (active) {
        uint4* d4 = reinterpret_cast<uint4*>(out + (size_t)task * 2048 + P * 1024);
        const uint4* s4 = reinterpret_cast<const uint4*>(acc + P * 1024);
        for (int q = lane; q < 256; q += 32)
            d4[q] = s4[q];
    }
}

// ---------------------------------------------------------------------------
// Latency-optimised blind rotation for narrow netlist levels (T <= ~2 x SMs), where
// br1024_kernel runs one dependent chain of n external products per warp and per-level
// latency is the chain length (630 x ~9 us).  Here FOUR warps share one task: warp r
// owns gadget row r = 2P + lvl (digit level lvl of accumulator polynomial P), so each
// external product is one forward transform deep instead of four:
//   1. warp r: digits of row r of (X^bara - 1) acc   (decomposePoly, poly.hpp:79-97)
//   2. warp r: forward transform, published to smem
//   3. warp 0 forms A = sum_r z_r bkA_r, warp 1 B = sum_r z_r bkB_r (own row from
//      registers), in row order as in br1024_kernel
//   4. warps 0 / 1: inverse transform, round, acc.a / acc.b += (ops.cpp:587-597)
// Every coefficient is an integer the FP64 error (<< 1/2) rounds back to exactly, so the
// outputs equal the reference's.  All four BK rows of step i are staged together (64 KiB)
// by the bulk-copy engine, two steps in flight; warp 3 refills a slot once warps 0 and 1
// have released it (mbarrier `empty`).
constexpr int kLatBuf = kFftXbufStride;  // double2 per exchange / transpose buffer
constexpr int kLatThreads = 160;          // 4 transform warps + 1 producer warp
constexpr int kLatProducerSleepNs = 1024;  // producer back-off between empty-slot probes

struct BrLatSmem {
    double2 ring[2][4 * 1024];
    double2 tw2[kTw2Entries * 32];
    double2 bufA[4][kLatBuf];  // transformed row z_r (also warp r's forward transposes)
    double2 bufB[2][kLatBuf];  // inverse-transform transposes of warps 0 / 1
    // accumulator polynomial P at acc[P * stride]: EXT = 1 keeps its negacyclic extension
    // (acc, -acc, acc: 3072 words), so a coefficient of X^-bara acc is one load at a lane
    // base plus an immediate offset (no index wrap / sign select in the digit pass); EXT = 2
    // keeps (acc, -acc) and applies one per-lane sign instead of the third copy
    uint32_t acc[2 * 3072];
    uint64_t full[2];
    uint64_t empty[2];  // slot consumed by the four transform warps (count 4)
    __device__ double2* xbuf(int r) { return bufA[r]; }
};


// PROBE: per-warp clock64 totals of the step phases -> probe[task][warp][16] (tuning).
// EXT: negacyclic-extension accumulator (see BrLatSmem).  Measured per 140-task level:
// 1.889 ms (EXT 0, the round-1 layout: 1024 words per polynomial, rot_coef1024), 1.679 ms
// (EXT 1), 1.672 ms (EXT 2, default); the others stay for A/B (VSP_LAT_EXT=0 / 1).
template <int BG, bool PROBE = false, int EXT = 2>
__global__ void __launch_bounds__(kLatThreads, 1)
    br_lat_kernel(const uint32_t* __restrict__ tasks, const double2* __restrict__ bkfd,
                  const double2* __restrict__ tw2g, uint32_t* __restrict__ out, int n,
                  unsigned long long* __restrict__ probe = nullptr)
{
    unsigned long long ph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tprev = PROBE ? clock64() : 0;
    auto mark = [&](int k) {
        if constexpr (PROBE) {
            const long long t = clock64();
            ph[k] += (unsigned long long)(t - tprev);
            tprev = t;
        }
    };
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<BrLatSmem*>(smem_raw);
    const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int task = blockIdx.x;
    const uint32_t* lwe = tasks + (size_t)task * (n + 1);

    for (int i = threadIdx.x; i < kTw2Entries * 32; i += blockDim.x)
        sm.tw2[i] = tw2g[i];
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2; q++) {
            mbar_init(&sm.full[q], 1);
            mbar_init(&sm.empty[q], 4);
        }
    }
    constexpr int kStride = EXT == 1 ? 3072 : EXT == 2 ? 2048 : 1024;  // words per polynomial
    {
        const uint32_t rot = (2048u - mod_switch_2n(lwe[n], 11)) & 2047u;
        for (int q = threadIdx.x; q < 1024; q += blockDim.x) {
            sm.acc[q] = 0;
            uint32_t val;
            if (rot < 1024)
                val = ((uint32_t)q < rot) ? (0u - kMu32) : kMu32;
            else
                val = ((uint32_t)q < rot - 1024) ? kMu32 : (0u - kMu32);
            sm.acc[kStride + q] = val;
            if constexpr (EXT) {
                sm.acc[1024 + q] = 0;
                sm.acc[kStride + 1024 + q] = 0u - val;
            }
            if constexpr (EXT == 1) {
                sm.acc[2048 + q] = 0;
                sm.acc[kStride + 2048 + q] = val;
            }
        }
    }
    __syncthreads();

    if (r == 4) {
        // producer warp: keeps the two-slot ring of bk rows full.  A warp issuing bulk
        // copies is slowed while they are in flight, so no transform warp issues them.
        if (lane == 0) {
            for (int i = 0; i < n; i++) {
                const int s = i & 1;
                if (i >= 2)
                    mbar_wait_sleep(&sm.empty[s], (uint32_t)(((i - 2) >> 1) & 1), kLatProducerSleepNs);
                mbar_arrive_expect_tx(&sm.full[s], 65536);
                bulk_g2s(sm.ring[s], bkfd + (size_t)i * 4096, 65536, &sm.full[s]);
            }
        }
    }
    else {
        constexpr uint32_t kHalf = 1u << (BG - 1);
        constexpr uint32_t kMask = (1u << BG) - 1;
        constexpr uint32_t kOffset = (kHalf << (32 - BG)) + (kHalf << (32 - 2 * BG));
        const int P = r >> 1, lvl = r & 1;
        const uint32_t* src = sm.acc + P * kStride;
        const uint32_t sh = (uint32_t)(32 - (lvl + 1) * BG);
        // MAC / inverse role: output o (0: a, 1: b) on the warp pair (o, o + 2), half h
        const int o = r & 1, h = r >> 1;
        const int L = 16 * h + (lane & 15), e = lane >> 4;

        // this lane's per-lane twiddles in registers for the whole rotation (the kernel has
        // the registers to spare; the loads were ~11% of its shared-memory wavefronts):
        // tangent forms for the forward transform, plain ones at the virtual lane L of the
        // pair inverse
        double2 twf[kTw2Plain], twi[kTw2Plain];
#pragma unroll
        for (int q = 0; q < kTw2Plain; q++) {
            twf[q] = sm.tw2[(kTw2Plain + q) * 32 + lane];
            twi[q] = sm.tw2[q * 32 + L];
        }
        // a_i is fetched one step ahead (lwe[i + 1] <= lwe[n] is in bounds) so the global
        // load latency hides behind the current external product
        uint32_t a_next = lwe[0];
#pragma unroll 1
        for (int i = 0; i < n; i++) {
            const uint32_t bara = mod_switch_2n(a_next, 11);
            a_next = lwe[i + 1];
            mark(9);
            double2 z[16];
            {
                const uint32_t lo = (uint32_t)lane + (uint32_t)opaque_zero();
                const uint32_t lk = lo - bara;
                const uint32_t* srcl = src + lo;
                // EXT: X^-bara acc at lane + 32 j is srcr[32 j] (EXT 2: times (-1)^sg)
                const uint32_t* srcr = src + (lk & (EXT == 1 ? 2047u : 1023u));
                const uint32_t sg = EXT == 2 ? (lk >> 10) & 1u : 0u;
                const uint32_t sm_ = 0u - sg, ko = kOffset + sg;
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    const uint32_t r0 = EXT ? srcr[32 * j] ^ sm_ : rot_coef1024(src, lk + 32 * j);
                    const uint32_t r1 = EXT ? srcr[32 * j + 512] ^ sm_ : rot_coef1024(src, lk + 32 * j + 512);
                    const uint32_t v0 = r0 - srcl[32 * j] + ko;
                    const uint32_t v1 = r1 - srcl[32 * j + 512] + ko;
                    // level-lvl digit = bits [32 - (lvl+1) BG, 32 - lvl BG) of v, recentred
                    // (the mask is a no-op for level 0); offset binary for ob_to_double
                    z[j].x = ob_to_double<31>(((v0 >> sh) & kMask) + (0x80000000u - kHalf));
                    z[j].y = ob_to_double<31>(((v1 >> sh) & kMask) + (0x80000000u - kHalf));
                }
            }
            mark(0);
            fft512_fwd_regs(z, sm.xbuf(r), twf, lane);
            mark(1);
            // publish the transformed row: z_r -> bufA[r] (warp r's own transpose buffer,
            // free again after the transform's last __syncwarp)
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++)
                sm.bufA[r][j * 32 + lane] = z[j];
            const int s = i & 1;
            // the key rows of this step: waited for before the barrier, so the wait overlaps
            // the slowest warp's transform instead of following it
            mbar_wait(&sm.full[s], (uint32_t)((i >> 1) & 1));
            mark(3);
            bar_group(1, 128);  // all four rows transformed
            mark(2);
            // output o at this lane's 8 slots: acc_o = sum_q z_q . bk[q][o], rows in order
            // 0..3 as in br1024_kernel
            const double2* bk = sm.ring[s] + o * 512;
            double2 u[8];
#pragma unroll
            for (int t = 0; t < 8; t++) {
                const int q = (2 * t + e) * 32 + L;
                const double2 z0 = sm.bufA[0][q], z1 = sm.bufA[1][q];
                const double2 z2 = sm.bufA[2][q], z3 = sm.bufA[3][q];
                const double2 b0 = bk[q], b1 = bk[1024 + q], b2 = bk[2048 + q], b3 = bk[3072 + q];
                double ax = fma(z0.x, b0.x, -z0.y * b0.y);
                double ay = fma(z0.x, b0.y, z0.y * b0.x);
                ax = fma(z1.x, b1.x, fma(-z1.y, b1.y, ax));
                ay = fma(z1.x, b1.y, fma(z1.y, b1.x, ay));
                ax = fma(z2.x, b2.x, fma(-z2.y, b2.y, ax));
                ay = fma(z2.x, b2.y, fma(z2.y, b2.x, ay));
                ax = fma(z3.x, b3.x, fma(-z3.y, b3.y, ax));
                ay = fma(z3.x, b3.y, fma(z3.y, b3.x, ay));
                u[t] = make_double2(ax, ay);
            }
            __syncwarp();
            if (lane == 0)
                mbar_arrive(&sm.empty[s]);  // this warp is done with slot s
            mark(5);
            fft512_inv_pair_regs(u, sm.bufB[o], twi, lane, h, 3 + o);
            mark(6);
            // (every warp read acc for its digits before barrier 1)
            uint32_t* dst = sm.acc + o * kStride;
#pragma unroll
            for (int t = 0; t < 8; t++) {
                const int p = L + 32 * (t + 8 * e);
                const uint32_t n0 = dst[p] + (uint32_t)__double2ll_rn(u[t].x);
                const uint32_t n1 = dst[p + 512] + (uint32_t)__double2ll_rn(u[t].y);
                dst[p] = n0;
                dst[p + 512] = n1;
                if constexpr (EXT) {
                    dst[p + 1024] = 0u - n0;
                    dst[p + 1536] = 0u - n1;
                }
                if constexpr (EXT == 1) {
                    dst[p + 2048] = n0;
                    dst[p + 2560] = n1;
                }
            }
            mark(7);
            bar_group(2, 128);  // acc updated before the next step's digits
            mark(8);
        }
    }
    if constexpr (PROBE) {
        if (lane == 0 && r < 4)
            for (int k = 0; k < 10; k++)
                probe[((size_t)task * 4 + r) * 16 + k] = ph[k];
    }
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(out + (size_t)task * 2048);
    for (int q = threadIdx.x; q < 512; q += blockDim.x)
        dst[q] = reinterpret_cast<const uint4*>(sm.acc + (q >> 8) * kStride)[q & 255];
}

// ---------------------------------------------------------------------------
// br_lat2_kernel: br_lat_kernel's four-warp task, TASKS tasks per CTA (one SM), all on the
// same key stream.  br_lat's step is bound by the shared-memory crossbar at ~58% of it
// with one warp per scheduler; two tasks per SM run two warps per scheduler and leave half
// of the SMs of a narrow level free (the netlist runner puts the RAM write bars there).
// The key arrives in 16 KiB chunks (one gadget row, both outputs) through an S-slot ring:
// chunk c = 4 i + q of step i lives in slot c % S; every MAC warp of the CTA releases the
// four slots of its step on `empty` (count 4 TASKS) and the producer warp refills them.
constexpr int kLat2Threads(int tasks) { return 128 * tasks + 32; }

template <int TASKS, int S>
struct BrLat2Smem {
    double2 ring[S][1024];
    double2 tw2[kTw2Entries * 32];
    double2 bufA[TASKS][4][kLatBuf];
    double2 bufB[TASKS][2][kLatBuf];
    uint32_t acc[TASKS][2048];
    uint64_t full[S];
    uint64_t empty[S];
};

template <int BG, int TASKS, int S>
__global__ void __launch_bounds__(128 * TASKS + 32, 1)
    br_lat2_kernel(const uint32_t* __restrict__ tasks, const double2* __restrict__ bkfd,
                   const double2* __restrict__ tw2g, uint32_t* __restrict__ out, int T, int n)
{
    static_assert(S >= 4, "one whole step of key rows must fit the ring");
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<BrLat2Smem<TASKS, S>*>(smem_raw);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tl = w >> 2;  // task slot of this warp (producer: tl == TASKS)
    const int r = w & 3;
    int task = blockIdx.x * TASKS + (tl < TASKS ? tl : 0);
    const bool active = task < T;
    if (!active)
        task = T - 1;  // shadow a real task: the ring protocol needs every warp
    const uint32_t* lwe = tasks + (size_t)task * (n + 1);
    const int nchunks = 4 * n;

    for (int i = threadIdx.x; i < kTw2Entries * 32; i += blockDim.x)
        sm.tw2[i] = tw2g[i];
    if (threadIdx.x == 0) {
        for (int q = 0; q < S; q++) {
            mbar_init(&sm.full[q], 1);
            mbar_init(&sm.empty[q], 4 * TASKS);
        }
    }
    if (tl < TASKS) {
        const uint32_t rot = (2048u - mod_switch_2n(lwe[n], 11)) & 2047u;
        uint32_t* a = sm.acc[tl];
        for (int q = threadIdx.x & 127; q < 1024; q += 128) {
            a[q] = 0;
            uint32_t val;
            if (rot < 1024)
                val = ((uint32_t)q < rot) ? (0u - kMu32) : kMu32;
            else
                val = ((uint32_t)q < rot - 1024) ? kMu32 : (0u - kMu32);
            a[1024 + q] = val;
        }
    }
    __syncthreads();

    if (tl == TASKS) {
        // producer warp (see br_lat_kernel: no transform warp issues bulk copies)
        if (lane == 0) {
            for (int c = 0; c < nchunks; c++) {
                const int q = c % S;
                if (c >= S)
                    mbar_wait(&sm.empty[q], (uint32_t)(((c / S) - 1) & 1));
                mbar_arrive_expect_tx(&sm.full[q], 16384);
                bulk_g2s(sm.ring[q], bkfd + (size_t)c * 1024, 16384, &sm.full[q]);
            }
        }
    }
    else {
        constexpr uint32_t kHalf = 1u << (BG - 1);
        constexpr uint32_t kMask = (1u << BG) - 1;
        constexpr uint32_t kOffset = (kHalf << (32 - BG)) + (kHalf << (32 - 2 * BG));
        const int P = r >> 1, lvl = r & 1;
        uint32_t* accT = sm.acc[tl];
        const uint32_t* src = accT + P * 1024;
        const uint32_t sh = (uint32_t)(32 - (lvl + 1) * BG);
        const int o = r & 1, h = r >> 1;
        const int L = 16 * h + (lane & 15), e = lane >> 4;
        const int barA = 1 + 4 * tl, barB = 2 + 4 * tl, barPair = 3 + 4 * tl + o;
        double2 (&bufA)[4][kLatBuf] = sm.bufA[tl];

        uint32_t a_next = lwe[0];
#pragma unroll 1
        for (int i = 0; i < n; i++) {
            const uint32_t bara = mod_switch_2n(a_next, 11);
            a_next = lwe[i + 1];
            double2 z[16];
            {
                const uint32_t lo = (uint32_t)lane + (uint32_t)opaque_zero();
                const uint32_t lk = lo - bara;
                const uint32_t* srcl = src + lo;
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    const uint32_t v0 = rot_coef1024(src, lk + 32 * j) - srcl[32 * j] + kOffset;
                    const uint32_t v1 = rot_coef1024(src, lk + 32 * j + 512) - srcl[32 * j + 512] + kOffset;
                    z[j].x = ob_to_double<31>(((v0 >> sh) & kMask) + (0x80000000u - kHalf));
                    z[j].y = ob_to_double<31>(((v1 >> sh) & kMask) + (0x80000000u - kHalf));
                }
            }
            fft512_fwd(z, bufA[r], sm.tw2, lane);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++)
                bufA[r][j * 32 + lane] = z[j];
            bar_group(barA, 128);  // this task's four rows transformed
            const int c0 = 4 * i;
#pragma unroll
            for (int q = 0; q < 4; q++)
                mbar_wait(&sm.full[(c0 + q) % S], (uint32_t)(((c0 + q) / S) & 1));
            const double2* b0p = sm.ring[(c0 + 0) % S] + o * 512;
            const double2* b1p = sm.ring[(c0 + 1) % S] + o * 512;
            const double2* b2p = sm.ring[(c0 + 2) % S] + o * 512;
            const double2* b3p = sm.ring[(c0 + 3) % S] + o * 512;
            double2 u[8];
#pragma unroll
            for (int t = 0; t < 8; t++) {
                const int q = (2 * t + e) * 32 + L;
                const double2 z0 = bufA[0][q], z1 = bufA[1][q];
                const double2 z2 = bufA[2][q], z3 = bufA[3][q];
                const double2 b0 = b0p[q], b1 = b1p[q], b2 = b2p[q], b3 = b3p[q];
                double ax = fma(z0.x, b0.x, -z0.y * b0.y);
                double ay = fma(z0.x, b0.y, z0.y * b0.x);
                ax = fma(z1.x, b1.x, fma(-z1.y, b1.y, ax));
                ay = fma(z1.x, b1.y, fma(z1.y, b1.x, ay));
                ax = fma(z2.x, b2.x, fma(-z2.y, b2.y, ax));
                ay = fma(z2.x, b2.y, fma(z2.y, b2.x, ay));
                ax = fma(z3.x, b3.x, fma(-z3.y, b3.y, ax));
                ay = fma(z3.x, b3.y, fma(z3.y, b3.x, ay));
                u[t] = make_double2(ax, ay);
            }
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < 4; q++)
                    mbar_arrive(&sm.empty[(c0 + q) % S]);
            }
            fft512_inv_pair(u, sm.bufB[tl][o], sm.tw2, lane, h, barPair);
            uint32_t* dst = accT + o * 1024;
#pragma unroll
            for (int t = 0; t < 8; t++) {
                const int p = L + 32 * (t + 8 * e);
                dst[p] += (uint32_t)__double2ll_rn(u[t].x);
                dst[p + 512] += (uint32_t)__double2ll_rn(u[t].y);
            }
            bar_group(barB, 128);  // acc updated before the next step's digits
        }
    }
    __syncthreads();
    if (tl < TASKS && active) {
        uint4* dst = reinterpret_cast<uint4*>(out + (size_t)task * 2048);
        const uint4* s4 = reinterpret_cast<const uint4*>(sm.acc[tl]);
        for (int q = threadIdx.x & 127; q < 512; q += 128)
            dst[q] = s4[q];
    }
}

// ---------------------------------------------------------------------------
// Gate linear combinations (linComb + per-kind coefficients, ops.cpp:774-893).
// Emits the level-0 TLWE input of each blind-rotation task; NOT is finished here
// (pure negation, ops.cpp:849-855).
// gtask[g] = (t0, t1): task slots of gate g (t1 >= 0 only for MUX; t0 < 0 for NOT).
__global__ void gate_prep_kernel(const int* __restrict__ kinds, const uint32_t* __restrict__ in,
                                 const int2* __restrict__ gtask, uint32_t* __restrict__ tasks,
                                 uint32_t* __restrict__ out, int G, int n)
{
    const int g = blockIdx.x;
    if (g >= G)
        return;
    const int kind = kinds[g];
    const int2 tt = gtask[g];
    const uint32_t* x = in + (size_t)g * 3 * (n + 1);
    const uint32_t* y = x + (n + 1);
    const uint32_t* z = y + (n + 1);
    const uint32_t mu = kMu32, nmu = 0u - kMu32;
    int c0 = 1, c1 = 1;
    uint32_t bias = nmu;
    switch (kind) {
    case kAnd: c0 = 1; c1 = 1; bias = nmu; break;
    case kNand: c0 = -1; c1 = -1; bias = mu; break;
    case kOr: c0 = 1; c1 = 1; bias = mu; break;
    case kNor: c0 = -1; c1 = -1; bias = nmu; break;
    case kXor: c0 = 2; c1 = 2; bias = 2 * mu; break;
    case kXnor: c0 = -2; c1 = -2; bias = 2 * nmu; break;
    case kAndNot: c0 = 1; c1 = -1; bias = nmu; break;
    case kOrNot: c0 = 1; c1 = -1; bias = mu; break;
    default: break;
    }
    for (int k = threadIdx.x; k <= n; k += blockDim.x) {
        const uint32_t bk = (k == n) ? 1u : 0u;
        if (kind == kNot) {
            out[(size_t)g * (n + 1) + k] = 0u - x[k];
        }
        else if (kind == kMux) {  // in = {sel, a, b}
            tasks[(size_t)tt.x * (n + 1) + k] = x[k] + y[k] + bk * nmu;
            tasks[(size_t)tt.y * (n + 1) + k] = z[k] - x[k] + bk * nmu;
        }
        else {
            tasks[(size_t)tt.x * (n + 1) + k] =
                (uint32_t)c0 * x[k] + (uint32_t)c1 * y[k] + bk * bias;
        }
    }
}

// The same, reading the gate inputs straight from the netlist runner's value table
// (innet[3 g + s]: net of input s, -1 for none) and writing NOT outputs to their net.
__global__ void gate_prep_idx_kernel(const int* __restrict__ kinds, const uint32_t* __restrict__ vals,
                                     const int* __restrict__ innet, const int* __restrict__ onet,
                                     const int2* __restrict__ gtask, uint32_t* __restrict__ tasks,
                                     uint32_t* __restrict__ outvals, int G, int n)
{
    const int g = blockIdx.x;
    if (g >= G)
        return;
    const int kind = kinds[g];
    const int2 tt = gtask[g];
    const size_t w = n + 1;
    const int i0 = innet[3 * g], i1 = innet[3 * g + 1], i2 = innet[3 * g + 2];
    const uint32_t* x = vals + (size_t)i0 * w;
    const uint32_t* y = vals + (size_t)(i1 >= 0 ? i1 : i0) * w;
    const uint32_t* z = vals + (size_t)(i2 >= 0 ? i2 : i0) * w;
    const uint32_t mu = kMu32, nmu = 0u - kMu32;
    int c0 = 1, c1 = 1;
    uint32_t bias = nmu;
    switch (kind) {
    case kAnd: c0 = 1; c1 = 1; bias = nmu; break;
    case kNand: c0 = -1; c1 = -1; bias = mu; break;
    case kOr: c0 = 1; c1 = 1; bias = mu; break;
    case kNor: c0 = -1; c1 = -1; bias = nmu; break;
    case kXor: c0 = 2; c1 = 2; bias = 2 * mu; break;
    case kXnor: c0 = -2; c1 = -2; bias = 2 * nmu; break;
    case kAndNot: c0 = 1; c1 = -1; bias = nmu; break;
    case kOrNot: c0 = 1; c1 = -1; bias = mu; break;
    default: break;
    }
    for (int k = threadIdx.x; k <= n; k += blockDim.x) {
        const uint32_t bk = (k == n) ? 1u : 0u;
        if (kind == kNot) {
            outvals[(size_t)onet[g] * w + k] = 0u - x[k];
        }
        else if (kind == kMux) {  // in = {sel, a, b}
            tasks[(size_t)tt.x * w + k] = x[k] + y[k] + bk * nmu;
            tasks[(size_t)tt.y * w + k] = z[k] - x[k] + bk * nmu;
        }
        else {
            tasks[(size_t)tt.x * w + k] = (uint32_t)c0 * x[k] + (uint32_t)c1 * y[k] + bk * bias;
        }
    }
}

// ---------------------------------------------------------------------------
// Batched identity key switch (ops.cpp:651-679) fused with sampleExtract(.,0)
// (ops.cpp:628-643) and the MUX level-1 sum (ops.cpp:886-892).
//
// out[g][k] = b'_g [k == n] - sum_{i,j} ksk[i][j][d_g(i,j) - 1][k]   (mod 2^32)
//
// Grid (ceil(Gl/GT), KSPLIT): CTA (x, y) handles GT gates x all n+1 coordinates over
// the slice y of the input index i.  For every (i, j) the CTA reads the (2^b - 1)
// candidate KSK rows once (coalesced) and each gate selects its row by digit, so the
// KSK is streamed once per GT gates; slices are combined with wrap-around u32
// atomics into `out`, which iks_init_kernel pre-sets to (0,...,0, b').  Integer
// addition is associative, so the result is independent of the order.
// Coefficient i of sampleExtract(TRLWE, k) (ops.cpp:628-643): a'[i] = A[k-i] (i <= k),
// -A[N+k-i] (i > k).
__device__ __forceinline__ uint32_t se_coef(const uint32_t* A, int N, int k, int i)
{
    return i <= k ? A[k - i] : 0u - A[N + k - i];
}

__device__ __forceinline__ void iks_level1_coef(const uint32_t* __restrict__ trlwe, int2 tt, int N,
                                                int k, int i, uint32_t& a)
{
    a = se_coef(trlwe + (size_t)tt.x * 2 * N, N, k, i);
    if (tt.y >= 0)
        a += se_coef(trlwe + (size_t)tt.y * 2 * N, N, k, i);
}

// oidx (optional, every key-switch kernel): output row of gate g is oidx[g] instead of g
// (the netlist runner writes straight into its value table, row = output net).
__global__ void iks_init_kernel(const uint32_t* __restrict__ trlwe, const int2* __restrict__ gtask,
                                const int* __restrict__ glist, const int* __restrict__ seidx,
                                int Gl, uint32_t* __restrict__ out, int n, int N,
                                const int* __restrict__ oidx = nullptr)
{
    const int gi = blockIdx.x;
    if (gi >= Gl)
        return;
    const int gate = glist[gi];
    const int2 tt = gtask[gate];
    const int se = seidx ? seidx[gate] : 0;
    for (int k = threadIdx.x; k <= n; k += blockDim.x) {
        uint32_t v = 0;
        if (k == n) {
            v = trlwe[(size_t)tt.x * 2 * N + N + se];
            if (tt.y >= 0)
                v += trlwe[(size_t)tt.y * 2 * N + N + se] + kMu32;
        }
        out[(size_t)(oidx ? oidx[gate] : gate) * (n + 1) + k] = v;
    }
}

template <int BASEBITS, int GT, int KPT>
__global__ void __launch_bounds__(256) iks_kernel(
    const uint32_t* __restrict__ trlwe, const int2* __restrict__ gtask,
    const int* __restrict__ glist, const int* __restrict__ seidx, int Gl,
    const uint32_t* __restrict__ ksk, uint32_t* __restrict__ out, int n, int N, int t,
    const int* __restrict__ oidx = nullptr)
{
    static_assert(GT * BASEBITS <= 64, "digit packing");
    constexpr uint32_t kMask = (1u << BASEBITS) - 1;
    constexpr int kPerBase = (1 << BASEBITS) - 1;
    extern __shared__ __align__(16) uint64_t dig[];  // [islice * t]
    const int g0 = blockIdx.x * GT;
    const int ng = min(GT, Gl - g0);
    const int islice = N / gridDim.y;
    const int i0 = blockIdx.y * islice;
    const uint32_t offset = (uint32_t)(BASEBITS * t >= 32 ? 0u : 1u << (32 - (1 + BASEBITS * t)));

    for (int ii = threadIdx.x; ii < islice; ii += blockDim.x) {
        uint64_t word[8];
#pragma unroll
        for (int j = 0; j < 8; j++)
            word[j] = 0;
        for (int g = 0; g < ng; g++) {
            uint32_t a;
            const int gate = glist[g0 + g];
            iks_level1_coef(trlwe, gtask[gate], N, seidx ? seidx[gate] : 0, i0 + ii, a);
            const uint32_t v = a + offset;
#pragma unroll
            for (int j = 0; j < 8; j++)
                if (j < t)
                    word[j] |= (uint64_t)((v >> (32 - (j + 1) * BASEBITS)) & kMask) << (g * BASEBITS);
        }
        for (int j = 0; j < t; j++)
            dig[ii * t + j] = word[j];
    }
    __syncthreads();

    uint32_t acc[GT][KPT];
#pragma unroll
    for (int g = 0; g < GT; g++)
#pragma unroll
        for (int kk = 0; kk < KPT; kk++)
            acc[g][kk] = 0u;

    const size_t rowStride = (size_t)n + 1;
    const uint32_t* kbase = ksk + (size_t)i0 * t * kPerBase * rowStride;
#pragma unroll 1
    for (int ij = 0; ij < islice * t; ij++) {
        const uint64_t dd = dig[ij];
        if (dd == 0)
            continue;
        const uint32_t* base = kbase + (size_t)ij * kPerBase * rowStride;
#pragma unroll
        for (int kk = 0; kk < KPT; kk++) {
            const int k = threadIdx.x + kk * 256;
            if (k > n)
                continue;
            if constexpr (BASEBITS == 2) {
                const uint32_t r1 = __ldg(base + k);
                const uint32_t r2 = __ldg(base + rowStride + k);
                const uint32_t r3 = __ldg(base + 2 * rowStride + k);
#pragma unroll
                for (int g = 0; g < GT; g++) {
                    const uint32_t d = (uint32_t)(dd >> (2 * g)) & 3u;
                    const uint32_t lo = (d & 1u) ? r1 : 0u;
                    const uint32_t hi = (d & 1u) ? r3 : r2;
                    acc[g][kk] += (d & 2u) ? hi : lo;
                }
            }
            else {
#pragma unroll
                for (int g = 0; g < GT; g++) {
                    const uint32_t d = (uint32_t)(dd >> (BASEBITS * g)) & kMask;
                    if (d)
                        acc[g][kk] += __ldg(base + (size_t)(d - 1) * rowStride + k);
                }
            }
        }
    }
#pragma unroll
    for (int g = 0; g < GT; g++) {
        if (g >= ng)
            break;
        const int gate = glist[g0 + g];
#pragma unroll
        for (int kk = 0; kk < KPT; kk++) {
            const int k = threadIdx.x + kk * 256;
            if (k <= n && acc[g][kk] != 0u)
                atomicAdd(out + (size_t)(oidx ? oidx[gate] : gate) * (n + 1) + k, 0u - acc[g][kk]);
        }
    }
}

// ---------------------------------------------------------------------------
// Identity key switch, base 2^2 x 8 (tfhe-80), register-tiled over gates.
//
// The 3 candidate KSK rows of one (i, j) are loaded ONCE per CTA into registers (lane =
// output coordinate k, coalesced) and reused by GT gates; each gate's 2-bit digit is
// warp-uniform (every lane works on the same gate), so the row choice is a uniform
// branch and the inner work is one u32 add per (gate, k) -- no per-element selects.
// Warp w of the CTA owns coordinates k = 32*KPT*w + 32*kk + lane; 4 warps cover
// 128*KPT >= n+1 coordinates.  blockIdx.y splits the input index i; the slices combine
// with u32 atomicAdd into `out` (pre-set by iks_init_kernel), associative mod 2^32 so
// bit-exact.  Loads for step (i, j+1) are issued before the adds of step (i, j).
template <int KPT, int GT>
__global__ void __launch_bounds__(128) iks_b2_kernel(
    const uint32_t* __restrict__ trlwe, const int2* __restrict__ gtask,
    const int* __restrict__ glist, const int* __restrict__ seidx, int Gl,
    const uint32_t* __restrict__ ksk, uint32_t* __restrict__ out, int n, int N,
    const int* __restrict__ oidx = nullptr)
{
    constexpr int T = 8;  // ksLen
    extern __shared__ __align__(16) uint16_t dig16[];  // [islice][GT]
    const int g0 = blockIdx.x * GT;
    const int ng = min(GT, Gl - g0);
    const int islice = N / gridDim.y;
    const int i0 = blockIdx.y * islice;
    constexpr uint32_t kOffset = 1u << 15;  // 2^(32 - (1 + 2*8)), ops.cpp:661-662

    for (int idx = threadIdx.x; idx < islice * GT; idx += blockDim.x) {
        const int ii = idx / GT, g = idx % GT;
        uint32_t w = 0;
        if (g < ng) {
            const int gate = glist[g0 + g];
            uint32_t a;
            iks_level1_coef(trlwe, gtask[gate], N, seidx ? seidx[gate] : 0, i0 + ii, a);
            w = (a + kOffset) >> 16;  // digits j = 0..7 at bits 14-2j (top 16 bits of v)
        }
        dig16[idx] = (uint16_t)w;
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kbase = warp * 32 * KPT + lane;
    const size_t rs = (size_t)n + 1;

    uint32_t acc[GT][KPT];
#pragma unroll
    for (int g = 0; g < GT; g++)
#pragma unroll
        for (int kk = 0; kk < KPT; kk++)
            acc[g][kk] = 0u;

    // Row pointers of digit d = 1..3 at this lane's first coordinate.  Coordinates past n
    // read into the next row (or the zeroed tail pad of the key buffer) and are never
    // stored, so the loads need no clamp and use immediate offsets 32*kk.
    const uint32_t* p0 = ksk + (size_t)i0 * T * 3 * rs + kbase;
    const uint32_t* p1 = p0 + rs;
    const uint32_t* p2 = p0 + 2 * rs;
    const size_t step = 3 * rs;
    uint32_t ra[3][KPT], rb[3][KPT];
    auto load = [&](uint32_t (&r)[3][KPT]) {
#pragma unroll
        for (int kk = 0; kk < KPT; kk++) {
            r[0][kk] = __ldg(p0 + 32 * kk);
            r[1][kk] = __ldg(p1 + 32 * kk);
            r[2][kk] = __ldg(p2 + 32 * kk);
        }
        p0 += step;
        p1 += step;
        p2 += step;
    };
    auto consume = [&](const uint32_t (&cur)[3][KPT], int s) {
        const int ii = s >> 3, j = s & 7;
        const uint4* dp = reinterpret_cast<const uint4*>(dig16 + ii * GT);
        uint32_t dw[GT / 2];
#pragma unroll
        for (int q = 0; q < GT / 8; q++) {
            const uint4 v = dp[q];
            dw[4 * q] = v.x;
            dw[4 * q + 1] = v.y;
            dw[4 * q + 2] = v.z;
            dw[4 * q + 3] = v.w;
        }
        const int sh = 14 - 2 * j;
        // all GT digits first (independent shifts, full ILP), then one uniform branch per gate
        uint32_t dg[GT];
#pragma unroll
        for (int g = 0; g < GT; g++)
            dg[g] = (dw[g >> 1] >> ((g & 1) * 16 + sh)) & 3u;
#pragma unroll
        for (int g = 0; g < GT; g++) {
            const uint32_t d = dg[g];
            if (d == 0)
                continue;
            if (d == 1) {
#pragma unroll
                for (int kk = 0; kk < KPT; kk++)
                    acc[g][kk] += cur[0][kk];
            }
            else if (d == 2) {
#pragma unroll
                for (int kk = 0; kk < KPT; kk++)
                    acc[g][kk] += cur[1][kk];
            }
            else {
#pragma unroll
                for (int kk = 0; kk < KPT; kk++)
                    acc[g][kk] += cur[2][kk];
            }
        }
    };

    const int steps = islice * T;  // multiple of 8 (T = 8)
    load(ra);
#pragma unroll 1
    for (int s = 0; s < steps; s += 2) {
        load(rb);
        consume(ra, s);
        if (s + 2 < steps)
            load(ra);
        consume(rb, s + 1);
    }
#pragma unroll
    for (int g = 0; g < GT; g++) {
        if (g >= ng)
            break;
        const int gate = glist[g0 + g];
#pragma unroll
        for (int kk = 0; kk < KPT; kk++) {
            const int k = kbase + 32 * kk;
            if (k <= n && acc[g][kk] != 0u)
                atomicAdd(out + (size_t)(oidx ? oidx[gate] : gate) * rs + k, 0u - acc[g][kk]);  // RED.ADD
        }
    }
}

}  // namespace vsp
