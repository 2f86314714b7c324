// CMUX chains (level 1): the RAM read tree layers, the RAM write bars and the ROM
// tree / rotation chain of CMUX Memory (mem.cpp:49-177) are all chains of
//     acc <- c0' + ExtProd(c1' - c0', S_s)          (cmux, ops.cpp:606-614)
// with, per task, either
//   mode 0 (fixed base):  c1' = acc, c0' = base          (write bars mem.cpp:105-116;
//                          a single step is one tree CMUX  mem.cpp:60-70, 153-159)
//   mode 1 (rotation):    c1' = X^{rot_s} acc, c0' = acc  (ROM low-bit rotations,
//                          mem.cpp:164-170)
// acc starts at c1 (mode 0) or init (mode 1).  One warp per task (FFT path, N1=1024)
// or one CTA per task (exact path, test-det).  Selectors are prepared TRGSWs in the
// FFT slot layout (64 KiB each), read through L1/L2 by each warp.
#pragma once

#include "exact.cuh"
#include "fft512.cuh"

namespace vsp {

constexpr int kChainMax = 16;

struct ChainTask {
    const uint32_t* c1;  // initial accumulator (TRLWE, 2N words)
    const uint32_t* c0;  // fixed base for mode 0 (TRLWE), unused in mode 1
    uint32_t* out;       // result TRLWE
    int32_t sel[kChainMax];  // selector index per step (into the selector table)
    int32_t rot[kChainMax];  // mode 1: rotation exponent per step
    int32_t nsteps;
    int32_t mode;
};

template <int WARPS>
struct Chain1024Smem {
    double2 tw2[kTw2Entries * 32];
    double2 xbuf[WARPS][kFftXbufStride];
    uint32_t acc[WARPS][2048];
    uint32_t dig[WARPS][512];  // level-1 digits of the current polynomial (2 x 16 bit)
};

// MODE is the chains' mode (every task of a launch has the same one: run_chains splits
// mixed batches), so the digit loop carries one code path.
template <int WARPS, int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1)
    cmux_chain1024_kernel(const ChainTask* __restrict__ tasks, int T,
                          const double2* __restrict__ sels, const double2* __restrict__ tw2g,
                          int bgbits)
{
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<Chain1024Smem<WARPS>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kTw2Entries * 32; i += blockDim.x)
        sm.tw2[i] = tw2g[i];
    __syncthreads();
    const int t = blockIdx.x * WARPS + warp;
    if (t >= T)
        return;
    const ChainTask& task = tasks[t];
    uint32_t* acc = sm.acc[warp];
    {
        // one round trip: 16 independent 16-byte loads per lane (a rolled word loop
        // serialised 64 global-load latencies per chain, ~30 us per single-step layer)
        const uint4* c1 = reinterpret_cast<const uint4*>(task.c1);
        uint4* a4 = reinterpret_cast<uint4*>(acc);
        uint4 v[16];
#pragma unroll
        for (int k = 0; k < 16; k++)
            v[k] = __ldg(c1 + lane + 32 * k);
#pragma unroll
        for (int k = 0; k < 16; k++)
            a4[lane + 32 * k] = v[k];
    }
    __syncwarp();
    const uint32_t half = 1u << (bgbits - 1);
    const uint32_t mask = (1u << bgbits) - 1;
    const uint32_t offset = (half << (32 - bgbits)) + (half << (32 - 2 * bgbits));
    const int sh1 = 32 - bgbits, sh2 = 32 - 2 * bgbits;
    double2* xbuf = sm.xbuf[warp];
    const uint32_t* base = task.c0;
    constexpr int mode = MODE;

#pragma unroll 1
    for (int s = 0; s < task.nsteps; s++) {
        const uint32_t rot = mode == 1 ? (uint32_t)task.rot[s] : 0u;
        const double2* S = sels + (size_t)task.sel[s] * 4 * 1024;
        double2 accA[16], accB[16];
#pragma unroll
        for (int j = 0; j < 16; j++) {
            accA[j] = make_double2(0.0, 0.0);
            accB[j] = make_double2(0.0, 0.0);
        }
#pragma unroll 1
        for (int P = 0; P < 2; P++) {
            const uint32_t* src = acc + P * 1024;
            const uint32_t* bsrc = base + P * 1024;
            // d = c1' - c0' once per polynomial; level 0 digits straight into z, level 1
            // parked as 16-bit offset-binary pairs (decomposePoly, poly.hpp:79-97)
            double2 z[16];
            // lane + 32 j from an opaque base so the compiler does not hoist 32 indices
            // into registers (mode 1 spilled with them)
            const uint32_t lo = (uint32_t)lane + (uint32_t)opaque_zero();
            const uint32_t lk = lo - rot;
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const uint32_t p0 = lo + 32 * j, p1 = p0 + 512;
                uint32_t d0, d1;
                if (mode == 0) {
                    d0 = src[p0] - __ldg(bsrc + p0);
                    d1 = src[p1] - __ldg(bsrc + p1);
                }
                else {  // (X^rot acc - acc) (polyMulByXkMinusOne, poly.hpp:51-57)
                    d0 = rot_coef1024(src, lk + 32 * j) - src[p0];
                    d1 = rot_coef1024(src, lk + 32 * j + 512) - src[p1];
                }
                const uint32_t v0 = d0 + offset, v1 = d1 + offset;
                z[j].x = ob_to_double<15>((v0 >> sh1) + (32768u - half));
                z[j].y = ob_to_double<15>((v1 >> sh1) + (32768u - half));
                sm.dig[warp][j * 32 + lane] = (((v0 >> sh2) & mask) + (32768u - half)) |
                                              ((((v1 >> sh2) & mask) + (32768u - half)) << 16);
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
                fft512_fwd<0, false, false>(z, xbuf, sm.tw2, lane);
                const double2* row = S + (size_t)(P * 2 + lvl) * 1024;
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    const double2 ba = __ldg(row + j * 32 + lane);
                    const double2 bb = __ldg(row + 512 + j * 32 + lane);
                    accA[j].x = fma(z[j].x, ba.x, fma(-z[j].y, ba.y, accA[j].x));
                    accA[j].y = fma(z[j].x, ba.y, fma(z[j].y, ba.x, accA[j].y));
                    accB[j].x = fma(z[j].x, bb.x, fma(-z[j].y, bb.y, accB[j].x));
                    accB[j].y = fma(z[j].x, bb.y, fma(z[j].y, bb.x, accB[j].y));
                }
            }
            __syncwarp();
        }
        // acc <- c0' + round(inverse): mode 0 c0' = base, mode 1 c0' = acc
        fft512_inv<0, false, false>(accA, xbuf, sm.tw2, lane);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int p = lane + 32 * j;
            const uint32_t b0 = mode == 0 ? __ldg(base + p) : acc[p];
            const uint32_t b1 = mode == 0 ? __ldg(base + p + 512) : acc[p + 512];
            acc[p] = b0 + round_u32(accA[j].x);
            acc[p + 512] = b1 + round_u32(accA[j].y);
        }
        fft512_inv<0, false, false>(accB, xbuf, sm.tw2, lane);
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int p = lane + 32 * j;
            const uint32_t b0 = mode == 0 ? __ldg(base + 1024 + p) : acc[1024 + p];
            const uint32_t b1 = mode == 0 ? __ldg(base + 1024 + p + 512) : acc[1024 + p + 512];
            acc[1024 + p] = b0 + round_u32(accB[j].x);
            acc[1024 + p + 512] = b1 + round_u32(accB[j].y);
        }
        __syncwarp();
    }
    {
        uint4* o4 = reinterpret_cast<uint4*>(task.out);
        const uint4* a4 = reinterpret_cast<const uint4*>(acc);
#pragma unroll
        for (int k = 0; k < 16; k++)
            o4[lane + 32 * k] = a4[lane + 32 * k];
    }
}

// Exact-path chain (test-det): one CTA of N threads per task; selectors raw TRGSW words.
__global__ void cmux_chain_exact_kernel(const ChainTask* __restrict__ tasks,
                                        const uint32_t* __restrict__ sels, int N, int l,
                                        int bgbits)
{
    extern __shared__ __align__(16) uint8_t sm[];
    uint32_t* acc = reinterpret_cast<uint32_t*>(sm);
    uint32_t* diff = acc + 2 * N;
    uint32_t* ep = diff + 2 * N;
    int32_t* dig = reinterpret_cast<int32_t*>(ep + 2 * N);
    const ChainTask& task = tasks[blockIdx.x];
    const int q = threadIdx.x;
    const uint32_t twoN = 2u * N;
    acc[q] = task.c1[q];
    acc[N + q] = task.c1[N + q];
    __syncthreads();
    const size_t per = (size_t)2 * l * 2 * N;
    for (int s = 0; s < task.nsteps; s++) {
        uint32_t c0a, c0b;
        if (task.mode == 0) {
            c0a = task.c0[q];
            c0b = task.c0[N + q];
            diff[q] = acc[q] - c0a;
            diff[N + q] = acc[N + q] - c0b;
        }
        else {
            c0a = acc[q];
            c0b = acc[N + q];
            const uint32_t rot = (uint32_t)task.rot[s];
            for (int P = 0; P < 2; P++) {
                const uint32_t idx = ((uint32_t)q + twoN - rot) % twoN;
                const uint32_t r = idx < (uint32_t)N ? acc[P * N + idx] : 0u - acc[P * N + idx - N];
                diff[P * N + q] = r - acc[P * N + q];
            }
        }
        __syncthreads();
        ext_prod_exact_block<uint32_t>(diff, sels + (size_t)task.sel[s] * per, ep, dig, N, l,
                                       bgbits);
        acc[q] = c0a + ep[q];
        acc[N + q] = c0b + ep[N + q];
        __syncthreads();
    }
    task.out[q] = acc[q];
    task.out[N + q] = acc[N + q];
}

// trgswNot (ops.cpp:937-947): out = trivial(1) - in, for `count` TRGSWs.
__global__ void trgsw_not_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                 int count, int N, int l, int bgbits)
{
    const size_t per = (size_t)2 * l * 2 * N;
    const size_t total = per * count;
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total;
         x += (size_t)gridDim.x * blockDim.x) {
        const size_t w = x % per;
        const int row = (int)(w / (2 * N));
        const int col = (int)(w % (2 * N));
        uint32_t v = 0u - in[x];
        if (row < l && col == 0)
            v += 1u << (32 - (row + 1) * bgbits);
        if (row >= l && col == N)
            v += 1u << (32 - (row - l + 1) * bgbits);
        out[x] = v;
    }
}

// TRLWE-wise helpers for the RAM control unit (homMuxNoSeIks, ops.cpp:898-909):
// out = t1 + t2, out.b[0] += mu.
__global__ void trlwe_sum_mu_kernel(const uint32_t* __restrict__ trlwe, const int2* __restrict__ pairs,
                                    uint32_t* __restrict__ out, int count, int N)
{
    const int c = blockIdx.x;
    if (c >= count)
        return;
    const int2 p = pairs[c];
    const uint32_t* a = trlwe + (size_t)p.x * 2 * N;
    const uint32_t* b = trlwe + (size_t)p.y * 2 * N;
    for (int q = threadIdx.x; q < 2 * N; q += blockDim.x)
        out[(size_t)c * 2 * N + q] = a[q] + b[q] + (q == N ? kMu32 : 0u);
}

// Linear combinations of homMuxNoSeIks (ops.cpp:898-905) for the RAM control unit:
// task 2j = wflag + wdata[j] - mu, task 2j+1 = -wflag + readOut[j] - mu.
// sel_stride = 0: one selector (the write flag) for all j; n + 1: selector j per item
// (the batched homMuxNoSeIks entry point).
__global__ void mux_prep_kernel(const uint32_t* __restrict__ wflag, const uint32_t* __restrict__ wdata,
                                const uint32_t* __restrict__ readout, uint32_t* __restrict__ out,
                                int w, int n, int sel_stride = 0)
{
    const int t = blockIdx.x;
    if (t >= 2 * w)
        return;
    const int j = t >> 1;
    const uint32_t* x = (t & 1) ? readout + (size_t)j * (n + 1) : wdata + (size_t)j * (n + 1);
    const uint32_t* sel = wflag + (size_t)j * sel_stride;
    for (int k = threadIdx.x; k <= n; k += blockDim.x) {
        const uint32_t f = (t & 1) ? 0u - sel[k] : sel[k];
        out[(size_t)t * (n + 1) + k] = f + x[k] + (k == n ? 0u - kMu32 : 0u);
    }
}

}  // namespace vsp
