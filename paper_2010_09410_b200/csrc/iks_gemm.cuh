// Identity key switching (identityKeySwitch, ops.cpp:651-679) of a batch as ONE INT8
// tensor-core GEMM.  For tfhe-80's key switch (base 2^2, t = 8 digits per coefficient):
//
//   out_g = (0, ..., 0, b_g) - sum_{i < N1, j < 8, d_gij != 0} KSK[i][j][d_gij - 1]
//
// is  out = base - S x K  where
//   S  (G x K_, K_ = N1 * 8 * 3): one-hot digit selectors, S[g][(i*8 + j)*3 + d - 1] = 1,
//   K  (K_ x 4(n+1)): the key-switching key in four signed-byte planes,
//      ksk word w = sum_b s_b 256^b (mod 2^32), s_b in [-128, 128) (balanced base 256).
// The int32 accumulation is exact (at most 8,192 terms of |s| <= 128 per entry) and the
// planes recombine mod 2^32, so the result is the reference's key switch word for word.
// The GEMM itself is a plain library GEMM (cuBLASLt, int8 x int8 -> int32 on the 5th-gen
// tensor cores); this file holds the operand preparation and the epilogue.
#pragma once

#include <cublasLt.h>

namespace vsp {

constexpr int kIksGemmK = 1024 * 8 * 3;  // N1 * ksLen * (2^ksBaseBits - 1) for tfhe-80

// Key preparation (once per upload): K4t[col][k], col = b * (n + 1) + kk (plane b,
// coordinate kk; cols padded to npad with zeros), k = KSK row (i * 8 + j) * 3 + d - 1.
// Column-major K_ x npad for the GEMM (K contiguous per column).
__global__ void iks_gemm_prep_key_kernel(const uint32_t* __restrict__ ksk, int8_t* __restrict__ k4t,
                                         int n, int npad)
{
    const int r = blockIdx.x;  // KSK row
    for (int col = threadIdx.x; col < npad; col += blockDim.x) {
        const int b = col / (n + 1), kk = col % (n + 1);
        int8_t v = 0;
        if (b < 4) {
            uint32_t w = ksk[(size_t)r * (n + 1) + kk];
            int8_t s = 0;
            for (int q = 0; q <= b; q++) {  // balanced base-256 digit q of w
                s = (int8_t)((int)((w + 128u) & 255u) - 128);
                w = (w - (uint32_t)(int32_t)s) >> 8;
            }
            v = s;
        }
        k4t[(size_t)col * kIksGemmK + r] = v;
    }
}

// S rows (one CTA per key switch of the batch): the level-1 sample of gate glist[gi]
// (sample extraction at seidx, MUX: sum of its two blind-rotation outputs) digit-
// decomposed like identityKeySwitch (offset 2^15, 2-bit digits, no rounding beyond it).
// Each thread writes 96 contiguous bytes (4 coefficients x 8 digits x 3 candidates).
__global__ void __launch_bounds__(256) iks_gemm_selectors_kernel(
    const uint32_t* __restrict__ trlwe, const int2* __restrict__ gtask, const int* __restrict__ glist,
    const int* __restrict__ seidx, int8_t* __restrict__ S, int N)
{
    const int gi = blockIdx.x;
    const int gate = glist[gi];
    const int2 tt = gtask[gate];
    const int se = seidx ? seidx[gate] : 0;
    constexpr uint32_t kOffset = 1u << 15;  // ops.cpp:661-662
    for (int i0 = threadIdx.x * 4; i0 < N; i0 += blockDim.x * 4) {
        uint32_t bytes[24];  // 96 bytes, little endian
#pragma unroll
        for (int q = 0; q < 24; q++)
            bytes[q] = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            uint32_t a;
            iks_level1_coef(trlwe, tt, N, se, i0 + u, a);
            const uint32_t v = a + kOffset;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const uint32_t d = (v >> (30 - 2 * j)) & 3u;
                if (d) {
                    const int pos = (u * 8 + j) * 3 + (int)d - 1;  // byte within the 96
                    bytes[pos >> 2] |= 1u << (8 * (pos & 3));
                }
            }
        }
        uint4* dst = reinterpret_cast<uint4*>(S + (size_t)gi * kIksGemmK + (size_t)i0 * 24);
#pragma unroll
        for (int q = 0; q < 6; q++)
            dst[q] = make_uint4(bytes[4 * q], bytes[4 * q + 1], bytes[4 * q + 2], bytes[4 * q + 3]);
    }
}

// out[glist[gi]] = (0, ..., 0, b') - sum_b 256^b C[gi][b (n+1) + kk]  (mod 2^32), with b'
// the extracted b (MUX: both plus mu, ops.cpp:886-892) exactly as iks_init_kernel.
// Split-K: the nsplit partial products C_b = C + b * cstride are summed mod 2^32 first.
// Grid (key switches, coordinate chunks of 128): one coordinate per thread, its 4 x nsplit
// partial words loaded together (one round trip; a per-gate loop over the coordinates
// serialised ~5 of them).
__global__ void __launch_bounds__(128) iks_gemm_epilogue_kernel(
    const int32_t* __restrict__ C, int npad, int nsplit, size_t cstride,
    const uint32_t* __restrict__ trlwe, const int2* __restrict__ gtask,
    const int* __restrict__ glist, const int* __restrict__ seidx, uint32_t* __restrict__ out,
    int n, int N, const int* __restrict__ oidx = nullptr)
{
    const int gi = blockIdx.x;
    const int kk = blockIdx.y * 128 + threadIdx.x;
    if (kk > n)
        return;
    const int gate = glist[gi];
    const int32_t* c = C + (size_t)gi * npad;
    uint32_t v = 0;
    if (kk == n) {
        const int2 tt = gtask[gate];
        const int se = seidx ? seidx[gate] : 0;
        v = trlwe[(size_t)tt.x * 2 * N + N + se];
        if (tt.y >= 0)
            v += trlwe[(size_t)tt.y * 2 * N + N + se] + kMu32;
    }
    uint32_t s = 0;
    if (nsplit == 4) {
        uint32_t w[4][4];
#pragma unroll
        for (int b = 0; b < 4; b++)
#pragma unroll
            for (int q = 0; q < 4; q++)
                w[b][q] = (uint32_t)__ldg(c + (size_t)b * cstride + (size_t)q * (n + 1) + kk);
#pragma unroll
        for (int b = 0; b < 4; b++)
            s += w[b][0] + (w[b][1] << 8) + (w[b][2] << 16) + (w[b][3] << 24);
    }
    else {
        for (int b = 0; b < nsplit; b++) {
            const int32_t* cb = c + (size_t)b * cstride;
            s += (uint32_t)cb[kk] + ((uint32_t)cb[(n + 1) + kk] << 8) +
                 ((uint32_t)cb[2 * (n + 1) + kk] << 16) + ((uint32_t)cb[3 * (n + 1) + kk] << 24);
        }
    }
    out[(size_t)(oidx ? oidx[gate] : gate) * (n + 1) + kk] = v - s;
}

}  // namespace vsp
