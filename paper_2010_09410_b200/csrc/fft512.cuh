// Warp-cooperative negacyclic transform for T[X]/(X^1024 + 1) (M = 512 complex points).
//
// The reference folds a real polynomial of degree < N into M = N/2 complex points,
// twists by e^{i pi j / N} and runs a radix-2 DIF FFT (fft.hpp:64-75, fft.cpp:33-55);
// the inverse is a DIT FFT, 1/M scaling, untwist and llrint (fft.hpp:77-97).
// This kernel evaluates the SAME M evaluation points (the roots of Y^M = i) by a
// recursive negacyclic split  Y^2m - c = (Y^m - s)(Y^m + s),  s^2 = c, starting from
// c = i, so no twist pass is needed; outputs come in a fixed permuted order that the
// bootstrapping key is prepared in as well (prepare kernel uses this same routine).
// Products are exact integers < 2^53 for tfhe-80, so rounding reproduces the
// reference (and its Exact backend) bit-for-bit.
//
// Data layout per warp: lane L holds 16 complex values v[j].
//   input / inverse output: position p = L + 32 j          (z_p = x_p + i x_{p+512})
//   stages 0-3 (position bits 8..5) are register-internal with lane-uniform twiddles
//   (compile-time constants from c_tw1); one shared-memory transpose; stages 4-7
//   (bits 4..1) register-internal with per-lane twiddles (tw2 table in smem);
//   stage 8 (bit 0) pairs lanes L, L^1 through __shfl_xor.
#pragma once

#include "vsp_common.cuh"

namespace vsp {

// zeta_{d,b} for stages 0..3 (index (1<<d)-1+b) of the 512-point transform rooted at
// Y^512 = c_ROOT, for the three roots in use (filled by the host):
//   ROOT 0: c = i            (level 1: X^1024 + 1 folded to Y^512 = i)
//   ROOT 1: c = e^{i pi/4}   (level 2, branch 0 of Y^1024 = i)
//   ROOT 2: c = e^{i 5pi/4}  (level 2, branch 1)
// The per-lane table tw2 (stages 4-8) is likewise per root.
__constant__ double2 c_tw1[3][15];

constexpr int kFftXbufStride = 544;  // 512 + 32 swizzle pad (double2 units)
constexpr int kTw2Entries = 23;      // 1+2+4+8 (stages 4-7) + 8 (stage 8)

__device__ __forceinline__ void bf_fwd(double2& u, double2& v, const double2 w)
{
    const double tx = w.x * v.x - w.y * v.y;
    const double ty = w.x * v.y + w.y * v.x;
    v.x = u.x - tx;
    v.y = u.y - ty;
    u.x = u.x + tx;
    u.y = u.y + ty;
}

// Inverse (Gentleman-Sande) butterfly without the 1/2: (a, b) -> (a + b, (a - b) conj(w)).
__device__ __forceinline__ void bf_inv(double2& a, double2& b, const double2 w)
{
    const double dx = a.x - b.x, dy = a.y - b.y;
    a.x = a.x + b.x;
    a.y = a.y + b.y;
    b.x = dx * w.x + dy * w.y;
    b.y = dy * w.x - dx * w.y;
}

__device__ __forceinline__ double2 shfl_xor_d2(double2 v, int m)
{
    v.x = __shfl_xor_sync(0xffffffffu, v.x, m);
    v.y = __shfl_xor_sync(0xffffffffu, v.y, m);
    return v;
}

// Forward transform in place.  xbuf: per-warp smem, kFftXbufStride double2.
// tw2: smem table [kTw2Entries][32] double2.
template <int ROOT = 0>
__device__ __forceinline__ void fft512_fwd(double2 (&v)[16], double2* xbuf,
                                           const double2* tw2, int lane)
{
#pragma unroll
    for (int d = 0; d < 4; d++) {
        const int h = 8 >> d;
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0)
                bf_fwd(v[j], v[j + h], c_tw1[ROOT][(1 << d) - 1 + (j >> (4 - d))]);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; j++)
        xbuf[lane + 34 * j] = v[j];
    __syncwarp();
    const int rbase = (lane & 1) + 34 * (lane >> 1);
#pragma unroll
    for (int j = 0; j < 16; j++)
        v[j] = xbuf[rbase + 2 * j];
#pragma unroll
    for (int d = 4; d < 8; d++) {
        const int h = 8 >> (d - 4);
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0)
                bf_fwd(v[j], v[j + h], tw2[((1 << (d - 4)) - 1 + (j >> (8 - d))) * 32 + lane]);
    }
    const bool odd = lane & 1;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const double2 send = odd ? v[k] : v[k + 8];
        const double2 recv = shfl_xor_d2(send, 1);
        double2 u = odd ? recv : v[k];
        double2 w = odd ? v[k + 8] : recv;
        bf_fwd(u, w, tw2[(15 + k) * 32 + lane]);
        v[k] = u;
        v[k + 8] = w;
    }
}

// Exact inverse of fft512_fwd up to the factor 512 (folded into the key).
template <int ROOT = 0>
__device__ __forceinline__ void fft512_inv(double2 (&v)[16], double2* xbuf,
                                           const double2* tw2, int lane)
{
    const bool odd = lane & 1;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        double2 a = v[k], b = v[k + 8];
        bf_inv(a, b, tw2[(15 + k) * 32 + lane]);
        const double2 send = odd ? a : b;
        const double2 recv = shfl_xor_d2(send, 1);
        v[k] = odd ? recv : a;
        v[k + 8] = odd ? b : recv;
    }
#pragma unroll
    for (int d = 7; d >= 4; d--) {
        const int h = 8 >> (d - 4);
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0)
                bf_inv(v[j], v[j + h], tw2[((1 << (d - 4)) - 1 + (j >> (8 - d))) * 32 + lane]);
    }
    __syncwarp();
    const int rbase = (lane & 1) + 34 * (lane >> 1);
#pragma unroll
    for (int j = 0; j < 16; j++)
        xbuf[rbase + 2 * j] = v[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; j++)
        v[j] = xbuf[lane + 34 * j];
#pragma unroll
    for (int d = 3; d >= 0; d--) {
        const int h = 8 >> d;
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0)
                bf_inv(v[j], v[j + h], c_tw1[ROOT][(1 << d) - 1 + (j >> (4 - d))]);
    }
}

}  // namespace vsp
