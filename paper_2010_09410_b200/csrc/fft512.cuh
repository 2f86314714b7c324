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
// The same twiddles in "tangent" form for the forward butterflies: (kappa, tau) with
// zeta = kappa (1 + i tau) (form A, |tan| <= 1) or zeta = kappa (tau + i) (form B,
// |cot| < 1); the form of each (root, d, b) is known at compile time (tw_form_a).
__constant__ double2 c_tw1t[3][15];

__host__ __device__ constexpr int bitrev_const(int b, int d)
{
    int r = 0;
    for (int i = 0; i < d; i++)
        r = (r << 1) | ((b >> i) & 1);
    return r;
}

// Angle of zeta_{d,b} for root ROOT in units of pi/64 (exact for d <= 3), and whether
// |tan| <= 1 (angle mod pi within [0, pi/4] or [3pi/4, pi)).
__host__ __device__ constexpr bool tw_form_a(int root, int d, int b)
{
    const int theta0 = root == 0 ? 32 : root == 1 ? 16 : 80;  // pi/2, pi/4, 5pi/4
    const int ang = theta0 / (2 << d) + 64 * bitrev_const(b, d) / (1 << d);
    const int m = ang % 64;  // mod pi (64 units)
    return m <= 16 || m >= 48;
}
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

// Forward butterfly with a tangent-form twiddle: 6 FMAs instead of 2 MUL + 2 FMA + 4 ADD.
template <bool FORM_A>
__device__ __forceinline__ void bf_fwd_tan(double2& u, double2& v, const double2 kt)
{
    const double k = kt.x, t = kt.y;
    double tx, ty;
    if (FORM_A) {  // zeta v = k (v.x - t v.y, v.y + t v.x)
        tx = fma(-t, v.y, v.x);
        ty = fma(t, v.x, v.y);
    }
    else {  // zeta v = k (t v.x - v.y, t v.y + v.x)
        tx = fma(t, v.x, -v.y);
        ty = fma(t, v.y, v.x);
    }
    v.x = fma(-k, tx, u.x);
    v.y = fma(-k, ty, u.y);
    u.x = fma(k, tx, u.x);
    u.y = fma(k, ty, u.y);
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

// An opaque zero: keeps the compiler from hoisting the per-stage twiddle loads out of
// the blind-rotation loop (which would pin ~60 registers for the whole kernel).
__device__ __forceinline__ int opaque_zero()
{
    int z;
    asm volatile("mov.u32 %0, 0;" : "=r"(z));
    return z;
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
    const double2* tw1t = &c_tw1t[ROOT][0] + opaque_zero();
#pragma unroll
    for (int d = 0; d < 4; d++) {
        const int h = 8 >> d;
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0) {
                const int b = j >> (4 - d);
                const double2 kt = tw1t[(1 << d) - 1 + b];
                if (tw_form_a(ROOT, d, b))
                    bf_fwd_tan<true>(v[j], v[j + h], kt);
                else
                    bf_fwd_tan<false>(v[j], v[j + h], kt);
            }
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
    const double2* tw1 = &c_tw1[ROOT][0] + opaque_zero();
#pragma unroll
    for (int d = 3; d >= 0; d--) {
        const int h = 8 >> d;
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0)
                bf_inv(v[j], v[j + h], tw1[(1 << d) - 1 + (j >> (4 - d))]);
    }
}

}  // namespace vsp
