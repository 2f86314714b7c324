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
// The same twiddles, all in form A (kappa, tau) = (cos, tan) of the half angle: used where
// the twiddle is chosen per lane (fft512_fwd_pair) so one butterfly formula serves both
// candidates.  tau may be large (angle near pi/2); kappa*tau keeps the rounding bound and
// no angle here is exactly pi/2.
__constant__ double2 c_tw1a[3][15];

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
// Per-lane twiddle table: stage d (4..7) of the second pass splits block
// b = (L' << (d-4)) | jt (L' = lane >> 1, jt = top d-4 bits of the register index) and
// zeta_{d,b} = zeta_{d,L'<<(d-4)} * exp(i pi br(jt) / 2^(d-4)) = entry[d][m] * i^q with
// k = br(jt) << (7-d) = 4q + m: only the q = 0 values are stored (1, 1, 2, 4 for
// stages 4-7 and 4 for stage 8); multiplying by i is a swap/negate folded into the
// butterfly.  12 loads per transform instead of 23 (the kernels are shared-memory bound).
// Entries [0, kTw2Plain) hold zeta (inverse butterflies); entries [kTw2Plain, 2 kTw2Plain)
// hold the same twiddles in tangent form (kappa, tau), zeta = kappa (1 + i tau), for the
// forward butterflies (6 FMAs).  tau may be large where zeta is near +-i; the products
// kappa * tau v stay within the same rounding bound, and zeta is never exactly +-i here.
constexpr int kTw2Plain = 12;
constexpr int kTw2Entries = 2 * kTw2Plain;

__host__ __device__ constexpr int tw_k(int d, int jt) { return bitrev_const(jt, d - 4) << (7 - d); }
__host__ __device__ constexpr int tw_entry(int d, int m)
{
    return d == 4 ? 0 : d == 5 ? 1 : d == 6 ? 2 + (m >> 1) : d == 7 ? 4 + m : 8 + m;
}

__device__ __forceinline__ void bf_fwd(double2& u, double2& v, const double2 w)
{
    const double tx = w.x * v.x - w.y * v.y;
    const double ty = w.x * v.y + w.y * v.x;
    v.x = u.x - tx;
    v.y = u.y - ty;
    u.x = u.x + tx;
    u.y = u.y + ty;
}

// Forward butterfly with twiddle i*w.
__device__ __forceinline__ void bf_fwd_i(double2& u, double2& v, const double2 w)
{
    const double tx = w.x * v.x - w.y * v.y;
    const double ty = w.x * v.y + w.y * v.x;
    v.x = u.x + ty;
    v.y = u.y - tx;
    u.x = u.x - ty;
    u.y = u.y + tx;
}

template <int Q>
__device__ __forceinline__ void bf_fwd_q(double2& u, double2& v, const double2 w)
{
    if (Q)
        bf_fwd_i(u, v, w);
    else
        bf_fwd(u, v, w);
}

// Forward butterfly with a per-lane tangent-form twiddle kt = (kappa, tau) of zeta, times
// i^Q: t = (1 + i tau) v (Q = 0) or (i - tau) v (Q = 1); v' = u - kappa t, u' = u + kappa t.
template <int Q>
__device__ __forceinline__ void bf_fwd_tq(double2& u, double2& v, const double2 kt)
{
    const double k = kt.x, t = kt.y;
    double tx, ty;
    if (Q) {
        tx = fma(-t, v.x, -v.y);
        ty = fma(-t, v.y, v.x);
    }
    else {
        tx = fma(-t, v.y, v.x);
        ty = fma(t, v.x, v.y);
    }
    v.x = fma(-k, tx, u.x);
    v.y = fma(-k, ty, u.y);
    u.x = fma(k, tx, u.x);
    u.y = fma(k, ty, u.y);
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

// Inverse butterfly with twiddle i*w: (a, b) -> (a + b, (a - b) conj(w) (-i)).
__device__ __forceinline__ void bf_inv_i(double2& a, double2& b, const double2 w)
{
    const double dx = a.x - b.x, dy = a.y - b.y;
    a.x = a.x + b.x;
    a.y = a.y + b.y;
    b.y = -(dx * w.x + dy * w.y);
    b.x = dy * w.x - dx * w.y;
}

template <int Q>
__device__ __forceinline__ void bf_inv_q(double2& a, double2& b, const double2 w)
{
    if (Q)
        bf_inv_i(a, b, w);
    else
        bf_inv(a, b, w);
}

// Exact small-integer -> double without I2F: for an offset-binary word u = d + 2^k (k < 52),
// (2^52 + u) - (2^52 + 2^k) = d exactly (one DADD; the I2F.F64 conversion is quarter rate).
template <int K>
__device__ __forceinline__ double ob_to_double(uint32_t u)
{
    return __hiloint2double(0x43300000, (int)u) - (4503599627370496.0 + (double)(1ull << K));
}

// Round-half-even of x to an integer, mod 2^32, in ONE DADD instead of the quarter-rate
// F2I.S64.F64 of __double2ll_rn: for |x| < 2^51, x + 1.5 * 2^52 lies in [2^52, 2^53), where
// doubles are exactly the integers, so the addition rounds x half-to-even (the default
// mode, as llrint, fft.hpp:47-50) and the low mantissa word is round(x) + 2^51 = round(x)
// mod 2^32.  The level-1 inverse outputs are sums of 4,096 products of digits |d| <= 2^9
// and key words < 2^31: ~2^45 for uniform key words, the bound 2^51 is ~100 sigma away.
__device__ __forceinline__ uint32_t round_u32(double x)
{
    return (uint32_t)__double2loint(__dadd_rn(x, 6755399441055744.0));
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

// Per-lane select as ONE LOP3 per 32-bit word: m = 0 -> a, m = ~0 -> b.  Written as the
// ternary, the compiler emits a move plus a predicated move per word -- in the lane-pair
// exchanges of the last forward / first inverse stage that was ~1,000 of the ~6,600
// instructions of an external product.
__device__ __forceinline__ uint32_t lop_sel(uint32_t m, uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xD8;" : "=r"(r) : "r"(a), "r"(b), "r"(m));  // (a & ~m) | (b & m)
    return r;
}
__device__ __forceinline__ double dsel(uint32_t m, double a, double b)
{
    return __hiloint2double((int)lop_sel(m, (uint32_t)__double2hiint(a), (uint32_t)__double2hiint(b)),
                            (int)lop_sel(m, (uint32_t)__double2loint(a), (uint32_t)__double2loint(b)));
}
__device__ __forceinline__ double2 d2sel(uint32_t m, double2 a, double2 b)
{
    return make_double2(dsel(m, a.x, b.x), dsel(m, a.y, b.y));
}
// LS = false: the plain ternary (kernels whose register allocation prefers it).
template <bool LS>
__device__ __forceinline__ double2 sel2(uint32_t m, double2 a, double2 b)
{
    if constexpr (LS)
        return d2sel(m, a, b);
    else
        return m ? b : a;
}

// The one data exchange of the transform: lane L's value j sits at position L + 32 j
// before it and at (L & 1) + 2 j + 32 (L >> 1) after it (stride-34 padding keeps both
// phases bank-conflict free).  HALF moves the real parts, then the imaginary parts,
// through a 16 x 34 double buffer (4.3 KB per warp instead of 8.7 KB).
template <bool HALF>
__device__ __forceinline__ void xpose_fwd(double2 (&v)[16], void* buf, int lane)
{
    const int rbase = (lane & 1) + 34 * (lane >> 1);
    if constexpr (HALF) {
        double* xb = static_cast<double*>(buf);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            xb[lane + 34 * j] = v[j].x;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            v[j].x = xb[rbase + 2 * j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            xb[lane + 34 * j] = v[j].y;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            v[j].y = xb[rbase + 2 * j];
    }
    else {
        double2* xb = static_cast<double2*>(buf);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            xb[lane + 34 * j] = v[j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            v[j] = xb[rbase + 2 * j];
    }
}

template <bool HALF>
__device__ __forceinline__ void xpose_inv(double2 (&v)[16], void* buf, int lane)
{
    const int rbase = (lane & 1) + 34 * (lane >> 1);
    if constexpr (HALF) {
        double* xb = static_cast<double*>(buf);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            xb[rbase + 2 * j] = v[j].x;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            v[j].x = xb[lane + 34 * j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            xb[rbase + 2 * j] = v[j].y;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            v[j].y = xb[lane + 34 * j];
    }
    else {
        double2* xb = static_cast<double2*>(buf);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            xb[rbase + 2 * j] = v[j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++)
            v[j] = xb[lane + 34 * j];
    }
}

// Forward transform in place.  xbuf: per-warp smem, kFftXbufStride double2 (HALF:
// kFftXbufStride doubles).  twt(e): this lane's tangent-form per-lane twiddle of entry
// e < kTw2Plain (a shared-memory load, or a register when the kernel has room to keep
// all twelve: fft512_fwd_regs).
template <int ROOT, bool HALF, class TWT, bool LS = true>
__device__ __forceinline__ void fft512_fwd_g(double2 (&v)[16], void* xbuf, const TWT& twt, int lane)
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
    xpose_fwd<HALF>(v, xbuf, lane);
#pragma unroll
    for (int d = 4; d < 8; d++) {
        const int h = 8 >> (d - 4);
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0) {
                const int k = tw_k(d, j >> (8 - d));
                const double2 w = twt(tw_entry(d, k & 3));
                if (k >> 2)
                    bf_fwd_tq<1>(v[j], v[j + h], w);
                else
                    bf_fwd_tq<0>(v[j], v[j + h], w);
            }
    }
    const uint32_t odd = 0u - (uint32_t)(lane & 1);  // select mask
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const double2 send = sel2<LS>(odd, v[k + 8], v[k]);
        const double2 recv = shfl_xor_d2(send, 1);
        double2 u = sel2<LS>(odd, v[k], recv);
        double2 w = sel2<LS>(odd, recv, v[k + 8]);
        const int br = bitrev_const(k, 3);
        const double2 t = twt(tw_entry(8, br & 3));
        if (br >> 2)
            bf_fwd_tq<1>(u, w, t);
        else
            bf_fwd_tq<0>(u, w, t);
        v[k] = u;
        v[k + 8] = w;
    }
}

// tw2: smem table [kTw2Entries][32] double2 (plain, then tangent).
template <int ROOT = 0, bool HALF = false, bool LS = true>
__device__ __forceinline__ void fft512_fwd(double2 (&v)[16], void* xbuf,
                                           const double2* tw2, int lane)
{
    const double2* tw2t = tw2 + kTw2Plain * 32;
    auto twt = [&](int e) { return tw2t[e * 32 + lane]; };
    fft512_fwd_g<ROOT, HALF, decltype(twt), LS>(v, xbuf, twt, lane);
}

// Same with the twelve tangent twiddles of this lane held in registers (twr[e]).
template <int ROOT = 0>
__device__ __forceinline__ void fft512_fwd_regs(double2 (&v)[16], void* xbuf,
                                                const double2 (&twr)[kTw2Plain], int lane)
{
    fft512_fwd_g<ROOT, false>(v, xbuf, [&](int e) { return twr[e]; }, lane);
}

// Exact inverse of fft512_fwd up to the factor 512 (folded into the key).
template <int ROOT = 0, bool HALF = false, bool LS = true>
__device__ __forceinline__ void fft512_inv(double2 (&v)[16], void* xbuf,
                                           const double2* tw2, int lane)
{
    const uint32_t odd = 0u - (uint32_t)(lane & 1);  // select mask
#pragma unroll
    for (int k = 0; k < 8; k++) {
        double2 a = v[k], b = v[k + 8];
        const int br = bitrev_const(k, 3);
        const double2 t = tw2[tw_entry(8, br & 3) * 32 + lane];
        if (br >> 2)
            bf_inv_q<1>(a, b, t);
        else
            bf_inv_q<0>(a, b, t);
        const double2 send = sel2<LS>(odd, b, a);
        const double2 recv = shfl_xor_d2(send, 1);
        v[k] = sel2<LS>(odd, a, recv);
        v[k + 8] = sel2<LS>(odd, recv, b);
    }
#pragma unroll
    for (int d = 7; d >= 4; d--) {
        const int h = 8 >> (d - 4);
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0) {
                const int k = tw_k(d, j >> (8 - d));
                const double2 w = tw2[tw_entry(d, k & 3) * 32 + lane];
                if (k >> 2)
                    bf_inv_q<1>(v[j], v[j + h], w);
                else
                    bf_inv_q<0>(v[j], v[j + h], w);
            }
    }
    xpose_inv<HALF>(v, xbuf, lane);
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

// Two inverse transforms at once (the accumulator pair of an external product): every
// per-lane twiddle is loaded once for both, and the two independent butterfly streams
// give the scheduler FP64 work to overlap with the other's shuffles and transposes.
template <int ROOT = 0>
__device__ __forceinline__ void fft512_inv2(double2 (&va)[16], double2 (&vb)[16], void* xbuf,
                                            const double2* tw2, int lane)
{
    const uint32_t odd = 0u - (uint32_t)(lane & 1);  // select mask
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const int br = bitrev_const(k, 3);
        const double2 t = tw2[tw_entry(8, br & 3) * 32 + lane];
        double2 a = va[k], b = va[k + 8];
        double2 c = vb[k], d = vb[k + 8];
        if (br >> 2) {
            bf_inv_q<1>(a, b, t);
            bf_inv_q<1>(c, d, t);
        }
        else {
            bf_inv_q<0>(a, b, t);
            bf_inv_q<0>(c, d, t);
        }
        const double2 ra = shfl_xor_d2(d2sel(odd, b, a), 1);
        const double2 rb = shfl_xor_d2(d2sel(odd, d, c), 1);
        va[k] = d2sel(odd, a, ra);
        va[k + 8] = d2sel(odd, ra, b);
        vb[k] = d2sel(odd, c, rb);
        vb[k + 8] = d2sel(odd, rb, d);
    }
#pragma unroll
    for (int d = 7; d >= 4; d--) {
        const int h = 8 >> (d - 4);
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0) {
                const int k = tw_k(d, j >> (8 - d));
                const double2 w = tw2[tw_entry(d, k & 3) * 32 + lane];
                if (k >> 2) {
                    bf_inv_q<1>(va[j], va[j + h], w);
                    bf_inv_q<1>(vb[j], vb[j + h], w);
                }
                else {
                    bf_inv_q<0>(va[j], va[j + h], w);
                    bf_inv_q<0>(vb[j], vb[j + h], w);
                }
            }
    }
    xpose_inv<false>(va, xbuf, lane);
    xpose_inv<false>(vb, xbuf, lane);
    const double2* tw1 = &c_tw1[ROOT][0] + opaque_zero();
#pragma unroll
    for (int d = 3; d >= 0; d--) {
        const int h = 8 >> d;
#pragma unroll
        for (int j = 0; j < 16; j++)
            if ((j & h) == 0) {
                const double2 w = tw1[(1 << d) - 1 + (j >> (4 - d))];
                bf_inv(va[j], va[j + h], w);
                bf_inv(vb[j], vb[j + h], w);
            }
    }
}

// Inverse transform of one block split over a warp pair (64 lanes x 8 values), for the
// latency kernel.  Lane l of pair half h stands for virtual lane L = 16h + (l & 15) of
// fft512_inv's layout and half e = l >> 4 of that lane's 16 values:
//   input  u[t] = v_L[2t + e]                    (frequency slot (2t + e) * 32 + L)
//   output u[t] = z at time position L + 32 (t + 8e)   (z_p = x_p + i x_{p+512})
// The butterflies are fft512_inv's, in the same order with the same twiddles; the two
// stages that pair the halves (7, and 0 after the transpose) go through __shfl_xor 16,
// stage 8's lane pairs (L, L^1) through __shfl_xor 1.  xbuf: kFftXbufStride double2
// shared by the pair, synchronised by named barrier bar_id over its 64 threads.
__device__ __forceinline__ double2 cmul(const double2 a, const double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

template <int ROOT, class TWP>
__device__ __forceinline__ void fft512_inv_pair_g(double2 (&u)[8], double2* xbuf, const TWP& twp,
                                                  int lane, int h, int bar_id)
{
    const int L = 16 * h + (lane & 15);
    const int e = lane >> 4;
    const bool oddL = L & 1;
    const double sg = e ? -1.0 : 1.0;
    // stage 8: butterflies (k, k + 8), k = 2 tp + e; bitrev3(k) = (e << 2) | bitrev2(tp)
#pragma unroll
    for (int tp = 0; tp < 4; tp++) {
        double2 w = twp(tw_entry(8, bitrev_const(tp, 2)));
        if (e)
            w = make_double2(-w.y, w.x);  // i^Q with Q = e
        double2 a = u[tp], b = u[tp + 4];
        bf_inv(a, b, w);
        const double2 recv = shfl_xor_d2(oddL ? a : b, 1);
        u[tp] = oddL ? recv : a;
        u[tp + 4] = oddL ? b : recv;
    }
    // stage 7: pairs (2t, 2t + 1) = the two halves; half 0 keeps a + b, half 1 (a - b) conj(w)
#pragma unroll
    for (int t = 0; t < 8; t++) {
        const int k = tw_k(7, t);
        double2 w = twp(tw_entry(7, k & 3));
        if (k >> 2)
            w = make_double2(-w.y, w.x);
        const double2 c = e ? make_double2(w.x, -w.y) : make_double2(1.0, 0.0);
        const double2 o = shfl_xor_d2(u[t], 16);
        const double2 d = make_double2(fma(sg, u[t].x, o.x), fma(sg, u[t].y, o.y));
        u[t] = cmul(d, c);
    }
    // stages 6, 5, 4: local pairs (t, t + hh)
#pragma unroll
    for (int d = 6; d >= 4; d--) {
        const int hh = 1 << (6 - d);
#pragma unroll
        for (int t = 0; t < 8; t++)
            if ((t & hh) == 0) {
                const int k = tw_k(d, t >> (7 - d));
                const double2 w = twp(tw_entry(d, k & 3));
                if (k >> 2)
                    bf_inv_q<1>(u[t], u[t + hh], w);
                else
                    bf_inv_q<0>(u[t], u[t + hh], w);
            }
    }
    // transpose through the pair's buffer (fft512_inv's xpose_inv element mapping)
    const int wbase = (L & 1) + 34 * (L >> 1) + 2 * e;
#pragma unroll
    for (int t = 0; t < 8; t++)
        xbuf[wbase + 4 * t] = u[t];
    asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
#pragma unroll
    for (int t = 0; t < 8; t++)
        u[t] = xbuf[L + 34 * (t + 8 * e)];
    // stages 3, 2, 1 local (j = t + 8e: twiddle index depends on the half), stage 0 pairs
    // the halves
    const double2* tw1 = &c_tw1[ROOT][0] + opaque_zero();
#pragma unroll
    for (int d = 3; d >= 1; d--) {
        const int hh = 8 >> d;
#pragma unroll
        for (int t = 0; t < 8; t++)
            if ((t & hh) == 0) {
                const int base = (1 << d) - 1 + (t >> (4 - d));
                const double2 w0 = tw1[base], w1 = tw1[base + (8 >> (4 - d))];
                bf_inv(u[t], u[t + hh], e ? w1 : w0);
            }
    }
    {
        const double2 w = tw1[0];
        const double2 c = e ? make_double2(w.x, -w.y) : make_double2(1.0, 0.0);
#pragma unroll
        for (int t = 0; t < 8; t++) {
            const double2 o = shfl_xor_d2(u[t], 16);
            const double2 d = make_double2(fma(sg, u[t].x, o.x), fma(sg, u[t].y, o.y));
            u[t] = cmul(d, c);
        }
    }
}

// twp(e): plain per-lane twiddle of entry e at virtual lane L = 16 h + (lane & 15).
template <int ROOT = 0>
__device__ __forceinline__ void fft512_inv_pair(double2 (&u)[8], double2* xbuf,
                                                const double2* tw2, int lane, int h, int bar_id)
{
    const int L = 16 * h + (lane & 15);
    fft512_inv_pair_g<ROOT>(u, xbuf, [&](int e) { return tw2[e * 32 + L]; }, lane, h, bar_id);
}

template <int ROOT = 0>
__device__ __forceinline__ void fft512_inv_pair_regs(double2 (&u)[8], double2* xbuf,
                                                     const double2 (&twr)[kTw2Plain], int lane,
                                                     int h, int bar_id)
{
    fft512_inv_pair_g<ROOT>(u, xbuf, [&](int e) { return twr[e]; }, lane, h, bar_id);
}

// Forward transform of one block split over a warp pair (the mirror of fft512_inv_pair).
// Lane l of pair half h: virtual lane L = 16h + (l & 15), half e = l >> 4:
//   input  u[t] = z at time position L + 32 (t + 8e)   (z_p = x_p + i x_{p+512})
//   output u[t] = v_L[2t + e]                          (frequency slot (2t + e) * 32 + L)
// i.e. exactly fft512_fwd's butterflies, twiddles and output slots.  Stage 0 and stage 7
// pair the halves through __shfl_xor 16, stage 8's lane pairs (L, L^1) use __shfl_xor 1.
template <int ROOT = 0>
__device__ __forceinline__ void fft512_fwd_pair(double2 (&u)[8], double2* xbuf,
                                                const double2* tw2, int lane, int h, int bar_id)
{
    const int L = 16 * h + (lane & 15);
    const int e = lane >> 4;
    const bool oddL = L & 1;
    const double2* tw2t = tw2 + kTw2Plain * 32;
    // cross-half butterfly (a = half 0's value, b = half 1's): half 0 keeps a + zeta b,
    // half 1 a - zeta b; zeta = k (1 + i t) in form A, Q multiplies it by i
    auto cross = [&](double2& mine, const double2 kt, bool Q) {
        const double2 o = shfl_xor_d2(mine, 16);
        const double2 a = e ? o : mine;
        double2 b = e ? mine : o;
        if (Q)
            b = make_double2(-b.y, b.x);
        const double tx = fma(-kt.y, b.y, b.x), ty = fma(kt.y, b.x, b.y);
        const double sk = e ? -kt.x : kt.x;
        mine = make_double2(fma(sk, tx, a.x), fma(sk, ty, a.y));
    };
    // ---- pass 1 (stages 0..3) on j = t + 8e
    {
        const double2* tw1a = &c_tw1a[ROOT][0] + opaque_zero();
        const double2 k0 = tw1a[0];
#pragma unroll
        for (int t = 0; t < 8; t++)
            cross(u[t], k0, false);
#pragma unroll
        for (int d = 1; d < 4; d++) {
            const int hh = 8 >> d;
#pragma unroll
            for (int t = 0; t < 8; t++)
                if ((t & hh) == 0) {
                    const int base = (1 << d) - 1 + (t >> (4 - d));
                    const double2 w0 = tw1a[base], w1 = tw1a[base + (8 >> (4 - d))];
                    bf_fwd_tan<true>(u[t], u[t + hh], e ? w1 : w0);
                }
        }
    }
    // ---- transpose through the pair's buffer (fft512_fwd's xpose_fwd element mapping)
#pragma unroll
    for (int t = 0; t < 8; t++)
        xbuf[L + 34 * (t + 8 * e)] = u[t];
    asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
    {
        const int rbase = (L & 1) + 34 * (L >> 1) + 2 * e;
#pragma unroll
        for (int t = 0; t < 8; t++)
            u[t] = xbuf[rbase + 4 * t];
    }
    // ---- pass 2 on j = 2t + e: stages 4, 5, 6 local, stage 7 across the halves
#pragma unroll
    for (int d = 4; d < 7; d++) {
        const int hh = 1 << (6 - d);
#pragma unroll
        for (int t = 0; t < 8; t++)
            if ((t & hh) == 0) {
                const int k = tw_k(d, t >> (7 - d));
                const double2 w = tw2t[tw_entry(d, k & 3) * 32 + L];
                if (k >> 2)
                    bf_fwd_tq<1>(u[t], u[t + hh], w);
                else
                    bf_fwd_tq<0>(u[t], u[t + hh], w);
            }
    }
#pragma unroll
    for (int t = 0; t < 8; t++) {
        const int k = tw_k(7, t);
        cross(u[t], tw2t[tw_entry(7, k & 3) * 32 + L], (k >> 2) != 0);
    }
    // ---- stage 8: k = 2 tp + e, Q = e (bitrev3(k) = (e << 2) | bitrev2(tp))
#pragma unroll
    for (int tp = 0; tp < 4; tp++) {
        const double2 recv = shfl_xor_d2(oddL ? u[tp] : u[tp + 4], 1);
        double2 a = oddL ? recv : u[tp];
        double2 b = oddL ? u[tp + 4] : recv;
        const double2 kt = tw2t[tw_entry(8, bitrev_const(tp, 2)) * 32 + L];
        const double2 bq = e ? make_double2(-b.y, b.x) : b;  // i^Q b, Q = e
        const double tx = fma(-kt.y, bq.y, bq.x), ty = fma(kt.y, bq.x, bq.y);
        b = make_double2(fma(-kt.x, tx, a.x), fma(-kt.x, ty, a.y));
        a = make_double2(fma(kt.x, tx, a.x), fma(kt.x, ty, a.y));
        u[tp] = a;
        u[tp + 4] = b;
    }
}

}  // namespace vsp
