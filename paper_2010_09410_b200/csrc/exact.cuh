// Exact (integer schoolbook) kernels for parameter sets whose MulBackend is Exact
// (test-det, params.cpp:58-86).  The reference multiplies with polyMulAccExact
// (poly.hpp:15-29); with 16-bit gadget digits the products exceed what FP64 can
// carry exactly, so these kernels keep the reference's exact semantics on the GPU:
// one CTA per ciphertext, one thread per output coefficient, wrapping arithmetic
// in the torus word type T (u32 level 1, u64 level 2).
#pragma once

#include <type_traits>
#include "vsp_common.cuh"

namespace vsp {

template <typename T>
struct TorusBits;
template <>
struct TorusBits<uint32_t> {
    static constexpr int W = 32;
};
template <>
struct TorusBits<uint64_t> {
    static constexpr int W = 64;
};

// decomposePoly (poly.hpp:79-97) of one coefficient into l signed digits.
template <typename T>
__device__ __forceinline__ int32_t digit_of(T v, int i, int bgbits)
{
    constexpr int W = TorusBits<T>::W;
    const T halfBg = (T)1 << (bgbits - 1);
    const T mask = ((T)1 << bgbits) - 1;
    return (int32_t)(typename std::conditional<sizeof(T) == 8, int64_t, int32_t>::type)(
        ((v >> (W - (i + 1) * bgbits)) & mask) - halfBg);
}

template <typename T>
__device__ __forceinline__ T gadget_offset(int l, int bgbits)
{
    constexpr int W = TorusBits<T>::W;
    const T halfBg = (T)1 << (bgbits - 1);
    T off = 0;
    for (int i = 1; i <= l; i++)
        off += halfBg << (W - i * bgbits);
    return off;
}

// Block-cooperative exact external product (externalProduct Exact branch,
// ops.cpp:566-572): out[0..2N) = sum_r digits_r (x) g.rows[r].  Must be called by
// exactly N threads; dig is smem scratch of 2l*N int32; in/out are smem.
template <typename T>
__device__ void ext_prod_exact_block(const T* in, const T* __restrict__ g, T* out,
                                     int32_t* dig, int N, int l, int bgbits)
{
    const int q = threadIdx.x;
    const T off = gadget_offset<T>(l, bgbits);
    for (int i = 0; i < l; i++) {
        dig[i * N + q] = digit_of<T>(in[q] + off, i, bgbits);
        dig[(l + i) * N + q] = digit_of<T>(in[N + q] + off, i, bgbits);
    }
    __syncthreads();
    T oa = 0, ob = 0;
    for (int r = 0; r < 2 * l; r++) {
        const int32_t* d = dig + r * N;
        const T* ga = g + (size_t)r * 2 * N;
        const T* gb = ga + N;
        for (int k = 0; k < N; k++) {
            const T dk = (T)(typename std::conditional<sizeof(T) == 8, int64_t, int32_t>::type)d[k];
            if (k <= q) {
                oa += dk * ga[q - k];
                ob += dk * gb[q - k];
            }
            else {
                oa -= dk * ga[q - k + N];
                ob -= dk * gb[q - k + N];
            }
        }
    }
    __syncthreads();
    out[q] = oa;
    out[N + q] = ob;
}

// Blind rotation (ops.cpp:713-742) with a caller-supplied test vector; one CTA
// (N threads) per task.  bk: n x 2l x 2 x N raw TRGSW words.
template <typename T>
__global__ void br_exact_kernel(const uint32_t* __restrict__ tasks, int n,
                                const T* __restrict__ bk, const T* __restrict__ tv,
                                T* __restrict__ out, int N, int log2_2N, int l, int bgbits)
{
    extern __shared__ __align__(16) uint8_t sm[];
    T* acc = reinterpret_cast<T*>(sm);
    T* diff = acc + 2 * N;
    T* ep = diff + 2 * N;
    int32_t* dig = reinterpret_cast<int32_t*>(ep + 2 * N);
    const uint32_t* lwe = tasks + (size_t)blockIdx.x * (n + 1);
    const int q = threadIdx.x;
    const uint32_t twoN = 2u * N;
    const uint32_t rot = (twoN - mod_switch_2n(lwe[n], log2_2N)) % twoN;
    // polyRotate (poly.hpp:32-48): (X^rot p)[q] = +-p[(q - rot) mod 2N]
    for (int P = 0; P < 2; P++) {
        const uint32_t idx = ((uint32_t)q + twoN - rot) % twoN;
        const T val = idx < (uint32_t)N ? tv[P * N + idx] : (T)0 - tv[P * N + idx - N];
        acc[P * N + q] = val;
    }
    __syncthreads();
    const size_t per = (size_t)2 * l * 2 * N;
    for (int i = 0; i < n; i++) {
        const uint32_t bara = mod_switch_2n(lwe[i], log2_2N);
        if (bara == 0)
            continue;
        for (int P = 0; P < 2; P++) {
            const uint32_t idx = ((uint32_t)q + twoN - bara) % twoN;
            const T r = idx < (uint32_t)N ? acc[P * N + idx] : (T)0 - acc[P * N + idx - N];
            diff[P * N + q] = r - acc[P * N + q];
        }
        __syncthreads();
        ext_prod_exact_block<T>(diff, bk + (size_t)i * per, ep, dig, N, l, bgbits);
        acc[q] += ep[q];
        acc[N + q] += ep[N + q];
        __syncthreads();
    }
    T* dst = out + (size_t)blockIdx.x * 2 * N;
    dst[q] = acc[q];
    dst[N + q] = acc[N + q];
}

}  // namespace vsp
