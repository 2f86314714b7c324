// Common device/host helpers for the VSP B200 engine (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#define VSP_CUDA_CHECK(expr)                                                         \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess)                                                       \
            throw std::runtime_error(std::string("CUDA error: ") +                   \
                                     cudaGetErrorString(_e) + " at " #expr);         \
    } while (0)

namespace vsp {

// Torus offset mu = 1/8 (params.hpp:12-13).
constexpr uint32_t kMu32 = 1u << 29;
constexpr uint64_t kMu64 = 1ull << 61;

// Parameter set, mirrors hvp::tfhe::ParameterSet (params.hpp:23-66).
struct Params {
    uint32_t n, N1, l1, Bg1Bits, N2, l2, Bg2Bits, ksBaseBits, ksLen, pksBaseBits, pksLen;
    int fft;  // MulBackend: 1 = Fft, 0 = Exact
};

// ---------------------------------------------------------------------------
// PTX wrappers: mbarrier + 1D bulk async copy (TMA engine, cp.async.bulk).

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Bulk global->shared copy completed on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// modSwitch(2N, phase) (ops.cpp:49-55) for 2N = 2^log2_2N: the reference computes
// ((phase<<32) + interval/2) / interval with interval = 2^(64-log2_2N), wrapping
// mod 2^64; that equals (phase + 2^(31-log2_2N)) >> (32-log2_2N) in u32 arithmetic.
__device__ __forceinline__ uint32_t mod_switch_2n(uint32_t phase, int log2_2N)
{
    return (phase + (1u << (31 - log2_2N))) >> (32 - log2_2N);
}

}  // namespace vsp
