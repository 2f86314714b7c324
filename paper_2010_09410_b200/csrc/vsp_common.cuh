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

// Wait with a sleeping back-off between probes: for producer warps that wait most of a
// step, so their spinning does not take issue slots from the compute warp sharing their
// scheduler.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, int ns)
{
    uint32_t ok;
    for (;;) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok)
            return;
        __nanosleep(ns);
    }
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

// ---------------------------------------------------------------------------
// Tensor memory (tcgen05) helpers: allocation, smem -> TMEM copies, TMEM -> register loads.

// Shared-memory matrix descriptor (no swizzle, sm100 version 1) for tcgen05.cp: rows of
// 16 bytes, 8-row core matrices `sbo` bytes apart.
__device__ __forceinline__ uint64_t tmem_desc_noswizzle(const void* p, uint32_t sbo)
{
    uint64_t d = (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
    d |= (uint64_t)((128u >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// 32 rows x 16 bytes of smem (row r = lane r) -> TMEM columns [col, col + 4) of lanes
// 32q + r in all four warp quadrants (multicast).
__device__ __forceinline__ void tmem_cp_32x128b_x4(uint32_t taddr, const void* src)
{
    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr),
                 "l"(tmem_desc_noswizzle(src, 128))
                 : "memory");
}

__device__ __forceinline__ void tmem_commit(uint64_t* bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 16 consecutive TMEM columns of this thread's lane -> 4 double2 (after tmem_wait_ld).
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// Named barrier over `nthreads` threads (a warp group of the CTA).
__device__ __forceinline__ void bar_group(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// (X^k p)[q] mod X^N + 1 (polyRotate, poly.hpp:32-48) = +-p[(q-k) mod 2N]; qk = q - k.
__device__ __forceinline__ uint32_t rot_coef1024(const uint32_t* src, uint32_t qk)
{
    const uint32_t idx = qk & 2047u;
    const uint32_t x = src[idx & 1023u];
    const uint32_t neg = idx >> 10;  // 0 or 1
    return (x ^ (0u - neg)) + neg;
}

// modSwitch(2N, phase) (ops.cpp:49-55) for 2N = 2^log2_2N: the reference computes
// ((phase<<32) + interval/2) / interval with interval = 2^(64-log2_2N), wrapping
// mod 2^64; that equals (phase + 2^(31-log2_2N)) >> (32-log2_2N) in u32 arithmetic.
__device__ __forceinline__ uint32_t mod_switch_2n(uint32_t phase, int log2_2N)
{
    return (phase + (1u << (31 - log2_2N))) >> (32 - log2_2N);
}

}  // namespace vsp
