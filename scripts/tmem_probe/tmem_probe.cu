// Probe: smem (32 lanes x 16 B rows, contiguous) -> TMEM via tcgen05.cp.32x128b.warpx4 ->
// tcgen05.ld.32x32b.x4 by 8 warps; checks every value.  Build: nvcc -arch=sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_noswizzle(const void* p, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
    d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;   // LBO (unused for one column)
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;   // SBO: next 8-row core matrix
    d |= (uint64_t)1 << 46;                        // version (sm100)
    return d;                                      // base offset 0, lbo mode 0, no swizzle
}

__global__ void probe(const double2* __restrict__ src, int* bad)
{
    __shared__ __align__(128) double2 buf[32 * 32];   // 32 chunks of (32 lanes x 16 B)
    __shared__ uint32_t taddr_sh;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 1024; i += blockDim.x) buf[i] = src[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&taddr_sh)), "n"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = taddr_sh;
    if (tid == 0) {
        for (int c = 0; c < 32; c++) {
            const uint64_t d = desc_noswizzle(&buf[c * 32], 128);
            const uint32_t dst = tbase + (uint32_t)(c * 4);   // 4 columns per 16-byte row
            asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" :: "r"(dst), "l"(d));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    }
    // wait for the copies
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" :: "r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    int nb = 0;
    for (int c = 0; c < 32; c++) {
        uint32_t r0, r1, r2, r3;
        const uint32_t a = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(c * 4);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        double2 v;
        v.x = __hiloint2double((int)r1, (int)r0);
        v.y = __hiloint2double((int)r3, (int)r2);
        const double2 w = buf[c * 32 + lane];
        if (v.x != w.x || v.y != w.y) nb++;
    }
    if (nb) atomicAdd(bad, nb);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase), "n"(128));
}

int main()
{
    double2 h[1024];
    for (int i = 0; i < 1024; i++) h[i] = make_double2(i * 1.5 + 0.25, -i * 3.0 - 0.5);
    double2* d; int* bad;
    cudaMalloc(&d, sizeof h); cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    probe<<<2, 256>>>(d, bad);
    cudaError_t e = cudaDeviceSynchronize();
    int hb = -1; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("err=%s bad=%d\n", cudaGetErrorString(e), hb);
    return 0;
}
