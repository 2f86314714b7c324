// Host runtime + C ABI of the VSP B200 engine (include/vsp_b200.h).
//
// One translation unit: the kernels live in the included .cuh files.  Built for
// sm_100a only (paper_2010_09410_b200/build.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <type_traits>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vsp_b200.h"
#include "bootstrap.cuh"
#include "exact.cuh"
#include "vsp_common.cuh"

using namespace vsp;

namespace {

thread_local std::string g_err;

struct InvalidArg : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

template <class F>
int guard(F&& f)
{
    try {
        f();
        return VSP_OK;
    }
    catch (const std::invalid_argument& e) {
        g_err = std::string("invalid_argument: ") + e.what();
        return VSP_EINVAL;
    }
    catch (const std::out_of_range& e) {
        g_err = std::string("out_of_range: ") + e.what();
        return VSP_ERANGE;
    }
    catch (const std::exception& e) {
        g_err = std::string("runtime_error: ") + e.what();
        return VSP_ERUNTIME;
    }
}

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* ensure(size_t bytes)
    {
        if (bytes > cap) {
            if (p)
                cudaFree(p);
            p = nullptr;
            cap = 0;
            VSP_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
            cap = std::max<size_t>(bytes, 256);
        }
        return p;
    }
    template <class T>
    T* as(size_t count)
    {
        return static_cast<T*>(ensure(count * sizeof(T)));
    }
    void release()
    {
        if (p)
            cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

int ilog2(uint32_t x)
{
    int r = 0;
    while ((1u << r) < x)
        r++;
    return r;
}

// zeta_{d,b} = exp(i pi (2^-(d+2) + bitrev_d(b) / 2^d)): the root used by the
// butterfly that splits block b at depth d of the negacyclic transform.
double2 zeta(int d, uint32_t b)
{
    uint32_t r = 0;
    for (int i = 0; i < d; i++)
        r = (r << 1) | ((b >> i) & 1u);
    const long double pi = 3.141592653589793238462643383279502884L;
    const long double ang =
        pi * (1.0L / (long double)(1u << (d + 2)) + (long double)r / (long double)(1u << d));
    return make_double2((double)cosl(ang), (double)sinl(ang));
}

}  // namespace

struct vsp_ctx {
    Params p{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool has_keys = false, has_cb = false;
    // key material
    double2* d_bk1fd = nullptr;    // FFT path: n x 4 x 1024 double2
    uint32_t* d_bk1raw = nullptr;  // Exact path: raw TRGSW words
    uint32_t* d_ksk = nullptr;
    uint64_t* d_bk2raw = nullptr;
    uint32_t* d_pks[2] = {nullptr, nullptr};
    double2* d_tw2 = nullptr;      // [23][32] per-lane twiddles of the 512-point transform
    uint32_t* d_tv1 = nullptr;     // level-1 test vector (0, mu...mu) for the exact path
    // scratch
    DevBuf tasks, trlwe, in, out, kinds, gtask, glist;
    uint64_t counters[5] = {0, 0, 0, 0, 0};
    uint64_t launches = 0;
    std::mutex mu;
    // optional per-kernel CUDA-event timing (bench.py's live roofline)
    bool profiling = false;
    struct KTimer {
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
        double total_ms = 0;
        uint64_t count = 0;
    };
    std::map<std::string, KTimer> timers;

    void set_device() const { VSP_CUDA_CHECK(cudaSetDevice(device)); }
    size_t ksk_words() const
    {
        return (size_t)p.N1 * p.ksLen * ((1u << p.ksBaseBits) - 1) * (p.n + 1);
    }
    size_t pks_words() const
    {
        return ((size_t)p.N2 + 1) * p.pksLen * ((1u << p.pksBaseBits) - 1) * 2 * p.N1;
    }
};

namespace {

template <class F>
void timed(vsp_ctx* c, const char* name, cudaStream_t st, F&& launch)
{
    if (!c->profiling) {
        launch();
        return;
    }
    cudaEvent_t a, b;
    VSP_CUDA_CHECK(cudaEventCreate(&a));
    VSP_CUDA_CHECK(cudaEventCreate(&b));
    VSP_CUDA_CHECK(cudaEventRecord(a, st));
    launch();
    VSP_CUDA_CHECK(cudaEventRecord(b, st));
    c->timers[name].pending.emplace_back(a, b);
}

void validate(const Params& p)  // ParameterSet::validate (params.cpp:17-29)
{
    auto pow2 = [](uint32_t x) { return x != 0 && (x & (x - 1)) == 0; };
    if (p.n == 0 || p.N1 == 0 || p.N2 == 0)
        throw std::invalid_argument("parameter set: zero dimension");
    if (!pow2(p.N1) || !pow2(p.N2))
        throw std::invalid_argument("parameter set: N1, N2 must be powers of two");
    if (p.l1 * p.Bg1Bits > 32 || p.l2 * p.Bg2Bits > 64)
        throw std::invalid_argument("parameter set: gadget exceeds torus word");
    if (p.ksBaseBits * p.ksLen > 32 || p.pksBaseBits * p.pksLen > 64)
        throw std::invalid_argument("parameter set: key switch digits exceed torus word");
}

// Kernel configuration of the level-1 FFT blind rotation.
constexpr int kBrWarps = 8;
constexpr int kBrSlots = 4;

void launch_br(vsp_ctx* c, const uint32_t* d_tasks, uint32_t* d_trlwe, int T, cudaStream_t st)
{
    if (T == 0)
        return;
    const Params& p = c->p;
    if (p.fft) {
        const size_t smem = sizeof(Br1024Smem<kBrWarps, kBrSlots>);
        const int grid = (T + kBrWarps - 1) / kBrWarps;
        timed(c, "br1024", st, [&] {
            br1024_kernel<kBrWarps, kBrSlots><<<grid, kBrWarps * 32, smem, st>>>(
                d_tasks, c->d_bk1fd, c->d_tw2, d_trlwe, T, (int)p.n, (int)p.Bg1Bits);
        });
    }
    else {
        const int N = (int)p.N1;
        const size_t smem = (size_t)6 * N * sizeof(uint32_t) + (size_t)2 * p.l1 * N * 4;
        timed(c, "br_exact", st, [&] {
            br_exact_kernel<uint32_t><<<T, N, smem, st>>>(d_tasks, (int)p.n, c->d_bk1raw,
                                                          c->d_tv1, d_trlwe, N, ilog2(2 * N),
                                                          (int)p.l1, (int)p.Bg1Bits);
        });
    }
    VSP_CUDA_CHECK(cudaGetLastError());
    c->launches++;
    c->counters[1] += (uint64_t)T;
}

void launch_iks(vsp_ctx* c, const uint32_t* d_trlwe, const int2* d_gtask, const int* d_glist,
                int Gl, uint32_t* d_out, cudaStream_t st)
{
    if (Gl == 0)
        return;
    const Params& p = c->p;
    const size_t smem = (size_t)p.N1 * p.ksLen * sizeof(uint64_t);
    const int kpt = (int)((p.n + 1 + 255) / 256);
    timed(c, "iks", st, [&] {
    if (p.ksBaseBits == 2) {
        constexpr int GT = 32;
        const int grid = (Gl + GT - 1) / GT;
        if (kpt == 1)
            iks_kernel<2, GT, 1><<<grid, 256, smem, st>>>(d_trlwe, d_gtask, d_glist, Gl, c->d_ksk,
                                                          d_out, p.n, p.N1, p.ksLen);
        else if (kpt == 2)
            iks_kernel<2, GT, 2><<<grid, 256, smem, st>>>(d_trlwe, d_gtask, d_glist, Gl, c->d_ksk,
                                                          d_out, p.n, p.N1, p.ksLen);
        else if (kpt == 3)
            iks_kernel<2, GT, 3><<<grid, 256, smem, st>>>(d_trlwe, d_gtask, d_glist, Gl, c->d_ksk,
                                                          d_out, p.n, p.N1, p.ksLen);
        else
            throw std::invalid_argument("identity key switch: n too large");
    }
    else if (p.ksBaseBits == 4 && kpt == 1) {
        constexpr int GT = 16;
        const int grid = (Gl + GT - 1) / GT;
        iks_kernel<4, GT, 1><<<grid, 256, smem, st>>>(d_trlwe, d_gtask, d_glist, Gl, c->d_ksk,
                                                      d_out, p.n, p.N1, p.ksLen);
    }
    else {
        throw std::invalid_argument("identity key switch: unsupported base");
    }
    });
    VSP_CUDA_CHECK(cudaGetLastError());
    c->launches++;
    c->counters[2] += (uint64_t)Gl;
}

void configure_kernels(size_t br_smem, size_t iks_smem)
{
    static std::once_flag once;
    std::call_once(once, [&] {
        VSP_CUDA_CHECK(cudaFuncSetAttribute(br1024_kernel<kBrWarps, kBrSlots>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)br_smem));
        const int ik = (int)iks_smem;
        VSP_CUDA_CHECK(cudaFuncSetAttribute(iks_kernel<2, 32, 1>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, ik));
        VSP_CUDA_CHECK(cudaFuncSetAttribute(iks_kernel<2, 32, 2>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, ik));
        VSP_CUDA_CHECK(cudaFuncSetAttribute(iks_kernel<2, 32, 3>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, ik));
        VSP_CUDA_CHECK(cudaFuncSetAttribute(iks_kernel<4, 16, 1>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, ik));
    });
}

void require_keys(const vsp_ctx* c)
{
    if (!c->has_keys)
        throw std::runtime_error("no bootstrapping key uploaded");
}

// Host-side plan of a gate batch: task slots per gate, gates that need an IKS.
struct GatePlan {
    std::vector<int2> gtask;
    std::vector<int> glist;
    int T = 0;
};

GatePlan plan_gates(const int32_t* kinds, size_t G)
{
    GatePlan pl;
    pl.gtask.resize(G);
    for (size_t g = 0; g < G; g++) {
        const int k = kinds[g];
        if (k < 0 || k > kXor)
            throw std::invalid_argument("homGate: unknown kind");
        if (k == kNot) {
            pl.gtask[g] = make_int2(-1, -1);
        }
        else if (k == kMux) {
            pl.gtask[g] = make_int2(pl.T, pl.T + 1);
            pl.T += 2;
            pl.glist.push_back((int)g);
        }
        else {
            pl.gtask[g] = make_int2(pl.T, -1);
            pl.T += 1;
            pl.glist.push_back((int)g);
        }
    }
    return pl;
}

void hom_gate_dev(vsp_ctx* c, const int32_t* kinds, const uint32_t* d_in, uint32_t* d_out,
                  size_t G, cudaStream_t st)
{
    require_keys(c);
    if (G == 0)
        return;
    const Params& p = c->p;
    GatePlan pl = plan_gates(kinds, G);
    int* d_kinds = c->kinds.as<int>(G);
    int2* d_gtask = c->gtask.as<int2>(G);
    int* d_glist = c->glist.as<int>(std::max<size_t>(pl.glist.size(), 1));
    VSP_CUDA_CHECK(cudaMemcpyAsync(d_kinds, kinds, G * sizeof(int), cudaMemcpyHostToDevice, st));
    VSP_CUDA_CHECK(cudaMemcpyAsync(d_gtask, pl.gtask.data(), G * sizeof(int2),
                                   cudaMemcpyHostToDevice, st));
    if (!pl.glist.empty())
        VSP_CUDA_CHECK(cudaMemcpyAsync(d_glist, pl.glist.data(), pl.glist.size() * sizeof(int),
                                       cudaMemcpyHostToDevice, st));
    uint32_t* d_tasks = c->tasks.as<uint32_t>((size_t)std::max(pl.T, 1) * (p.n + 1));
    uint32_t* d_trlwe = c->trlwe.as<uint32_t>((size_t)std::max(pl.T, 1) * 2 * p.N1);
    timed(c, "gate_prep", st, [&] {
        gate_prep_kernel<<<(unsigned)G, 128, 0, st>>>(d_kinds, d_in, d_gtask, d_tasks, d_out,
                                                      (int)G, (int)p.n);
    });
    VSP_CUDA_CHECK(cudaGetLastError());
    c->launches++;
    launch_br(c, d_tasks, d_trlwe, pl.T, st);
    launch_iks(c, d_trlwe, d_gtask, d_glist, (int)pl.glist.size(), d_out, st);
}

}  // namespace

// DFMA throughput probe: 16 independent FMA chains per thread.
__global__ void fp64_probe_kernel(double* out, int iters, double m)
{
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; k++)
        x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < 16; k++)
            x[k] = fma(x[k], m, 1e-9);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; k++)
        s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

extern "C" {

const char* vsp_last_error(void) { return g_err.c_str(); }

int vsp_params_by_name(const char* name, uint32_t n_override, vsp_params* out)
{
    return guard([&] {
        Params p{};
        const std::string s = name ? name : "";
        if (s == "tfhe-80") {  // params.cpp:31-56
            p = Params{500, 1024, 2, 10, 2048, 4, 9, 2, 8, 3, 10, 1};
        }
        else if (s == "test-det") {  // params.cpp:58-86
            p = Params{16, 64, 2, 16, 128, 4, 16, 4, 8, 4, 8, 0};
        }
        else {
            throw std::invalid_argument("unknown parameter set: " + s);
        }
        if (n_override)
            p.n = n_override;
        validate(p);
        std::memcpy(out, &p, sizeof(vsp_params));
    });
}

vsp_ctx* vsp_create(const vsp_params* params, int device)
{
    vsp_ctx* out = nullptr;
    guard([&] {
        auto c = std::make_unique<vsp_ctx>();
        std::memcpy(&c->p, params, sizeof(vsp_params));
        validate(c->p);
        if (c->p.fft && (c->p.N1 != 1024 || c->p.l1 != 2))
            throw std::invalid_argument("FFT path is specialised for N1 = 1024, l1 = 2");
        c->device = device;
        c->set_device();
        VSP_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        // twiddles of the 512-point negacyclic transform
        double2 tw1[15];
        for (int d = 0; d < 4; d++)
            for (int b = 0; b < (1 << d); b++)
                tw1[(1 << d) - 1 + b] = zeta(d, (uint32_t)b);
        VSP_CUDA_CHECK(cudaMemcpyToSymbol(c_tw1, tw1, sizeof(tw1)));
        std::vector<double2> tw2(kTw2Entries * 32);
        for (int L = 0; L < 32; L++) {
            const uint32_t hi = L >> 1, odd = L & 1;
            int e = 0;
            for (int d = 4; d < 8; d++)
                for (uint32_t s = 0; s < (1u << (d - 4)); s++)
                    tw2[(e++) * 32 + L] = zeta(d, (hi << (d - 4)) | s);
            for (uint32_t k = 0; k < 8; k++)
                tw2[(e++) * 32 + L] = zeta(8, hi * 16 + k + 8 * odd);
        }
        VSP_CUDA_CHECK(cudaMalloc(&c->d_tw2, tw2.size() * sizeof(double2)));
        VSP_CUDA_CHECK(cudaMemcpy(c->d_tw2, tw2.data(), tw2.size() * sizeof(double2),
                                  cudaMemcpyHostToDevice));
        std::vector<uint32_t> tv(2 * c->p.N1, 0);
        for (uint32_t i = 0; i < c->p.N1; i++)
            tv[c->p.N1 + i] = kMu32;
        VSP_CUDA_CHECK(cudaMalloc(&c->d_tv1, tv.size() * 4));
        VSP_CUDA_CHECK(cudaMemcpy(c->d_tv1, tv.data(), tv.size() * 4, cudaMemcpyHostToDevice));
        configure_kernels(sizeof(Br1024Smem<kBrWarps, kBrSlots>),
                          (size_t)c->p.N1 * c->p.ksLen * sizeof(uint64_t));
        out = c.release();
    });
    return out;
}

void vsp_destroy(vsp_ctx* c)
{
    if (!c)
        return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (void* q : {(void*)c->d_bk1fd, (void*)c->d_bk1raw, (void*)c->d_ksk, (void*)c->d_bk2raw,
                    (void*)c->d_pks[0], (void*)c->d_pks[1], (void*)c->d_tw2, (void*)c->d_tv1})
        if (q)
            cudaFree(q);
    for (DevBuf* b : {&c->tasks, &c->trlwe, &c->in, &c->out, &c->kinds, &c->gtask, &c->glist})
        b->release();
    cudaStreamDestroy(c->stream);
    delete c;
}

int vsp_upload_keys(vsp_ctx* c, const uint32_t* bk1, const uint32_t* ksk, const uint64_t* bk2,
                    const uint32_t* pks_negs, const uint32_t* pks_id, int has_cb)
{
    return guard([&] {
        std::lock_guard<std::mutex> lk(c->mu);
        c->set_device();
        const Params& p = c->p;
        if (!bk1 || !ksk)
            throw std::invalid_argument("bk1 and ksk are required");
        if (has_cb && (!bk2 || !pks_negs || !pks_id))
            throw std::invalid_argument("circuit-bootstrapping material incomplete");
        const size_t bk1_words = (size_t)p.n * 2 * p.l1 * 2 * p.N1;
        uint32_t* d_raw = nullptr;
        VSP_CUDA_CHECK(cudaMalloc(&d_raw, bk1_words * 4));
        VSP_CUDA_CHECK(cudaMemcpy(d_raw, bk1, bk1_words * 4, cudaMemcpyHostToDevice));
        if (p.fft) {
            if (c->d_bk1fd)
                cudaFree(c->d_bk1fd);
            VSP_CUDA_CHECK(cudaMalloc(&c->d_bk1fd, (size_t)p.n * 4 * 1024 * sizeof(double2)));
            const int npolys = (int)(p.n * 4 * 2);
            prepare_poly1024_kernel<<<(npolys + 3) / 4, 128, 0, c->stream>>>(
                d_raw, c->d_tw2, c->d_bk1fd, npolys);
            VSP_CUDA_CHECK(cudaGetLastError());
            c->launches++;
            VSP_CUDA_CHECK(cudaStreamSynchronize(c->stream));
            cudaFree(d_raw);
        }
        else {
            if (c->d_bk1raw)
                cudaFree(c->d_bk1raw);
            c->d_bk1raw = d_raw;
        }
        if (c->d_ksk)
            cudaFree(c->d_ksk);
        VSP_CUDA_CHECK(cudaMalloc(&c->d_ksk, c->ksk_words() * 4));
        VSP_CUDA_CHECK(cudaMemcpy(c->d_ksk, ksk, c->ksk_words() * 4, cudaMemcpyHostToDevice));
        c->has_cb = false;
        if (has_cb) {
            const size_t bk2_words = (size_t)p.n * 2 * p.l2 * 2 * p.N2;
            if (c->d_bk2raw)
                cudaFree(c->d_bk2raw);
            VSP_CUDA_CHECK(cudaMalloc(&c->d_bk2raw, bk2_words * 8));
            VSP_CUDA_CHECK(cudaMemcpy(c->d_bk2raw, bk2, bk2_words * 8, cudaMemcpyHostToDevice));
            for (int w = 0; w < 2; w++) {
                if (c->d_pks[w])
                    cudaFree(c->d_pks[w]);
                VSP_CUDA_CHECK(cudaMalloc(&c->d_pks[w], c->pks_words() * 4));
                VSP_CUDA_CHECK(cudaMemcpy(c->d_pks[w], w == 0 ? pks_negs : pks_id,
                                          c->pks_words() * 4, cudaMemcpyHostToDevice));
            }
            c->has_cb = true;
        }
        c->has_keys = true;
    });
}

int vsp_hom_gate_batch_dev(vsp_ctx* c, const int32_t* kinds, const uint32_t* d_in,
                           uint32_t* d_out, size_t G, void* stream)
{
    return guard([&] {
        std::lock_guard<std::mutex> lk(c->mu);
        c->set_device();
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
        hom_gate_dev(c, kinds, d_in, d_out, G, st);
    });
}

int vsp_hom_gate_batch(vsp_ctx* c, const int32_t* kinds, const uint32_t* in, uint32_t* out,
                       size_t G)
{
    return guard([&] {
        std::lock_guard<std::mutex> lk(c->mu);
        c->set_device();
        for (size_t g = 0; g < G; g++)
            if (kinds[g] < 0 || kinds[g] > kXor)
                throw std::invalid_argument("homGate: unknown kind");
        if (G == 0)
            return;
        const size_t w = c->p.n + 1;
        uint32_t* d_in = c->in.as<uint32_t>(G * 3 * w);
        uint32_t* d_out = c->out.as<uint32_t>(G * w);
        VSP_CUDA_CHECK(cudaMemcpyAsync(d_in, in, G * 3 * w * 4, cudaMemcpyHostToDevice, c->stream));
        hom_gate_dev(c, kinds, d_in, d_out, G, c->stream);
        VSP_CUDA_CHECK(cudaMemcpyAsync(out, d_out, G * w * 4, cudaMemcpyDeviceToHost, c->stream));
        VSP_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int vsp_bootstrap_to_trlwe_batch(vsp_ctx* c, const uint32_t* in, uint32_t* out, size_t G)
{
    return guard([&] {
        std::lock_guard<std::mutex> lk(c->mu);
        c->set_device();
        require_keys(c);
        if (G == 0)
            return;
        const size_t w = c->p.n + 1;
        uint32_t* d_in = c->in.as<uint32_t>(G * w);
        uint32_t* d_tr = c->trlwe.as<uint32_t>(G * 2 * c->p.N1);
        VSP_CUDA_CHECK(cudaMemcpyAsync(d_in, in, G * w * 4, cudaMemcpyHostToDevice, c->stream));
        launch_br(c, d_in, d_tr, (int)G, c->stream);
        VSP_CUDA_CHECK(cudaMemcpyAsync(out, d_tr, G * 2 * c->p.N1 * 4, cudaMemcpyDeviceToHost,
                                       c->stream));
        VSP_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int vsp_gate_bootstrap_batch(vsp_ctx* c, const uint32_t* in, uint32_t* out, size_t G)
{
    return guard([&] {
        std::lock_guard<std::mutex> lk(c->mu);
        c->set_device();
        require_keys(c);
        if (G == 0)
            return;
        const size_t w = c->p.n + 1;
        uint32_t* d_in = c->in.as<uint32_t>(G * w);
        uint32_t* d_tr = c->trlwe.as<uint32_t>(G * 2 * c->p.N1);
        uint32_t* d_out = c->out.as<uint32_t>(G * w);
        std::vector<int2> gt(G);
        std::vector<int> gl(G);
        for (size_t g = 0; g < G; g++) {
            gt[g] = make_int2((int)g, -1);
            gl[g] = (int)g;
        }
        int2* d_gt = c->gtask.as<int2>(G);
        int* d_gl = c->glist.as<int>(G);
        VSP_CUDA_CHECK(cudaMemcpyAsync(d_gt, gt.data(), G * sizeof(int2), cudaMemcpyHostToDevice,
                                       c->stream));
        VSP_CUDA_CHECK(cudaMemcpyAsync(d_gl, gl.data(), G * sizeof(int), cudaMemcpyHostToDevice,
                                       c->stream));
        VSP_CUDA_CHECK(cudaMemcpyAsync(d_in, in, G * w * 4, cudaMemcpyHostToDevice, c->stream));
        launch_br(c, d_in, d_tr, (int)G, c->stream);
        launch_iks(c, d_tr, d_gt, d_gl, (int)G, d_out, c->stream);
        VSP_CUDA_CHECK(cudaMemcpyAsync(out, d_out, G * w * 4, cudaMemcpyDeviceToHost, c->stream));
        VSP_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int vsp_identity_key_switch_batch(vsp_ctx* c, const uint32_t* in, uint32_t* out, size_t G)
{
    return guard([&] {
        std::lock_guard<std::mutex> lk(c->mu);
        c->set_device();
        require_keys(c);
        if (G == 0)
            return;
        // Express each level-1 TLWE as a TRLWE whose sample extract at 0 returns it:
        // a'[0] = A[0], a'[i] = -A[N-i]  =>  A[0] = a'[0], A[N-i] = -a'[i]; B[0] = b'.
        const uint32_t N = c->p.N1;
        std::vector<uint32_t> tr((size_t)G * 2 * N, 0);
        for (size_t g = 0; g < G; g++) {
            const uint32_t* a = in + g * (N + 1);
            uint32_t* A = tr.data() + g * 2 * N;
            A[0] = a[0];
            for (uint32_t i = 1; i < N; i++)
                A[N - i] = 0u - a[i];
            A[N] = a[N];
        }
        std::vector<int2> gt(G);
        std::vector<int> gl(G);
        for (size_t g = 0; g < G; g++) {
            gt[g] = make_int2((int)g, -1);
            gl[g] = (int)g;
        }
        uint32_t* d_tr = c->trlwe.as<uint32_t>(tr.size());
        uint32_t* d_out = c->out.as<uint32_t>(G * (c->p.n + 1));
        int2* d_gt = c->gtask.as<int2>(G);
        int* d_gl = c->glist.as<int>(G);
        VSP_CUDA_CHECK(cudaMemcpyAsync(d_tr, tr.data(), tr.size() * 4, cudaMemcpyHostToDevice,
                                       c->stream));
        VSP_CUDA_CHECK(cudaMemcpyAsync(d_gt, gt.data(), G * sizeof(int2), cudaMemcpyHostToDevice,
                                       c->stream));
        VSP_CUDA_CHECK(cudaMemcpyAsync(d_gl, gl.data(), G * sizeof(int), cudaMemcpyHostToDevice,
                                       c->stream));
        launch_iks(c, d_tr, d_gt, d_gl, (int)G, d_out, c->stream);
        VSP_CUDA_CHECK(cudaMemcpyAsync(out, d_out, G * (c->p.n + 1) * 4, cudaMemcpyDeviceToHost,
                                       c->stream));
        VSP_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int vsp_counters(vsp_ctx* c, uint64_t out[5])
{
    std::memcpy(out, c->counters, sizeof(c->counters));
    return 0;
}

int vsp_counters_reset(vsp_ctx* c)
{
    std::memset(c->counters, 0, sizeof(c->counters));
    return 0;
}

uint64_t vsp_kernel_launches(vsp_ctx* c) { return c->launches; }

int vsp_profile_enable(vsp_ctx* c, int on)
{
    c->profiling = on != 0;
    return 0;
}

int vsp_profile_read(vsp_ctx* c, const char* name, double* total_ms, uint64_t* count)
{
    return guard([&] {
        c->set_device();
        auto it = c->timers.find(name);
        if (it == c->timers.end()) {
            *total_ms = 0;
            *count = 0;
            return;
        }
        auto& t = it->second;
        for (auto& e : t.pending) {
            VSP_CUDA_CHECK(cudaEventSynchronize(e.second));
            float ms = 0;
            VSP_CUDA_CHECK(cudaEventElapsedTime(&ms, e.first, e.second));
            t.total_ms += ms;
            t.count++;
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        t.pending.clear();
        *total_ms = t.total_ms;
        *count = t.count;
    });
}

int vsp_profile_reset(vsp_ctx* c)
{
    return guard([&] {
        c->set_device();
        for (auto& kv : c->timers)
            for (auto& e : kv.second.pending) {
                cudaEventSynchronize(e.second);
                cudaEventDestroy(e.first);
                cudaEventDestroy(e.second);
            }
        c->timers.clear();
    });
}

int vsp_fp64_peak_probe(int device, double* tflops)
{
    return guard([&] {
        VSP_CUDA_CHECK(cudaSetDevice(device));
        int sms = 0;
        VSP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        const int blocks = sms * 8, threads = 256, iters = 4096;
        double* d = nullptr;
        VSP_CUDA_CHECK(cudaMalloc(&d, (size_t)blocks * threads * sizeof(double)));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        fp64_probe_kernel<<<blocks, threads>>>(d, iters, 1.0000001);
        VSP_CUDA_CHECK(cudaGetLastError());
        float best = 1e30f;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(a);
            fp64_probe_kernel<<<blocks, threads>>>(d, iters, 1.0000001);
            cudaEventRecord(b);
            VSP_CUDA_CHECK(cudaEventSynchronize(b));
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            best = std::min(best, ms);
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(d);
        const double flops = 2.0 * 16.0 * iters * (double)blocks * threads;
        *tflops = flops / (best * 1e-3) / 1e12;
    });
}

int vsp_synchronize(vsp_ctx* c)
{
    return guard([&] {
        c->set_device();
        VSP_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"
