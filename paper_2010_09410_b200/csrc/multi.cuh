// Multi-GPU: one process per GPU, keys replicated, every netlist level's
// gates split into per-rank slices of equal TASK count (a MUX is two blind rotations, a
// NOT none), the level's output TLWEs all-gathered so every rank holds the full value
// table for the next level; the RAM is sharded by bit-block (rank r owns blocks
// [r w / world, (r + 1) w / world): its read trees, control bits and write bars), the
// read-out TLWEs joining the all-gather.  Included by vsp_capi.cu after hom_gate_dev.
//
// Exchange backends:
//  - NCCL (vsp_attach_comm): ncclAllGather on the engine stream, over NVLink / NVSwitch.
//    NCCL is loaded with dlopen at first use, so a single-GPU process never needs it and a
//    process that already loaded torch's NCCL reuses that copy.
//  - host callback (vsp_attach_exchange): the engine stages the slice in host memory and
//    calls an all-gather the caller provides (e.g. torch.distributed over gloo / TCP); the
//    tests drive the engine's sharded C++ path this way with two processes on one GPU.
#pragma once

namespace {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl()
{
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL not loadable: ") + dlerror();
            return;
        }
        api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
        api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
        api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
        api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
        if (!api.getUniqueId || !api.commInitRank || !api.allGather || !api.commDestroy)
            err = "NCCL symbols missing";
    });
    if (!err.empty())
        throw std::runtime_error(err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what)
{
    if (r != ncclSuccess)
        throw std::runtime_error(std::string(what) + ": " +
                                 (nccl().getErrorString ? nccl().getErrorString(r) : "NCCL error"));
}

// A communicator or exchange is attached: the level / RAM sharding is active (also at world 1
// with VSP_NCCL_SINGLE, which the tests use to run the sharded path on one GPU).
bool sharded(const vsp_ctx* c) { return c->comm || c->xchg; }

// All-gather of `bytes` per rank: recv[r * bytes ...] = rank r's send.  send may alias
// recv + rank * bytes (in place).  Device buffers, ordered on `st`.
void exchange_allgather(vsp_ctx* c, const void* send, void* recv, size_t bytes, cudaStream_t st)
{
    if (c->comm) {
        nccl_check(nccl().allGather(send, recv, bytes, ncclUint8, (ncclComm_t)c->comm, st),
                   "ncclAllGather");
        return;
    }
    if (!c->xchg)
        throw std::logic_error("exchange_allgather without a communicator");
    uint8_t* hs = c->xchg_host.as<uint8_t>(bytes * (1 + (size_t)c->world));
    uint8_t* hr = hs + bytes;
    VSP_CUDA_CHECK(cudaMemcpyAsync(hs, send, bytes, cudaMemcpyDeviceToHost, st));
    VSP_CUDA_CHECK(cudaStreamSynchronize(st));
    if (c->xchg(hs, hr, bytes, c->xchg_user) != 0)
        throw std::runtime_error("exchange callback failed");
    VSP_CUDA_CHECK(cudaMemcpyAsync(recv, hr, bytes * c->world, cudaMemcpyHostToDevice, st));
    VSP_CUDA_CHECK(cudaStreamSynchronize(st));  // hr is reused by the next exchange
}

// Per-rank slices of a G-gate level with equal TASK counts: cut points at r T / world in
// task space (tasks of gate g = 2 for MUX, 0 for NOT, else 1), a gate belonging to the
// slice in which its first task falls (NOT gates: where their position falls).  `per` =
// the largest slice (the all-gather's per-rank count).
struct Slice {
    size_t lo, hi, per;
};

std::vector<size_t> level_cuts(const int32_t* kinds, size_t G, int world)
{
    std::vector<size_t> start(G + 1, 0);
    for (size_t g = 0; g < G; g++) {
        const int k = kinds ? kinds[g] : 3;
        start[g + 1] = start[g] + (k == kMux ? 2 : k == kNot ? 0 : 1);
    }
    const size_t T = start[G];
    std::vector<size_t> cut(world + 1, G);
    cut[0] = 0;
    for (int r = 1; r < world; r++) {
        if (T == 0) {  // all NOT: split by gate count
            cut[r] = G * (size_t)r / world;
            continue;
        }
        const size_t b = (T * (size_t)r + world - 1) / world;  // first task of slice r
        cut[r] = (size_t)(std::lower_bound(start.begin(), start.begin() + G, b) - start.begin());
        cut[r] = std::max(cut[r], cut[r - 1]);
    }
    return cut;
}

Slice level_slice(const int32_t* kinds, size_t G, int world, int rank)
{
    const std::vector<size_t> cut = level_cuts(kinds, G, world);
    size_t per = 0;
    for (int r = 0; r < world; r++)
        per = std::max(per, cut[r + 1] - cut[r]);
    return {cut[rank], cut[rank + 1], per};
}

// Scatter the padded all-gather blocks (rank r's gates at recv[r * per]) to their level
// positions out[cut[r] ...].
__global__ void repack_slices_kernel(const uint32_t* __restrict__ recv, uint32_t* __restrict__ out,
                                     const int64_t* __restrict__ cut, int world, size_t per, int n1)
{
    const size_t g = blockIdx.x;  // destination gate
    int r = 0;
    while (r + 1 < world && (size_t)cut[r + 1] <= g)
        r++;
    const size_t src = (size_t)r * per + (g - (size_t)cut[r]);
    for (int k = threadIdx.x; k < n1; k += blockDim.x)
        out[g * n1 + k] = recv[src * n1 + k];
}

// homGate over one whole level, sharded across the ranks: this rank bootstraps its slice,
// then one all-gather assembles all G outputs (d_out_all, G x (n+1)) on every rank.
// d_in_all holds all G gates' inputs (every rank has the full value table).  Equal slices
// (e.g. uniform gates, G a multiple of world) are all-gathered in place into d_out_all.
void hom_gate_level_dev(vsp_ctx* c, const int32_t* kinds, const uint32_t* d_in_all,
                        uint32_t* d_out_all, size_t G, cudaStream_t st)
{
    if (!sharded(c) || G == 0) {
        hom_gate_dev(c, kinds, d_in_all, d_out_all, G, st);
        return;
    }
    const size_t n1 = c->p.n + 1;
    const std::vector<size_t> cut = level_cuts(kinds, G, c->world);
    size_t per = 0;
    bool equal = true;
    for (int r = 0; r < c->world; r++) {
        per = std::max(per, cut[r + 1] - cut[r]);
        equal = equal && cut[r] == (size_t)r * (G / c->world);
    }
    equal = equal && G % c->world == 0;
    const size_t lo = cut[c->rank], hi = cut[c->rank + 1];
    if (equal) {
        uint32_t* mine = d_out_all + lo * n1;
        if (hi > lo)
            hom_gate_dev(c, kinds + lo, d_in_all + lo * 3 * n1, mine, hi - lo, st);
        exchange_allgather(c, mine, d_out_all, per * n1 * 4, st);
        return;
    }
    uint32_t* recv = c->mg_recv.as<uint32_t>(per * n1 * c->world);
    uint32_t* mine = recv + (size_t)c->rank * per * n1;
    if (hi > lo)
        hom_gate_dev(c, kinds + lo, d_in_all + lo * 3 * n1, mine, hi - lo, st);
    exchange_allgather(c, mine, recv, per * n1 * 4, st);
    std::vector<int64_t> hcut(cut.begin(), cut.end());
    int64_t* d_cut = c->mg_send.as<int64_t>(hcut.size());
    VSP_CUDA_CHECK(cudaMemcpyAsync(d_cut, hcut.data(), hcut.size() * 8, cudaMemcpyHostToDevice, st));
    repack_slices_kernel<<<(unsigned)G, 128, 0, st>>>(recv, d_out_all, d_cut, c->world, per, (int)n1);
    VSP_CUDA_CHECK(cudaGetLastError());
    c->launches++;
}

// RAM bit-block ownership: rank r owns blocks [j0, j1) when the word width divides evenly
// over the ranks (otherwise every rank runs the whole RAM, replicated).
struct BlockRange {
    int j0, j1;
    bool shard;
};

BlockRange ram_blocks(const vsp_ctx* c, int w)
{
    if (!sharded(c) || w % c->world != 0)
        return {0, w, false};
    const int per = w / c->world;
    return {c->rank * per, (c->rank + 1) * per, true};
}

// All-gather the owned bit-blocks of a sharded RAM image in place, so every rank holds the
// whole current image (getter / snapshot / host API).
void ram_gather_dev(vsp_ctx* c, uint32_t* d_ram, int v, int w, cudaStream_t st)
{
    const BlockRange br = ram_blocks(c, w);
    if (!br.shard)
        return;
    const size_t cw = 2 * (size_t)c->p.N1;
    const size_t cells = (size_t)(br.j1 - br.j0) << v;
    exchange_allgather(c, d_ram + ((size_t)br.j0 << v) * cw, d_ram, cells * cw * 4, st);
}

}  // namespace
