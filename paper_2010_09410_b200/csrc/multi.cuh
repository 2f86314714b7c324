// Multi-GPU level sharding: one process per GPU, keys replicated, every
// netlist level's gates split into contiguous per-rank slices, the level's output TLWEs
// all-gathered over NCCL (NVLink / NVSwitch) so every rank holds the full value table
// for the next level.  Included by vsp_capi.cu after hom_gate_dev.
//
// NCCL is loaded with dlopen at first use, so a single-GPU process never needs it and a
// process that already loaded torch's NCCL reuses that copy (one libnccl.so.2 per
// process).  Only the C types of nccl.h are used at compile time.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

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

// Contiguous slice of a G-gate level for `rank` of `world`: every rank owns `per` =
// ceil(G / world) slots (the all-gather needs equal counts); slots past G are padding.
struct Slice {
    size_t lo, hi, per;
};

Slice level_slice(size_t G, int world, int rank)
{
    const size_t per = (G + world - 1) / world;
    const size_t lo = std::min(G, per * (size_t)rank);
    const size_t hi = std::min(G, lo + per);
    return {lo, hi, per};
}

// homGate over one whole level, sharded across the ranks of c's communicator: this rank
// bootstraps gates [lo, hi) of the level, then one ncclAllGather assembles all G outputs
// (d_out_all, G x (n+1)) on every rank.  d_in_all holds all G gates' inputs (every rank
// has the full value table).  Single rank: plain hom_gate_dev.
void hom_gate_level_dev(vsp_ctx* c, const int32_t* kinds, const uint32_t* d_in_all,
                        uint32_t* d_out_all, size_t G, cudaStream_t st)
{
    if (!c->comm || G == 0) {
        hom_gate_dev(c, kinds, d_in_all, d_out_all, G, st);
        return;
    }
    const size_t n1 = c->p.n + 1;
    const Slice sl = level_slice(G, c->world, c->rank);
    uint32_t* send = c->mg_send.as<uint32_t>(sl.per * n1);
    uint32_t* recv = c->mg_recv.as<uint32_t>(sl.per * n1 * c->world);
    if (sl.hi > sl.lo)
        hom_gate_dev(c, kinds + sl.lo, d_in_all + sl.lo * 3 * n1, send, sl.hi - sl.lo, st);
    nccl_check(nccl().allGather(send, recv, sl.per * n1, ncclUint32, (ncclComm_t)c->comm, st),
               "ncclAllGather");
    VSP_CUDA_CHECK(cudaMemcpyAsync(d_out_all, recv, G * n1 * sizeof(uint32_t),
                                   cudaMemcpyDeviceToDevice, st));
}

}  // namespace
