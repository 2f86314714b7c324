// Internal (C++ linkage) hook between the client keygen (client.cpp, host compiler) and
// the CUDA runtime (vsp_capi.cu): the keygen's deferred b += a*s products can run on a
// GPU.  Not part of the C ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>

#include "../../include/vsp_b200.h"

namespace vsp_internal {

// fin(bits, trlwes, count, N, key): for each of `count` consecutive (a[N], b[N]) pairs of
// `bits`-bit torus words at `trlwes`, b += a * key (negacyclic, binary key; polyMulBinary,
// poly.hpp:61-75).
using Finalizer = std::function<void(int bits, void* trlwes, size_t count, size_t N,
                                     const uint32_t* key)>;

void keygen(const vsp_params& p, uint64_t seed, int with_cb, uint32_t* lv0, uint32_t* lv1,
            uint32_t* lv2, uint32_t* bk1, uint32_t* ksk, uint64_t* bk2, uint32_t* pks_negs,
            uint32_t* pks_id, const Finalizer& fin);

}  // namespace vsp_internal
