// k_layout.cu — K3: the inverted-file layout in HBM (ivf_index.hpp:15-41).
// Lists are stored back to back in list order, each list start padded to a
// multiple of 16 entries (128 B of m=8 codes) so scans start on aligned,
// coalesced addresses.  Per entry: m code bytes, a u32 id, m' refine-code
// bytes — all position-aligned, so the scanner carries positions and ids are
// gathered only for shortlist candidates.  Within a list ids ascend
// (ivf_index.hpp:15-16): old entries keep their order and staged entries, which
// carry larger ids (id-ascending adds), are appended in stable id order.
#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

__device__ __forceinline__ void copy_bytes(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                           uint32_t nb) {
    if (nb == 8) {
        *reinterpret_cast<u64*>(dst) = *reinterpret_cast<const u64*>(src);
    } else if (nb % 4 == 0) {
        for (uint32_t i = 0; i < nb; i += 4)
            *reinterpret_cast<uint32_t*>(dst + i) = *reinterpret_cast<const uint32_t*>(src + i);
    } else {
        for (uint32_t i = 0; i < nb; ++i) dst[i] = src[i];
    }
}

__global__ void copy_old_kernel(const uint64_t* __restrict__ old_off, const uint32_t* __restrict__ old_len,
                                const uint64_t* __restrict__ new_off,
                                const uint8_t* __restrict__ old_codes, const uint32_t* __restrict__ old_ids,
                                const uint8_t* __restrict__ old_rcodes, uint32_t m, uint32_t mprime,
                                uint8_t* __restrict__ codes, uint32_t* __restrict__ ids,
                                uint8_t* __restrict__ rcodes) {
    const uint32_t l = blockIdx.x;
    const uint32_t len = old_len[l];
    const uint64_t src0 = old_off[l], dst0 = new_off[l];
    for (uint32_t r = blockIdx.y * blockDim.x + threadIdx.x; r < len; r += gridDim.y * blockDim.x) {
        const uint64_t src = src0 + r, dst = dst0 + r;
        ids[dst] = old_ids[src];
        copy_bytes(codes + dst * m, old_codes + src * m, m);
        if (mprime) copy_bytes(rcodes + dst * mprime, old_rcodes + src * mprime, mprime);
    }
}

__global__ void place_new_kernel(const uint32_t* __restrict__ sorted_list,
                                 const uint32_t* __restrict__ sorted_idx, size_t n,
                                 const uint32_t* __restrict__ stage_off,
                                 const uint64_t* __restrict__ new_off,
                                 const uint32_t* __restrict__ old_len,
                                 const uint8_t* __restrict__ st_codes,
                                 const uint8_t* __restrict__ st_rcodes, const uint32_t* __restrict__ st_ids, uint32_t m,
                                 uint32_t mprime, uint8_t* __restrict__ codes,
                                 uint32_t* __restrict__ ids, uint8_t* __restrict__ rcodes) {
    size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint32_t l = sorted_list[s], idx = sorted_idx[s];
    const uint64_t pos = new_off[l] + old_len[l] + (s - stage_off[l]);
    ids[pos] = st_ids[idx];
    copy_bytes(codes + pos * m, st_codes + (size_t)idx * m, m);
    if (mprime) copy_bytes(rcodes + pos * mprime, st_rcodes + (size_t)idx * mprime, mprime);
}

}  // namespace

void launch_layout_copy_old(const uint64_t* old_off, const uint32_t* old_len, uint32_t nlists,
                            const uint64_t* new_off, const uint8_t* old_codes,
                            const uint32_t* old_ids, const uint8_t* old_rcodes, uint32_t m,
                            uint32_t mprime, uint8_t* codes, uint32_t* ids, uint8_t* rcodes,
                            uint32_t max_len, cudaStream_t s) {
    if (nlists == 0 || max_len == 0) return;
    dim3 grid(nlists, std::min<uint32_t>((max_len + 255) / 256, 64));
    copy_old_kernel<<<grid, 256, 0, s>>>(old_off, old_len, new_off, old_codes, old_ids, old_rcodes, m,
                                         mprime, codes, ids, rcodes);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_layout_place_new(const uint32_t* sorted_list, const uint32_t* sorted_idx, size_t n,
                             const uint32_t* stage_off, const uint64_t* new_off,
                             const uint32_t* old_len, const uint8_t* st_codes,
                             const uint8_t* st_rcodes, const uint32_t* st_ids, uint32_t m,
                             uint32_t mprime, uint8_t* codes, uint32_t* ids, uint8_t* rcodes,
                             cudaStream_t s) {
    if (n == 0) return;
    place_new_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        sorted_list, sorted_idx, n, stage_off, new_off, old_len, st_codes, st_rcodes, st_ids, m,
        mprime, codes, ids, rcodes);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
