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

// Parity vector of an m = 8 code: bit j = code byte j & 1.  A 16-query LUT row
// is 64 B, i.e. exactly one half of the 32 banks, and the half is selected by
// the parity of the code byte; two entries of one warp step collide iff their
// bytes share parity.
__global__ void parity_keys_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                   const uint8_t* __restrict__ codes, uint32_t* __restrict__ keys,
                                   uint32_t* __restrict__ vals) {
    const uint32_t l = blockIdx.x;
    const uint64_t o = off[l];
    for (uint32_t r = threadIdx.x; r < len[l]; r += blockDim.x) {
        const u64 c = *reinterpret_cast<const u64*>(codes + (o + r) * 8);
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) v |= (uint32_t)((c >> (8 * j)) & 1ull) << j;
        keys[o + r] = v;
        vals[o + r] = (uint32_t)(o + r);
    }
}

// XOR masks of 8 bits ordered by decreasing popcount (Hamming distance 8..1).
__constant__ uint8_t c_masks[255];
__constant__ uint16_t c_mask_off[10];  // masks with popcount d: [c_mask_off[8-d], c_mask_off[9-d])

// One CTA per list: the scanner's LDS.128 is served in quarter-warp phases of
// 8 lanes = 2 consecutive entries (measured: tools/microbench/lds128.cu), so a
// phase is conflict-free in sub-quantizer j iff the two entries' code bytes
// differ in parity.  The list's entries, stably sorted by parity vector v, are
// matched greedily into pairs of maximal Hamming distance (complements first,
// then distance 7, ...), pairs laid out at even offsets, same-bucket leftovers
// last.  Every bucket-pair step exhausts a bucket, so the plan has <= 512 rows.
__global__ void pair_perm_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                 const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
                                 uint32_t* __restrict__ perm) {
    __shared__ uint32_t cnt[256], start[256], taken[256];
    __shared__ uint32_t p_a[512], p_b[512], p_k[512], p_out[512];
    __shared__ uint32_t s_np;
    const uint32_t l = blockIdx.x;
    const uint64_t o = off[l];
    const uint32_t n = len[l];
    for (uint32_t v = threadIdx.x; v < 256; v += blockDim.x) {
        cnt[v] = 0;
        taken[v] = 0;
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) atomicAdd(&cnt[skeys[o + r]], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t v = 0; v < 256; ++v) {
            start[v] = acc;
            acc += cnt[v];
        }
        uint32_t out = 0, np = 0;
        for (int d = 8; d >= 1; --d) {
            const uint32_t m0 = c_mask_off[8 - d], m1 = c_mask_off[9 - d];
            for (uint32_t v = 0; v < 256; ++v) {
                for (uint32_t mi = m0; mi < m1 && taken[v] < cnt[v]; ++mi) {
                    const uint32_t u = v ^ c_masks[mi];
                    const uint32_t k = min(cnt[v] - taken[v], cnt[u] - taken[u]);
                    if (k == 0) continue;
                    p_a[np] = start[v] + taken[v];
                    p_b[np] = start[u] + taken[u];
                    p_k[np] = k;
                    p_out[np] = out;
                    ++np;
                    out += 2 * k;
                    taken[v] += k;
                    taken[u] += k;
                }
            }
        }
        for (uint32_t v = 0; v < 256; ++v) {  // same-bucket leftovers
            const uint32_t k = cnt[v] - taken[v];
            if (!k) continue;
            p_a[np] = start[v] + taken[v];
            p_b[np] = 0xffffffffu;
            p_k[np] = k;
            p_out[np] = out;
            ++np;
            out += k;
        }
        s_np = np;
    }
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (uint32_t p = warp; p < s_np; p += nw) {
        const uint32_t a = p_a[p], b = p_b[p], k = p_k[p], dst = p_out[p];
        for (uint32_t i = lane; i < k; i += 32) {
            if (b == 0xffffffffu) {
                perm[o + dst + i] = svals[o + a + i];
            } else {
                perm[o + dst + 2 * i] = svals[o + a + i];
                perm[o + dst + 2 * i + 1] = svals[o + b + i];
            }
        }
    }
}

void upload_masks() {
    static int done_dev[64] = {0};
    int dev = 0;
    PQRR_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && done_dev[dev]) return;
    uint8_t masks[255];
    uint16_t moff[10];
    int k = 0;
    for (int d = 8; d >= 1; --d) {
        moff[8 - d] = (uint16_t)k;
        for (int m = 1; m < 256; ++m)
            if (__builtin_popcount(m) == d) masks[k++] = (uint8_t)m;
    }
    moff[8] = (uint16_t)k;
    moff[9] = (uint16_t)k;
    PQRR_CUDA(cudaMemcpyToSymbol(c_masks, masks, sizeof(masks)));
    PQRR_CUDA(cudaMemcpyToSymbol(c_mask_off, moff, sizeof(moff)));
    if (dev < 64) done_dev[dev] = 1;
}

__global__ void gather_layout_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                     const uint32_t* __restrict__ perm, const uint8_t* __restrict__ codes,
                                     const uint32_t* __restrict__ ids, const uint8_t* __restrict__ rcodes,
                                     uint32_t m, uint32_t mprime, uint8_t* __restrict__ o_codes,
                                     uint32_t* __restrict__ o_ids, uint8_t* __restrict__ o_rcodes) {
    const uint32_t l = blockIdx.x;
    const uint64_t o = off[l];
    for (uint32_t r = threadIdx.x; r < len[l]; r += blockDim.x) {
        const uint64_t dst = o + r, src = perm[o + r];
        o_ids[dst] = ids[src];
        copy_bytes(o_codes + dst * m, codes + src * m, m);
        if (mprime) copy_bytes(o_rcodes + dst * mprime, rcodes + src * mprime, mprime);
    }
}

__global__ void list_keys_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                 const uint32_t* __restrict__ ids, uint32_t* __restrict__ keys,
                                 uint32_t* __restrict__ vals) {
    const uint32_t l = blockIdx.x;
    const uint64_t o = off[l];
    for (uint32_t r = threadIdx.x; r < len[l]; r += blockDim.x) {
        keys[o + r] = ids[o + r];
        vals[o + r] = (uint32_t)(o + r);
    }
}

}  // namespace

namespace {
// block_list[pos >> 4] = list owning position pos (list starts are 16-aligned).
__global__ void block_list_kernel(const uint64_t* __restrict__ off, uint32_t nlists,
                                  uint16_t* __restrict__ bl) {
    const uint32_t l = blockIdx.x;
    if (l >= nlists) return;
    const uint64_t b0 = off[l] >> 4, b1 = off[l + 1] >> 4;
    for (uint64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) bl[b] = (uint16_t)l;
}
}  // namespace

void launch_block_list(const uint64_t* off, uint32_t nlists, uint16_t* bl, cudaStream_t s) {
    if (!nlists) return;
    block_list_kernel<<<nlists, 256, 0, s>>>(off, nlists, bl);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_parity_keys(const uint64_t* off, const uint32_t* len, uint32_t nlists,
                        const uint8_t* codes, uint32_t* keys, uint32_t* vals, cudaStream_t s) {
    parity_keys_kernel<<<nlists, 256, 0, s>>>(off, len, codes, keys, vals);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_list_id_keys(const uint64_t* off, const uint32_t* len, uint32_t nlists,
                         const uint32_t* ids, uint32_t* keys, uint32_t* vals, cudaStream_t s) {
    list_keys_kernel<<<nlists, 256, 0, s>>>(off, len, ids, keys, vals);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_pair_perm(const uint64_t* off, const uint32_t* len, uint32_t nlists,
                      const uint32_t* skeys, const uint32_t* svals, uint32_t* perm, cudaStream_t s) {
    upload_masks();
    pair_perm_kernel<<<nlists, 256, 0, s>>>(off, len, skeys, svals, perm);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_gather_layout(const uint64_t* off, const uint32_t* len, uint32_t nlists,
                          const uint32_t* perm, const uint8_t* codes, const uint32_t* ids,
                          const uint8_t* rcodes, uint32_t m, uint32_t mprime, uint8_t* o_codes,
                          uint32_t* o_ids, uint8_t* o_rcodes, cudaStream_t s) {
    gather_layout_kernel<<<nlists, 256, 0, s>>>(off, len, perm, codes, ids, rcodes, m, mprime, o_codes,
                                                o_ids, o_rcodes);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void segmented_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                          uint32_t* vals_out, size_t n, uint32_t nseg, const uint64_t* seg_begin,
                          const uint64_t* seg_end, int bits, cudaStream_t s);

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
