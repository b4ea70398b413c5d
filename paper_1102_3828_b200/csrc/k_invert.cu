// k_invert.cu — the probe inversion of a SMALL batch in two launches.
//
// ivf_search probes w lists per query (ivf_index.hpp:58-61); the list-major
// scan needs the (query, list) pairs sorted by list and cut into work items.
// For thousands of queries that is a radix sort, a histogram and a handful of
// scans (pqrr_dev.cu: items_phase1 / items_phase2, ~20 launches).  A serving
// batch of 1-32 queries holds at most a few thousand pairs, and those 20
// launches cost more than the scan they prepare (C5 batch 1: 0.17 of
// 0.55 ms).  Here one CTA does the whole inversion in shared memory:
//   invert_small_kernel      pairs sorted by (list, sampling tier, coarse gap)
//                            -> pair_sorted, per-list counts / first pair,
//                            item offsets of the 16-query (LUT pass) and the
//                            64-query (K4f) item sets;
//   items_finish_small_kernel  one CTA per item set: the items and their
//                            longest-first order.
// Both produce exactly what the large-batch kernels produce (same sort keys,
// ties in pair / item order), so everything downstream is shared.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int IV_THREADS = 1024;

__device__ __forceinline__ void bitonic_u64(u64* a, uint32_t n2) {
    for (uint32_t k = 2; k <= n2; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (j - 1)), hi = lo + j;
                const bool up = (lo & k) == 0;
                const u64 x = a[lo], y = a[hi];
                if ((x > y) == up) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
            __syncthreads();
        }
}

// Exclusive scan of three per-thread triples across the CTA.
struct U3 {
    uint32_t a, b, c;
};
__device__ __forceinline__ U3 add3(U3 x, U3 y) { return U3{x.a + y.a, x.b + y.b, x.c + y.c}; }
__device__ __forceinline__ U3 shfl_up3(U3 v, int o) {
    return U3{__shfl_up_sync(0xffffffffu, v.a, o), __shfl_up_sync(0xffffffffu, v.b, o),
              __shfl_up_sync(0xffffffffu, v.c, o)};
}
__device__ U3 block_excl_scan3(U3 v, U3* s_warp /* [32] */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    U3 incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const U3 t = shfl_up3(incl, o);
        if (lane >= o) incl = add3(incl, t);
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        U3 w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : U3{0, 0, 0};
        U3 wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const U3 t = shfl_up3(wi, o);
            if (lane >= o) wi = add3(wi, t);
        }
        s_warp[lane] = U3{wi.a - w.a, wi.b - w.b, wi.c - w.c};
    }
    __syncthreads();
    const U3 base = s_warp[warp];
    return U3{base.a + incl.a - v.a, base.b + incl.b - v.b, base.c + incl.c - v.c};
}

__global__ __launch_bounds__(IV_THREADS) void invert_small_kernel(
    const uint32_t* __restrict__ probes, uint32_t np, uint32_t w, const float* __restrict__ D, uint32_t c,
    const uint32_t* __restrict__ list_len, uint32_t qt_a, uint32_t qt_b, uint32_t chunk_b,
    uint32_t* __restrict__ pair_sorted, uint32_t* __restrict__ list_cnt, uint32_t* __restrict__ list_first,
    uint32_t* __restrict__ item_off_a, uint32_t* __restrict__ item_off_b) {
    extern __shared__ u64 iv_keys[];  // [n2]
    __shared__ U3 s_warp[32];
    uint32_t n2 = 1;
    while (n2 < np) n2 <<= 1;
    for (uint32_t i = threadIdx.x; i <= c; i += blockDim.x) list_cnt[i] = 0;
    // sort key of pair p = (q, r): (list, sampling tier of r, coarse gap to the
    // query's nearest probe) — pair_key_kernel's key; ties by pair id
    for (uint32_t p = threadIdx.x; p < n2; p += blockDim.x) {
        u64 k = ~0ull;
        if (p < np) {
            const uint32_t q = p / w, l = probes[p];
            const float gap = fmaxf(__fsub_rn(D[(size_t)q * c + l], D[(size_t)q * c + probes[q * w]]), 0.f);
            const uint32_t tier = sample_tier(p % w, w, 1);
            const uint32_t key = (l << 14) | (tier << 12) | (__float_as_uint(gap) >> 19);
            k = ((u64)key << 32) | p;
        }
        iv_keys[p] = k;
    }
    __syncthreads();
    bitonic_u64(iv_keys, n2);
    for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
        const u64 k = iv_keys[i];
        pair_sorted[i] = (uint32_t)k;
        atomicAdd(&list_cnt[(uint32_t)(k >> 46)], 1u);
    }
    __syncthreads();
    // per-list counts -> first pair; items per list of both sets -> offsets
    const uint32_t per = (c + 1 + blockDim.x - 1) / blockDim.x;
    const uint32_t l0 = threadIdx.x * per, l1 = min(c + 1, l0 + per);
    U3 sum{0, 0, 0};
    for (uint32_t l = l0; l < l1; ++l) {
        const uint32_t cnt = l < c ? list_cnt[l] : 0u;
        const uint32_t len = l < c ? list_len[l] : 0u;
        const uint32_t chunks = max(1u, (len + chunk_b - 1) / chunk_b);
        sum = add3(sum, U3{cnt, (cnt + qt_a - 1) / qt_a, ((cnt + qt_b - 1) / qt_b) * chunks});
    }
    U3 run = block_excl_scan3(sum, s_warp);
    for (uint32_t l = l0; l < l1; ++l) {
        const uint32_t cnt = l < c ? list_cnt[l] : 0u;
        const uint32_t len = l < c ? list_len[l] : 0u;
        const uint32_t chunks = max(1u, (len + chunk_b - 1) / chunk_b);
        list_first[l] = run.a;
        item_off_a[l] = run.b;
        item_off_b[l] = run.c;
        run = add3(run, U3{cnt, (cnt + qt_a - 1) / qt_a, ((cnt + qt_b - 1) / qt_b) * chunks});
    }
}

struct ItemOut {
    const uint32_t* item_off;
    uint32_t *item_list, *item_start, *item_nq, *item_e0, *item_e1, *item_order;
    uint32_t qt, chunk, bound;
};

// blockIdx.x = item set.  Items as items_build_kernel, order = items sorted by
// length descending (ties by item index), as the stable radix sort gives.
__global__ __launch_bounds__(IV_THREADS) void items_finish_small_kernel(
    const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ first, const uint32_t* __restrict__ len,
    uint32_t nlists, ItemOut oa, ItemOut ob) {
    extern __shared__ u64 iv_keys[];
    const ItemOut o = blockIdx.x == 0 ? oa : ob;
    const uint32_t n = min(o.item_off[nlists], o.bound);
    uint32_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
        u64 key = ~0ull;
        if (i < n) {
            uint32_t lo = 0, hi = nlists;  // last list with item_off[l] <= i
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (o.item_off[mid] <= i) lo = mid;
                else hi = mid;
            }
            const uint32_t l = lo, c = cnt[l], L = len[l];
            const uint32_t chunks = max(1u, (L + o.chunk - 1) / o.chunk);
            const uint32_t k = i - o.item_off[l];
            const uint32_t grp = k / chunks, ch = k % chunks;
            const uint32_t e0 = ch * o.chunk, e1 = min(L, e0 + o.chunk);
            o.item_list[i] = l;
            o.item_start[i] = first[l] + grp * o.qt;
            o.item_nq[i] = min(o.qt, c - grp * o.qt);
            o.item_e0[i] = e0;
            o.item_e1[i] = e1;
            key = ((u64)(0xffffffffu - (e1 - e0)) << 32) | i;
        }
        iv_keys[i] = key;
    }
    __syncthreads();
    bitonic_u64(iv_keys, n2);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) o.item_order[i] = (uint32_t)iv_keys[i];
}

}  // namespace

bool invert_small_supported(size_t np, uint32_t c) {
    return np >= 1 && np <= kInvertSmallMaxPairs && c < (1u << 18) && (size_t)c + 1 <= (size_t)IV_THREADS * 64;
}

void launch_invert_small(const uint32_t* probes, uint32_t np, uint32_t w, const float* D, uint32_t c,
                         const uint32_t* list_len, uint32_t qt_a, uint32_t qt_b, uint32_t chunk_b,
                         uint32_t* pair_sorted, uint32_t* list_cnt, uint32_t* list_first,
                         uint32_t* item_off_a, uint32_t* item_off_b, cudaStream_t s) {
    uint32_t n2 = 1;
    while (n2 < np) n2 <<= 1;
    invert_small_kernel<<<1, IV_THREADS, (size_t)n2 * sizeof(u64), s>>>(
        probes, np, w, D, c, list_len, qt_a, qt_b, chunk_b, pair_sorted, list_cnt, list_first, item_off_a,
        item_off_b);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_items_finish_small(const uint32_t* list_cnt, const uint32_t* list_first, const uint32_t* list_len,
                               uint32_t nlists, const SmallItems& a, const SmallItems* b, cudaStream_t s) {
    auto conv = [](const SmallItems& x) {
        return ItemOut{x.item_off, x.item_list, x.item_start, x.item_nq, x.item_e0, x.item_e1, x.item_order,
                       x.qt, x.chunk, x.bound};
    };
    const uint32_t mx = std::max(a.bound, b ? b->bound : 0u);
    uint32_t n2 = 1;
    while (n2 < mx) n2 <<= 1;
    items_finish_small_kernel<<<b ? 2 : 1, IV_THREADS, (size_t)n2 * sizeof(u64), s>>>(
        list_cnt, list_first, list_len, nlists, conv(a), conv(b ? *b : a));
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
