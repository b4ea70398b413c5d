// k_invert.cu — the probe inversion of a SMALL batch in one launch.
//
// ivf_search probes w lists per query (ivf_index.hpp:58-61); the list-major
// scan needs the (query, list) pairs sorted by list and cut into work items.
// For thousands of queries that is a radix sort, a histogram and a handful of
// scans (pqrr_dev.cu: items_phase1 / items_phase2, ~20 launches).  A serving
// batch of 1-32 queries holds at most a few thousand pairs, and those 20
// launches cost more than the scan they prepare (C5 batch 1: 0.17 of
// 0.55 ms).  Here one CTA does the whole inversion in shared memory:
// pairs sorted by (list, sampling tier, coarse gap) -> pair_sorted, per-list
// counts / first pair, the item offsets of the 16-query (LUT pass) and the
// 64-query (K4f) item sets, the items themselves and their longest-first
// order.  It produces exactly what the large-batch kernels produce (same sort
// keys, ties in pair / item order), so everything downstream is shared.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int IV_THREADS = 1024;

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

struct ItemOut {
    uint32_t* item_off;  // [c + 1], written here
    uint32_t *item_list, *item_start, *item_nq, *item_e0, *item_e1, *item_order;
    uint32_t qt, chunk, bound;  // bound = 0: offsets only (the items are built by the large-batch kernels)
};

// First index i in [0, n) with a[i] >= v (a ascending); n if none.
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One CTA.  Global reads: the P probes, their coarse distances and the lengths
// of the probed lists, all issued in parallel; everything per list (the c + 1
// entries of list_cnt / list_first / item_off the scan kernels index) is
// derived from the run table of the sorted pairs in shared memory, so no
// thread walks the lists through dependent global loads.
__global__ __launch_bounds__(IV_THREADS) void invert_small_kernel(
    const uint32_t* __restrict__ probes, uint32_t np, uint32_t w, const float* __restrict__ D, uint32_t c,
    const uint32_t* __restrict__ list_len, uint32_t* __restrict__ pair_sorted,
    uint32_t* __restrict__ list_cnt, uint32_t* __restrict__ list_first, ItemOut oa, ItemOut ob) {
    extern __shared__ u64 iv_keys[];  // [max(n2, item bound pow2)]
    __shared__ U3 s_warp[32];
    __shared__ uint32_t s_nruns;
    uint32_t n2 = 32;
    while (n2 < np) n2 <<= 1;
    // run table (<= np runs): list id, first pair, then per set the item prefix
    uint32_t* run_list = reinterpret_cast<uint32_t*>(iv_keys + kInvertSmallMaxPairs);
    uint32_t* run_first = run_list + kInvertSmallMaxPairs + 1;
    uint32_t* run_len = run_first + kInvertSmallMaxPairs + 1;
    uint32_t* run_pa = run_len + kInvertSmallMaxPairs + 1;
    uint32_t* run_pb = run_pa + kInvertSmallMaxPairs + 1;
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
    if (threadIdx.x == 0) s_nruns = 0;
    __syncthreads();
    cta_bitonic_sort(iv_keys, n2);
    // runs of equal list: flag heads, scan, scatter
    {
        const uint32_t per = (np + blockDim.x - 1) / blockDim.x;
        const uint32_t i0 = min(np, threadIdx.x * per), i1 = min(np, i0 + per);
        uint32_t heads = 0;
        for (uint32_t i = i0; i < i1; ++i) {
            const uint32_t l = (uint32_t)(iv_keys[i] >> 46);
            heads += (i == 0 || (uint32_t)(iv_keys[i - 1] >> 46) != l) ? 1u : 0u;
        }
        U3 ex = block_excl_scan3(U3{heads, 0, 0}, s_warp);
        uint32_t r = ex.a;
        for (uint32_t i = i0; i < i1; ++i) {
            const uint32_t l = (uint32_t)(iv_keys[i] >> 46);
            if (i == 0 || (uint32_t)(iv_keys[i - 1] >> 46) != l) {
                run_list[r] = l;
                run_first[r] = i;
                run_len[r] = list_len[l];
                ++r;
            }
        }
        if (i1 == np && i0 < np) s_nruns = r;  // the thread holding the last pair
    }
    for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) pair_sorted[i] = (uint32_t)iv_keys[i];
    __syncthreads();
    const uint32_t nr = s_nruns;
    if (threadIdx.x == 0) run_first[nr] = np;
    __syncthreads();
    // item prefix of both sets over the runs
    {
        const uint32_t per = (nr + blockDim.x - 1) / blockDim.x;
        const uint32_t r0 = min(nr, threadIdx.x * per), r1 = min(nr, r0 + per);
        U3 sum{0, 0, 0};
        for (uint32_t r = r0; r < r1; ++r) {
            const uint32_t cnt = run_first[r + 1] - run_first[r];
            const uint32_t ca = max(1u, (run_len[r] + oa.chunk - 1) / oa.chunk);
            const uint32_t cb = max(1u, (run_len[r] + ob.chunk - 1) / ob.chunk);
            sum = add3(sum, U3{((cnt + oa.qt - 1) / oa.qt) * ca, ((cnt + ob.qt - 1) / ob.qt) * cb, 0});
        }
        U3 run = block_excl_scan3(sum, s_warp);
        for (uint32_t r = r0; r < r1; ++r) {
            const uint32_t cnt = run_first[r + 1] - run_first[r];
            const uint32_t ca = max(1u, (run_len[r] + oa.chunk - 1) / oa.chunk);
            const uint32_t cb = max(1u, (run_len[r] + ob.chunk - 1) / ob.chunk);
            run_pa[r] = run.a;
            run_pb[r] = run.b;
            run = add3(run, U3{((cnt + oa.qt - 1) / oa.qt) * ca, ((cnt + ob.qt - 1) / ob.qt) * cb, 0});
        }
        if (r0 < nr && r1 == nr) {  // the thread holding the last run: totals
            run_pa[nr] = run.a;
            run_pb[nr] = run.b;
        }
    }
    __syncthreads();
    // per list (coalesced): the run at or after it gives every offset
    for (uint32_t l = threadIdx.x; l <= c; l += blockDim.x) {
        const uint32_t r = lower_bound_u32(run_list, nr, l);
        const bool hit = r < nr && run_list[r] == l;
        list_cnt[l] = hit ? run_first[r + 1] - run_first[r] : 0u;
        list_first[l] = run_first[r];
        oa.item_off[l] = run_pa[r];
        ob.item_off[l] = run_pb[r];
    }
    // items of both sets from the run table, then their longest-first order
    for (int set = 0; set < 2; ++set) {
        const ItemOut o = set == 0 ? oa : ob;
        const uint32_t* run_p = set == 0 ? run_pa : run_pb;
        if (o.bound == 0) continue;
        __syncthreads();
        const uint32_t n = min(run_p[nr], o.bound);
        uint32_t m2 = 32;
        while (m2 < n) m2 <<= 1;
        for (uint32_t i = threadIdx.x; i < m2; i += blockDim.x) {
            u64 key = ~0ull;
            if (i < n) {
                // last run with run_p[r] <= i (item counts are positive)
                const uint32_t r = lower_bound_u32(run_p, nr, i + 1) - 1;
                const uint32_t cnt = run_first[r + 1] - run_first[r], L = run_len[r];
                const uint32_t chunks = max(1u, (L + o.chunk - 1) / o.chunk);
                const uint32_t k = i - run_p[r];
                const uint32_t grp = k / chunks, ch = k % chunks;
                const uint32_t e0 = ch * o.chunk, e1 = min(L, e0 + o.chunk);
                o.item_list[i] = run_list[r];
                o.item_start[i] = run_first[r] + grp * o.qt;
                o.item_nq[i] = min(o.qt, cnt - grp * o.qt);
                o.item_e0[i] = e0;
                o.item_e1[i] = e1;
                key = ((u64)(0xffffffffu - (e1 - e0)) << 32) | i;
            }
            iv_keys[i] = key;
        }
        __syncthreads();
        cta_bitonic_sort(iv_keys, m2);
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) o.item_order[i] = (uint32_t)iv_keys[i];
    }
}

}  // namespace

bool invert_small_supported(size_t np, uint32_t c) {
    return np >= 1 && np <= kInvertSmallMaxPairs && c < (1u << 18);
}

void launch_invert_small(const uint32_t* probes, uint32_t np, uint32_t w, const float* D, uint32_t c,
                         const uint32_t* list_len, uint32_t* pair_sorted, uint32_t* list_cnt,
                         uint32_t* list_first, const SmallItems& a, const SmallItems& b, cudaStream_t s) {
    auto conv = [](const SmallItems& x) {
        return ItemOut{x.item_off, x.item_list, x.item_start, x.item_nq, x.item_e0, x.item_e1, x.item_order,
                       x.qt, x.chunk, x.bound};
    };
    if (a.bound > kInvertSmallMaxItems || b.bound > kInvertSmallMaxItems)
        throw ArgError("invert_small: item bound above the shared-memory sort");
    // sort buffer (pairs, then items) + the run table
    const size_t smem = kInvertSmallMaxPairs * sizeof(u64) + 5 * (kInvertSmallMaxPairs + 1) * sizeof(uint32_t);
    static_assert(kInvertSmallMaxItems <= kInvertSmallMaxPairs, "items are sorted in the pair buffer");
    set_max_smem((const void*)invert_small_kernel, smem);
    invert_small_kernel<<<1, IV_THREADS, smem, s>>>(probes, np, w, D, c, list_len, pair_sorted, list_cnt,
                                                    list_first, conv(a), conv(b));
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
