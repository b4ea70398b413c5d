// k_select.cu — threshold estimation, exact top-k' shortlist selection and the
// K5 re-ranker (ivf_rerank, ivf_index.hpp:79-81).
//
// Selection is exact under the reference total order (types.hpp:47-50): every
// candidate becomes a 64-bit key (dist bits << 32 | id) — distances are
// non-negative so the IEEE pattern orders like the value — and a CTA-wide
// MSB-first radix select finds the k'-th key; ties on distance are therefore
// broken by id exactly like TopK (topk.hpp:18-29).
#include <float.h>

#include <cstdlib>
#include <string>
#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int SEL_THREADS = 256;
constexpr int RADIX_BITS = 11;
constexpr int NBINS = 1 << RADIX_BITS;

__global__ void query_sizes_kernel(const uint32_t* __restrict__ probes, size_t nq, uint32_t w,
                                   const uint32_t* __restrict__ list_len, uint32_t stride,
                                   int tiered, uint32_t cap, uint64_t* __restrict__ n_entries,
                                   uint8_t* __restrict__ sampled, uint64_t* __restrict__ pair_samples,
                                   unsigned long long* __restrict__ grand_total, uint32_t max_rank) {
    // one warp per query: the probes' list lengths are dependent loads
    const size_t q = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= nq) return;
    unsigned long long tot = 0;
    for (uint32_t r = lane; r < w; r += 32) tot += list_len[probes[q * w + r]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    // every query whose candidates may not fit the buffer gets a threshold
    // (stride 1 samples every entry: still exact, only slower)
    const bool samp = tot > cap;
    unsigned long long ssum = 0;
    for (uint32_t r = lane; r < w; r += 32) {
        const uint32_t len = list_len[probes[q * w + r]];
        const uint32_t st = stride << tier_shift(sample_tier(r, w, tiered), w);
        const uint64_t ns = (samp && r < max_rank) ? (len + st - 1) / st : 0;
        pair_samples[q * w + r] = ns;
        ssum += ns;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    if (lane == 0) {
        n_entries[q] = tot;
        atomicAdd(grand_total, tot);
        sampled[q] = samp ? 1 : 0;
        atomicMax(grand_total + 1, ssum);
    }
}

// query_sizes_kernel + the exclusive scan of the pairs' sample counts in one
// CTA, for the few thousand pairs of a small batch (two launches and the
// library scan less on the serving path).  sample_off has nq * w + 1 entries.
constexpr int QS_THREADS = 1024;
__global__ __launch_bounds__(QS_THREADS) void query_sizes_small_kernel(
    const uint32_t* __restrict__ probes, uint32_t nq, uint32_t w, const uint32_t* __restrict__ list_len,
    uint32_t stride, int tiered, uint32_t cap, uint64_t* __restrict__ n_entries,
    uint8_t* __restrict__ sampled, uint64_t* __restrict__ sample_off,
    unsigned long long* __restrict__ grand_total, uint32_t max_rank) {
    extern __shared__ uint32_t qs_ns[];  // [nq * w] samples per pair
    __shared__ unsigned long long s_warp[QS_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t np = nq * w;
    for (uint32_t q = warp; q < nq; q += QS_THREADS / 32) {
        unsigned long long tot = 0;
        for (uint32_t r = lane; r < w; r += 32) tot += list_len[probes[q * w + r]];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        const bool samp = tot > cap;
        unsigned long long ssum = 0;
        for (uint32_t r = lane; r < w; r += 32) {
            const uint32_t len = list_len[probes[q * w + r]];
            const uint32_t st = stride << tier_shift(sample_tier(r, w, tiered), w);
            const uint32_t ns = (samp && r < max_rank) ? (len + st - 1) / st : 0u;
            qs_ns[q * w + r] = ns;
            ssum += ns;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
        if (lane == 0) {
            n_entries[q] = tot;
            atomicAdd(grand_total, tot);
            sampled[q] = samp ? 1 : 0;
            atomicMax(grand_total + 1, ssum);
        }
    }
    __syncthreads();
    // exclusive scan over the pairs: contiguous chunk per thread
    const uint32_t per = (np + QS_THREADS - 1) / QS_THREADS;
    const uint32_t i0 = min(np, threadIdx.x * per), i1 = min(np, i0 + per);
    unsigned long long sum = 0;
    for (uint32_t i = i0; i < i1; ++i) sum += qs_ns[i];
    unsigned long long incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long v = s_warp[lane];
        unsigned long long wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        s_warp[lane] = wi - v;
    }
    __syncthreads();
    unsigned long long run = s_warp[warp] + incl - sum;
    for (uint32_t i = i0; i < i1; ++i) {
        sample_off[i] = run;
        run += qs_ns[i];
    }
    if (i0 < np && i1 == np) sample_off[np] = run;  // the thread holding the last pair: the total
}

// Block-wide search of the bin holding the rank-th element (1-based) of a
// 2048-bin histogram; returns bin and rank within the bin.
__device__ void find_bin(const uint32_t* hist, uint32_t rank, uint32_t* s_bin, uint32_t* s_rank,
                         uint32_t* s_cnt = nullptr) {
    // one warp: lane l owns bins [64 l, 64 l + 64); it reads them rotated by
    // l so the 32 lanes hit 32 banks (unrotated, lane * 64 + b is one bank)
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        uint32_t sum = 0;
#pragma unroll 8
        for (int b = 0; b < 64; ++b) sum += hist[lane * 64 + ((b + lane) & 63)];
        uint32_t incl = sum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        const uint32_t excl = incl - sum;
        const bool mine = excl < rank && rank <= incl;
        const unsigned who = __ballot_sync(0xffffffffu, mine);
        if (who) {
            // the owner's 64 bins, two per lane, scanned by the whole warp
            const int owner = __ffs(who) - 1;
            const uint32_t base = __shfl_sync(0xffffffffu, excl, owner);
            const uint32_t h0 = hist[owner * 64 + 2 * lane], h1 = hist[owner * 64 + 2 * lane + 1];
            uint32_t inc2 = h0 + h1;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                uint32_t v = __shfl_up_sync(0xffffffffu, inc2, off);
                if (lane >= off) inc2 += v;
            }
            const uint32_t c0 = base + inc2 - h0 - h1;  // entries before this lane's two bins
            const bool hit0 = c0 < rank && rank <= c0 + h0;
            const bool hit1 = c0 + h0 < rank && rank <= c0 + h0 + h1;
            if (hit0 || hit1) {  // exactly one lane
                *s_bin = owner * 64 + 2 * lane + (hit0 ? 0 : 1);
                *s_rank = rank - (hit0 ? c0 : c0 + h0);
                if (s_cnt) *s_cnt = hit0 ? h0 : h1;
            }
        }
    }
}

// Applies f to every u32 of src[0, n) with 16-byte loads, 4 in flight per
// thread (the passes over the sample are latency bound).  src may start at any
// 4-byte alignment.
template <class F>
__device__ __forceinline__ void for_each_u32(const uint32_t* __restrict__ src, uint32_t n, F f) {
    const uint32_t head = min((uint32_t)((4 - ((reinterpret_cast<uintptr_t>(src) >> 2) & 3)) & 3), n);
    for (uint32_t i = threadIdx.x; i < head; i += blockDim.x) f(__ldg(src + i));
    const uint32_t nv = (n - head) / 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint32_t v = threadIdx.x;
    for (; v + 3 * blockDim.x < nv; v += 4 * blockDim.x) {
        uint4 x[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) x[t] = __ldg(s4 + v + t * blockDim.x);
#pragma unroll
        for (int t = 0; t < 4; ++t) { f(x[t].x); f(x[t].y); f(x[t].z); f(x[t].w); }
    }
    for (; v < nv; v += blockDim.x) {
        const uint4 x = __ldg(s4 + v);
        f(x.x); f(x.y); f(x.z); f(x.w);
    }
    for (uint32_t i = head + 4 * nv + threadIdx.x; i < n; i += blockDim.x) f(__ldg(src + i));
}

// tau_q: the distance at which the weighted count of samples reaches alpha*k'
// entries (each sample stands for its pair's stride, see sample_tier); +inf
// for queries scanned without sampling or with too few entries.  A weighted
// MSB-first radix select (11/11/10 bits): pass 1 histograms the top bits
// straight from global memory, the selected bin is compacted into shared
// memory when it fits stage_cap (with each element's tier), and the remaining
// passes run over that small set only.
constexpr int THR_THREADS_MAX = 1024;
__global__ __launch_bounds__(THR_THREADS_MAX, 1) void sample_threshold_kernel(
    const float* __restrict__ sample, const uint64_t* __restrict__ sample_off, uint32_t w,
    const uint8_t* __restrict__ sampled, float alpha_k, uint32_t stride, int tiered,
    uint32_t stage_cap, float* __restrict__ tau) {
    extern __shared__ uint32_t stage[];  // [stage_cap] values, then [stage_cap] tiers (bytes)
    uint8_t* stage_t = reinterpret_cast<uint8_t*>(stage + stage_cap);
    __shared__ uint32_t hist[NBINS];
    __shared__ uint32_t s_bin, s_rank, s_fill;
    __shared__ uint32_t s_mins[THR_THREADS_MAX];
    __shared__ unsigned long long s_seg[5];
    const size_t q = blockIdx.x;
    if (!sampled[q]) {
        if (threadIdx.x == 0) tau[q] = __int_as_float(0x7f800000);
        return;
    }
    // tier segments: contiguous ranges of the query's sample slots
    if (threadIdx.x == 0) {
        uint32_t r = 0;
        for (uint32_t t = 0; t < 4; ++t) {
            while (r < w && sample_tier(r, w, tiered) < t) ++r;
            s_seg[t] = sample_off[q * w + r];
        }
        s_seg[4] = sample_off[q * w + w];
    }
    __syncthreads();
    unsigned long long total = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) total += (s_seg[t + 1] - s_seg[t]) * ((unsigned long long)stride << tier_shift(t, w));
    const uint32_t rank = (uint32_t)max(1.0, ceil((double)alpha_k));
    if (total < rank) {
        if (threadIdx.x == 0) tau[q] = __int_as_float(0x7f800000);
        return;
    }
    const uint32_t* gsrc = reinterpret_cast<const uint32_t*>(sample);
    for (int b = threadIdx.x; b < NBINS; b += blockDim.x) hist[b] = 0;
    if (threadIdx.x == 0) s_fill = 0;
    __syncthreads();
    // The target rank sits in the far lower tail (~64-128 samples of 10^4-10^6),
    // and a histogram over all samples serialises its shared-memory atomics on
    // the two or three bins that hold nearly everything.  So first bound the
    // answer from above without atomics: each thread keeps the minimum of the
    // tier-0 samples it reads (tier 0 carries the smallest weight, `stride`);
    // the R0-th smallest of those minima, R0 = ceil(rank / stride), has at
    // least R0 tier-0 samples at or below it, i.e. weight >= rank.  Only the
    // samples <= that bound (a few hundred) are staged, and the exact weighted
    // select runs over the stage.  Same tau as the full radix select.
    const uint32_t n0 = (uint32_t)(s_seg[1] - s_seg[0]);
    const uint32_t R0 = (rank + stride - 1) / stride;
    bool staged = false;
    uint32_t cnt = 0, prefix = 0, r = rank;
    if (R0 <= blockDim.x / 2 && n0 >= 8 * blockDim.x) {
        uint32_t mn = 0xffffffffu;
        for_each_u32(gsrc + s_seg[0], n0, [&](uint32_t u) { mn = min(mn, u); });
        const uint32_t T0 = cta_tail_bound(mn, R0, s_mins);
        for (int t = 0; t < 4; ++t) {
            const uint32_t n = (uint32_t)(s_seg[t + 1] - s_seg[t]);
            if (n)
                for_each_u32(gsrc + s_seg[t], n, [&](uint32_t u) {
                    if (u <= T0) {
                        const uint32_t k = atomicAdd(&s_fill, 1u);
                        if (k < stage_cap) {
                            stage[k] = u;
                            stage_t[k] = (uint8_t)t;
                        }
                    }
                });
        }
        __syncthreads();
        cnt = s_fill;
        staged = cnt <= stage_cap;
        __syncthreads();
        if (!staged && threadIdx.x == 0) s_fill = 0;
        __syncthreads();
    }
    if (staged) {  // top 11 bits over the stage
        for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x)
            atomicAdd(&hist[stage[i] >> 21], stride << tier_shift(stage_t[i], w));
        __syncthreads();
        find_bin(hist, rank, &s_bin, &s_rank);
        __syncthreads();
        prefix = s_bin;
        r = s_rank;
    } else {
        for (int t = 0; t < 4; ++t) {
            const uint32_t wt = stride << tier_shift(t, w);
            const uint32_t n = (uint32_t)(s_seg[t + 1] - s_seg[t]);
            if (n) for_each_u32(gsrc + s_seg[t], n, [&](uint32_t u) { atomicAdd(&hist[u >> 21], wt); });
        }
        __syncthreads();
        find_bin(hist, rank, &s_bin, &s_rank);
        __syncthreads();
        prefix = s_bin;
        r = s_rank;
        // optimistic compaction of the selected bin (with each element's tier);
        // an overfull stage falls back to reading global memory
        {
            const uint32_t top = prefix;
            for (int t = 0; t < 4; ++t) {
                const uint32_t n = (uint32_t)(s_seg[t + 1] - s_seg[t]);
                if (n)
                    for_each_u32(gsrc + s_seg[t], n, [&](uint32_t u) {
                        if ((u >> 21) == top) {
                            const uint32_t k = atomicAdd(&s_fill, 1u);
                            if (k < stage_cap) {
                                stage[k] = u;
                                stage_t[k] = (uint8_t)t;
                            }
                        }
                    });
            }
        }
        __syncthreads();
        cnt = s_fill;
        staged = cnt <= stage_cap;
        if (cnt == 1) {  // the bin holds a single value: it is the answer
            if (threadIdx.x == 0) tau[q] = __uint_as_float(stage[0]);
            return;
        }
    }
    const int shifts[2] = {10, 0};
    const int widths[2] = {11, 10};
    for (int pass = 0; pass < 2; ++pass) {
        for (int b = threadIdx.x; b < NBINS; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const int sh = shifts[pass], wd = widths[pass];
        const uint32_t msk = (1u << wd) - 1u;
        auto add = [&](uint32_t u, uint32_t t) {
            if ((u >> (sh + wd)) == prefix) atomicAdd(&hist[(u >> sh) & msk], stride << tier_shift(t, w));
        };
        if (staged) {
            for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) add(stage[i], stage_t[i]);
        } else {
            for (int t = 0; t < 4; ++t)
                for (uint64_t i = s_seg[t] + threadIdx.x; i < s_seg[t + 1]; i += blockDim.x) add(gsrc[i], t);
        }
        __syncthreads();
        find_bin(hist, r, &s_bin, &s_rank);
        __syncthreads();
        prefix = (prefix << wd) | s_bin;
        r = s_rank;
        __syncthreads();
    }
    if (threadIdx.x == 0) tau[q] = __uint_as_float(prefix);
}

__device__ void bitonic_sort_kv(u64* keys, uint32_t* vals, uint32_t n2) {
    for (uint32_t k = 2; k <= n2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (j - 1));
                const uint32_t hi = lo + j;
                const bool up = (lo & k) == 0;
                const u64 a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                    if (vals) {
                        const uint32_t t = vals[lo];
                        vals[lo] = vals[hi];
                        vals[hi] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// Exact k'-smallest (dist, id) keys among a query's candidates.
__global__ __launch_bounds__(SEL_THREADS, 4) void select_topk_kernel(
    const float* __restrict__ cand_dist, const uint32_t* __restrict__ cand_pos,
    const uint32_t* __restrict__ cand_cnt, uint32_t cap, uint32_t slots,
    const uint32_t* __restrict__ ids, uint32_t kprime, int sorted, u64* __restrict__ sl_key,
    uint32_t* __restrict__ sl_pos, uint32_t* __restrict__ sl_cnt) {
    extern __shared__ u64 skeys[];
    __shared__ uint32_t hist[NBINS];
    __shared__ uint32_t s_bin, s_rank, s_out, s_bincnt;
    __shared__ u64 s_kth;
    __shared__ u64 s_mm[2 * SEL_THREADS / 32];
    const size_t q = blockIdx.x;
    const uint32_t n = min(cand_cnt[q], cap);
    uint32_t* spos = reinterpret_cast<uint32_t*>(skeys + slots);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t p = cand_pos[q * cap + i];
        skeys[i] = nb_key(cand_dist[q * cap + i], ids[p]);
        spos[i] = p;
    }
    if (threadIdx.x == 0) s_out = 0;
    __syncthreads();
    u64 kth = ~0ull;
    if (n > kprime) {
        // the candidates' distances share their leading bits (all are <= tau and
        // >= the nearest entry): start below the common prefix of the smallest
        // and the largest key, or the first pass would put every atomic on one bin
        u64 kmin = ~0ull, kmax = 0ull;
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            kmin = min(kmin, skeys[i]);
            kmax = max(kmax, skeys[i]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
            kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
        }
        if ((threadIdx.x & 31) == 0) {
            s_mm[2 * (threadIdx.x >> 5)] = kmin;
            s_mm[2 * (threadIdx.x >> 5) + 1] = kmax;
        }
        __syncthreads();
        for (uint32_t i = 0; i < blockDim.x / 32; ++i) {
            kmin = min(kmin, s_mm[2 * i]);
            kmax = max(kmax, s_mm[2 * i + 1]);
        }
        int consumed = kmin == kmax ? 0 : __clzll((long long)(kmin ^ kmax));
        u64 prefix = consumed ? kmin >> (64 - consumed) : 0ull;
        uint32_t r = kprime;
        while (consumed < 64) {
            const int wd = min(RADIX_BITS, 64 - consumed);
            const int sh = 64 - consumed - wd;
            for (int b = threadIdx.x; b < NBINS; b += blockDim.x) hist[b] = 0;
            __syncthreads();
            const u64 msk = (1ull << wd) - 1ull;
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
                const u64 k = skeys[i];
                const bool match = consumed == 0 ? true : ((k >> (sh + wd)) == prefix);
                if (match) atomicAdd(&hist[(uint32_t)((k >> sh) & msk)], 1u);
            }
            __syncthreads();
            find_bin(hist, r, &s_bin, &s_rank, &s_bincnt);
            __syncthreads();
            prefix = (prefix << wd) | s_bin;
            r = s_rank;
            consumed += wd;
            if (s_bincnt == 1 && consumed < 64) {
                // the rank-th key is the only one left with this prefix
                const int rem = 64 - consumed;
                for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
                    if ((skeys[i] >> rem) == prefix) s_kth = skeys[i];
                __syncthreads();
                prefix = s_kth;
                break;
            }
            __syncthreads();
        }
        kth = prefix;
    }
    const uint32_t cnt = min(n, kprime);
    // compaction of the keys <= kth (exactly cnt of them: keys are unique)
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const u64 k = skeys[i];
        if (k <= kth) {
            const uint32_t o = atomicAdd(&s_out, 1u);
            sl_key[q * kprime + o] = k;
            sl_pos[q * kprime + o] = spos[i];
        }
    }
    if (threadIdx.x == 0) sl_cnt[q] = cnt;
    if (!sorted) return;
    __syncthreads();
    uint32_t n2 = 1;
    while (n2 < cnt) n2 <<= 1;
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
        skeys[i] = i < cnt ? sl_key[q * kprime + i] : ~0ull;
        spos[i] = i < cnt ? sl_pos[q * kprime + i] : 0u;
    }
    __syncthreads();
    bitonic_sort_kv(skeys, spos, n2);
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        sl_key[q * kprime + i] = skeys[i];
        sl_pos[q * kprime + i] = spos[i];
    }
}

// Radix select over 32-bit keys produced by `key(i)` for the entries `pred(i)`
// accepts; returns the rank-th smallest key and its rank among equal keys.
template <class KeyF, class PredF>
__device__ void radix_select32(uint32_t n, uint32_t rank, KeyF key, PredF pred, uint32_t* hist,
                               uint32_t* s_bin, uint32_t* s_rank, uint32_t* s_cnt, uint32_t* s_val,
                               uint32_t& out_key, uint32_t& out_rank, uint32_t& out_cnt) {
    uint32_t prefix = 0, r = rank, cnt = 0;
    const int shifts[3] = {21, 10, 0};
    const int widths[3] = {11, 11, 10};
    for (int pass = 0; pass < 3; ++pass) {
        for (int b = threadIdx.x; b < NBINS; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const int sh = shifts[pass], wd = widths[pass];
        const uint32_t msk = (1u << wd) - 1u;
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            if (!pred(i)) continue;
            const uint32_t u = key(i);
            if (pass == 0 || (u >> (sh + wd)) == prefix) atomicAdd(&hist[(u >> sh) & msk], 1u);
        }
        __syncthreads();
        find_bin(hist, r, s_bin, s_rank, s_cnt);
        __syncthreads();
        prefix = (prefix << wd) | *s_bin;
        r = *s_rank;
        cnt = *s_cnt;
        if (cnt == 1 && sh > 0) {  // a single key left under this prefix
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
                if (pred(i) && (key(i) >> sh) == prefix) *s_val = key(i);
            __syncthreads();
            prefix = *s_val;
            break;
        }
        __syncthreads();
    }
    out_key = prefix;
    out_rank = r;
    out_cnt = cnt;
}

// Exact top-k' for candidate sets too large for shared memory (k' up to 1e4):
// radix select on the distance bits streamed from global memory, then the
// boundary distance's ties resolved by a second radix select on ids; ids are
// gathered only for the selected entries and the ties.
__global__ __launch_bounds__(SEL_THREADS, 4) void select_large_kernel(
    const float* __restrict__ cand_dist, const uint32_t* __restrict__ cand_pos,
    const uint32_t* __restrict__ cand_cnt, uint32_t cap, const uint32_t* __restrict__ ids,
    uint32_t kprime, u64* __restrict__ sl_key, uint32_t* __restrict__ sl_pos,
    uint32_t* __restrict__ sl_cnt) {
    __shared__ uint32_t hist[NBINS];
    __shared__ uint32_t s_bin, s_rank, s_cnt, s_val, s_out;
    const size_t q = blockIdx.x;
    const uint32_t n = min(cand_cnt[q], cap);
    const uint32_t* db = reinterpret_cast<const uint32_t*>(cand_dist) + q * cap;
    const uint32_t* pb = cand_pos + q * cap;
    if (threadIdx.x == 0) s_out = 0;
    uint32_t dstar = 0xffffffffu, r = 0, ceq = 0;
    if (n > kprime) {
        radix_select32(n, kprime, [&](uint32_t i) { return db[i]; }, [](uint32_t) { return true; },
                       hist, &s_bin, &s_rank, &s_cnt, &s_val, dstar, r, ceq);
    }
    __syncthreads();
    // entries strictly below the boundary distance are all in
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t u = db[i];
        if (n <= kprime || u < dstar) {
            const uint32_t p = pb[i];
            const uint32_t o = atomicAdd(&s_out, 1u);
            sl_key[q * kprime + o] = ((u64)u << 32) | ids[p];
            sl_pos[q * kprime + o] = p;
        }
    }
    if (n > kprime) {
        // r of the entries at exactly dstar, smallest ids first (types.hpp:47-50)
        uint32_t idstar = 0xffffffffu, r2 = 0, c2 = 0;
        const bool all_ties = (r == ceq);
        if (!all_ties) {
            radix_select32(n, r, [&](uint32_t i) { return ids[pb[i]]; },
                           [&](uint32_t i) { return db[i] == dstar; }, hist, &s_bin, &s_rank,
                           &s_cnt, &s_val, idstar, r2, c2);
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            if (db[i] != dstar) continue;
            const uint32_t p = pb[i];
            const uint32_t id = ids[p];
            if (all_ties || id <= idstar) {
                const uint32_t o = atomicAdd(&s_out, 1u);
                sl_key[q * kprime + o] = ((u64)dstar << 32) | id;
                sl_pos[q * kprime + o] = p;
            }
        }
    }
    if (threadIdx.x == 0) sl_cnt[q] = min(n, kprime);
}

// In-place ascending sort of each query's selected (key, pos) rows.
__global__ __launch_bounds__(256) void sort_rows_kernel(u64* __restrict__ sl_key,
                                                        uint32_t* __restrict__ sl_pos,
                                                        const uint32_t* __restrict__ sl_cnt,
                                                        uint32_t kprime) {
    extern __shared__ u64 rkeys2[];
    const size_t q = blockIdx.x;
    const uint32_t cnt = sl_cnt[q];
    uint32_t n2 = 1;
    while (n2 < cnt) n2 <<= 1;
    uint32_t* rpos = reinterpret_cast<uint32_t*>(rkeys2 + n2);
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
        rkeys2[i] = i < cnt ? sl_key[q * kprime + i] : ~0ull;
        rpos[i] = i < cnt ? sl_pos[q * kprime + i] : 0u;
    }
    __syncthreads();
    bitonic_sort_kv(rkeys2, rpos, n2);
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        sl_key[q * kprime + i] = rkeys2[i];
        sl_pos[q * kprime + i] = rpos[i];
    }
}

// l2_sq(x, yhat) with yhat[t] = (C_l[t] + B(code)[t]) + R(rcode)[t].
template <bool FAST>
__device__ __forceinline__ float rerank_dist(const float* __restrict__ xs, uint32_t d,
                                             const float* __restrict__ crow,
                                             const float* __restrict__ books, const uint8_t* code,
                                             uint32_t ds, const float* __restrict__ rbooks,
                                             const uint8_t* rcode, uint32_t dsr, uint32_t ks,
                                             u64 nz) {
    if constexpr (FAST) {
        u64 s01 = 0, s23 = 0;
#pragma unroll 8
        for (uint32_t t = 0; t < d; t += 4) {
            const uint32_t jj = t / ds, jr = t / dsr;
            const float4 c = __ldg(reinterpret_cast<const float4*>(crow + t));
            const float4 b = __ldg(reinterpret_cast<const float4*>(
                books + ((size_t)jj * ks + code[jj]) * ds + (t - jj * ds)));
            const float4 rr = __ldg(reinterpret_cast<const float4*>(
                rbooks + ((size_t)jr * ks + rcode[jr]) * dsr + (t - jr * dsr)));
            const float y0 = __fadd_rn(__fadd_rn(c.x, b.x), rr.x);
            const float y1 = __fadd_rn(__fadd_rn(c.y, b.y), rr.y);
            const float y2 = __fadd_rn(__fadd_rn(c.z, b.z), rr.z);
            const float y3 = __fadd_rn(__fadd_rn(c.w, b.w), rr.w);
            const float4 x = *reinterpret_cast<const float4*>(xs + t);
            s01 = acc_sq2(s01, pk2(x.x, x.y), pk2(y0, y1), nz);
            s23 = acc_sq2(s23, pk2(x.z, x.w), pk2(y2, y3), nz);
        }
        return __fadd_rn(__fadd_rn(lo2(s01), hi2(s01)), __fadd_rn(lo2(s23), hi2(s23)));
    } else {
        float s[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t full = d & ~3u;
        for (uint32_t t = 0; t < d; ++t) {
            const uint32_t jj = t / ds, jr = t / dsr;
            const float rec1 = __fadd_rn(crow[t], books[((size_t)jj * ks + code[jj]) * ds + (t - jj * ds)]);
            const float yh = __fadd_rn(rec1, rbooks[((size_t)jr * ks + rcode[jr]) * dsr + (t - jr * dsr)]);
            const float df = __fsub_rn(xs[t], yh);
            const int slot = t < full ? (int)(t & 3) : (int)(t - full);
            s[slot] = __fadd_rn(s[slot], __fmul_rn(df, df));
        }
        return __fadd_rn(__fadd_rn(s[0], s[1]), __fadd_rn(s[2], s[3]));
    }
}

template <bool FAST>
__global__ __launch_bounds__(256, 3) void rerank_kernel(
    const u64* __restrict__ sl_key, const uint32_t* __restrict__ sl_pos,
    const uint32_t* __restrict__ sl_cnt, uint32_t sl_stride, const float* __restrict__ xq, uint32_t d,
    const uint16_t* __restrict__ block_list, const float* __restrict__ coarse,
    const uint8_t* __restrict__ codes, const float* __restrict__ books, uint32_t m,
    const uint8_t* __restrict__ rcodes, const float* __restrict__ rbooks, uint32_t mprime,
    uint32_t ks, uint32_t k, uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
    uint32_t* __restrict__ out_cnt, u64 nz) {
    extern __shared__ u64 rkeys[];
    float* xs = reinterpret_cast<float*>(rkeys);  // first d floats (rounded up to 16 B)
    const uint32_t xwords = ((d + 3) & ~3u) / 2;  // u64 words taken by xs
    u64* keys = rkeys + xwords;
    const size_t q = blockIdx.x;
    const uint32_t n = sl_cnt[q];
    for (uint32_t t = threadIdx.x; t < d; t += blockDim.x) xs[t] = xq[q * d + t];
    uint32_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    __syncthreads();
    const uint32_t ds = d / m, dsr = d / mprime;
    for (uint32_t i = n + threadIdx.x; i < n2; i += blockDim.x) keys[i] = ~0ull;
    // two candidates per thread in flight: their gathers (position, list
    // search, code bytes, centroid rows) overlap
    for (uint32_t i0 = threadIdx.x; i0 < n; i0 += 2 * blockDim.x) {
        const uint32_t i1 = i0 + blockDim.x;
        const bool has1 = i1 < n;
        const uint32_t p0 = sl_pos[q * sl_stride + i0];
        const uint32_t p1 = has1 ? sl_pos[q * sl_stride + i1] : p0;
        const uint32_t id0 = key_id(sl_key[q * sl_stride + i0]);
        const uint32_t id1 = has1 ? key_id(sl_key[q * sl_stride + i1]) : 0u;
        const uint32_t l0 = block_list[p0 >> 4];
        const uint32_t l1 = block_list[p1 >> 4];
        const float d0 = rerank_dist<FAST>(xs, d, coarse + (size_t)l0 * d, books, codes + (size_t)p0 * m, ds,
                                           rbooks, rcodes + (size_t)p0 * mprime, dsr, ks, nz);
        const float d1 = rerank_dist<FAST>(xs, d, coarse + (size_t)l1 * d, books, codes + (size_t)p1 * m, ds,
                                           rbooks, rcodes + (size_t)p1 * mprime, dsr, ks, nz);
        keys[i0] = nb_key(d0, id0);
        if (has1) keys[i1] = nb_key(d1, id1);
    }
    __syncthreads();
    bitonic_sort_kv(keys, nullptr, n2);
    const uint32_t cnt = min(n, k);
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        const bool live = i < cnt;
        out_ids[q * k + i] = live ? key_id(keys[i]) : 0xffffffffu;
        out_dists[q * k + i] = live ? key_dist(keys[i]) : __int_as_float(0x7f800000);
    }
    if (threadIdx.x == 0) out_cnt[q] = cnt;
}


// K5b: top-k of (rdist, rid) rows under (dist, id): radix select on the
// distance bits (rows streamed from L2), ties at the boundary broken by id,
// then the k winners sorted in shared memory.
__global__ __launch_bounds__(SEL_THREADS) void rerank_topk_kernel(
    const float* __restrict__ rdist, const uint32_t* __restrict__ rid,
    const uint32_t* __restrict__ cnt_in, uint32_t stride, uint32_t k, uint32_t k2,
    uint32_t* __restrict__ out_ids, float* __restrict__ out_dists, uint32_t* __restrict__ out_cnt) {
    extern __shared__ u64 tk_keys[];
    __shared__ uint32_t hist[NBINS];
    __shared__ uint32_t s_bin, s_rank, s_cnt, s_val, s_out;
    const size_t q = blockIdx.x;
    const uint32_t n = cnt_in[q];
    const uint32_t* db = reinterpret_cast<const uint32_t*>(rdist) + q * stride;
    const uint32_t* ib = rid + q * stride;
    for (uint32_t i = threadIdx.x; i < k2; i += blockDim.x) tk_keys[i] = ~0ull;
    if (threadIdx.x == 0) s_out = 0;
    __syncthreads();
    uint32_t dstar = 0xffffffffu, r = 0, ceq = 0;
    if (n > k)
        radix_select32(n, k, [&](uint32_t i) { return db[i]; }, [](uint32_t) { return true; }, hist,
                       &s_bin, &s_rank, &s_cnt, &s_val, dstar, r, ceq);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t u = db[i];
        if (n <= k || u < dstar) tk_keys[atomicAdd(&s_out, 1u)] = ((u64)u << 32) | ib[i];
    }
    if (n > k) {
        uint32_t idstar = 0xffffffffu, r2 = 0, c2 = 0;
        const bool all_ties = (r == ceq);
        if (!all_ties)
            radix_select32(n, r, [&](uint32_t i) { return ib[i]; },
                           [&](uint32_t i) { return db[i] == dstar; }, hist, &s_bin, &s_rank, &s_cnt,
                           &s_val, idstar, r2, c2);
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
            if (db[i] == dstar && (all_ties || ib[i] <= idstar))
                tk_keys[atomicAdd(&s_out, 1u)] = ((u64)dstar << 32) | ib[i];
    }
    __syncthreads();
    bitonic_sort_kv(tk_keys, nullptr, k2);
    const uint32_t cnt = min(n, k);
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        const bool live = i < cnt;
        out_ids[q * k + i] = live ? key_id(tk_keys[i]) : 0xffffffffu;
        out_dists[q * k + i] = live ? key_dist(tk_keys[i]) : __int_as_float(0x7f800000);
    }
    if (threadIdx.x == 0) out_cnt[q] = cnt;
}

// K7: merge of per-shard ranked lists (all-gathered [parts][nq][width]) into
// the global top-k under (dist, id) — one CTA per query, bitonic in smem.
__global__ __launch_bounds__(256) void merge_topk_kernel(
    const uint32_t* __restrict__ ids, const float* __restrict__ dists,
    const uint32_t* __restrict__ counts, size_t nq, uint32_t parts, uint32_t width, size_t ps,
    size_t cs, uint32_t k, uint32_t n2, uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
    uint32_t* __restrict__ out_cnt) {
    extern __shared__ u64 mkeys[];
    const size_t q = blockIdx.x;
    __shared__ uint32_t s_total;
    if (threadIdx.x == 0) s_total = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
        u64 key = ~0ull;
        if (i < parts * width) {
            const uint32_t p = i / width, j = i % width;
            const size_t e = p * ps + q * width + j;
            if (j < counts[p * cs + q]) {
                key = nb_key(dists[e], ids[e]);
                atomicAdd(&s_total, 1u);
            }
        }
        mkeys[i] = key;
    }
    __syncthreads();
    bitonic_sort_kv(mkeys, nullptr, n2);
    const uint32_t cnt = min(s_total, k);
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        const bool live = i < cnt;
        out_ids[q * k + i] = live ? key_id(mkeys[i]) : 0xffffffffu;
        out_dists[q * k + i] = live ? key_dist(mkeys[i]) : __int_as_float(0x7f800000);
    }
    if (threadIdx.x == 0) out_cnt[q] = cnt;
}

// Large K7 inputs (parts * width above the smem bitonic): pack each query's
// valid entries of all parts contiguously for select_large_kernel.
__global__ void merge_pack_kernel(const uint32_t* __restrict__ ids, const float* __restrict__ dists,
                                  const uint32_t* __restrict__ counts, size_t nq, uint32_t parts,
                                  uint32_t width, size_t ps, size_t cs, float* __restrict__ cd, uint32_t* __restrict__ cp,
                                  uint32_t* __restrict__ cid, uint32_t* __restrict__ ccnt) {
    const size_t q = blockIdx.x;
    const size_t cap = (size_t)parts * width;
    uint32_t off = 0;
    for (uint32_t p = 0; p < parts; ++p) {
        const size_t row = p * ps + q * width;
        const uint32_t c = min(counts[p * cs + q], width);
        for (uint32_t j = threadIdx.x; j < c; j += blockDim.x) {
            const size_t o = q * cap + off + j;
            cd[o] = dists[row + j];
            cid[o] = ids[row + j];
            cp[o] = (uint32_t)o;
        }
        off += c;
    }
    if (threadIdx.x == 0) ccnt[q] = off;
}

__global__ void unpack_keys_kernel(const u64* __restrict__ keys, const uint32_t* __restrict__ cnt,
                                   size_t nq, uint32_t stride, uint32_t* __restrict__ ids,
                                   float* __restrict__ dists) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nq * stride) return;
    size_t q = idx / stride;
    uint32_t i = (uint32_t)(idx % stride);
    if (i < cnt[q]) {
        ids[idx] = key_id(keys[idx]);
        dists[idx] = key_dist(keys[idx]);
    } else {  // rows shorter than the width: (UINT32_MAX, +inf) sentinels
        ids[idx] = 0xffffffffu;
        dists[idx] = __int_as_float(0x7f800000);
    }
}

void set_smem(const void* f, size_t bytes) {
    set_max_smem((const void*)f, (size_t)((int)bytes));
}

}  // namespace

void launch_query_sizes(const uint32_t* probes, size_t nq, uint32_t w, const uint32_t* list_len,
                        uint32_t stride, int tiered, uint32_t cap, uint64_t* nq_entries,
                        uint8_t* query_sampled, uint64_t* pair_samples, uint64_t* grand_total,
                        cudaStream_t s, uint32_t max_rank) {
    if (nq == 0) return;
    query_sizes_kernel<<<(unsigned)((nq + 3) / 4), 128, 0, s>>>(
        probes, nq, w, list_len, stride, tiered, cap, nq_entries, query_sampled, pair_samples,
        reinterpret_cast<unsigned long long*>(grand_total), max_rank);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

bool launch_query_sizes_small(const uint32_t* probes, size_t nq, uint32_t w, const uint32_t* list_len,
                              uint32_t stride, int tiered, uint32_t cap, uint64_t* nq_entries,
                              uint8_t* query_sampled, uint64_t* sample_off, uint64_t* grand_total,
                              cudaStream_t s, uint32_t max_rank) {
    const size_t np = nq * (size_t)w;
    if (nq == 0 || np > 8192) return false;
    query_sizes_small_kernel<<<1, QS_THREADS, np * sizeof(uint32_t), s>>>(
        probes, (uint32_t)nq, w, list_len, stride, tiered, cap, nq_entries, query_sampled, sample_off,
        reinterpret_cast<unsigned long long*>(grand_total), max_rank);
    PQRR_LAUNCH_CHECK();
    count_launch();
    return true;
}

void launch_sample_threshold(const float* sample_dist, const uint64_t* sample_off, uint32_t w,
                             size_t nq, const uint8_t* query_sampled, float alpha_k,
                             uint32_t stride, int tiered, uint32_t max_samples, float* tau,
                             cudaStream_t s) {
    if (nq == 0) return;
    // warp per query when the batch fills the GPU with warps; a small batch
    // (C5 latency points) spreads each query's samples over a CTA instead
    if (nq >= (size_t)2 * sm_count() * 8) {
        launch_threshold_warp(sample_dist, sample_off, w, nq, query_sampled, alpha_k, stride, tiered, tau, s);
        return;
    }
    const uint32_t stage_cap = std::min<uint32_t>(max_samples, 8 * 1024);
    const size_t smem = (size_t)std::max<uint32_t>(stage_cap, 1) * (sizeof(uint32_t) + 1) + 16;
    set_smem((const void*)sample_threshold_kernel, smem);
    // few queries: 1024 threads each (the passes over a query's samples are latency bound)
    const int thr = nq <= (size_t)2 * sm_count() ? THR_THREADS_MAX : SEL_THREADS;
    sample_threshold_kernel<<<(unsigned)nq, thr, smem, s>>>(
        sample_dist, sample_off, w, query_sampled, alpha_k, stride, tiered, stage_cap, tau);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_select_topk(const float* cand_dist, const uint32_t* cand_pos, const uint32_t* cand_cnt,
                        uint32_t cap, uint32_t max_n, size_t nq, const uint32_t* ids,
                        uint32_t kprime, bool sorted, uint64_t* sl_key, uint32_t* sl_pos,
                        uint32_t* sl_cnt, cudaStream_t s,
                        const uint32_t* cand_mm, bool need_ids) {
    if (nq == 0) return;
    if (!sorted) {
        // unsorted shortlist (re-ranked next): warp per query; a batch too
        // small to fill the GPU with warps gives each query a CTA (C5 batch 1:
        // 0.052 -> 0.012 ms)
        const bool cta = nq < (size_t)2 * sm_count() && need_ids && (size_t)cap * 12 <= 96 * 1024;
        if (!cta) {
            launch_select_warp(cand_dist, cand_pos, cand_cnt, cap, nq, ids, kprime, sl_key, sl_pos, sl_cnt, s,
                               cand_mm, need_ids);
            return;
        }
        max_n = cap;
    }
    uint32_t kp2 = 1;
    while (kp2 < kprime) kp2 <<= 1;
    // smem sized by the largest candidate set of this batch (max_n <= cap)
    const uint32_t slots = std::max(std::max(std::min(max_n, cap), 1u), sorted ? kp2 : 0u);
    const size_t smem = (size_t)slots * (sizeof(u64) + sizeof(uint32_t));
    if (smem > 96 * 1024) {
        // large k' (C4: 1e4): candidates stay in global memory
        select_large_kernel<<<(unsigned)nq, SEL_THREADS, 0, s>>>(
            cand_dist, cand_pos, cand_cnt, cap, ids, kprime, reinterpret_cast<u64*>(sl_key), sl_pos,
            sl_cnt);
        PQRR_LAUNCH_CHECK();
        count_launch();
        if (sorted) {
            const size_t ssm = (size_t)kp2 * (sizeof(u64) + sizeof(uint32_t));
            if (ssm > 200 * 1024) throw ArgError("kprime too large for a sorted device shortlist");
            set_smem((const void*)sort_rows_kernel, ssm);
            sort_rows_kernel<<<(unsigned)nq, 256, ssm, s>>>(reinterpret_cast<u64*>(sl_key), sl_pos,
                                                           sl_cnt, kprime);
            PQRR_LAUNCH_CHECK();
            count_launch();
        }
        return;
    }
    set_smem((const void*)select_topk_kernel, smem);
    select_topk_kernel<<<(unsigned)nq, SEL_THREADS, smem, s>>>(
        cand_dist, cand_pos, cand_cnt, cap, slots, ids, kprime, sorted ? 1 : 0,
        reinterpret_cast<u64*>(sl_key), sl_pos, sl_cnt);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_rerank(const uint64_t* sl_key, const uint32_t* sl_pos, const uint32_t* sl_cnt,
                   uint32_t sl_stride, size_t nq, const float* xq, uint32_t d,
                   const uint16_t* block_list, const float* coarse,
                   const uint8_t* codes, const float* books, uint32_t m, const uint8_t* rcodes,
                   const float* rbooks, uint32_t mprime, uint32_t ks, uint32_t k,
                   uint32_t* out_ids, float* out_dists, uint32_t* out_cnt, cudaStream_t s,
                   cudaEvent_t ev_dist_done, const uint32_t* ids_for_keys) {
    if (nq == 0) return;
    uint32_t n2 = 1;
    while (n2 < sl_stride) n2 <<= 1;
    uint32_t k2 = 1;
    while (k2 < k) k2 <<= 1;
    // every BASELINE shape (d = 128, m = 8, ks = 256, m' in {8, 16, 32}):
    // refined distances on CTA pairs (k_rerank.cu) + per-query top-k; other
    // shapes: CTA per query
    if (rerank_pair_supported(d, m, ks, mprime) && (size_t)k2 * 8 <= 200 * 1024) {
        const size_t tot = nq * (size_t)sl_stride;
        float* rd = nullptr;
        uint32_t* ri = nullptr;
        PQRR_CUDA(cudaMallocAsync(&rd, tot * sizeof(float), s));
        PQRR_CUDA(cudaMallocAsync(&ri, tot * sizeof(uint32_t), s));
        launch_rerank_pair(sl_key, sl_pos, sl_cnt, sl_stride, nq, xq, block_list, coarse, codes, books,
                           rcodes, rbooks, mprime, rd, ri, s, ids_for_keys);
        if (ev_dist_done) PQRR_CUDA(cudaEventRecord(ev_dist_done, s));
        // (a batch too small to fill the GPU with warps gives each query a CTA)
        if (nq < (size_t)2 * sm_count() ||
            !launch_rerank_topk_warp(rd, ri, sl_cnt, sl_stride, nq, k, out_ids, out_dists, out_cnt, s)) {
            set_smem((const void*)rerank_topk_kernel, (size_t)k2 * 8);
            rerank_topk_kernel<<<(unsigned)nq, SEL_THREADS, (size_t)k2 * 8, s>>>(
                rd, ri, sl_cnt, sl_stride, k, k2, out_ids, out_dists, out_cnt);
            PQRR_LAUNCH_CHECK();
            count_launch();
        }
        PQRR_CUDA(cudaFreeAsync(rd, s));
        PQRR_CUDA(cudaFreeAsync(ri, s));
        return;
    }
    const size_t smem = ((d + 3) & ~3u) * sizeof(float) + (size_t)n2 * sizeof(u64);
    if (smem > 200 * 1024) throw ArgError("shortlist too large for the device re-ranker");
    const bool fast = d % 4 == 0 && (d / m) % 4 == 0 && (d / mprime) % 4 == 0;
    auto go = [&](auto kern) {
        set_smem((const void*)kern, smem);
        kern<<<(unsigned)nq, 256, smem, s>>>(
            reinterpret_cast<const u64*>(sl_key), sl_pos, sl_cnt, sl_stride, xq, d, block_list,
            coarse, codes, books, m, rcodes, rbooks, mprime, ks, k, out_ids, out_dists,
            out_cnt, kNegZero2);
    };
    if (fast) go(rerank_kernel<true>);
    else go(rerank_kernel<false>);
    PQRR_LAUNCH_CHECK();
    count_launch();
    if (ev_dist_done) PQRR_CUDA(cudaEventRecord(ev_dist_done, s));
}

void launch_merge_topk(const uint32_t* ids, const float* dists, const uint32_t* counts, size_t nq,
                       uint32_t parts, uint32_t width, uint32_t k, uint32_t* out_ids,
                       float* out_dists, uint32_t* out_cnt, cudaStream_t s, size_t ps, size_t cs) {
    if (nq == 0) return;
    if (!ps) ps = nq * width;  // [parts, nq, width] + [parts, nq] by default
    if (!cs) cs = nq;
    uint32_t n2 = 1;
    while (n2 < parts * width) n2 <<= 1;
    const size_t smem = (size_t)n2 * sizeof(u64);
    if (smem > 200 * 1024) {
        // exact multi-shard mode merges k'-wide shortlists (C4: 8 x 1e4): pack,
        // radix-select from global memory (select_large_kernel), sort the k rows
        const size_t cap = (size_t)parts * width;
        if (nq * cap > 0xffffffffull) throw ArgError("nq * parts * width too large for the device merge");
        uint32_t k2 = 1;
        while (k2 < k) k2 <<= 1;
        const size_t ssm = (size_t)k2 * (sizeof(u64) + sizeof(uint32_t));
        if (ssm > 200 * 1024) throw ArgError("k too large for the device merge");
        float* cd = nullptr;
        uint32_t *cp = nullptr, *cid = nullptr, *ccnt = nullptr, *spos = nullptr;
        u64* skey = nullptr;
        PQRR_CUDA(cudaMallocAsync(&cd, nq * cap * 4, s));
        PQRR_CUDA(cudaMallocAsync(&cp, nq * cap * 4, s));
        PQRR_CUDA(cudaMallocAsync(&cid, nq * cap * 4, s));
        PQRR_CUDA(cudaMallocAsync(&ccnt, nq * 4, s));
        PQRR_CUDA(cudaMallocAsync(&skey, nq * k * 8, s));
        PQRR_CUDA(cudaMallocAsync(&spos, nq * k * 4, s));
        merge_pack_kernel<<<(unsigned)nq, 256, 0, s>>>(ids, dists, counts, nq, parts, width, ps, cs, cd, cp,
                                                       cid, ccnt);
        PQRR_LAUNCH_CHECK();
        count_launch();
        select_large_kernel<<<(unsigned)nq, SEL_THREADS, 0, s>>>(cd, cp, ccnt, (uint32_t)cap, cid, k,
                                                                 skey, spos, out_cnt);
        PQRR_LAUNCH_CHECK();
        count_launch();
        set_smem((const void*)sort_rows_kernel, ssm);
        sort_rows_kernel<<<(unsigned)nq, 256, ssm, s>>>(skey, spos, out_cnt, k);
        PQRR_LAUNCH_CHECK();
        count_launch();
        launch_unpack_keys(reinterpret_cast<const uint64_t*>(skey), out_cnt, nq, k, out_ids, out_dists, s);
        for (void* p : {(void*)cd, (void*)cp, (void*)cid, (void*)ccnt, (void*)skey, (void*)spos})
            PQRR_CUDA(cudaFreeAsync(p, s));
        return;
    }
    set_smem((const void*)merge_topk_kernel, smem);
    merge_topk_kernel<<<(unsigned)nq, 256, smem, s>>>(ids, dists, counts, nq, parts, width, ps, cs, k, n2,
                                                      out_ids, out_dists, out_cnt);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_unpack_keys(const uint64_t* keys, const uint32_t* cnt, size_t nq, uint32_t stride,
                        uint32_t* ids, float* dists, cudaStream_t s) {
    size_t total = nq * stride;
    if (!total) return;
    unpack_keys_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const u64*>(keys), cnt, nq, stride, ids, dists);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
