// k_wselect.cu — warp-per-query exact selections (one query per warp, no
// block-wide barriers):
//   * topw_warp_kernel      K1 epilogue: the w nearest coarse centroids of a
//                           query under (dist, index) (ties -> lowest index,
//                           SPEC.md:125), w <= 64, sorted;
//   * select_warp_kernel    exact top-k' of a query's candidates under the
//                           reference order (dist, id) (types.hpp:47-50,
//                           topk.hpp:18-29), unsorted;
//   * rerank_topk_warp_kernel  top-k of the re-ranked distances under
//                           (dist, id), sorted, with sentinels past the count.
// All three find the boundary key with a 4-pass 8-bit radix select on the
// distance bits (non-negative floats order like their bit patterns) using a
// warp-private 256-bin histogram in shared memory, then compact the keys below
// the boundary plus the boundary's tied entries in (index / id) order.
#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int WS_WARPS = 8;  // queries per CTA
constexpr uint32_t TIE_CAP = 256;  // boundary ties sorted in shared memory

// Rank-th (1-based) smallest of n 32-bit keys key(i); on return `kth` is that
// key and `r_eq` the number of entries equal to it that belong to the
// rank smallest (1 <= r_eq).  The leading bits shared by the smallest and the
// largest key are skipped (a query's candidate distances sit in a narrow band,
// and equal leading digits would pile every lane's atomic onto one bin); the
// remaining bits are resolved 8 at a time.
template <class KeyF>
__device__ __forceinline__ void warp_radix_select(uint32_t n, uint32_t rank, KeyF key,
                                                  uint32_t* __restrict__ hist, uint32_t& kth,
                                                  uint32_t& r_eq, uint32_t kmin0 = 0xffffffffu,
                                                  uint32_t kmax0 = 0u) {
    const int lane = threadIdx.x & 31;
    constexpr int U = 8;  // loads in flight per lane
    // the key range, when the producer already knows it (K4r), saves a pass
    const bool known = kmin0 <= kmax0 && kmax0 != 0xffffffffu;  // (all-ones = not provided)
    uint32_t kmin = known ? kmin0 : 0xffffffffu, kmax = known ? kmax0 : 0u;
    for (uint32_t base = 0; !known && base < n; base += 32 * U) {
        uint32_t v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t i = base + k * 32 + lane;
            v[k] = i < n ? key(i) : 0u;
        }
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (base + k * 32 + lane < n) {
                kmin = min(kmin, v[k]);
                kmax = max(kmax, v[k]);
            }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (kmin == kmax) {  // all keys equal
        kth = kmin;
        r_eq = rank;
        return;
    }
    int consumed = __clz(kmin ^ kmax);  // leading bits common to every key
    uint32_t prefix = consumed ? kmin >> (32 - consumed) : 0u;
    uint32_t r = rank;
#pragma unroll 1
    while (consumed < 32) {
        const int wd = min(8, 32 - consumed);
        const int sh = 32 - consumed - wd;
        const uint32_t msk = (1u << wd) - 1u;
#pragma unroll
        for (int b = 0; b < 8; ++b) hist[lane * 8 + b] = 0;
        __syncwarp();
        for (uint32_t base = 0; base < n; base += 32 * U) {
            uint32_t v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                v[k] = i < n ? key(i) : 0u;
            }
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (base + k * 32 + lane < n && (consumed == 0 || (v[k] >> (sh + wd)) == prefix))
                    atomicAdd(&hist[(v[k] >> sh) & msk], 1u);
        }
        __syncwarp();
        uint32_t h[8], sum = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            h[b] = hist[lane * 8 + b];
            sum += h[b];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - sum;
        const bool mine = excl < r && r <= incl;
        const int owner = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        uint32_t bin = 0, before = excl, bcnt = 0;
        if (mine) {
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                if (r > before + h[b]) {
                    before += h[b];
                } else {
                    bin = lane * 8 + b;
                    bcnt = h[b];
                    break;
                }
            }
        }
        bin = __shfl_sync(0xffffffffu, bin, owner);
        before = __shfl_sync(0xffffffffu, before, owner);
        bcnt = __shfl_sync(0xffffffffu, bcnt, owner);
        prefix = (prefix << wd) | bin;
        r -= before;
        consumed += wd;
        __syncwarp();
        if (bcnt == 1 && consumed < 32) {  // a single key left under this prefix
            uint32_t v = 0;
            for (uint32_t base = 0; base < n; base += 32 * U) {
                uint32_t vv[U];
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const uint32_t i = base + k * 32 + lane;
                    vv[k] = i < n ? key(i) : 0u;
                }
#pragma unroll
                for (int k = 0; k < U; ++k)
                    if (base + k * 32 + lane < n && (vv[k] >> (32 - consumed)) == prefix) v = vv[k];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
            prefix = v;
            break;
        }
    }
    kth = prefix;
    r_eq = r;
}

// In-warp bitonic sort of n2 (power of two, <= 1024) 64-bit keys in smem.
__device__ __forceinline__ void warp_bitonic(u64* keys, uint32_t n2) {
    const int lane = threadIdx.x & 31;
    for (uint32_t k = 2; k <= n2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < n2 / 2; i += 32) {
                const uint32_t lo = 2 * i - (i & (j - 1));
                const uint32_t hi = lo + j;
                const bool up = (lo & k) == 0;
                const u64 a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncwarp();
        }
    }
}

// Top-w of a coarse distance row in three passes over the row (the rows of a
// large batch do not fit L2): min / max, one 8-bit histogram below their
// common leading bits, then one pass that emits every entry of a lower bin (in
// index order) and compacts the boundary bin's entries (value, index) into a
// per-warp buffer, from which a small sort takes the remaining rank.  A
// boundary bin larger than the buffer falls back to the full radix select.
constexpr uint32_t TW_BIN_CAP = 256;

__global__ __launch_bounds__(WS_WARPS * 32) void topw_warp_kernel(const float* __restrict__ D, size_t nq,
                                                                   uint32_t nc, uint32_t w,
                                                                   uint32_t* __restrict__ out_idx,
                                                                   float* __restrict__ out_dist) {
    __shared__ uint32_t hist_all[WS_WARPS][256];
    __shared__ u64 keys_all[WS_WARPS][64];
    __shared__ u64 bin_all[WS_WARPS][TW_BIN_CAP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t q = (size_t)blockIdx.x * WS_WARPS + warp;
    if (q >= nq) return;
    const uint32_t* row = reinterpret_cast<const uint32_t*>(D + q * nc);
    uint32_t* hist = hist_all[warp];
    u64* keys = keys_all[warp];
    u64* binb = bin_all[warp];
    const unsigned lt_mask = (1u << lane) - 1u;
    constexpr int U = 8;
    // ---- pass 1: min / max
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (uint32_t base = 0; base < nc; base += 32 * U) {
        uint32_t v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t i = base + k * 32 + lane;
            v[k] = i < nc ? __ldg(row + i) : 0u;
        }
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (base + k * 32 + lane < nc) {
                kmin = min(kmin, v[k]);
                kmax = max(kmax, v[k]);
            }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    bool fast = kmin != kmax;
    uint32_t lo_key = 0, r_bin = 0;
    int sh = 0;
    if (fast) {
        // ---- pass 2: 8-bit histogram of the bits below the common prefix
        const int consumed = __clz(kmin ^ kmax);
        const int wd = min(8, 32 - consumed);
        sh = 32 - consumed - wd;
        const uint32_t base_key = consumed ? (kmin >> (32 - consumed)) << (32 - consumed) : 0u;
#pragma unroll
        for (int b = 0; b < 8; ++b) hist[lane * 8 + b] = 0;
        __syncwarp();
        for (uint32_t base = 0; base < nc; base += 32 * U) {
            uint32_t v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                v[k] = i < nc ? __ldg(row + i) : 0u;
            }
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (base + k * 32 + lane < nc) atomicAdd(&hist[(v[k] >> sh) & ((1u << wd) - 1u)], 1u);
        }
        __syncwarp();
        uint32_t h[8], sum = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            h[b] = hist[lane * 8 + b];
            sum += h[b];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t excl = incl - sum;
        const bool mine = excl < w && w <= incl;
        const int owner = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        uint32_t bin = 0, before = excl, bc = 0;
        if (mine) {
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                if (w > before + h[b]) {
                    before += h[b];
                } else {
                    bin = lane * 8 + b;
                    bc = h[b];
                    break;
                }
            }
        }
        bin = __shfl_sync(0xffffffffu, bin, owner);
        before = __shfl_sync(0xffffffffu, before, owner);
        bc = __shfl_sync(0xffffffffu, bc, owner);
        lo_key = base_key | (bin << sh);  // first key of the boundary bin
        r_bin = w - before;               // entries to take from the boundary bin
        fast = bc <= TW_BIN_CAP;
    }
    uint32_t n_out = 0;
    if (fast) {
        // ---- pass 3: keys below the boundary bin in index order; the bin's
        // entries (value, index) to the per-warp buffer
        const uint32_t hi_key = lo_key + ((1u << sh) - 1u);  // last key of the bin
        uint32_t nb = 0;
        for (uint32_t base = 0; base < nc; base += 32 * U) {
            uint32_t v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                v[k] = i < nc ? __ldg(row + i) : 0xffffffffu;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                const bool valid = i < nc;
                const bool lt = valid && v[k] < lo_key;
                const bool inb = valid && v[k] >= lo_key && v[k] <= hi_key;
                const unsigned mlt = __ballot_sync(0xffffffffu, lt), mb = __ballot_sync(0xffffffffu, inb);
                if (lt) keys[n_out + __popc(mlt & lt_mask)] = ((u64)v[k] << 32) | i;
                if (inb) binb[nb + __popc(mb & lt_mask)] = ((u64)v[k] << 32) | i;
                n_out += __popc(mlt);
                nb += __popc(mb);
            }
        }
        __syncwarp();
        uint32_t b2 = 1;
        while (b2 < nb) b2 <<= 1;
        for (uint32_t i = nb + lane; i < b2; i += 32) binb[i] = ~0ull;
        __syncwarp();
        warp_bitonic(binb, b2);
        for (uint32_t t = lane; t < r_bin; t += 32) keys[n_out + t] = binb[t];
        n_out += r_bin;
    } else {
        // fallback: full radix select, then compaction in index order
        uint32_t kth, r_eq;
        warp_radix_select(nc, w, [&](uint32_t i) { return __ldg(row + i); }, hist, kth, r_eq);
        uint32_t eq_taken = 0;
        for (uint32_t base = 0; base < nc; base += 32) {
            const uint32_t i = base + lane;
            const uint32_t u = i < nc ? __ldg(row + i) : 0xffffffffu;
            const bool lt = i < nc && u < kth;
            const bool eq = i < nc && u == kth;
            const unsigned meq = __ballot_sync(0xffffffffu, eq);
            const uint32_t eq_rank = eq_taken + __popc(meq & lt_mask);
            const bool take = lt || (eq && eq_rank < r_eq);
            const unsigned mtake = __ballot_sync(0xffffffffu, take);
            if (take) keys[n_out + __popc(mtake & lt_mask)] = ((u64)u << 32) | i;
            n_out += __popc(mtake);
            eq_taken += __popc(meq);
        }
    }
    uint32_t w2 = 1;
    while (w2 < w) w2 <<= 1;
    __syncwarp();
    for (uint32_t i = w + lane; i < w2; i += 32) keys[i] = ~0ull;
    __syncwarp();
    warp_bitonic(keys, w2);
    for (uint32_t i = lane; i < w; i += 32) {
        out_idx[q * w + i] = key_id(keys[i]);
        if (out_dist) out_dist[q * w + i] = key_dist(keys[i]);
    }
}

// Shortlist selection (unsorted): candidates (dist, pos) of query q, ids
// gathered for the selected entries only.  Ties at the boundary distance are
// resolved by id with a small warp loop (they are rare).
__global__ __launch_bounds__(WS_WARPS * 32) void select_warp_kernel(
    const float* __restrict__ cand_dist, const uint32_t* __restrict__ cand_pos,
    const uint32_t* __restrict__ cand_cnt, uint32_t cap, size_t nq, const uint32_t* __restrict__ ids,
    uint32_t kprime, u64* __restrict__ sl_key, uint32_t* __restrict__ sl_pos,
    uint32_t* __restrict__ sl_cnt, const uint32_t* __restrict__ cand_mm, int need_ids) {
    __shared__ uint32_t hist_all[WS_WARPS][256];
    __shared__ u64 tie_all[WS_WARPS][TIE_CAP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t q = (size_t)blockIdx.x * WS_WARPS + warp;
    if (q >= nq) return;
    const uint32_t n = min(cand_cnt[q], cap);
    const uint32_t* dq = reinterpret_cast<const uint32_t*>(cand_dist) + q * cap;
    const uint32_t* pq = cand_pos + q * cap;
    u64* ok = sl_key + q * kprime;
    uint32_t* op = sl_pos + q * kprime;
    const unsigned lt_mask = (1u << lane) - 1u;
    if (n <= kprime) {
        for (uint32_t i = lane; i < n; i += 32) {
            const uint32_t p = pq[i];
            ok[i] = ((u64)dq[i] << 32) | (need_ids ? ids[p] : 0u);
            op[i] = p;
        }
        if (lane == 0) sl_cnt[q] = n;
        return;
    }
    uint32_t kth, r_eq;
    warp_radix_select(n, kprime, [&](uint32_t i) { return dq[i]; }, hist_all[warp], kth, r_eq,
                      cand_mm ? cand_mm[2 * q] : 0xffffffffu, cand_mm ? cand_mm[2 * q + 1] : 0u);
    // one pass, 8 chunks of 32 per iteration (loads hoisted): entries strictly
    // below the boundary go out directly; entries at the boundary distance go
    // to a per-warp tie buffer as (id, pos) (exact ADC ties are common: equal
    // codes in one list); the r_eq smallest ids among them are taken after.
    constexpr int U = 8;
    u64* tie = tie_all[warp];
    uint32_t n_out = 0, n_eq = 0;
    for (uint32_t base = 0; base < n; base += 32 * U) {
        uint32_t u[U], p[U], id[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t i = base + k * 32 + lane;
            u[k] = i < n ? dq[i] : 0xffffffffu;
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t i = base + k * 32 + lane;
            p[k] = (i < n && u[k] <= kth) ? pq[i] : 0u;
        }
#pragma unroll
        // ids only where they decide (the boundary ties) unless the caller
        // needs them in the keys (the re-ranker with records reads its own)
        for (int k = 0; k < U; ++k) id[k] = (u[k] == kth || (need_ids && u[k] < kth)) ? ids[p[k]] : 0u;
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const bool lt = u[k] < kth, eq = u[k] == kth;  // padding lanes carry 0xffffffff
            const unsigned mlt = __ballot_sync(0xffffffffu, lt), meq = __ballot_sync(0xffffffffu, eq);
            if (lt) {
                const uint32_t o = n_out + __popc(mlt & lt_mask);
                ok[o] = ((u64)u[k] << 32) | id[k];
                op[o] = p[k];
            }
            if (eq) {
                const uint32_t t = n_eq + __popc(meq & lt_mask);
                if (t < TIE_CAP) tie[t] = ((u64)id[k] << 32) | p[k];
            }
            n_out += __popc(mlt);
            n_eq += __popc(meq);
        }
    }
    __syncwarp();
    if (n_eq <= TIE_CAP) {
        if (n_eq != r_eq) {
            uint32_t t2 = 1;
            while (t2 < n_eq) t2 <<= 1;
            for (uint32_t i = n_eq + lane; i < t2; i += 32) tie[i] = ~0ull;
            __syncwarp();
            warp_bitonic(tie, t2);
        }
        for (uint32_t t = lane; t < r_eq; t += 32) {
            ok[n_out + t] = ((u64)kth << 32) | (uint32_t)(tie[t] >> 32);
            op[n_out + t] = (uint32_t)tie[t];
        }
    } else {
        // many ties (duplicate vectors): radix-select the r_eq-th smallest id
        // among them (non-tied entries map to 0xffffffff, above every id)
        uint32_t idk, dummy;
        warp_radix_select(n, r_eq, [&](uint32_t i) { return dq[i] == kth ? ids[pq[i]] : 0xffffffffu; },
                          hist_all[warp], idk, dummy);
        uint32_t nt = 0;
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t i = base + lane;
            uint32_t pp = 0, idd = 0xffffffffu;
            if (i < n && dq[i] == kth) {
                pp = pq[i];
                idd = ids[pp];
            }
            const bool take = idd <= idk && idd != 0xffffffffu;
            const unsigned m = __ballot_sync(0xffffffffu, take);
            if (take) {
                const uint32_t o = n_out + nt + __popc(m & lt_mask);
                ok[o] = ((u64)kth << 32) | idd;
                op[o] = pp;
            }
            nt += __popc(m);
        }
    }
    if (lane == 0) sl_cnt[q] = kprime;
}

// One pass over a row for its k smallest (dist, id) keys when k << n (C4: 100
// of 10^4): the warp keeps a bound >= the k-th smallest distance, stages by
// ballot compaction the entries at or below it, and when the stage fills, the
// exact k-th smallest staged distance becomes the bound (the k-th of a subset
// is >= the k-th of the row) and the stage keeps its entries <= it.  The final
// stage holds every entry <= the bound, so its first k keys in (dist, id)
// order are the row's.  false: the stage cannot hold k plus a round (or masses
// of ties); the caller runs the multi-pass select.
constexpr uint32_t RT_CAP = 512;
__device__ __forceinline__ bool rerank_topk_stream(uint32_t n, uint32_t k, const uint32_t* __restrict__ db,
                                                   const uint32_t* __restrict__ ib, u64* stage, uint32_t cap,
                                                   uint32_t* hist, uint32_t& n_out) {
    constexpr int U = 4;  // (8 loads in flight need a 1024-entry stage: 64 KiB per CTA, measured slower)
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    if (cap < RT_CAP || k + 32 * U > cap / 2) return false;
    uint32_t bound = 0xffffffffu, cnt = 0;
    auto tighten = [&]() {
        __syncwarp();
        uint32_t kth, r_eq;
        warp_radix_select(cnt, k, [&](uint32_t j) { return (uint32_t)(stage[j] >> 32); }, hist, kth, r_eq);
        bound = kth;
        __syncwarp();
        uint32_t kept = 0;
        for (uint32_t j0 = 0; j0 < cnt; j0 += 32) {
            const uint32_t j = j0 + lane;
            const u64 e = j < cnt ? stage[j] : ~0ull;
            const bool keep = j < cnt && (uint32_t)(e >> 32) <= bound;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            __syncwarp();
            if (keep) stage[kept + __popc(m & lt_mask)] = e;
            kept += __popc(m);
            __syncwarp();
        }
        cnt = kept;
    };
    for (uint32_t base = 0; base < n; base += 32 * U) {
        uint32_t v[U];
#pragma unroll
        for (int t = 0; t < U; ++t) {
            const uint32_t i = base + t * 32 + lane;
            v[t] = i < n ? __ldg(db + i) : 0xffffffffu;
        }
#pragma unroll
        for (int t = 0; t < U; ++t) {
            const uint32_t i = base + t * 32 + lane;
            const bool pass = i < n && v[t] <= bound;
            const unsigned m = __ballot_sync(0xffffffffu, pass);
            if (m) {
                if (pass) stage[cnt + __popc(m & lt_mask)] = ((u64)v[t] << 32) | __ldg(ib + i);
                cnt += __popc(m);
            }
        }
        if (cnt > cap - 32 * U) {
            tighten();
            if (cnt > cap / 2) return false;
        }
    }
    if (cnt > 2 * k + 64) tighten();  // keep the final sort small
    n_out = cnt;
    return true;
}

// Re-rank top-k: (rdist, rid) rows of width `stride`, n = cnt[q] valid.
__global__ __launch_bounds__(WS_WARPS * 32) void rerank_topk_warp_kernel(
    const float* __restrict__ rdist, const uint32_t* __restrict__ rid,
    const uint32_t* __restrict__ cnt_in, uint32_t stride, size_t nq, uint32_t k, uint32_t k2, uint32_t cap,
    uint32_t* __restrict__ out_ids, float* __restrict__ out_dists, uint32_t* __restrict__ out_cnt) {
    extern __shared__ u64 wkeys[];  // [WS_WARPS][cap], cap >= k2
    __shared__ uint32_t hist_all[WS_WARPS][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t q = (size_t)blockIdx.x * WS_WARPS + warp;
    if (q >= nq) return;
    u64* keys = wkeys + (size_t)warp * cap;
    const uint32_t n = cnt_in[q];
    const uint32_t* db = reinterpret_cast<const uint32_t*>(rdist) + q * stride;
    const uint32_t* ib = rid + q * stride;
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t n_out = 0;
    if (n <= k) {
        for (uint32_t i = lane; i < n; i += 32) keys[i] = ((u64)db[i] << 32) | ib[i];
        n_out = n;
    } else if (rerank_topk_stream(n, k, db, ib, keys, cap, hist_all[warp], n_out)) {
        // (one pass: the stage holds every entry at or below the k-th distance)
    } else {
        uint32_t kth, r_eq;
        warp_radix_select(n, k, [&](uint32_t i) { return db[i]; }, hist_all[warp], kth, r_eq);
        uint32_t n_eq = 0;
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t i = base + lane;
            const uint32_t u = i < n ? db[i] : 0xffffffffu;
            const bool lt = i < n && u < kth;
            const unsigned m = __ballot_sync(0xffffffffu, lt);
            if (lt) keys[n_out + __popc(m & lt_mask)] = ((u64)u << 32) | ib[i];
            n_out += __popc(m);
            n_eq += __popc(__ballot_sync(0xffffffffu, i < n && u == kth));
        }
        if (n_eq == r_eq) {
            for (uint32_t base = 0; base < n; base += 32) {
                const uint32_t i = base + lane;
                const bool eq = i < n && db[i] == kth;
                const unsigned m = __ballot_sync(0xffffffffu, eq);
                if (eq) keys[n_out + __popc(m & lt_mask)] = ((u64)kth << 32) | ib[i];
                n_out += __popc(m);
            }
        } else {
            // the r_eq smallest ids among the ties (radix select on ids)
            uint32_t idk, dummy;
            warp_radix_select(n, r_eq, [&](uint32_t i) { return db[i] == kth ? ib[i] : 0xffffffffu; },
                              hist_all[warp], idk, dummy);
            uint32_t nt = 0;
            for (uint32_t base = 0; base < n; base += 32) {
                const uint32_t i = base + lane;
                const bool take = i < n && db[i] == kth && ib[i] <= idk;
                const unsigned m = __ballot_sync(0xffffffffu, take);
                if (take) keys[n_out + nt + __popc(m & lt_mask)] = ((u64)kth << 32) | ib[i];
                nt += __popc(m);
            }
            n_out += r_eq;
        }
    }
    __syncwarp();
    uint32_t s2 = k2;  // (the streamed stage may hold more than k entries: ties and the last bound's slack)
    while (s2 < n_out) s2 <<= 1;
    for (uint32_t i = n_out + lane; i < s2; i += 32) keys[i] = ~0ull;
    __syncwarp();
    warp_bitonic(keys, s2);
    const uint32_t cnt = min(n, k);
    for (uint32_t i = lane; i < k; i += 32) {
        const bool live = i < cnt;
        out_ids[q * k + i] = live ? key_id(keys[i]) : 0xffffffffu;
        out_dists[q * k + i] = live ? key_dist(keys[i]) : __int_as_float(0x7f800000);
    }
    if (lane == 0) out_cnt[q] = cnt;
}

// Weighted variant for the threshold estimate: the smallest key at which the
// weights of the keys <= it reach `rank`.  weight(i) > 0, sums fit 32 bits.
template <class KeyF, class WtF>
__device__ __forceinline__ uint32_t warp_weighted_select(uint32_t n, uint32_t rank, KeyF key, WtF wt,
                                                         uint32_t* __restrict__ hist) {
    const int lane = threadIdx.x & 31;
    constexpr int U = 8;  // loads in flight per lane
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (uint32_t base = 0; base < n; base += 32 * U) {
        uint32_t v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t i = base + k * 32 + lane;
            v[k] = i < n ? key(i) : kmin;
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t i = base + k * 32 + lane;
            if (i < n) {
                kmin = min(kmin, v[k]);
                kmax = max(kmax, v[k]);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (kmin == kmax) return kmin;
    int consumed = __clz(kmin ^ kmax);
    uint32_t prefix = consumed ? kmin >> (32 - consumed) : 0u;
    uint32_t r = rank;
    // the threshold is an estimate (exactness is checked downstream): stop with
    // <= 8 low bits undecided and return the bin's upper edge (a relative
    // over-estimate below 2^-15), saving the last pass over the samples
#pragma unroll 1
    while (consumed < 24) {
        const int wd = min(8, 32 - consumed);
        const int sh = 32 - consumed - wd;
        const uint32_t msk = (1u << wd) - 1u;
#pragma unroll
        for (int b = 0; b < 8; ++b) hist[lane * 8 + b] = 0;
        __syncwarp();
        for (uint32_t base = 0; base < n; base += 32 * U) {
            uint32_t v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                v[k] = i < n ? key(i) : 0u;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                if (i < n && (consumed == 0 || (v[k] >> (sh + wd)) == prefix))
                    atomicAdd(&hist[(v[k] >> sh) & msk], wt(i));
            }
        }
        __syncwarp();
        uint32_t h[8], sum = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            h[b] = hist[lane * 8 + b];
            sum += h[b];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - sum;
        const bool mine = excl < r && r <= incl;
        const int owner = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        uint32_t bin = 0, before = excl;
        if (mine) {
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                if (r > before + h[b]) {
                    before += h[b];
                } else {
                    bin = lane * 8 + b;
                    break;
                }
            }
        }
        bin = __shfl_sync(0xffffffffu, bin, owner);
        before = __shfl_sync(0xffffffffu, before, owner);
        prefix = (prefix << wd) | bin;
        r -= before;
        consumed += wd;
        __syncwarp();
    }
    if (consumed >= 32) return prefix;
    const int rest = 32 - consumed;
    return (prefix << rest) | ((1u << rest) - 1u);
}

// tau_q (one query per warp): the distance at which the weighted count of the
// query's samples reaches alpha*k' entries; each sample weighs its pair's
// stride (sample_tier: the tiers are contiguous ranges of the query's slots).
// +inf for queries scanned without sampling or with too few entries.
constexpr int TH_CAP = 640;  // staged samples per warp (threshold_warp_kernel)
__global__ __launch_bounds__(WS_WARPS * 32) void threshold_warp_kernel(
    const float* __restrict__ sample, const uint64_t* __restrict__ sample_off, uint32_t w,
    size_t nq, const uint8_t* __restrict__ sampled, float alpha_k, uint32_t stride, int tiered,
    float* __restrict__ tau) {
    __shared__ uint32_t hist_all[WS_WARPS][256];
    __shared__ uint32_t stage_all[WS_WARPS][2 * TH_CAP];  // per warp: staged values, then their indices
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t q = (size_t)blockIdx.x * WS_WARPS + warp;
    if (q >= nq) return;
    const float inf = __int_as_float(0x7f800000);
    if (!sampled[q]) {
        if (lane == 0) tau[q] = inf;
        return;
    }
    // first probe rank of each tier: ceil(w/8), ceil(w/4), ceil(w/2) (sample_tier)
    uint32_t rb = w;
    if (tiered && lane >= 1 && lane <= 3) rb = min(w, (w * (1u << (lane - 1)) + 7u) / 8u);
    if (lane == 0) rb = 0;
    const uint64_t seg = lane <= 4 ? sample_off[q * w + (lane == 4 ? w : rb)] : 0ull;
    const uint64_t s0 = __shfl_sync(0xffffffffu, seg, 0), s1 = __shfl_sync(0xffffffffu, seg, 1);
    const uint64_t s2 = __shfl_sync(0xffffffffu, seg, 2), s3 = __shfl_sync(0xffffffffu, seg, 3);
    const uint64_t s4 = __shfl_sync(0xffffffffu, seg, 4);
    const uint32_t h1 = tier_shift(1, w), h2 = tier_shift(2, w), h3 = tier_shift(3, w);
    const unsigned long long total = ((s1 - s0) + ((s2 - s1) << h1) + ((s3 - s2) << h2) + ((s4 - s3) << h3)) *
                                     (unsigned long long)stride;
    const uint32_t rank = (uint32_t)max(1.0, ceil((double)alpha_k));
    if (total < rank) {
        if (lane == 0) tau[q] = inf;
        return;
    }
    const uint32_t n = (uint32_t)(s4 - s0);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(sample) + s0;
    const uint32_t b1 = (uint32_t)(s1 - s0), b2 = (uint32_t)(s2 - s0), b3 = (uint32_t)(s3 - s0);
    // One pass over the samples instead of four.  The target rank sits in the
    // far lower tail (rank / stride ~ 64-128 samples of 10^4-10^5), and at
    // large batches the samples stream from HBM (C5, 65536 queries: 16.5 GB per
    // pass).  The warp keeps a bound Tw >= the answer and stages (ballot
    // compaction, no atomics) only the samples <= Tw.  When the stage fills, a
    // weighted select over it gives a new bound — the rank-th of a subset is
    // >= the rank-th of all — and the stage keeps only its entries <= the new
    // bound.  Every sample dropped or skipped is above a bound, hence above the
    // answer, so the final select over the stage is the select over all
    // samples.  The stage fills ~4 times per query (512, 4k, 30k samples in).
    {
        constexpr int U = 8;
        uint32_t* st_v = stage_all[warp];
        uint32_t* st_i = st_v + TH_CAP;
        auto st_wt = [&](uint32_t j) {
            const uint32_t ix = st_i[j];
            return stride << tier_shift((ix >= b1) + (ix >= b2) + (ix >= b3), w);
        };
        uint32_t Tw = 0xffffffffu, cnt = 0;
        bool give_up = false;
        const uint32_t lt_mask = (1u << lane) - 1u;
        for (uint32_t base = 0; base < n && !give_up; base += 32 * U) {
            uint32_t v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                v[k] = i < n ? __ldg(src + i) : 0xffffffffu;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                const bool pass = i < n && v[k] <= Tw;
                const uint32_t m = __ballot_sync(0xffffffffu, pass);
                if (m) {
                    if (pass) {
                        const uint32_t pos = cnt + __popc(m & lt_mask);
                        st_v[pos] = v[k];
                        st_i[pos] = i;
                    }
                    cnt += __popc(m);
                }
            }
            if (cnt > TH_CAP - 32 * U) {  // (warp-uniform) the next round may not fit: tighten the bound
                __syncwarp();
                unsigned long long wsum = 0;
                for (uint32_t j = lane; j < cnt; j += 32) wsum += st_wt(j);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
                if (wsum < rank) {
                    give_up = true;  // (stage weight below the rank: tiny strides against a huge rank)
                    break;
                }
                Tw = warp_weighted_select(cnt, rank, [&](uint32_t j) { return st_v[j]; }, st_wt, hist_all[warp]);
                __syncwarp();
                uint32_t kept = 0;
                for (uint32_t j0 = 0; j0 < cnt; j0 += 32) {
                    const uint32_t j = j0 + lane;
                    const uint32_t vv = j < cnt ? st_v[j] : 0xffffffffu, ii = j < cnt ? st_i[j] : 0u;
                    const bool keep = j < cnt && vv <= Tw;
                    const uint32_t m = __ballot_sync(0xffffffffu, keep);
                    __syncwarp();
                    if (keep) {
                        const uint32_t pos = kept + __popc(m & lt_mask);
                        st_v[pos] = vv;
                        st_i[pos] = ii;
                    }
                    kept += __popc(m);
                    __syncwarp();
                }
                cnt = kept;
                if (cnt > TH_CAP / 2) give_up = true;  // (masses of equal values: the multi-pass select handles them)
            }
        }
        if (!give_up) {
            __syncwarp();
            const uint32_t t = warp_weighted_select(cnt, rank, [&](uint32_t j) { return st_v[j]; }, st_wt,
                                                    hist_all[warp]);
            if (lane == 0) tau[q] = __uint_as_float(t);
            return;
        }
        __syncwarp();
    }
    const uint32_t t = warp_weighted_select(
        n, rank, [&](uint32_t i) { return __ldg(src + i); },
        [&](uint32_t i) { return stride << tier_shift((i >= b1) + (i >= b2) + (i >= b3), w); }, hist_all[warp]);
    if (lane == 0) tau[q] = __uint_as_float(t);
}

}  // namespace

bool launch_topw_warp(const float* D, size_t nq, uint32_t nc, uint32_t w, uint32_t* out_idx,
                      float* out_dist, cudaStream_t s) {
    if (w > 64 || w == 0 || w > nc) return false;
    topw_warp_kernel<<<(unsigned)((nq + WS_WARPS - 1) / WS_WARPS), WS_WARPS * 32, 0, s>>>(
        D, nq, nc, w, out_idx, out_dist);
    PQRR_LAUNCH_CHECK();
    count_launch();
    return true;
}

void launch_select_warp(const float* cand_dist, const uint32_t* cand_pos, const uint32_t* cand_cnt,
                        uint32_t cap, size_t nq, const uint32_t* ids, uint32_t kprime,
                        uint64_t* sl_key, uint32_t* sl_pos, uint32_t* sl_cnt, cudaStream_t s,
                        const uint32_t* cand_mm, bool need_ids) {
    if (nq == 0) return;
    select_warp_kernel<<<(unsigned)((nq + WS_WARPS - 1) / WS_WARPS), WS_WARPS * 32, 0, s>>>(
        cand_dist, cand_pos, cand_cnt, cap, nq, ids, kprime, reinterpret_cast<u64*>(sl_key), sl_pos,
        sl_cnt, cand_mm, need_ids ? 1 : 0);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

bool launch_rerank_topk_warp(const float* rdist, const uint32_t* rid, const uint32_t* cnt,
                             uint32_t stride, size_t nq, uint32_t k, uint32_t* out_ids,
                             float* out_dists, uint32_t* out_cnt, cudaStream_t s) {
    uint32_t k2 = 1;
    while (k2 < k) k2 <<= 1;
    const uint32_t cap = std::max<uint32_t>(k2, RT_CAP);  // per-warp keys: the streaming stage or the k2 winners
    const size_t smem = (size_t)WS_WARPS * cap * sizeof(u64);
    if (k2 > 1024 || smem > 96 * 1024) return false;
    if (smem > 48 * 1024)
        set_max_smem((const void*)rerank_topk_warp_kernel, (size_t)((int)smem));
    rerank_topk_warp_kernel<<<(unsigned)((nq + WS_WARPS - 1) / WS_WARPS), WS_WARPS * 32, smem, s>>>(
        rdist, rid, cnt, stride, nq, k, k2, cap, out_ids, out_dists, out_cnt);
    PQRR_LAUNCH_CHECK();
    count_launch();
    return true;
}

}  // namespace pqrr_b200

namespace pqrr_b200 {
void launch_threshold_warp(const float* sample_dist, const uint64_t* sample_off, uint32_t w, size_t nq,
                           const uint8_t* query_sampled, float alpha_k, uint32_t stride, int tiered,
                           float* tau, cudaStream_t s) {
    if (nq == 0) return;
    threshold_warp_kernel<<<(unsigned)((nq + WS_WARPS - 1) / WS_WARPS), WS_WARPS * 32, 0, s>>>(
        sample_dist, sample_off, w, nq, query_sampled, alpha_k, stride, tiered, tau);
    PQRR_LAUNCH_CHECK();
    count_launch();
}
}  // namespace pqrr_b200
