// k_lutpass.cu — K2, the LUT pass of ivf_search (ivf_index.hpp:58-61;
// build_lut, product_quantizer.hpp:48-49; adc_distance, :53-57), as a
// warp-specialised persistent kernel.
//
// One work item = one inverted list and up to 16 probing queries.  Per item
// the consumer warps (16) build the 16 exact residual LUTs LUT[j][i][q] in
// shared memory (128 KiB), reduce every (j, q) sub-table's minimum / range,
// write the item's 8-bit LUT block for K4f with a TMA bulk store, and compute
// the exact ADC distance of every stride-th entry of the list for the sampled
// queries (threshold estimation).  A producer warp runs one item ahead: it
// claims the next item, gathers its metadata, stages the query / coarse rows
// and the sampled codes with cp.async, and writes the residual queries
// x - C_l into the other half of a double buffer.  Producer and consumers
// hand buffers over through full / empty mbarriers; the consumers synchronise
// among themselves with a named barrier.  So the dependent global-load chain
// at the start of an item (counter -> item -> pairs -> queries -> rows) is off
// the consumers' critical path.
#include <float.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int M = 8;
constexpr int KS = 256;
constexpr int QT = kQT;
constexpr int NC = kScanThreads;  // consumer threads
constexpr int NCW = NC / 32;      // consumer warps
constexpr int NTH = NC + 64;      // + the item producer warp + the book warp
constexpr int LUT_FLOATS = M * KS * QT;
constexpr int Q8_BYTES = M * KS * QT;  // 32 KiB
constexpr int SCAP = 1024;             // sampled codes staged per item (more: read from global)
constexpr int RING = 3;                // code-book slices in flight

struct ItemMeta {
    uint32_t it, l, e0, e1, nqi;
    uint32_t smin;  // smallest sampling stride among the item's sampled queries
    int q[QT];
    uint32_t pair[QT];
    unsigned long long sbase[QT];
    uint8_t samp[QT];
    uint8_t sshift[QT];  // the query's stride = smin << sshift (sample_tier)
};

__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory"); }

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Residual row q of an item: stride d + 4 floats (16 B mod 128 B) plus 16 B
// for rows 8..15, so the rows a quarter warp reads in the build (0, 2, .., 14
// or 1, 3, .., 15) fall on 8 distinct 16-byte bank groups.
__device__ __forceinline__ int xrow(int q, int xld) { return q * xld + ((q >> 3) << 2); }
constexpr int xbuf(int xld) { return QT * xld + 4; }  // floats per residual buffer

__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
    unsigned done;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
    return done != 0;
}

// Exact LUTs of the item (the reference order of l2_sq; consumer threads only)
// with the per-(j, q) minimum / maximum reduced into s_mnu / s_mxu.  The
// code-book slice of sub-space j arrives in a RING-slot ring filled by the
// book warp (TMA bulk copies, full / empty mbarriers), so the consumers never
// meet at a block barrier inside the build.  Register blocking: a thread
// computes 2 queries x CI codes per sub-space, so every code-book row it
// loads serves two entries (a broadcast LDS.128 still costs one wavefront per
// quarter warp); the LUT is written with conflict-free 8-byte stores.
template <int DSUB>
__device__ __forceinline__ void build_luts_ring(float* __restrict__ lut, const float* __restrict__ xr,
                                                int xld, const float* __restrict__ ring,
                                                unsigned long long* bfull, unsigned long long* bempty,
                                                uint32_t& gslice, u64 nz, bool mm,
                                                unsigned* __restrict__ s_mnu, unsigned* __restrict__ s_mxu) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int qa = 2 * (lane & 7), ic = lane >> 3;
    constexpr int BF = KS * DSUB;
    constexpr int NCODE = KS / NCW;  // codes per warp and sub-space
    constexpr int CI = NCODE / 4;    // codes per thread and sub-space
    constexpr int T4 = DSUB / 4;
#pragma unroll 1
    for (int j = 0; j < M; ++j, ++gslice) {
        const uint32_t slot = gslice % RING;
        mbar_wait(&bfull[slot], (gslice / RING) & 1u);
        const float* bj = ring + slot * BF;
        u64 a01[T4], a23[T4], b01[T4], b23[T4];
#pragma unroll
        for (int t4 = 0; t4 < T4; ++t4) {
            const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(xr + xrow(qa, xld) + j * DSUB + 4 * t4);
            const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(xr + xrow(qa + 1, xld) + j * DSUB + 4 * t4);
            a01[t4] = u.x;
            a23[t4] = u.y;
            b01[t4] = w.x;
            b23[t4] = w.y;
        }
        float va[CI], vb[CI];
#pragma unroll
        for (int ci = 0; ci < CI; ++ci) {
            const int i = warp * NCODE + ci * 4 + ic;
            const ulonglong2* bp = reinterpret_cast<const ulonglong2*>(bj + i * DSUB);
            u64 sa01 = 0, sa23 = 0, sb01 = 0, sb23 = 0;
#pragma unroll
            for (int t4 = 0; t4 < T4; ++t4) {
                const ulonglong2 c = bp[t4];
                if (t4 == 0) {  // 0 + x == x for the rounded square x >= +0
                    sa01 = sq2(sub2(a01[0], c.x), nz);
                    sa23 = sq2(sub2(a23[0], c.y), nz);
                    sb01 = sq2(sub2(b01[0], c.x), nz);
                    sb23 = sq2(sub2(b23[0], c.y), nz);
                } else {
                    sa01 = acc_sq2(sa01, a01[t4], c.x, nz);
                    sa23 = acc_sq2(sa23, a23[t4], c.y, nz);
                    sb01 = acc_sq2(sb01, b01[t4], c.x, nz);
                    sb23 = acc_sq2(sb23, b23[t4], c.y, nz);
                }
            }
            va[ci] = __fadd_rn(__fadd_rn(lo2(sa01), hi2(sa01)), __fadd_rn(lo2(sa23), hi2(sa23)));
            vb[ci] = __fadd_rn(__fadd_rn(lo2(sb01), hi2(sb01)), __fadd_rn(lo2(sb23), hi2(sb23)));
        }
        __syncwarp();  // every lane's reads of the slice are complete
        if (lane == 0) mbar_arrive(&bempty[slot]);
        float mna = __int_as_float(0x7f800000), mxa = 0.f, mnb = mna, mxb = 0.f;
#pragma unroll
        for (int ci = 0; ci < CI; ++ci) {
            const int i = warp * NCODE + ci * 4 + ic;
            *reinterpret_cast<float2*>(lut + (j * KS + i) * QT + qa) = make_float2(va[ci], vb[ci]);
            mna = fminf(mna, va[ci]);
            mxa = fmaxf(mxa, va[ci]);
            mnb = fminf(mnb, vb[ci]);
            mxb = fmaxf(mxb, vb[ci]);
        }
        if (mm) {
#pragma unroll
            for (int o = 8; o < 32; o <<= 1) {
                mna = fminf(mna, __shfl_xor_sync(0xffffffffu, mna, o));
                mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, o));
                mnb = fminf(mnb, __shfl_xor_sync(0xffffffffu, mnb, o));
                mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, o));
            }
            if (ic == 0) {
                atomicMin(s_mnu + j * QT + qa, __float_as_uint(mna));
                atomicMax(s_mxu + j * QT + qa, __float_as_uint(mxa));
                atomicMin(s_mnu + j * QT + qa + 1, __float_as_uint(mnb));
                atomicMax(s_mxu + j * QT + qa + 1, __float_as_uint(mxb));
            }
        }
    }
}

template <int DSUB>
__global__ __launch_bounds__(NTH, 1) void lut_pass_kernel(const ScanArgs a, const u64 nz) {
    extern __shared__ float4 smem4[];
    const int xld = (int)a.d + 4;
    float* lut = reinterpret_cast<float*>(smem4);
    float* xr0 = lut + LUT_FLOATS;                 // [2][xbuf] residual queries (xrow)
    float* raw = xr0 + 2 * xbuf(xld);              // [QT + 1][d] producer staging
    u64* scodes = reinterpret_cast<u64*>(raw + (QT + 1) * a.d);  // [2][SCAP] sampled codes
    float* ring = reinterpret_cast<float*>(scodes + 2 * SCAP);  // [RING][KS * DSUB] code-book slices
    __shared__ ItemMeta meta[2];
    __shared__ __align__(8) unsigned long long full_bar[2], empty_bar[2], bfull[RING], bempty[RING];
    __shared__ volatile int s_stop;
    __shared__ __align__(16) float s_min[M * QT], s_rng[M * QT], s_inv[QT];
    __shared__ unsigned s_mnu[M * QT], s_mxu[M * QT];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t n_items = *a.num_items;
    // per-lane (scale, sum of minima) whenever q8_param is set; the 8-bit
    // block too unless this is the bound pass of the two-phase LUT pass
    const bool store_q8 = a.q8_param != nullptr;
    const bool store_block = store_q8 && a.q8_cache != nullptr && a.q8_mode == 0;
    const bool sampling = a.sample_dist != nullptr;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full_bar[b], 1);
            mbar_init(&empty_bar[b], 1);
        }
        for (int r = 0; r < RING; ++r) {
            mbar_init(&bfull[r], 1);
            mbar_init(&bempty[r], NCW);
        }
        s_stop = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW + 1) {
        // ------------------------------------------------------- book warp
        // streams the code-book slices j = 0..M-1, 0..M-1, ... (the same for
        // every item) into the ring; a slot is refilled once all consumer
        // warps released it.  Stops when the consumers saw the last item.
        if (lane == 0) {
            constexpr unsigned BYTES = KS * DSUB * sizeof(float);
            uint32_t n = 0;
            for (;; ++n) {
                const uint32_t slot = n % RING;
                bool stop = false;
                if (n >= RING) {
                    while (!mbar_try(&bempty[slot], ((n / RING) - 1) & 1u)) {
                        if (s_stop) {
                            stop = true;
                            break;
                        }
                        __nanosleep(64);  // leave the issue slots to the consumer warps
                    }
                } else {
                    stop = s_stop != 0;
                }
                if (stop) break;
                const float* src = a.books + (size_t)(n % M) * KS * DSUB;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(smem_u32(&bfull[slot])), "r"(BYTES) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(ring + slot * KS * DSUB)), "l"(src), "r"(BYTES),
                               "r"(smem_u32(&bfull[slot])) : "memory");
            }
            // the slices still in flight land before the CTA exits
            for (uint32_t t = n > (uint32_t)RING ? n - RING : 0u; t < n; ++t) mbar_wait(&bfull[t % RING], (t / RING) & 1u);
        }
        return;
    }

    if (warp == NCW) {
        // ---------------------------------------------------------- producer
        uint32_t live_mask = 0, my_c = 0;  // skip_dead: claimed items found live
        for (uint32_t k = 0;; ++k) {
            const int b = k & 1;
            if (k >= 2) mbar_wait(&empty_bar[b], ((k >> 1) - 1) & 1);
            ItemMeta& mt = meta[b];
            uint32_t c, it, l, e0, e1, start, nqi, p;
            int q;
            for (;;) {
                c = 0;
                if (a.skip_dead) {
                    // round 2 of the two-phase pass skips most far items: the
                    // lanes claim 32 items at once and test one item each (the
                    // dependent loads of 32 items overlap instead of running one
                    // item after the other); live items are then taken in order
                    while (!live_mask) {
                        uint32_t cb = 0;
                        if (lane == 0) cb = atomicAdd(a.item_counter, 32u);
                        cb = __shfl_sync(0xffffffffu, cb, 0);
                        if (cb >= n_items) break;
                        my_c = cb + lane;
                        bool lv = false;
                        if (my_c < n_items) {
                            const uint32_t it2 = a.item_order[my_c];
                            const uint32_t st2 = a.item_start[it2], nq2 = a.item_nq[it2];
                            for (uint32_t j = 0; j < nq2 && j < (uint32_t)QT && !lv; ++j) {
                                const uint32_t p2 = a.pair_sorted[st2 + j];
                                const int q2 = (int)(p2 / a.w);
                                const float sm2 = a.pair_bound ? a.pair_bound[p2]
                                                               : a.q8_param[((size_t)it2 * QT + j) * 2 + 1];
                                lv = pair_live(a.tau[q2], sm2);
                            }
                        }
                        live_mask = __ballot_sync(0xffffffffu, lv);
                    }
                    if (!live_mask) {
                        c = n_items;
                        break;
                    }
                    const int src = __ffs(live_mask) - 1;
                    live_mask &= live_mask - 1u;
                    c = __shfl_sync(0xffffffffu, my_c, src);
                } else {
                    if (lane == 0) c = atomicAdd(a.item_counter, 1u);
                    c = __shfl_sync(0xffffffffu, c, 0);
                }
                if (c >= n_items) break;
                it = a.item_order[c];  // longest items first
                l = a.item_list[it];
                e0 = a.item_e0[it];
                e1 = a.item_e1[it];
                start = a.item_start[it];
                nqi = a.item_nq[it];
                q = -1;
                p = 0;
                if (lane < QT && (uint32_t)lane < nqi) {
                    p = a.pair_sorted[start + lane];
                    q = (int)(p / a.w);
                }
                break;  // (skip_dead: the item was found live above)
            }
            if (c >= n_items) {
                if (lane == 0) {
                    mt.it = 0xffffffffu;
                    mbar_arrive(&full_bar[b]);
                }
                break;
            }
            // per-query sampling stride for this list (probe rank tier)
            const uint8_t sm = (q >= 0 && a.query_sampled) ? a.query_sampled[q] : 0;
            // the lane's stride shift (tier_shift of its probe rank's tier)
            const uint32_t tier = (lane < QT && q >= 0) ? tier_shift(sample_tier(p % a.w, a.w, a.tiered), a.w) : 31u;
            uint32_t tmin = (sm && lane < QT) ? tier : 31u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
            if (lane < QT) {
                mt.q[lane] = q;
                mt.pair[lane] = p;
                mt.samp[lane] = sm;
                mt.sbase[lane] = (sampling && sm) ? a.sample_off[p] : 0ull;
                mt.sshift[lane] = (uint8_t)(sm ? tier - tmin : 0u);
            }
            if (lane == 0) {
                mt.it = it;
                mt.l = l;
                mt.e0 = e0;
                mt.e1 = e1;
                mt.nqi = nqi;
                mt.smin = tmin < 31u ? (a.stride << tmin) : 0u;
            }
            __syncwarp();
            // rows: 16 query rows + the coarse row, 16 B per cp.async
            const uint32_t dch = a.d / 4;
            for (uint32_t i = lane; i < (QT + 1) * dch; i += 32) {
                const uint32_t r = i / dch, cc = i % dch;
                if (r == QT) cp16(raw + r * a.d + 4 * cc, a.coarse + (size_t)l * a.d + 4 * cc);
                else if (mt.q[r] >= 0) cp16(raw + r * a.d + 4 * cc, a.xq + (size_t)mt.q[r] * a.d + 4 * cc);
            }
            // sampled codes of the item's entries at the smallest stride among
            // its sampled queries (items cover whole lists: e0 == 0)
            if (sampling && tmin < 31u) {
                const uint32_t smin = a.stride << tmin;
                const uint32_t ns = (e1 + smin - 1) / smin;
                const u64* lcodes = reinterpret_cast<const u64*>(a.codes) + a.list_off[l];
                for (uint32_t si = lane; si < min(ns, (uint32_t)SCAP); si += 32)
                    cp8(scodes + b * SCAP + si, lcodes + sample_pos(si, smin, e1));
                // the samples past the staged ones are read by the consumers one
                // item later: pull their sectors into L2 now, so those loads
                // wait an L2 hit instead of a DRAM access (all 16 consumer warps
                // sit in the sampling loop together, nothing else hides it)
                for (uint32_t si = SCAP + lane; si < ns; si += 32)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(lcodes + sample_pos(si, smin, e1)));
            }
            cp_commit();
            cp_wait<0>();
            __syncwarp();
            // residual queries x - C_l (ivf_index.hpp:58-59) into xr[b]
            float* xr = xr0 + b * xbuf(xld);
            const float* crow = raw + QT * a.d;
            for (uint32_t i = lane; i < QT * dch; i += 32) {
                const uint32_t r = i / dch, cc = i % dch;
                const bool live = r < nqi;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (live) {
                    const float4 x = *reinterpret_cast<const float4*>(raw + r * a.d + 4 * cc);
                    const float4 y = *reinterpret_cast<const float4*>(crow + 4 * cc);
                    v = make_float4(__fsub_rn(x.x, y.x), __fsub_rn(x.y, y.y), __fsub_rn(x.z, y.z),
                                    __fsub_rn(x.w, y.w));
                }
                *reinterpret_cast<float4*>(xr + xrow(r, xld) + 4 * cc) = v;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_bar[b]);
        }
        return;
    }

    // -------------------------------------------------------------- consumers
    const int slot = lane >> 2, qd = lane & 3;
    const float4* lut4 = reinterpret_cast<const float4*>(lut);
    uint32_t gslice = 0;  // code-book slices consumed
    for (uint32_t k = 0;; ++k) {
        const int b = k & 1;
        mbar_wait(&full_bar[b], (k >> 1) & 1);
        const ItemMeta& mt = meta[b];
        const uint32_t it = mt.it;
        if (it == 0xffffffffu) {
            if (threadIdx.x == 0) s_stop = 1;
            break;
        }
        if (store_q8 && threadIdx.x < M * QT) {
            s_mnu[threadIdx.x] = 0x7f800000u;
            s_mxu[threadIdx.x] = 0u;
        }
        csync();
        build_luts_ring<DSUB>(lut, xr0 + b * xbuf(xld), xld, ring, bfull, bempty, gslice, nz, store_q8, s_mnu,
                              s_mxu);
        csync();  // LUT and the (j, q) minima / maxima complete
#ifdef LP_NOQUANT  // timing experiment only
        if (false) {
#else
        if (store_q8) {
#endif
            // 8-bit LUT (see quantize_item in k_scan.cu)
            const int t = threadIdx.x;
            if (t < M * QT) {
                const float mn = __uint_as_float(s_mnu[t]), mx = __uint_as_float(s_mxu[t]);
                s_min[t] = mn;
                s_rng[t] = __fsub_rn(mx, mn);
            }
            csync();
            if (t < QT) {
                float rng = 0.f, sm = 0.f;
#pragma unroll
                for (int jj = 0; jj < M; ++jj) {
                    rng = fmaxf(rng, s_rng[jj * QT + t]);
                    sm = __fadd_rn(sm, s_min[jj * QT + t]);
                }
                const float sc = __fdiv_rn(rng, 255.f);
                s_inv[t] = sc > 0.f ? __frcp_rn(sc) : 0.f;
                float* prm = a.q8_param + (size_t)it * 2 * QT;
                prm[2 * t] = sc;
                prm[2 * t + 1] = sm;
            }
            csync();
            if (store_block) {
            // 8-bit block straight to global memory, lane-major (q8_put_rows):
            // a thread quantises 4 rows x 4 lanes and writes 4 lane words;
            // a warp's stores cover 4 lanes x 32 contiguous bytes
            uint32_t* block = reinterpret_cast<uint32_t*>(a.q8_cache + (size_t)it * Q8_BYTES);
            const int g = t & 3;
            // 1/s with the (1 - 2^-20) shrink folded in: fsub, rcp, this product
            // and the per-entry product are 4 roundings, (1 + 2^-24)^4 (1 - 2^-20) < 1,
            // so v8 = floor(x) <= (L - m) / s as before
            const float shrink = 0.99999904632568359375f;  // 1 - 2^-20
            const float4 inv0 = *reinterpret_cast<const float4*>(s_inv + 4 * g);
            const float4 inv = make_float4(__fmul_rn(inv0.x, shrink), __fmul_rn(inv0.y, shrink),
                                           __fmul_rn(inv0.z, shrink), __fmul_rn(inv0.w, shrink));
            // floor(x) for 0 <= x <= 255 without the quarter-rate F2I:
            // x + 2^23 rounded down has ulp 1, so its low byte is floor(x)
            auto q8 = [&](float L, float m, float ivs) -> uint32_t {
                const float x = fminf(__fmul_rn(__fsub_rn(L, m), ivs), 255.f);
                return __float_as_uint(__fadd_rd(x, 8388608.f));
            };
#pragma unroll 2
            for (int rq = t >> 2; rq < M * KS / 4; rq += NC / 4) {
                const float4 mn = *reinterpret_cast<const float4*>(s_min + (rq >> 6) * QT + 4 * g);
                uint32_t rw[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float4 v = lut4[(4 * rq + i) * 4 + g];
                    const uint32_t p01 = __byte_perm(q8(v.x, mn.x, inv.x), q8(v.y, mn.y, inv.y), 0x0040);
                    const uint32_t p23 = __byte_perm(q8(v.z, mn.z, inv.z), q8(v.w, mn.w, inv.w), 0x0040);
                    rw[i] = __byte_perm(p01, p23, 0x5410);
                }
                q8_put_rows(block, g, rq, rw[0], rw[1], rw[2], rw[3]);
            }
            }  // store_block
        }
#ifdef LP_NOSAMPLE  // timing experiment only
        if (false) {
#else
        if (sampling && mt.smin) {
#endif
            // entries i = si * smin of the list; query lane k samples those with
            // si % 2^sshift_k == 0 into its slot si >> sshift_k (i / its stride)
            const uint32_t smin = mt.smin;
            const uint32_t ns = (mt.e1 + smin - 1) / smin;
            const u64* lcodes = reinterpret_cast<const u64*>(a.codes) + a.list_off[mt.l];
            const u64* sc = scodes + b * SCAP;
            // An item of a small batch holds one or two probing queries: with
            // <= 4 live lanes (all in quad 0) every lane of a warp takes its
            // own sample for that quad (32 samples per warp step instead of 8
            // samples x 4 quads, three of them dead).  Codes are loaded four
            // steps ahead: past the staged ones they are random DRAM sectors.
            const bool narrow = mt.nqi <= 4;
            const int my_qd = narrow ? 0 : qd;
            const uint32_t nslot = narrow ? 32u : 8u;
            const uint32_t step = NCW * nslot;
            unsigned long long sbase[4];
            bool sw[4];
            uint32_t sh[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int qq = my_qd * 4 + kk;
                sw[kk] = mt.q[qq] >= 0 && mt.samp[qq];
                sbase[kk] = mt.sbase[qq];
                sh[kk] = mt.sshift[qq];
            }
            constexpr int SU = 4;
            for (uint32_t si0 = warp * nslot + (narrow ? (uint32_t)lane : (uint32_t)slot); si0 < ns;
                 si0 += SU * step) {
                u64 code[SU];
#pragma unroll
                for (int u = 0; u < SU; ++u) {
                    const uint32_t si = si0 + u * step;
                    code[u] = si >= ns ? 0ull
                                       : (si < (uint32_t)SCAP ? sc[si] : __ldg(lcodes + sample_pos(si, smin, mt.e1)));
                }
#pragma unroll
                for (int u = 0; u < SU; ++u) {
                    const uint32_t si = si0 + u * step;
                    if (si >= ns) break;
                    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int j = 0; j < M; ++j) {
                        const uint32_t cj = (uint32_t)(code[u] >> (8 * j)) & 0xffu;
                        const float4 v = lut4[(j * KS + cj) * (QT / 4) + my_qd];
                        acc[0] = __fadd_rn(acc[0], v.x);
                        acc[1] = __fadd_rn(acc[1], v.y);
                        acc[2] = __fadd_rn(acc[2], v.z);
                        acc[3] = __fadd_rn(acc[3], v.w);
                    }
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        if (sw[kk] && (si & ((1u << sh[kk]) - 1u)) == 0u)
                            a.sample_dist[sbase[kk] + (si >> sh[kk])] = acc[kk];
                }
            }
        }
        csync();  // all consumers are done with xr[b], meta[b], scodes[b] and the LUT
        if (threadIdx.x == 0) mbar_arrive(&empty_bar[b]);
    }
}

template <int DSUB>
void lut_pass_t(const ScanArgs& a, cudaStream_t s) {
    const size_t ring = (size_t)RING * KS * DSUB * sizeof(float);
    const size_t smem = (size_t)LUT_FLOATS * sizeof(float) + 2 * (size_t)xbuf((int)a.d + 4) * sizeof(float) +
                        (size_t)(QT + 1) * a.d * sizeof(float) + 2 * (size_t)SCAP * sizeof(u64) + ring;
    set_max_smem((const void*)lut_pass_kernel<DSUB>, (size_t)((int)smem));
    lut_pass_kernel<DSUB><<<sm_count(), NTH, smem, s>>>(a, kNegZero2);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace

bool lut_pass_supported(uint32_t d, uint32_t m, uint32_t ks) {
    if (m != M || ks != KS) return false;
    const uint32_t ds = d / m;
    if (ds != 4 && ds != 8 && ds != 16) return false;
    const size_t ring = (size_t)RING * KS * ds * sizeof(float);
    const size_t smem = (size_t)LUT_FLOATS * 4 + 2 * (size_t)xbuf((int)d + 4) * 4 + (size_t)(QT + 1) * d * 4 +
                        2 * (size_t)SCAP * 8 + ring;
    return smem <= 220 * 1024;
}

void launch_lut_pass(const ScanArgs& a, cudaStream_t s) {
    switch (a.d / a.m) {
        case 16: return lut_pass_t<16>(a, s);
        case 8: return lut_pass_t<8>(a, s);
        case 4: return lut_pass_t<4>(a, s);
        default: throw ArgError("LUT pass supports d/m in {4, 8, 16}");
    }
}

}  // namespace pqrr_b200
