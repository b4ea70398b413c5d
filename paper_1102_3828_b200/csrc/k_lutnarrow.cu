// k_lutnarrow.cu — K2, the LUT pass (build_lut, product_quantizer.hpp:48-49;
// adc_distance, :53-57; ivf_search, ivf_index.hpp:58-61) for SMALL batches.
//
// lut_pass_kernel (k_lutpass.cu) builds the LUTs of up to 16 queries that probe
// one list side by side: 128 KiB of LUT in shared memory, the code book
// streamed past it through a TMA ring.  A serving batch of 1-64 queries has
// about one probing query per list, so 15 of the 16 lanes are dead and an item
// still costs the 8 code-book slices through the ring plus the hand-overs
// between the specialised warps (measured: 12-20 us per item at C5, of which
// arithmetic is a small part).  Here the roles flip: the CODE BOOK is resident
// (128 KiB per CTA, loaded once, 16-byte chunks swizzled so a warp's 32 rows
// hit 8 bank groups evenly) and the LUT is two query lanes wide (16 KiB); an
// item with more lanes is processed two lanes at a time.  Per item a CTA
// gathers the metadata, forms the residual queries x - C_l, builds the exact
// LUT in the reference order, quantises it into the item's 8-bit block (the
// live lanes' columns of the lane-major layout K4f reads, q8_put_rows) and
// computes the exact ADC distance of the sampled entries.  Same values, same
// positions, same layouts as lut_pass_kernel — the two kernels are
// interchangeable per launch and chosen by batch size.
#include <float.h>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int M = 8;
constexpr int KS = 256;
constexpr int QT = kQT;
constexpr int DSUB = 16;
constexpr int D = M * DSUB;
constexpr int NT = 512;  // NG groups of NT / NG threads share the resident code book, each on its own item
constexpr int LANE_WORDS = M * KS / 4;  // one lane's 8-bit column (2 KiB)
constexpr int Q8_BYTES = M * KS * QT;

struct NarrowMeta {
    uint32_t it, l, len, nqi, smin;
    int q[QT];
    unsigned long long sbase[QT];
    uint8_t samp[QT], sshift[QT];
};

// chunk c (16 B) of code-book row r (64 B) lives at chunk (c + (r >> 1)) & 3:
// rows r .. r + 7 at one chunk index then cover 8 distinct 16-byte bank groups
__device__ __forceinline__ int book_chunk(int r, int c) { return (c + (r >> 1)) & 3; }

template <int NG>
__global__ __launch_bounds__(NT, 1) void lut_pass_narrow_kernel(const ScanArgs a, const u64 nz) {
    constexpr int GT = NT / NG;
    extern __shared__ float4 nl_smem[];
    float* book = reinterpret_cast<float*>(nl_smem);  // [M * KS][16], chunk-swizzled
    // NG = 2: two groups of 256 threads walk the items independently (named
    // barriers): an item is a chain of dependent loads (claim -> item -> pairs
    // -> rows, then the sampled codes at DRAM latency) with little arithmetic,
    // so two items in flight per SM overlap each other's latencies (C5 batch
    // 16: 0.494 -> 0.470 ms).  NG = 1 when there are no more items than SMs
    // (one query: the whole CTA on its one item).
    const int g = threadIdx.x / GT, t = threadIdx.x % GT, lane = t & 31;
    float* lut = book + M * KS * DSUB + g * (M * KS * 2);              // per group [M * KS][2]
    float* xr = book + M * KS * DSUB + NG * (M * KS * 2) + g * 2 * D;  // per group [2][D] residual queries
    __shared__ NarrowMeta mt_all[NG];
    __shared__ unsigned s_mnu_all[NG][M * 2], s_mxu_all[NG][M * 2];
    __shared__ float s_min_all[NG][M * 2], s_inv_all[NG][2];
    NarrowMeta& mt = mt_all[g];
    unsigned* s_mnu = s_mnu_all[g];
    unsigned* s_mxu = s_mxu_all[g];
    float* s_min = s_min_all[g];
    float* s_inv = s_inv_all[g];
    auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(GT) : "memory"); };
    const uint32_t n_items = *a.num_items;
    // the code book, once per CTA
    for (int i = threadIdx.x; i < M * KS * 4; i += NT) {
        const int r = i >> 2, c = i & 3;
        *reinterpret_cast<float4*>(book + r * DSUB + 4 * book_chunk(r & (KS - 1), c)) =
            __ldg(reinterpret_cast<const float4*>(a.books) + i);
    }
    __syncthreads();
    const bool sampling = a.sample_dist != nullptr;
    for (;;) {
        gsync();  // the previous item is done with mt / lut / xr
        if (t < 32) {
            // ---- claim an item and gather its metadata (one warp)
            uint32_t c = 0;
            if (lane == 0) c = atomicAdd(a.item_counter, 1u);
            c = __shfl_sync(0xffffffffu, c, 0);
            if (c >= n_items) {
                if (lane == 0) mt.it = 0xffffffffu;
            } else {
                const uint32_t it = a.item_order[c];
                const uint32_t l = a.item_list[it], start = a.item_start[it], nqi = a.item_nq[it];
                int q = -1;
                uint32_t p = 0;
                if (lane < QT && (uint32_t)lane < nqi) {
                    p = a.pair_sorted[start + lane];
                    q = (int)(p / a.w);
                }
                const uint8_t sm = (q >= 0 && a.query_sampled && sampling) ? a.query_sampled[q] : 0;
                const uint32_t tier = q >= 0 ? tier_shift(sample_tier(p % a.w, a.w, a.tiered), a.w) : 31u;
                uint32_t tmin = sm ? tier : 31u;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
                if (lane < QT) {
                    mt.q[lane] = q;
                    mt.samp[lane] = sm;
                    mt.sbase[lane] = sm ? a.sample_off[p] : 0ull;
                    mt.sshift[lane] = (uint8_t)(sm ? tier - tmin : 0u);
                }
                if (lane == 0) {
                    mt.it = it;
                    mt.l = l;
                    mt.len = a.item_e1[it];  // LUT-pass items cover whole lists (e0 == 0)
                    mt.nqi = nqi;
                    mt.smin = tmin < 31u ? (a.stride << tmin) : 0u;
                }
            }
        }
        gsync();
        const uint32_t it = mt.it;
        if (it == 0xffffffffu) break;
        const uint32_t l = mt.l, len = mt.len, nqi = mt.nqi;
        const u64* lcodes = reinterpret_cast<const u64*>(a.codes) + a.list_off[l];
        for (uint32_t lp = 0; lp < nqi; lp += 2) {
            if (lp) gsync();  // the previous lane pair is done with lut / xr
            // ---- residual queries x - C_l (ivf_index.hpp:58-59) of lanes lp, lp + 1
            if (t < 2 * D) {
                const int k = t / D, e = t % D, q = lp + k < nqi ? mt.q[lp + k] : -1;
                xr[t] = q >= 0 ? __fsub_rn(a.xq[(size_t)q * D + e], a.coarse[(size_t)l * D + e]) : 0.f;
            }
            if (t < M * 2) {
                s_mnu[t] = 0x7f800000u;
                s_mxu[t] = 0u;
            }
            gsync();
            // ---- exact LUT in the reference order: thread = 8 (j, code) entries x 2 lanes
#pragma unroll
            for (int r = 0; r < M * KS / GT; ++r) {
                const int idx = t + GT * r, j = idx >> 8, i = idx & (KS - 1);
                const float* brow = book + idx * DSUB;
                u64 sa01 = 0, sa23 = 0, sb01 = 0, sb23 = 0;
#pragma unroll
                for (int t4 = 0; t4 < DSUB / 4; ++t4) {
                    const ulonglong2 c = *reinterpret_cast<const ulonglong2*>(brow + 4 * book_chunk(i, t4));
                    const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(xr + j * DSUB + 4 * t4);
                    const ulonglong2 w2 = *reinterpret_cast<const ulonglong2*>(xr + D + j * DSUB + 4 * t4);
                    if (t4 == 0) {  // 0 + x == x for the rounded square x >= +0
                        sa01 = sq2(sub2(u.x, c.x), nz);
                        sa23 = sq2(sub2(u.y, c.y), nz);
                        sb01 = sq2(sub2(w2.x, c.x), nz);
                        sb23 = sq2(sub2(w2.y, c.y), nz);
                    } else {
                        sa01 = acc_sq2(sa01, u.x, c.x, nz);
                        sa23 = acc_sq2(sa23, u.y, c.y, nz);
                        sb01 = acc_sq2(sb01, w2.x, c.x, nz);
                        sb23 = acc_sq2(sb23, w2.y, c.y, nz);
                    }
                }
                const float va = __fadd_rn(__fadd_rn(lo2(sa01), hi2(sa01)), __fadd_rn(lo2(sa23), hi2(sa23)));
                const float vb = __fadd_rn(__fadd_rn(lo2(sb01), hi2(sb01)), __fadd_rn(lo2(sb23), hi2(sb23)));
                *reinterpret_cast<float2*>(lut + idx * 2) = make_float2(va, vb);
                // (a warp's 32 entries share j) per-(j, lane) minimum / maximum
                float mna = va, mxa = va, mnb = vb, mxb = vb;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mna = fminf(mna, __shfl_xor_sync(0xffffffffu, mna, o));
                    mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, o));
                    mnb = fminf(mnb, __shfl_xor_sync(0xffffffffu, mnb, o));
                    mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, o));
                }
                if (lane == 0) {
                    atomicMin(s_mnu + j * 2, __float_as_uint(mna));
                    atomicMax(s_mxu + j * 2, __float_as_uint(mxa));
                    atomicMin(s_mnu + j * 2 + 1, __float_as_uint(mnb));
                    atomicMax(s_mxu + j * 2 + 1, __float_as_uint(mxb));
                }
            }
            gsync();
            // ---- 8-bit block of the live lanes (quantize as lut_pass_kernel)
            if (a.q8_param) {
                if (t < 2) {
                    float rng = 0.f, sm = 0.f;
#pragma unroll
                    for (int jj = 0; jj < M; ++jj) {
                        const float mn = __uint_as_float(s_mnu[jj * 2 + t]), mx = __uint_as_float(s_mxu[jj * 2 + t]);
                        s_min[jj * 2 + t] = mn;
                        rng = fmaxf(rng, __fsub_rn(mx, mn));
                        sm = __fadd_rn(sm, mn);
                    }
                    const float sc = __fdiv_rn(rng, 255.f);
                    s_inv[t] = sc > 0.f ? __frcp_rn(sc) : 0.f;
                    if (lp + t < nqi) {
                        float* prm = a.q8_param + (size_t)it * 2 * QT + 2 * (lp + t);
                        prm[0] = sc;
                        prm[1] = sm;
                    }
                }
                gsync();
                if (a.q8_cache) {
                    uint32_t* block = reinterpret_cast<uint32_t*>(a.q8_cache + (size_t)it * Q8_BYTES);
                    const float shrink = 0.99999904632568359375f;  // 1 - 2^-20 (see lut_pass_kernel)
                    auto q8 = [&](float L, float m, float ivs) -> uint32_t {
                        const float x = fminf(__fmul_rn(__fsub_rn(L, m), ivs), 255.f);
                        return __float_as_uint(__fadd_rd(x, 8388608.f)) & 0xffu;
                    };
                    // word rq of a lane's column = rows 4 rq .. 4 rq + 3 (row = j * KS + code)
                    for (int wd = t; wd < 2 * LANE_WORDS; wd += GT) {
                        const int k = wd / LANE_WORDS, rq = wd % LANE_WORDS;
                        if (lp + k >= nqi) continue;
                        const int j = (4 * rq) >> 8;
                        const float mn = s_min[j * 2 + k], ivs = __fmul_rn(s_inv[k], shrink);
                        uint32_t word = 0;
#pragma unroll
                        for (int b = 0; b < 4; ++b) word |= q8(lut[(4 * rq + b) * 2 + k], mn, ivs) << (8 * b);
                        block[(lp + k) * LANE_WORDS + rq] = word;
                    }
                }
            }
            // ---- exact ADC of the sampled entries (positions as lut_pass_kernel:
            // entry sample_pos(s << sshift, smin) for the lane's slot s)
            if (sampling && mt.smin) {
                const uint32_t smin = mt.smin;
                constexpr int SU = 8;  // codes in flight per thread: random DRAM sectors, nothing else hides them
                const bool s0 = mt.samp[lp], s1 = lp + 1 < nqi && mt.samp[lp + 1];
                if (s0 && s1 && mt.sshift[lp] == mt.sshift[lp + 1]) {
                    // both lanes at the same stride (two queries at the same probe
                    // tier): one code per slot serves both
                    const uint32_t sh = mt.sshift[lp];
                    const uint32_t st = smin << sh, ns = (len + st - 1) / st;
                    float* out0 = a.sample_dist + mt.sbase[lp];
                    float* out1 = a.sample_dist + mt.sbase[lp + 1];
                    for (uint32_t sb = t; sb < ns; sb += SU * GT) {
                        u64 code[SU];
#pragma unroll
                        for (int u = 0; u < SU; ++u) {
                            const uint32_t s = sb + u * GT;
                            code[u] = s < ns ? __ldg(lcodes + sample_pos(s << sh, smin, len)) : 0ull;
                        }
#pragma unroll
                        for (int u = 0; u < SU; ++u) {
                            const uint32_t s = sb + u * GT;
                            if (s >= ns) break;
                            float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
                            for (int j = 0; j < M; ++j) {
                                const float2 v = *reinterpret_cast<const float2*>(
                                    lut + (j * KS + ((uint32_t)(code[u] >> (8 * j)) & 0xffu)) * 2);
                                acc0 = __fadd_rn(acc0, v.x);
                                acc1 = __fadd_rn(acc1, v.y);
                            }
                            out0[s] = acc0;
                            out1[s] = acc1;
                        }
                    }
                } else {
                    for (int k = 0; k < 2 && lp + k < nqi; ++k) {
                        if (!mt.samp[lp + k]) continue;
                        const uint32_t sh = mt.sshift[lp + k];
                        const uint32_t st = smin << sh, ns = (len + st - 1) / st;
                        float* out = a.sample_dist + mt.sbase[lp + k];
                        for (uint32_t sb = t; sb < ns; sb += SU * GT) {
                            u64 code[SU];
#pragma unroll
                            for (int u = 0; u < SU; ++u) {
                                const uint32_t s = sb + u * GT;
                                code[u] = s < ns ? __ldg(lcodes + sample_pos(s << sh, smin, len)) : 0ull;
                            }
#pragma unroll
                            for (int u = 0; u < SU; ++u) {
                                const uint32_t s = sb + u * GT;
                                if (s >= ns) break;
                                float acc = 0.f;
#pragma unroll
                                for (int j = 0; j < M; ++j)
                                    acc = __fadd_rn(acc, lut[(j * KS + ((uint32_t)(code[u] >> (8 * j)) & 0xffu)) * 2 + k]);
                                out[s] = acc;
                            }
                        }
                    }
                }
            }
        }
    }
}

}  // namespace

bool lut_pass_narrow_supported(uint32_t d, uint32_t m, uint32_t ks) { return d == D && m == M && ks == KS; }

void launch_lut_pass_narrow(const ScanArgs& a, cudaStream_t s, size_t max_items) {
    if (!lut_pass_narrow_supported(a.d, a.m, a.ks)) throw ArgError("narrow LUT pass supports d = 128, m = 8, ks = 256");
    if (a.q8_mode || a.skip_dead) throw ArgError("narrow LUT pass: single-phase only");
    const int ng = max_items <= (size_t)sm_count() ? 1 : 2;
    const size_t smem = ((size_t)M * KS * DSUB + (size_t)ng * (M * KS * 2 + 2 * D)) * sizeof(float);
    if (ng == 1) {
        set_max_smem((const void*)lut_pass_narrow_kernel<1>, smem);
        lut_pass_narrow_kernel<1><<<sm_count(), NT, smem, s>>>(a, kNegZero2);
    } else {
        set_max_smem((const void*)lut_pass_narrow_kernel<2>, smem);
        lut_pass_narrow_kernel<2><<<sm_count(), NT, smem, s>>>(a, kNegZero2);
    }
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
