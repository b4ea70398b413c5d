// k_scan.cu — K2 + K4: per-(list, query-group) LUT construction in shared
// memory fused with the ADC list scan (ivf_search's hot loop,
// ivf_index.hpp:58-61; adc_distance, product_quantizer.hpp:53-57).
//
// List-major, query-lane design.  A work item is one inverted list and up to
// 16 queries that probe it.  The CTA builds the 16 residual LUTs
// LUT[j][i][q] = l2_sq(x_q^j - C_l^j, B_j[i]) (query index fastest, 128 KiB),
// then streams the list's 8-byte codes once for all 16 queries: a warp covers
// 8 entries x 16 queries per step, each lane owning one entry and 4 queries,
// so every lookup is one LDS.128 returning 4 queries' table values.  Codes are
// read from HBM once per 16 queries instead of once per query; the kernel is
// bound by shared-memory LUT gathers (SURVEY.md §7 "Hard parts").
//
// ADC sums are j-ascending fp32 adds (acc = 0; acc += LUT[j][c_j]), bit-equal
// to the reference.  Candidates at or below the query's threshold tau_q are
// appended (dist, position) to the query's buffer with warp-aggregated
// atomics.  Sample mode (stride > 1) writes every stride-th entry's distance
// to a per-(query, probe) slot instead; it feeds the threshold estimate.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int M = 8;
constexpr int KS = 256;
constexpr int QT = kQT;
constexpr int NT = kScanThreads;
constexpr int NW = NT / 32;
constexpr int LUT_FLOATS = M * KS * QT;  // 32768 floats = 128 KiB

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Sub-codebook j (KS x DSUB floats) -> smem buffer, 16 B per cp.async.
template <int DSUB>
__device__ __forceinline__ void stage_book(float* __restrict__ dst, const float* __restrict__ books,
                                           int j) {
    constexpr int CH = KS * DSUB / 4;  // 16-byte chunks
    const float* src = books + (size_t)j * KS * DSUB;
    for (int c = threadIdx.x; c < CH; c += NT) cp_async16(dst + 4 * c, src + 4 * c);
    cp_async_commit();
}

// LUT[j][i][q] for the item's 16 queries.  B_j is double-buffered in shared
// memory (cp.async of B_{j+1} overlaps the arithmetic of j); every warp reads 2
// distinct centroid rows per LDS.128 (broadcast) and writes 32 contiguous LUT
// words.  The first square of each accumulator is not added to +0: 0 + x == x
// exactly for the x >= +0 a rounded square is.  With MM, the minimum and
// maximum of every (j, query lane) sub-table are reduced on the fly into
// s_mnu / s_mxu (float bits; the values are >= +0, so the bit patterns order
// like the values).
template <int DSUB, bool MM>
__device__ __forceinline__ void build_luts(float* __restrict__ lut, const float* __restrict__ xr,
                                           int xld, const float* __restrict__ books,
                                           float* __restrict__ bbuf, u64 nz,
                                           unsigned* __restrict__ s_mnu = nullptr,
                                           unsigned* __restrict__ s_mxu = nullptr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int qq = lane & 15, ih = lane >> 4;
    constexpr int BF = KS * DSUB;
    stage_book<DSUB>(bbuf, books, 0);
#pragma unroll 1
    for (int j = 0; j < M; ++j) {
        if (j + 1 < M) {
            stage_book<DSUB>(bbuf + ((j + 1) & 1) * BF, books, j + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float* bj = bbuf + (j & 1) * BF;
        float r[DSUB];
#pragma unroll
        for (int t = 0; t < DSUB; t += 4) {
            float4 v = *reinterpret_cast<const float4*>(xr + qq * xld + j * DSUB + t);
            r[t] = v.x; r[t + 1] = v.y; r[t + 2] = v.z; r[t + 3] = v.w;
        }
        float mn = __int_as_float(0x7f800000), mx = 0.f;
#pragma unroll
        for (int ib = 0; ib < KS / (2 * NW); ++ib) {
            const int i = (ib * NW + warp) * 2 + ih;
            const float* b = bj + i * DSUB;
            u64 s01 = 0, s23 = 0;
#pragma unroll
            for (int t = 0; t < DSUB; t += 4) {
                const float4 c = *reinterpret_cast<const float4*>(b + t);
                if (t == 0) {
                    s01 = sq2(sub2(pk2(r[t], r[t + 1]), pk2(c.x, c.y)), nz);
                    s23 = sq2(sub2(pk2(r[t + 2], r[t + 3]), pk2(c.z, c.w)), nz);
                } else {
                    s01 = acc_sq2(s01, pk2(r[t], r[t + 1]), pk2(c.x, c.y), nz);
                    s23 = acc_sq2(s23, pk2(r[t + 2], r[t + 3]), pk2(c.z, c.w), nz);
                }
            }
            const float v = __fadd_rn(__fadd_rn(lo2(s01), hi2(s01)), __fadd_rn(lo2(s23), hi2(s23)));
            lut[(j * KS + i) * QT + qq] = v;
            if (MM) {
                mn = fminf(mn, v);
                mx = fmaxf(mx, v);
            }
        }
        if (MM) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, 16));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
            if (ih == 0) {
                atomicMin(s_mnu + j * QT + qq, __float_as_uint(mn));
                atomicMax(s_mxu + j * QT + qq, __float_as_uint(mx));
            }
        }
        __syncthreads();  // buffer (j & 1) is refilled by the prefetch of j + 2
    }
}

// Plain per-lane append (hits are rare after the threshold: ~2k' per query).
__device__ __forceinline__ void emit1(bool hit, int q, float dist, uint32_t pos,
                                      uint32_t* __restrict__ cnt, float* __restrict__ cdist,
                                      uint32_t* __restrict__ cpos, uint32_t cap) {
    if (!hit) return;
    const unsigned slot = atomicAdd(cnt + q, 1u);
    if (slot < cap) {
        cdist[(size_t)q * cap + slot] = dist;
        cpos[(size_t)q * cap + slot] = pos;
    }
}

// Per (query lane, subspace) minimum and range of the item's exact LUT, then
// the 8-bit LUT the K4f filter derives its 4-bit tables from:
//   v8 = min(255, floor((L - min_j) / s)),  s = max_j range_j / 255
// computed so that v8 * s <= L - min_j holds in exact arithmetic (the
// (1 - 2^-20) factor covers the three roundings), which keeps the filter's
// lower bound conservative.  The block goes to q8 (32 KiB) through `stage`;
// per query lane (s, sum_j min_j) goes to param.
__device__ __forceinline__ void quantize_item(const float* __restrict__ lut, uint32_t* __restrict__ stage,
                                              const unsigned* __restrict__ s_mnu,
                                              const unsigned* __restrict__ s_mxu,
                                              float* __restrict__ s_min, float* __restrict__ s_rng,
                                              float* __restrict__ s_inv, float* __restrict__ param) {
    const int t = threadIdx.x;
    if (t < M * QT) {
        const float mn = __uint_as_float(s_mnu[t]), mx = __uint_as_float(s_mxu[t]);
        s_min[t] = mn;  // [j][q]
        s_rng[t] = __fsub_rn(mx, mn);
    }
    __syncthreads();
    if (t < QT) {
        float rng = 0.f, sm = 0.f;
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
            rng = fmaxf(rng, s_rng[jj * 16 + t]);
            sm = __fadd_rn(sm, s_min[jj * 16 + t]);
        }
        const float sc = __fdiv_rn(rng, 255.f);
        s_inv[t] = sc > 0.f ? __frcp_rn(sc) : 0.f;
        param[2 * t] = sc;
        param[2 * t + 1] = sm;
    }
    __syncthreads();
    const float4* lut4 = reinterpret_cast<const float4*>(lut);
    const int g = t & 3;
    const float4 inv = *reinterpret_cast<const float4*>(s_inv + 4 * g);
    const float shrink = 0.99999904632568359375f;  // 1 - 2^-20
    auto q8 = [&](float L, float m, float iv) -> uint32_t {
        const float x = fminf(__fmul_rn(__fmul_rn(__fsub_rn(L, m), iv), shrink), 255.f);
        return __float2uint_rz(x);
    };
    // lane-major block (q8_put_rows), staged in shared memory for the bulk store
    for (int rq = t >> 2; rq < M * KS / 4; rq += NT / 4) {
        const float4 mn = *reinterpret_cast<const float4*>(s_min + (rq >> 6) * 16 + 4 * g);
        uint32_t rw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float4 v = lut4[(4 * rq + i) * 4 + g];
            rw[i] = q8(v.x, mn.x, inv.x) | (q8(v.y, mn.y, inv.y) << 8) | (q8(v.z, mn.z, inv.z) << 16) |
                    (q8(v.w, mn.w, inv.w) << 24);
        }
        q8_put_rows(stage, g, rq, rw[0], rw[1], rw[2], rw[3]);
    }
}

template <int DSUB>
__global__ __launch_bounds__(NT, 1) void ivf_scan_kernel(const ScanArgs a, const u64 nz) {
    extern __shared__ float4 smem4[];
    float* lut = reinterpret_cast<float*>(smem4);
    const int xld = (int)a.d + 4;
    float* xr = lut + LUT_FLOATS;         // [QT][d + 4]
    float* bbuf = xr + QT * xld;          // [2][KS][DSUB] sub-codebook ring; q8 staging after the build
    __shared__ uint32_t s_item;
    __shared__ int s_q[QT];
    __shared__ uint32_t s_pair[QT];
    __shared__ float s_tau[QT];
    __shared__ uint8_t s_samp[QT];
    __shared__ __align__(16) float s_min[M * QT], s_rng[M * QT], s_inv[QT];
    __shared__ unsigned s_mnu[M * QT], s_mxu[M * QT];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int slot = lane >> 2, qd = lane & 3;
    const uint32_t n_items = *a.num_items;
    const float4* lut4 = reinterpret_cast<const float4*>(lut);
    const bool store_q8 = a.pass == 1 && a.q8_cache != nullptr;

    for (;;) {
        if (threadIdx.x == 0) {
            const uint32_t c = atomicAdd(a.item_counter, 1u);
            s_item = c < n_items ? a.item_order[c] : 0xffffffffu;  // longest items first
            // the previous item's bulk q8 store must have read smem before reuse
            if (store_q8) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncthreads();
        const uint32_t it = s_item;
        if (it == 0xffffffffu) break;
        const uint32_t l = a.item_list[it];
        const uint32_t e0 = a.item_e0[it], e1 = a.item_e1[it];
        const uint32_t start = a.item_start[it];
        const uint32_t nqi = a.item_nq[it];
        if (threadIdx.x < QT) {
            int q = -1;
            uint32_t p = 0;
            if (threadIdx.x < nqi) {
                p = a.pair_sorted[start + threadIdx.x];
                q = (int)(p / a.w);
            }
            s_q[threadIdx.x] = q;
            s_pair[threadIdx.x] = p;
            s_tau[threadIdx.x] = (q >= 0 && a.pass == 0) ? a.tau[q] : -1.0f;
            s_samp[threadIdx.x] = (q >= 0 && a.query_sampled) ? a.query_sampled[q] : 0;
        }
        __syncthreads();
        {
            // residual queries x - C_l (ivf_index.hpp:58-59)
            const float* crow = a.coarse + (size_t)l * a.d;
            for (uint32_t idx = threadIdx.x; idx < QT * a.d; idx += NT) {
                const uint32_t qq = idx / a.d, t = idx % a.d;
                const int q = s_q[qq];
                xr[qq * xld + t] = q >= 0 ? __fsub_rn(a.xq[(size_t)q * a.d + t], crow[t]) : 0.f;
            }
            if (store_q8 && threadIdx.x < M * QT) {
                s_mnu[threadIdx.x] = 0x7f800000u;
                s_mxu[threadIdx.x] = 0u;
            }
            __syncthreads();
            if (store_q8) build_luts<DSUB, true>(lut, xr, xld, a.books, bbuf, nz, s_mnu, s_mxu);
            else build_luts<DSUB, false>(lut, xr, xld, a.books, bbuf, nz);
            if (store_q8) {
                uint32_t* stage = reinterpret_cast<uint32_t*>(bbuf);
                quantize_item(lut, stage, s_mnu, s_mxu, s_min, s_rng, s_inv, a.q8_param + (size_t)it * 2 * QT);
                // async TMA bulk store of the 32 KiB block; it overlaps this
                // item's sampled scan and is waited for (read side) before the
                // staging buffer is rewritten
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncthreads();
                if (threadIdx.x == 0) {
                    const unsigned src = (unsigned)__cvta_generic_to_shared(stage);
                    uint8_t* dst = a.q8_cache + (size_t)it * (M * KS * QT);
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                 ::"l"(dst), "r"(src), "r"((unsigned)(M * KS * QT)) : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
        }

        // this item's entry range [e0, e1) of the list (long lists are chunked)
        const uint64_t off = a.list_off[l] + e0;
        const uint32_t len = e1 - e0;
        const u64* codes = reinterpret_cast<const u64*>(a.codes) + off;
        int qk[4];
        float tk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            qk[k] = s_q[qd * 4 + k];
            tk[k] = s_tau[qd * 4 + k];
        }
        if (a.pass == 0) {
            // ---------------- main mode: threshold filter + append.  Codes are
            // prefetched PF steps ahead in registers so the L2/HBM latency of
            // the stream hides behind the LUT gathers of earlier steps.
            // Two entry-steps (A, B = A + S) per iteration: 8 independent
            // j-ordered FADD chains per lane and one vote per two steps.
            constexpr uint32_t S = NW * 8;  // entries per CTA step
            const uint32_t wbase = warp * 8;
            u64 nA = 0ull, nB = 0ull, fA = 0ull, fB = 0ull;
            {
                const uint32_t e = wbase + slot;
                nA = e < len ? __ldg(codes + e) : 0ull;
                nB = e + S < len ? __ldg(codes + e + S) : 0ull;
                fA = e + 2 * S < len ? __ldg(codes + e + 2 * S) : 0ull;
                fB = e + 3 * S < len ? __ldg(codes + e + 3 * S) : 0ull;
            }
            for (uint32_t wb = wbase; wb < len; wb += 2 * S) {
                const uint32_t eA = wb + slot, eB = eA + S;
                const bool vA = eA < len, vB = eB < len;
                const u64 cA = nA, cB = nB;
                nA = fA;
                nB = fB;
                fA = eA + 4 * S < len ? __ldg(codes + eA + 4 * S) : 0ull;
                fB = eB + 4 * S < len ? __ldg(codes + eB + 4 * S) : 0ull;
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
                float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    const uint32_t ca = (uint32_t)(cA >> (8 * j)) & 0xffu;
                    const uint32_t cb = (uint32_t)(cB >> (8 * j)) & 0xffu;
                    const float4 va = lut4[(j * KS + ca) * (QT / 4) + qd];
                    const float4 vb = lut4[(j * KS + cb) * (QT / 4) + qd];
                    a0 = __fadd_rn(a0, va.x);
                    a1 = __fadd_rn(a1, va.y);
                    a2 = __fadd_rn(a2, va.z);
                    a3 = __fadd_rn(a3, va.w);
                    b0 = __fadd_rn(b0, vb.x);
                    b1 = __fadd_rn(b1, vb.y);
                    b2 = __fadd_rn(b2, vb.z);
                    b3 = __fadd_rn(b3, vb.w);
                }
                const bool hA0 = vA && a0 <= tk[0], hA1 = vA && a1 <= tk[1];
                const bool hA2 = vA && a2 <= tk[2], hA3 = vA && a3 <= tk[3];
                const bool hB0 = vB && b0 <= tk[0], hB1 = vB && b1 <= tk[1];
                const bool hB2 = vB && b2 <= tk[2], hB3 = vB && b3 <= tk[3];
                if (__any_sync(0xffffffffu, hA0 | hA1 | hA2 | hA3 | hB0 | hB1 | hB2 | hB3)) {
                    const uint32_t pA = (uint32_t)(off + eA), pB = (uint32_t)(off + eB);
                    emit1(hA0, qk[0], a0, pA, a.cand_cnt, a.cand_dist, a.cand_pos, a.cap);
                    emit1(hA1, qk[1], a1, pA, a.cand_cnt, a.cand_dist, a.cand_pos, a.cap);
                    emit1(hA2, qk[2], a2, pA, a.cand_cnt, a.cand_dist, a.cand_pos, a.cap);
                    emit1(hA3, qk[3], a3, pA, a.cand_cnt, a.cand_dist, a.cand_pos, a.cap);
                    emit1(hB0, qk[0], b0, pB, a.cand_cnt, a.cand_dist, a.cand_pos, a.cap);
                    emit1(hB1, qk[1], b1, pB, a.cand_cnt, a.cand_dist, a.cand_pos, a.cap);
                    emit1(hB2, qk[2], b2, pB, a.cand_cnt, a.cand_dist, a.cand_pos, a.cap);
                    emit1(hB3, qk[3], b3, pB, a.cand_cnt, a.cand_dist, a.cand_pos, a.cap);
                }
            }
        } else if (a.sample_dist) {
            // ---------------- sample mode: every stride-th entry, fixed slots
            const uint32_t ns = (e1 + a.stride - 1) / a.stride - (e0 + a.stride - 1) / a.stride;
            uint64_t sbase[4];
            bool sw[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                sw[k] = qk[k] >= 0 && s_samp[qd * 4 + k];
                sbase[k] = sw[k] ? a.sample_off[s_pair[qd * 4 + k]] : 0;
            }
            // sampled entries of the chunk: global indices i * stride in [e0, e1),
            // written at their fixed per-(query, probe) slot i
            const uint32_t i0 = (e0 + a.stride - 1) / a.stride;
            const u64* lcodes = reinterpret_cast<const u64*>(a.codes) + a.list_off[l];
            constexpr uint32_t S = NW * 8;
            constexpr int PF = 4;
            const uint32_t wbase = warp * 8;
            u64 cbuf[PF];
#pragma unroll
            for (int k = 0; k < PF; ++k) {
                const uint32_t si = wbase + k * S + slot;
                cbuf[k] = si < ns ? __ldg(lcodes + sample_pos(i0 + si, a.stride, a.list_len[l])) : 0ull;
            }
            for (uint32_t wb = wbase; wb < ns; wb += PF * S) {
#pragma unroll
                for (int kk = 0; kk < PF; ++kk) {
                    const uint32_t sb = wb + kk * S;
                    if (sb >= ns) break;
                    const uint32_t si = sb + slot;
                    const u64 code = cbuf[kk];
                    const uint32_t sn = si + PF * S;
                    cbuf[kk] = sn < ns ? __ldg(lcodes + sample_pos(i0 + sn, a.stride, a.list_len[l])) : 0ull;
                    if (si >= ns) continue;
                    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int j = 0; j < M; ++j) {
                        const uint32_t c = (uint32_t)(code >> (8 * j)) & 0xffu;
                        const float4 v = lut4[(j * KS + c) * (QT / 4) + qd];
                        acc[0] = __fadd_rn(acc[0], v.x);
                        acc[1] = __fadd_rn(acc[1], v.y);
                        acc[2] = __fadd_rn(acc[2], v.z);
                        acc[3] = __fadd_rn(acc[3], v.w);
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (sw[k]) a.sample_dist[sbase[k] + i0 + si] = acc[k];
                }
            }
        }
        __syncthreads();
    }
    // drain outstanding bulk q8 stores before the CTA retires
    if (threadIdx.x == 0 && store_q8) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Kernel seam helpers (kernels::scan_topk / build_lut parity).
__global__ void lut_scan_all_kernel(const float* __restrict__ lut, uint32_t m, uint32_t ks,
                                    const uint8_t* __restrict__ codes, size_t n,
                                    float* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float acc = 0.f;
    for (uint32_t j = 0; j < m; ++j) acc = __fadd_rn(acc, lut[(size_t)j * ks + codes[i * m + j]]);
    out[i] = acc;
}

__global__ void build_lut_kernel(const float* __restrict__ xr, size_t nx, uint32_t d,
                                 const float* __restrict__ books, uint32_t m, uint32_t ks,
                                 float* __restrict__ out) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nx * m * ks) return;
    size_t v = idx / ((size_t)m * ks);
    uint32_t r = (uint32_t)(idx % ((size_t)m * ks));
    uint32_t j = r / ks, i = r % ks;
    uint32_t ds = d / m;
    out[idx] = l2sq_scalar(xr + v * d + (size_t)j * ds, books + ((size_t)j * ks + i) * ds, (int)ds);
}

// Work items: (list, group of <= qt probing queries, chunk of <= `chunk`
// entries).  Chunking bounds the longest item so the longest-first schedule
// leaves no tail of one huge list on one SM; it is used for the K4f items of
// small batches only (the LUT-pass items cover whole lists: chunks would
// rebuild the same LUT).

__global__ void items_per_list_kernel(const uint32_t* __restrict__ cnt,
                                      const uint32_t* __restrict__ len, uint32_t nlists,
                                      uint32_t* __restrict__ items, uint32_t qt, uint32_t chunk) {
    uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < nlists) {
        const uint32_t chunks = max(1u, (len[l] + chunk - 1) / chunk);
        items[l] = ((cnt[l] + qt - 1) / qt) * chunks;
    }
    if (l == nlists) items[l] = 0;
}

// One thread per item: its list by binary search over item_off (items of a
// list are contiguous: groups of qt pairs x entry chunks).
__global__ void items_build_kernel(const uint32_t* __restrict__ cnt,
                                   const uint32_t* __restrict__ first,
                                   const uint32_t* __restrict__ len, uint32_t nlists,
                                   const uint32_t* __restrict__ item_off,
                                   uint32_t* __restrict__ item_list, uint32_t* __restrict__ item_start,
                                   uint32_t* __restrict__ item_nq, uint32_t* __restrict__ item_e0,
                                   uint32_t* __restrict__ item_e1, uint32_t* __restrict__ sort_key,
                                   uint32_t qt, uint32_t chunk) {
    const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= item_off[nlists]) return;
    uint32_t lo = 0, hi = nlists;  // last list with item_off[l] <= o
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (item_off[mid] <= o) lo = mid;
        else hi = mid;
    }
    const uint32_t l = lo, c = cnt[l], L = len[l];
    const uint32_t chunks = max(1u, (L + chunk - 1) / chunk);
    const uint32_t k = o - item_off[l];
    const uint32_t grp = k / chunks, ch = k % chunks;
    const uint32_t e0 = ch * chunk, e1 = min(L, e0 + chunk);
    item_list[o] = l;
    item_start[o] = first[l] + grp * qt;
    item_nq[o] = min(qt, c - grp * qt);
    item_e0[o] = e0;
    item_e1[o] = e1;
    sort_key[o] = 0xffffffffu - (e1 - e0);  // ascending sort = longest first
}

template <int DSUB>
void scan_t(const ScanArgs& a, cudaStream_t s) {
    // the sub-codebook ring doubles as the 32 KiB q8 staging buffer
    const size_t ring = std::max<size_t>(2 * (size_t)KS * DSUB * sizeof(float), (size_t)M * KS * QT);
    const size_t smem = (size_t)LUT_FLOATS * sizeof(float) + (size_t)QT * (a.d + 4) * sizeof(float) + ring;
    set_max_smem((const void*)ivf_scan_kernel<DSUB>, (size_t)((int)smem));
    ivf_scan_kernel<DSUB><<<sm_count(), NT, smem, s>>>(a, kNegZero2);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace

void launch_ivf_scan(const ScanArgs& a, cudaStream_t s) {
    if (a.m != M || a.ks != KS) throw ArgError("device scan supports m = 8, ks = 256");
    switch (a.d / a.m) {
        case 16: return scan_t<16>(a, s);
        case 8: return scan_t<8>(a, s);
        case 4: return scan_t<4>(a, s);
        case 32: return scan_t<32>(a, s);
        default: throw ArgError("device scan supports d/m in {4, 8, 16, 32}");
    }
}

void launch_items_per_list(const uint32_t* list_cnt, const uint32_t* list_len, uint32_t nlists,
                           uint32_t* items, uint32_t qt, cudaStream_t s, uint32_t chunk) {
    items_per_list_kernel<<<(nlists + 1 + 255) / 256, 256, 0, s>>>(list_cnt, list_len, nlists, items,
                                                                   qt, chunk);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_items_build(const uint32_t* list_cnt, const uint32_t* list_first,
                        const uint32_t* list_len, uint32_t nlists, const uint32_t* item_off,
                        uint32_t* item_list, uint32_t* item_start, uint32_t* item_nq,
                        uint32_t* item_e0, uint32_t* item_e1, uint32_t* sort_key, uint32_t qt,
                        cudaStream_t s, uint32_t chunk, uint32_t n_items) {
    if (n_items == 0) return;
    items_build_kernel<<<(n_items + 255) / 256, 256, 0, s>>>(list_cnt, list_first, list_len, nlists,
                                                             item_off, item_list, item_start, item_nq,
                                                             item_e0, item_e1, sort_key, qt, chunk);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_lut_scan_all(const float* lut, uint32_t m, uint32_t ks, const uint8_t* codes, size_t n,
                         float* out_dist, cudaStream_t s) {
    if (n == 0) return;
    lut_scan_all_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lut, m, ks, codes, n, out_dist);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_build_lut(const float* xr, size_t nx, uint32_t d, const float* books, uint32_t m,
                      uint32_t ks, float* out, cudaStream_t s) {
    size_t total = nx * m * ks;
    if (!total) return;
    build_lut_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(xr, nx, d, books, m, ks, out);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
