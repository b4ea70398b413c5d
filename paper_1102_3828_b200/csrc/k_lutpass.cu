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
constexpr int NTH = NC + 32;      // + one producer warp
constexpr int LUT_FLOATS = M * KS * QT;
constexpr int Q8_BYTES = M * KS * QT;  // 32 KiB
constexpr int SCAP = 2048;             // sampled codes staged per item (more: read from global)

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

template <int DSUB>
__device__ __forceinline__ void stage_book(float* __restrict__ dst, const float* __restrict__ books, int j) {
    constexpr int CH = KS * DSUB / 4;
    const float* src = books + (size_t)j * KS * DSUB;
    for (int c = threadIdx.x; c < CH; c += NC) cp16(dst + 4 * c, src + 4 * c);
    cp_commit();
}

// Exact LUTs of the item (see build_luts in k_scan.cu; consumer threads only)
// with the per-(j, q) minimum / maximum reduced into s_mnu / s_mxu.
template <int DSUB>
__device__ __forceinline__ void build_luts_mm(float* __restrict__ lut, const float* __restrict__ xr,
                                              int xld, const float* __restrict__ books,
                                              float* __restrict__ bbuf, u64 nz, bool mm,
                                              unsigned* __restrict__ s_mnu, unsigned* __restrict__ s_mxu) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int qq = lane & 15, ih = lane >> 4;
    constexpr int BF = KS * DSUB;
    stage_book<DSUB>(bbuf, books, 0);
#pragma unroll 1
    for (int j = 0; j < M; ++j) {
        if (j + 1 < M) {
            stage_book<DSUB>(bbuf + ((j + 1) & 1) * BF, books, j + 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        csync();
        const float* bj = bbuf + (j & 1) * BF;
        // operands as packed f32x2 pairs: one 16-byte load gives (t, t+1) and
        // (t+2, t+3) ready for the packed arithmetic (LDS.128, not 2 x LDS.64)
        u64 r01[DSUB / 4], r23[DSUB / 4];
#pragma unroll
        for (int t4 = 0; t4 < DSUB / 4; ++t4) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(xr + qq * xld + j * DSUB + 4 * t4);
            r01[t4] = v.x;
            r23[t4] = v.y;
        }
        float mn = __int_as_float(0x7f800000), mx = 0.f;
#pragma unroll
        for (int ib = 0; ib < KS / (2 * NCW); ++ib) {
            const int i = (ib * NCW + warp) * 2 + ih;
            const ulonglong2* b = reinterpret_cast<const ulonglong2*>(bj + i * DSUB);
            u64 s01 = 0, s23 = 0;
#pragma unroll
            for (int t4 = 0; t4 < DSUB / 4; ++t4) {
                const ulonglong2 c = b[t4];
                if (t4 == 0) {  // 0 + x == x for the rounded square x >= +0
                    s01 = sq2(sub2(r01[t4], c.x), nz);
                    s23 = sq2(sub2(r23[t4], c.y), nz);
                } else {
                    s01 = acc_sq2(s01, r01[t4], c.x, nz);
                    s23 = acc_sq2(s23, r23[t4], c.y, nz);
                }
            }
            const float v = __fadd_rn(__fadd_rn(lo2(s01), hi2(s01)), __fadd_rn(lo2(s23), hi2(s23)));
            lut[(j * KS + i) * QT + qq] = v;
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
        if (mm) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, 16));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
            if (ih == 0) {
                atomicMin(s_mnu + j * QT + qq, __float_as_uint(mn));
                atomicMax(s_mxu + j * QT + qq, __float_as_uint(mx));
            }
        }
        csync();  // buffer (j & 1) is refilled by the prefetch of j + 2
    }
}

template <int DSUB>
__global__ __launch_bounds__(NTH, 1) void lut_pass_kernel(const ScanArgs a, const u64 nz) {
    extern __shared__ float4 smem4[];
    const int xld = (int)a.d + 4;
    float* lut = reinterpret_cast<float*>(smem4);
    float* xr0 = lut + LUT_FLOATS;                 // [2][QT][xld] residual queries
    float* raw = xr0 + 2 * QT * xld;               // [QT + 1][d] producer staging
    u64* scodes = reinterpret_cast<u64*>(raw + (QT + 1) * a.d);  // [2][SCAP] sampled codes
    float* bbuf = reinterpret_cast<float*>(scodes + 2 * SCAP);  // code-book ring / q8 staging
    __shared__ ItemMeta meta[2];
    __shared__ __align__(8) unsigned long long full_bar[2], empty_bar[2];
    __shared__ __align__(16) float s_min[M * QT], s_rng[M * QT], s_inv[QT];
    __shared__ unsigned s_mnu[M * QT], s_mxu[M * QT];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t n_items = *a.num_items;
    const bool store_q8 = a.q8_cache != nullptr;
    const bool sampling = a.sample_dist != nullptr;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full_bar[b], 1);
            mbar_init(&empty_bar[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {
        // ---------------------------------------------------------- producer
        for (uint32_t k = 0;; ++k) {
            const int b = k & 1;
            if (k >= 2) mbar_wait(&empty_bar[b], ((k >> 1) - 1) & 1);
            uint32_t c = 0;
            if (lane == 0) c = atomicAdd(a.item_counter, 1u);
            c = __shfl_sync(0xffffffffu, c, 0);
            ItemMeta& mt = meta[b];
            if (c >= n_items) {
                if (lane == 0) {
                    mt.it = 0xffffffffu;
                    mbar_arrive(&full_bar[b]);
                }
                break;
            }
            const uint32_t it = a.item_order[c];  // longest items first
            const uint32_t l = a.item_list[it];
            const uint32_t e0 = a.item_e0[it], e1 = a.item_e1[it];
            const uint32_t start = a.item_start[it], nqi = a.item_nq[it];
            int q = -1;
            uint32_t p = 0;
            if (lane < QT && (uint32_t)lane < nqi) {
                p = a.pair_sorted[start + lane];
                q = (int)(p / a.w);
            }
            // per-query sampling stride for this list (probe rank tier)
            const uint8_t sm = (q >= 0 && a.query_sampled) ? a.query_sampled[q] : 0;
            const uint32_t tier = (lane < QT && q >= 0) ? sample_tier(p % a.w, a.w, a.tiered) : 7u;
            uint32_t tmin = (sm && lane < QT) ? tier : 7u;
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
                mt.smin = tmin < 7u ? (a.stride << tmin) : 0u;
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
            if (sampling && tmin < 7u) {
                const uint32_t smin = a.stride << tmin;
                const uint32_t ns = (e1 + smin - 1) / smin;
                const u64* lcodes = reinterpret_cast<const u64*>(a.codes) + a.list_off[l];
                for (uint32_t si = lane; si < min(ns, (uint32_t)SCAP); si += 32)
                    cp8(scodes + b * SCAP + si, lcodes + (size_t)si * smin);
            }
            cp_commit();
            cp_wait<0>();
            __syncwarp();
            // residual queries x - C_l (ivf_index.hpp:58-59) into xr[b]
            float* xr = xr0 + b * QT * xld;
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
                *reinterpret_cast<float4*>(xr + r * xld + 4 * cc) = v;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_bar[b]);
        }
        return;
    }

    // -------------------------------------------------------------- consumers
    const int slot = lane >> 2, qd = lane & 3;
    const float4* lut4 = reinterpret_cast<const float4*>(lut);
    for (uint32_t k = 0;; ++k) {
        const int b = k & 1;
        mbar_wait(&full_bar[b], (k >> 1) & 1);
        const ItemMeta& mt = meta[b];
        const uint32_t it = mt.it;
        if (it == 0xffffffffu) break;
        if (threadIdx.x == 0 && store_q8)  // previous bulk store has read the staging buffer
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (store_q8 && threadIdx.x < M * QT) {
            s_mnu[threadIdx.x] = 0x7f800000u;
            s_mxu[threadIdx.x] = 0u;
        }
        csync();
        build_luts_mm<DSUB>(lut, xr0 + b * QT * xld, xld, a.books, bbuf, nz, store_q8, s_mnu, s_mxu);
        if (store_q8) {
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
            uint32_t* stage = reinterpret_cast<uint32_t*>(bbuf);
            const int g = t & 3;
            const float4 inv = *reinterpret_cast<const float4*>(s_inv + 4 * g);
            const float shrink = 0.99999904632568359375f;  // 1 - 2^-20
#pragma unroll 4
            for (int row = t >> 2; row < M * KS; row += NC / 4) {
                const float4 v = lut4[row * 4 + g];
                const float4 mn = *reinterpret_cast<const float4*>(s_min + (row >> 8) * QT + 4 * g);
                auto q8 = [&](float L, float m, float iv) -> uint32_t {
                    const float x = fminf(__fmul_rn(__fmul_rn(__fsub_rn(L, m), iv), shrink), 255.f);
                    return __float2uint_rz(x);
                };
                stage[row * 4 + g] = q8(v.x, mn.x, inv.x) | (q8(v.y, mn.y, inv.y) << 8) |
                                     (q8(v.z, mn.z, inv.z) << 16) | (q8(v.w, mn.w, inv.w) << 24);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            csync();
            if (threadIdx.x == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(a.q8_cache + (size_t)it * Q8_BYTES), "r"(smem_u32(stage)),
                             "r"((unsigned)Q8_BYTES) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
        if (sampling && mt.smin) {
            // entries i = si * smin of the list; query lane k samples those with
            // si % 2^sshift_k == 0 into its slot si >> sshift_k (i / its stride)
            const uint32_t smin = mt.smin;
            const uint32_t ns = (mt.e1 + smin - 1) / smin;
            const u64* lcodes = reinterpret_cast<const u64*>(a.codes) + a.list_off[mt.l];
            const u64* sc = scodes + b * SCAP;
            unsigned long long sbase[4];
            bool sw[4];
            uint32_t sh[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int qq = qd * 4 + kk;
                sw[kk] = mt.q[qq] >= 0 && mt.samp[qq];
                sbase[kk] = mt.sbase[qq];
                sh[kk] = mt.sshift[qq];
            }
            for (uint32_t si = warp * 8 + slot; si < ns; si += NCW * 8) {
                const u64 code = si < (uint32_t)SCAP ? sc[si] : __ldg(lcodes + (size_t)si * smin);
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    const uint32_t cj = (uint32_t)(code >> (8 * j)) & 0xffu;
                    const float4 v = lut4[(j * KS + cj) * (QT / 4) + qd];
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
        csync();  // all consumers are done with xr[b], meta[b], scodes[b] and the LUT
        if (threadIdx.x == 0) mbar_arrive(&empty_bar[b]);
    }
    if (threadIdx.x == 0 && store_q8) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int DSUB>
void lut_pass_t(const ScanArgs& a, cudaStream_t s) {
    const size_t ring = std::max<size_t>(2 * (size_t)KS * DSUB * sizeof(float), (size_t)Q8_BYTES);
    const size_t smem = (size_t)LUT_FLOATS * sizeof(float) + 2 * (size_t)QT * (a.d + 4) * sizeof(float) +
                        (size_t)(QT + 1) * a.d * sizeof(float) + 2 * (size_t)SCAP * sizeof(u64) + ring;
    PQRR_CUDA(cudaFuncSetAttribute(lut_pass_kernel<DSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    lut_pass_kernel<DSUB><<<sm_count(), NTH, smem, s>>>(a, kNegZero2);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace

bool lut_pass_supported(uint32_t d, uint32_t m, uint32_t ks) {
    if (m != M || ks != KS) return false;
    const uint32_t ds = d / m;
    if (ds != 4 && ds != 8 && ds != 16) return false;
    const size_t ring = std::max<size_t>(2 * (size_t)KS * ds * sizeof(float), (size_t)Q8_BYTES);
    const size_t smem = (size_t)LUT_FLOATS * 4 + 2 * (size_t)QT * (d + 4) * 4 + (size_t)(QT + 1) * d * 4 +
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
