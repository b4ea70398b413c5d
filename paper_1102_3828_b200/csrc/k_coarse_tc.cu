// k_coarse_tc.cu — K1 on the tensor cores with a certified exact result:
// the w nearest coarse centroids of every query (ivf_index.hpp:58, coarse
// probe selection; ties to the lowest index), exactly as the
// reference's l2_sq order ranks them.
//
// 1. coarse_gemm_kernel: D~[q][c] = |x_q|^2 + |c|^2 - 2 <x_q, c> with the dot
//    products on the tensor cores (mma.sync m16n8k8 TF32, fp32 accumulation).
//    The centroids round to TF32 (cvt.rna, relative 2^-11).  Queries from u8
//    are exact in TF32; float queries round too.  sum_i |x_i c_i| <=
//    (|x|^2 + |c|^2) / 2 bounds every error term: the operand rounding (2^-11
//    per rounded operand), the fp32 accumulation (< 2^-16), the epilogue and
//    the reference's own fp32 l2_sq (< 40 u), so
//        |D~ - d_ref| <= delta = 2^-10 (|x|^2 + |c|^2)   (u8 queries)
//        |D~ - d_ref| <= delta = 2^-9  (|x|^2 + |c|^2)   (any float query);
//    the certify kernel picks the scale per query by checking its components.
// 2. topw_certify_kernel (one query per warp): T~ >= the w-th smallest D~;
//    every true top-w centroid c has D~_c <= d_w + delta_c and
//    d_w <= T~ + delta_max, so the candidate set {c : D~_c <= T~ + 2 delta_max}
//    contains the exact top-w.  The candidates' exact distances are computed
//    in the reference order (l2sq_packed) and sorted by (dist, index).  A
//    candidate set larger than the buffer marks the query for the exact path.
#include <float.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int GM = 64;    // queries per CTA
constexpr int GN = 128;   // centroids per CTA
constexpr int GW = 8;     // warps: 16 queries x 64 centroids each (4 x 2 warp grid)
constexpr int GLD = 144;  // smem row stride (floats): conflict-free fragment loads

__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = valid ? 16 : 0;  // zero-fill rows past the end
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(sz));
}

// D = 128: one CTA = 64 queries x 128 centroids, all 128 dims staged at once.
// Lane (g, tig)'s k-slots (tig, tig + 4) of the k-step pair (2p, 2p + 1) carry
// the contiguous dims 16p + 4 tig .. + 3 of a row (one LDS.128 each for A and
// B); a dot product is independent of the k order as long as A and B agree.
__global__ __launch_bounds__(GW * 32) void coarse_gemm_kernel(const float* __restrict__ x, size_t nq,
                                                              const float* __restrict__ c, uint32_t nc,
                                                              const float* __restrict__ cnorm,
                                                              float* __restrict__ out) {
    constexpr int D = 128;
    extern __shared__ float4 sm_g[];
    float* As = reinterpret_cast<float*>(sm_g);  // [GM][GLD]
    float* Bs = As + GM * GLD;                   // [GN][GLD]
    __shared__ float s_nx[GM], s_nc[GN];
    const size_t q0 = (size_t)blockIdx.y * GM;
    const uint32_t c0 = blockIdx.x * GN;
    for (int i = threadIdx.x; i < GM * (D / 4); i += blockDim.x) {
        const int r = i / (D / 4), k = i % (D / 4);
        const bool v = q0 + r < nq;
        cp16(As + r * GLD + 4 * k, x + (v ? (q0 + r) * D : 0) + 4 * k, v);
    }
    for (int i = threadIdx.x; i < GN * (D / 4); i += blockDim.x) {
        const int r = i / (D / 4), k = i % (D / 4);
        const bool v = c0 + r < nc;
        cp16(Bs + r * GLD + 4 * k, c + (size_t)(v ? c0 + r : 0) * D + 4 * k, v);
    }
    asm volatile("cp.async.commit_group;");
    for (int i = threadIdx.x; i < GN; i += blockDim.x) s_nc[i] = c0 + i < nc ? cnorm[c0 + i] : 0.f;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < GM) {  // |x|^2 of the tile's queries
        const float* r = As + threadIdx.x * GLD;
        float acc = 0.f;
#pragma unroll 16
        for (int t = 0; t < D; ++t) acc = fmaf(r[t], r[t], acc);
        s_nx[threadIdx.x] = acc;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int m0 = (warp & 3) * 16, n0w = (warp >> 2) * (GN / 2);
    constexpr int NT = GN / 2 / 8;  // n-tiles per warp
    float acc[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
#pragma unroll
    for (int p = 0; p < D / 16; ++p) {
        const float4 a0 = *reinterpret_cast<const float4*>(As + (m0 + g) * GLD + 16 * p + 4 * tig);
        const float4 a1 = *reinterpret_cast<const float4*>(As + (m0 + g + 8) * GLD + 16 * p + 4 * tig);
        const uint32_t A0[4] = {to_tf32(a0.x), to_tf32(a1.x), to_tf32(a0.y), to_tf32(a1.y)};
        const uint32_t A1[4] = {to_tf32(a0.z), to_tf32(a1.z), to_tf32(a0.w), to_tf32(a1.w)};
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const float4 b = *reinterpret_cast<const float4*>(Bs + (n0w + t * 8 + g) * GLD + 16 * p + 4 * tig);
            mma_tf32(acc[t], A0, to_tf32(b.x), to_tf32(b.y));
            mma_tf32(acc[t], A1, to_tf32(b.z), to_tf32(b.w));
        }
    }
    // epilogue: acc[t][i] = <x_q, c> for q = m0 + g + 8 (i >> 1), c = 8 t + 2 tig + (i & 1)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int ql = m0 + g + 8 * h;
        const size_t q = q0 + ql;
        if (q >= nq) continue;
        const float nx = s_nx[ql];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int cl = n0w + t * 8 + 2 * tig;
            const float v0 = nx + s_nc[cl] - 2.f * acc[t][2 * h];
            const float v1 = nx + s_nc[cl + 1] - 2.f * acc[t][2 * h + 1];
            const uint32_t cc = c0 + cl;
            if (cc + 1 < nc) {
                *reinterpret_cast<float2*>(out + q * nc + cc) = make_float2(v0, v1);
            } else if (cc < nc) {
                out[q * nc + cc] = v0;
            }
        }
    }
}

__global__ void sq_norms_kernel(const float* __restrict__ c, uint32_t n, uint32_t d, float* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float acc = 0.f;
    for (uint32_t t = 0; t < d; ++t) acc = fmaf(c[(size_t)i * d + t], c[(size_t)i * d + t], acc);
    out[i] = acc;
}

constexpr int CW = 8;            // queries (warps) per CTA
constexpr uint32_t CCAP = 256;   // candidate buffer per query (more: exact path)
constexpr uint32_t SCAP = 512;   // staged (key, index) entries of the streaming select

// In-warp bitonic sort of n2 (power of two) 64-bit keys in shared memory.
__device__ __forceinline__ void wbitonic(u64* keys, uint32_t n2) {
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

// Upper edge of the bin (two 8-bit radix steps below the keys' common prefix)
// that holds the rank-th smallest of n keys: a value >= that key.  One warp;
// hist = 256 words of its shared memory.  have_mm: kmin / kmax are given.
template <class KeyF>
__device__ __forceinline__ uint32_t warp_rank_key(uint32_t n, uint32_t rank, KeyF key, uint32_t* hist,
                                                  bool have_mm, uint32_t kmin, uint32_t kmax) {
    const int lane = threadIdx.x & 31;
    constexpr int U = 4;
    // ---- pass 1: min / max of the keys (unless given)
    for (uint32_t base = 0; !have_mm && base < n; base += 32 * U) {
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
    // ---- passes 2-3: two 8-bit radix steps below the common prefix narrow the
    // bin holding the w-th key; T~ = the top key of that bin (>= the w-th key)
    uint32_t tkey = kmax;
    if (kmin != kmax) {
        int consumed = __clz(kmin ^ kmax);
        uint32_t prefix = consumed ? kmin >> (32 - consumed) : 0u;
        uint32_t r = rank;
#pragma unroll 1
        for (int step = 0; step < 2 && consumed < 32; ++step) {
            const int wd = min(8, 32 - consumed);
            const int sh = 32 - consumed - wd;
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
                        atomicAdd(&hist[(v[k] >> sh) & ((1u << wd) - 1u)], 1u);
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
        tkey = consumed >= 32 ? prefix : ((prefix << (32 - consumed)) | ((1u << (32 - consumed)) - 1u));
    }
    return tkey;
}

__global__ __launch_bounds__(CW * 32, 4) void topw_certify_kernel(
    const float* __restrict__ Dt, size_t nq, uint32_t nc, uint32_t w, const float* __restrict__ x,
    const float* __restrict__ c, float cnorm_max, uint32_t* __restrict__ out_idx,
    uint32_t* __restrict__ overflow, const u64 nz, const uint32_t* __restrict__ kmm, float dscale_tc) {
    constexpr int D = 128;
    __shared__ uint32_t hist_all[CW][256];
    __shared__ __align__(16) u64 cand_all[CW][SCAP];  // the streaming stage, then the candidates
    __shared__ __align__(16) float xs_all[CW][D];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t q = (size_t)blockIdx.x * CW + warp;
    if (q >= nq) return;
    const uint32_t* row = reinterpret_cast<const uint32_t*>(Dt + q * nc);
    uint32_t* hist = hist_all[warp];
    u64* cand = cand_all[warp];
    u64* stage = cand;
    float* xs = xs_all[warp];
    reinterpret_cast<float4*>(xs)[lane] = reinterpret_cast<const float4*>(x + q * D)[lane];
    constexpr int U = 8;
    // D~ may be slightly negative: order keys as signed floats
    auto key = [&](uint32_t i) {
        const uint32_t u = __ldg(row + i);
        return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    };
    // |x|^2 and the certification window first (the streaming select needs them)
    float nx = 0.f;
    bool tf32_exact = true;  // zero or normal with the low 13 mantissa bits clear
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const float v = xs[4 * lane + t];
        const uint32_t b = __float_as_uint(v);
        tf32_exact &= (b & 0x1fffu) == 0 && ((b & 0x7f800000u) != 0 || (b & 0x7fffffffu) == 0);
        nx = fmaf(v, v, nx);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nx += __shfl_xor_sync(0xffffffffu, nx, o);
    // 2^-10 when the query is exact in TF32 (u8 queries); 2^-9 when its
    // components round too (float queries through pqrr_dev_search_f32); + 1%
    // slack for this sum and an absolute floor for underflowing products
    // (the tcgen05 path passes its own, 2^-13: fp16 hi/lo centroid split)
    const float dscale = dscale_tc > 0.f ? dscale_tc
                                         : (__all_sync(0xffffffffu, tf32_exact) ? 9.765625e-04f : 1.953125e-03f);
    const float delta_max = dscale * (nx + cnorm_max) * 1.01f + 0x1p-100f;
    auto fkey = [](float f) {
        const uint32_t u = __float_as_uint(f);
        return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    };
    auto kfloat = [](uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); };
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t ncand = 0;
    // ---- one pass over the row.  The warp keeps a bound Tw >= the w-th
    // smallest D~ and stages (ballot compaction) the entries with
    // D~ <= Tw + 2 delta_max; when the stage fills, the w-th smallest staged
    // key tightens Tw (the w-th of a subset is >= the w-th of the row) and the
    // stage is filtered.  What is skipped or dropped lies above a bound + 2
    // delta_max, so the final stage holds every certified candidate.
    bool streamed = w + 64 <= SCAP / 2;
    if (streamed) {
        uint32_t bkey = 0xffffffffu;  // key of Tw + 2 delta_max
        uint32_t cnt = 0;
        auto tighten = [&]() {
            const uint32_t tk = warp_rank_key(cnt, w, [&](uint32_t j) { return (uint32_t)(stage[j] >> 32); }, hist,
                                              false, 0xffffffffu, 0u);
            bkey = fkey(kfloat(tk) + 2.f * delta_max);
            __syncwarp();
            uint32_t kept = 0;
            for (uint32_t j0 = 0; j0 < cnt; j0 += 32) {
                const uint32_t j = j0 + lane;
                const u64 e = j < cnt ? stage[j] : ~0ull;
                const bool keep = j < cnt && (uint32_t)(e >> 32) <= bkey;
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                __syncwarp();
                if (keep) stage[kept + __popc(m & lt_mask)] = e;
                kept += __popc(m);
                __syncwarp();
            }
            cnt = kept;
        };
        for (uint32_t base = 0; base < nc && streamed; base += 32 * U) {
            uint32_t v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                v[k] = i < nc ? key(i) : 0xffffffffu;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t i = base + k * 32 + lane;
                const bool pass = i < nc && v[k] <= bkey;
                const unsigned m = __ballot_sync(0xffffffffu, pass);
                if (m) {
                    if (pass) stage[cnt + __popc(m & lt_mask)] = ((u64)v[k] << 32) | i;
                    cnt += __popc(m);
                }
            }
            if (cnt > SCAP - 32 * U) {
                __syncwarp();
                tighten();
                if (cnt > SCAP / 2) streamed = false;  // (a wide window or masses of ties: the multi-pass select)
            }
        }
        if (streamed && cnt >= w) {
            __syncwarp();
            tighten();  // final T~ and window; the stage now holds exactly the candidates
            ncand = cnt;
            for (uint32_t t = lane; t < ncand; t += 32) cand[t] = stage[t] & 0xffffffffull;  // indices
            __syncwarp();
        } else {
            streamed = false;
        }
    }
    if (!streamed) {
    // ---- multi-pass select (fallback).  pass 1: min / max of the keys (given by the tcgen05 epilogue when kmm)
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    if (kmm) {  // [min keys nq][max keys nq]
        kmin = kmm[q];
        kmax = kmm[nq + q];
    }
    const uint32_t tkey = warp_rank_key(nc, w, key, hist, kmm != nullptr, kmin, kmax);
    // back to a float: T~ (>= the w-th smallest D~), candidate bound T~ + 2 delta_max
    const float bound = kfloat(tkey) + 2.f * delta_max;
    // ---- pass 3: candidates D~ <= bound (index order)
    ncand = 0;
    for (uint32_t base = 0; base < nc; base += 32 * U) {
        float v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t i = base + k * 32 + lane;
            v[k] = i < nc ? __uint_as_float(__ldg(row + i)) : __int_as_float(0x7f800000);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint32_t i = base + k * 32 + lane;
            const bool take = v[k] <= bound;
            const unsigned m = __ballot_sync(0xffffffffu, take);
            const uint32_t o = ncand + __popc(m & lt_mask);
            if (take && o < CCAP) cand[o] = i;
            ncand += __popc(m);
        }
    }
    }
    if (ncand > CCAP || ncand < w) {
        // the batch is redone on the exact path; emit valid probes meanwhile
        for (uint32_t t = lane; t < w; t += 32) out_idx[q * w + t] = t % nc;
        if (lane == 0) atomicAdd(overflow, 1u);
        return;
    }
    __syncwarp();
    // exact distances (reference order) of the candidates
    for (uint32_t t = lane; t < ncand; t += 32) {
        const uint32_t ci = (uint32_t)cand[t];
        // l2_sq(x, C_ci) in the reference order (as l2sq_packed), 2-way unrolled
        const float* cr = c + (size_t)ci * D;
        u64 s01 = 0, s23 = 0;
#pragma unroll 2
        for (int e = 0; e < D; e += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(xs + e);
            const float4 cv = __ldg(reinterpret_cast<const float4*>(cr + e));
            s01 = acc_sq2(s01, pk2(xv.x, xv.y), pk2(cv.x, cv.y), nz);
            s23 = acc_sq2(s23, pk2(xv.z, xv.w), pk2(cv.z, cv.w), nz);
        }
        const float dd = __fadd_rn(__fadd_rn(lo2(s01), hi2(s01)), __fadd_rn(lo2(s23), hi2(s23)));
        cand[t] = nb_key(dd, ci);
    }
    uint32_t n2 = 1;
    while (n2 < ncand) n2 <<= 1;
    for (uint32_t t = ncand + lane; t < n2; t += 32) cand[t] = ~0ull;
    __syncwarp();
    wbitonic(cand, n2);
    for (uint32_t t = lane; t < w; t += 32) out_idx[q * w + t] = key_id(cand[t]);
}

}  // namespace

bool coarse_tc_supported(uint32_t d, uint32_t w) { return d == 128 && w >= 1 && w <= CCAP; }

void launch_coarse_norms(const float* c, uint32_t n, uint32_t d, float* out, cudaStream_t s) {
    if (!n) return;
    sq_norms_kernel<<<(n + 255) / 256, 256, 0, s>>>(c, n, d, out);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_coarse_tc(const float* x, size_t nq, const float* c, uint32_t nc, const float* cnorm,
                      float cnorm_max, uint32_t w, float* Dt, uint32_t* out_idx, uint32_t* overflow,
                      cudaStream_t s, AssignTc* atc) {
    if (!nq) return;
    if (atc) {
        // D~ on the 5th-generation tensor cores; the window shrinks from
        // 2^-10 to 2^-13 (|x|^2 + max |c|^2), the min / max pass is folded in
        uint32_t* kmm = nullptr;
        PQRR_CUDA(cudaMallocAsync(&kmm, nq * 2 * sizeof(uint32_t), s));
        atc->dtilde(x, nq, Dt, kmm, s);
        topw_certify_kernel<<<(unsigned)((nq + CW - 1) / CW), CW * 32, 0, s>>>(
            Dt, nq, nc, w, x, c, atc->cmax, out_idx, overflow, kNegZero2, kmm, 0x1p-13f);
        PQRR_LAUNCH_CHECK();
        count_launch();
        PQRR_CUDA(cudaFreeAsync(kmm, s));
        return;
    }
    const size_t smem = (size_t)(GM + GN) * GLD * sizeof(float);
    static bool attr = false;
    if (!attr) {
        set_max_smem((const void*)coarse_gemm_kernel, (size_t)((int)smem));
        attr = true;
    }
    dim3 grid((nc + GN - 1) / GN, (unsigned)((nq + GM - 1) / GM));
    coarse_gemm_kernel<<<grid, GW * 32, smem, s>>>(x, nq, c, nc, cnorm, Dt);
    PQRR_LAUNCH_CHECK();
    topw_certify_kernel<<<(unsigned)((nq + CW - 1) / CW), CW * 32, 0, s>>>(Dt, nq, nc, w, x, c, cnorm_max,
                                                                           out_idx, overflow, kNegZero2,
                                                                           nullptr, 0.f);
    PQRR_LAUNCH_CHECK();
    count_launch(2);
}

}  // namespace pqrr_b200
