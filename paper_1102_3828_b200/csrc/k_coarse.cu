// k_coarse.cu — K1: exact-order query x centroid distance tiles with fused
// epilogues: (a) the full distance matrix for coarse probe selection
// (ivf_index.hpp:58-61), (b) fused argmin for the add path and
// k-means assignment (kernels::assign_batch, kernels.cpp:21-39).
//
// Distances follow distance.hpp:16-33 exactly (see common.cuh): each pair
// keeps (s0,s1) and (s2,s3) as two packed f32x2 accumulators, dims ascending.
// Tiles: 64 rows x 64 centroids per CTA, 256 threads, each thread a 4x4
// micro-tile with rows ty+16i and centroids tx+16j so that the LDS.128 reads
// of a warp hit 2 distinct rows (broadcast) and 16 centroid rows spread over
// all banks (rows padded to D+4 floats).
#include <float.h>

#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int TB = 64;  // tile rows / centroids

__global__ void widen_u8_kernel(const uint8_t* __restrict__ in, float* __restrict__ out,
                                size_t count) {
    size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i + 4 <= count) {
        uint32_t w = *reinterpret_cast<const uint32_t*>(in + i);
        float4 f = make_float4((float)(w & 0xff), (float)((w >> 8) & 0xff),
                               (float)((w >> 16) & 0xff), (float)(w >> 24));
        *reinterpret_cast<float4*>(out + i) = f;
    } else {
        for (; i < count; ++i) out[i] = (float)in[i];
    }
}

template <int D>
__device__ __forceinline__ void load_tile(float* __restrict__ dst, const float* __restrict__ src,
                                          size_t row0, size_t nrows) {
    constexpr int LD = D + 4;
    constexpr int V = D / 4;
    for (int idx = threadIdx.x; idx < TB * V; idx += blockDim.x) {
        int r = idx / V, c = idx % V;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row0 + r < nrows) v = reinterpret_cast<const float4*>(src + (row0 + r) * D)[c];
        *reinterpret_cast<float4*>(dst + r * LD + c * 4) = v;
    }
}

// acc[i][j] = (s01, s23) of pair (row ty+16i, centroid tx+16j).
template <int D>
__device__ __forceinline__ void tile_dists(const float* __restrict__ Xs, const float* __restrict__ Cs,
                                           int ty, int tx, u64 nz, float out[4][4]) {
    constexpr int LD = D + 4;
    u64 a01[4][4], a23[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) a01[i][j] = a23[i][j] = 0ull;
#pragma unroll 4
    for (int t = 0; t < D; t += 4) {
        float4 x[4], c[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = *reinterpret_cast<const float4*>(Xs + (ty + 16 * i) * LD + t);
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = *reinterpret_cast<const float4*>(Cs + (tx + 16 * j) * LD + t);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const u64 x01 = pk2(x[i].x, x[i].y), x23 = pk2(x[i].z, x[i].w);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                a01[i][j] = acc_sq2(a01[i][j], x01, pk2(c[j].x, c[j].y), nz);
                a23[i][j] = acc_sq2(a23[i][j], x23, pk2(c[j].z, c[j].w), nz);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
            out[i][j] = __fadd_rn(__fadd_rn(lo2(a01[i][j]), hi2(a01[i][j])),
                                  __fadd_rn(lo2(a23[i][j]), hi2(a23[i][j])));
}

template <int D>
__global__ __launch_bounds__(256) void pair_dists_kernel(const float* __restrict__ x, size_t nx,
                                                         const float* __restrict__ c, uint32_t nc,
                                                         float* __restrict__ out, u64 nz) {
    extern __shared__ float4 sm4[];
    float* Xs = reinterpret_cast<float*>(sm4);
    float* Cs = Xs + TB * (D + 4);
    const size_t row0 = (size_t)blockIdx.x * TB;
    const size_t col0 = (size_t)blockIdx.y * TB;
    load_tile<D>(Xs, x, row0, nx);
    load_tile<D>(Cs, c, col0, nc);
    __syncthreads();
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
    float dd[4][4];
    tile_dists<D>(Xs, Cs, ty, tx, nz, dd);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        size_t r = row0 + ty + 16 * i;
        if (r >= nx) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            size_t k = col0 + tx + 16 * j;
            if (k < nc) out[r * nc + k] = dd[i][j];
        }
    }
}

__device__ __forceinline__ bool lex_less(float d1, uint32_t i1, float d2, uint32_t i2) {
    return d1 < d2 || (d1 == d2 && i1 < i2);
}

template <int D>
__global__ __launch_bounds__(256) void argmin_kernel(const float* __restrict__ x, size_t nx,
                                                     const float* __restrict__ c, uint32_t nc,
                                                     uint32_t* __restrict__ out_idx,
                                                     float* __restrict__ out_dist, u64 nz) {
    extern __shared__ float4 sm4[];
    float* Xs = reinterpret_cast<float*>(sm4);
    float* Cs = Xs + TB * (D + 4);
    const size_t row0 = (size_t)blockIdx.x * TB;
    load_tile<D>(Xs, x, row0, nx);
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
    float best[4];
    uint32_t bidx[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        best[i] = __int_as_float(0x7f800000);
        bidx[i] = 0xffffffffu;
    }
    for (uint32_t col0 = 0; col0 < nc; col0 += TB) {
        __syncthreads();
        load_tile<D>(Cs, c, col0, nc);
        __syncthreads();
        float dd[4][4];
        tile_dists<D>(Xs, Cs, ty, tx, nz, dd);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t k = col0 + tx + 16 * j;
            if (k >= nc) continue;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (lex_less(dd[i][j], k, best[i], bidx[i])) {
                    best[i] = dd[i][j];
                    bidx[i] = k;
                }
        }
    }
    // reduce over the 16 tx lanes of this half warp (lexicographic (dist, idx))
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) {
            float od = __shfl_xor_sync(0xffffffffu, best[i], off);
            uint32_t oi = __shfl_xor_sync(0xffffffffu, bidx[i], off);
            if (lex_less(od, oi, best[i], bidx[i])) {
                best[i] = od;
                bidx[i] = oi;
            }
        }
        size_t r = row0 + ty + 16 * i;
        if (tx == 0 && r < nx) {
            out_idx[r] = bidx[i];
            if (out_dist) out_dist[r] = best[i];
        }
    }
}

// Generic fallback for any d: one thread per (row, centroid) pair.
__global__ void pair_dists_generic(const float* __restrict__ x, size_t nx,
                                   const float* __restrict__ c, uint32_t nc, uint32_t d,
                                   float* __restrict__ out) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nx * nc) return;
    size_t r = idx / nc, k = idx % nc;
    out[idx] = l2sq_scalar(x + r * d, c + k * d, (int)d);
}

__global__ void argmin_generic(const float* __restrict__ x, size_t nx, const float* __restrict__ c,
                               uint32_t nc, uint32_t d, uint32_t* __restrict__ out_idx,
                               float* __restrict__ out_dist) {
    size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nx) return;
    uint32_t best = 0;
    float bd = l2sq_scalar(x + r * d, c, (int)d);
    for (uint32_t k = 1; k < nc; ++k) {
        float dd = l2sq_scalar(x + r * d, c + (size_t)k * d, (int)d);
        if (dd < bd) {
            bd = dd;
            best = k;
        }
    }
    out_idx[r] = best;
    if (out_dist) out_dist[r] = bd;
}

// One CTA per row: bitonic sort of (dist, idx) keys, emit the w smallest.
__global__ __launch_bounds__(512) void topw_kernel(const float* __restrict__ D, uint32_t nc,
                                                   uint32_t n2, uint32_t w,
                                                   uint32_t* __restrict__ out_idx,
                                                   float* __restrict__ out_dist) {
    extern __shared__ u64 keys[];
    const size_t q = blockIdx.x;
    const float* row = D + q * nc;
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x)
        keys[i] = i < nc ? nb_key(row[i], i) : ~0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= n2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                uint32_t lo = 2 * i - (i & (j - 1));
                uint32_t hi = lo + j;
                bool up = (lo & k) == 0;
                u64 a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < w; i += blockDim.x) {
        out_idx[q * w + i] = key_id(keys[i]);
        if (out_dist) out_dist[q * w + i] = key_dist(keys[i]);
    }
}

// Top-w by radix select (K1 epilogue for probe selection): the w-th smallest
// distance D* is found with three 11/11/10-bit histogram passes over the row
// staged in smem; the row's entries below D* plus the lowest-index entries
// equal to D* (ties -> lowest centroid index) are compacted and
// only those w keys are sorted.  Replaces a full sort of Kc keys per query.
constexpr int TW_THREADS = 256;
constexpr uint32_t TW_TAIL = 1024;  // keys of the sorted-tail shortcut (the 2048-word histogram)

__device__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t* s_total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < TW_THREADS / 32; ++i) {
            const uint32_t t = s_warp[i];
            s_warp[i] = acc;
            acc += t;
        }
        *s_total = acc;
    }
    __syncthreads();
    return s_warp[warp] + incl - v;
}

__global__ __launch_bounds__(TW_THREADS) void topw_radix_kernel(const float* __restrict__ D,
                                                                uint32_t nc, uint32_t w, uint32_t w2,
                                                                uint32_t* __restrict__ out_idx,
                                                                float* __restrict__ out_dist) {
    extern __shared__ uint32_t tw_smem[];
    uint32_t* bits = tw_smem;                                 // [nc]
    u64* sel = reinterpret_cast<u64*>(tw_smem + ((nc + 1) & ~1u));  // [w2]
    __shared__ __align__(16) uint32_t hist[2048];
    __shared__ uint32_t s_bin, s_rank, s_out, s_total, s_warp[TW_THREADS / 32];
    const size_t q = blockIdx.x;
    const uint32_t* row = reinterpret_cast<const uint32_t*>(D + q * nc);
    uint32_t mn = 0xffffffffu;
    for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
        const uint32_t u = row[i];
        bits[i] = u;
        mn = min(mn, u);
    }
    for (uint32_t i = threadIdx.x; i < w2; i += blockDim.x) sel[i] = ~0ull;
    if (threadIdx.x == 0) s_out = 0;
    __syncthreads();
    // a query's coarse distances share their top bits: count only the low
    // tail (values <= a bound on the w-th smallest, see cta_tail_bound) or the
    // first pass serialises 8192 atomics on two or three bins (41 -> 9 us)
    uint32_t T0 = 0xffffffffu;
    if (w <= blockDim.x / 2 && nc >= blockDim.x) T0 = cta_tail_bound(mn, w, hist);
    __syncthreads();
    // the tail itself (a little over w entries) usually fits a small buffer:
    // sort it by (distance, index) and take the first w — no radix passes
    if (T0 != 0xffffffffu) {
        u64* tail = reinterpret_cast<u64*>(hist);  // 2048 words = TW_TAIL keys
        for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
            const uint32_t u = bits[i];
            if (u <= T0) {
                const uint32_t k = atomicAdd(&s_out, 1u);
                if (k < TW_TAIL) tail[k] = ((u64)u << 32) | i;
            }
        }
        __syncthreads();
        const uint32_t cnt = s_out;
        __syncthreads();
        if (cnt <= TW_TAIL) {
            uint32_t n2 = 32;
            while (n2 < cnt) n2 <<= 1;
            for (uint32_t i = cnt + threadIdx.x; i < n2; i += blockDim.x) tail[i] = ~0ull;
            __syncthreads();
            cta_bitonic_sort(tail, n2);
            for (uint32_t i = threadIdx.x; i < w; i += blockDim.x) {
                out_idx[q * w + i] = key_id(tail[i]);
                if (out_dist) out_dist[q * w + i] = key_dist(tail[i]);
            }
            return;
        }
        if (threadIdx.x == 0) s_out = 0;
        __syncthreads();
    }
    uint32_t prefix = 0, r = w;
    const int shifts[3] = {21, 10, 0}, widths[3] = {11, 11, 10};
    for (int pass = 0; pass < 3; ++pass) {
        for (int b = threadIdx.x; b < 2048; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const int sh = shifts[pass], wd = widths[pass];
        const uint32_t msk = (1u << wd) - 1u;
        for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
            const uint32_t u = bits[i];
            if (pass == 0 ? u <= T0 : (u >> (sh + wd)) == prefix) atomicAdd(&hist[(u >> sh) & msk], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // bin holding rank r: lane l owns 64 bins
            const int lane = threadIdx.x;
            uint32_t sum = 0;
            for (int b = 0; b < 64; ++b) sum += hist[lane * 64 + b];
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const uint32_t excl = incl - sum;
            const bool mine = excl < r && r <= incl;
            const unsigned who = __ballot_sync(0xffffffffu, mine);
            if (mine && lane == __ffs(who) - 1) {
                uint32_t cacc = excl;
                for (int b = 0; b < 64; ++b) {
                    const uint32_t h = hist[lane * 64 + b];
                    if (r <= cacc + h) {
                        s_bin = lane * 64 + b;
                        s_rank = r - cacc;
                        break;
                    }
                    cacc += h;
                }
            }
        }
        __syncthreads();
        prefix = (prefix << wd) | s_bin;
        r = s_rank;
        __syncthreads();
    }
    const uint32_t dstar = prefix;  // exact w-th smallest distance bits; r of its ties are in
    // strictly smaller entries: any order
    for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x)
        if (bits[i] < dstar) sel[atomicAdd(&s_out, 1u)] = ((u64)bits[i] << 32) | i;
    // ties at dstar: the r lowest indices, in index order (contiguous chunks per thread)
    const uint32_t chunk = (nc + TW_THREADS - 1) / TW_THREADS;
    const uint32_t lo = threadIdx.x * chunk, hi = min(nc, lo + chunk);
    uint32_t mine = 0;
    for (uint32_t i = lo; i < hi; ++i) mine += bits[i] == dstar;
    __syncthreads();
    const uint32_t before = block_excl_scan(mine, s_warp, &s_total);
    const uint32_t base_lt = w - r;
    uint32_t k = before;
    for (uint32_t i = lo; i < hi && k < r; ++i)
        if (bits[i] == dstar) sel[base_lt + k++] = ((u64)dstar << 32) | i;
    __syncthreads();
    // sort the w selected keys (w2 = next pow2, >= 32)
    cta_bitonic_sort(sel, w2);
    for (uint32_t i = threadIdx.x; i < w; i += blockDim.x) {
        out_idx[q * w + i] = key_id(sel[i]);
        if (out_dist) out_dist[q * w + i] = key_dist(sel[i]);
    }
}

template <int D>
void pair_dists_t(const float* x, size_t nx, const float* c, uint32_t nc, float* out,
                  cudaStream_t s) {
    size_t smem = 2 * TB * (D + 4) * sizeof(float);
    static bool attr = false;
    if (!attr) {
        set_max_smem((const void*)pair_dists_kernel<D>, (size_t)((int)smem));
        attr = true;
    }
    dim3 grid((unsigned)((nx + TB - 1) / TB), (nc + TB - 1) / TB);
    pair_dists_kernel<D><<<grid, 256, smem, s>>>(x, nx, c, nc, out, kNegZero2);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

template <int D>
void argmin_t(const float* x, size_t nx, const float* c, uint32_t nc, uint32_t* out_idx,
              float* out_dist, cudaStream_t s) {
    size_t smem = 2 * TB * (D + 4) * sizeof(float);
    static bool attr = false;
    if (!attr) {
        set_max_smem((const void*)argmin_kernel<D>, (size_t)((int)smem));
        attr = true;
    }
    argmin_kernel<D><<<(unsigned)((nx + TB - 1) / TB), 256, smem, s>>>(x, nx, c, nc, out_idx,
                                                                        out_dist, kNegZero2);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace

void launch_widen_u8(const uint8_t* in, float* out, size_t count, cudaStream_t s) {
    if (count == 0) return;
    size_t threads = (count + 3) / 4;
    widen_u8_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(in, out, count);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_pair_dists(const float* x, size_t nx, const float* c, uint32_t nc, uint32_t d,
                       float* out, cudaStream_t s) {
    if (nx == 0 || nc == 0) return;
    switch (d) {
        case 128: return pair_dists_t<128>(x, nx, c, nc, out, s);
        case 64: return pair_dists_t<64>(x, nx, c, nc, out, s);
        case 32: return pair_dists_t<32>(x, nx, c, nc, out, s);
        case 16: return pair_dists_t<16>(x, nx, c, nc, out, s);
        case 8: return pair_dists_t<8>(x, nx, c, nc, out, s);
        case 4: return pair_dists_t<4>(x, nx, c, nc, out, s);
        default: break;
    }
    size_t total = nx * nc;
    pair_dists_generic<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(x, nx, c, nc, d, out);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_argmin(const float* x, size_t nx, const float* c, uint32_t nc, uint32_t d,
                   uint32_t* out_idx, float* out_dist, cudaStream_t s) {
    if (nx == 0) return;
    switch (d) {
        case 128: return argmin_t<128>(x, nx, c, nc, out_idx, out_dist, s);
        case 64: return argmin_t<64>(x, nx, c, nc, out_idx, out_dist, s);
        case 32: return argmin_t<32>(x, nx, c, nc, out_idx, out_dist, s);
        case 16: return argmin_t<16>(x, nx, c, nc, out_idx, out_dist, s);
        case 8: return argmin_t<8>(x, nx, c, nc, out_idx, out_dist, s);
        case 4: return argmin_t<4>(x, nx, c, nc, out_idx, out_dist, s);
        default: break;
    }
    argmin_generic<<<(unsigned)((nx + 127) / 128), 128, 0, s>>>(x, nx, c, nc, d, out_idx, out_dist);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_topw(const float* D, size_t nq, uint32_t nc, uint32_t w, uint32_t* out_idx,
                 float* out_dist, cudaStream_t s) {
    if (nq == 0) return;
    // default: warp-per-query radix select (w <= 64); a batch too small to
    // fill the GPU with warps gives each query a CTA instead
    if (nq >= (size_t)2 * sm_count() && launch_topw_warp(D, nq, nc, w, out_idx, out_dist, s)) return;
    // radix select wins for large Kc (8192: 5.65 -> 2.33 ms per 10k queries);
    // the full bitonic sort is faster for Kc <= 2048 (measured 0.54 vs 0.61 ms)
    if (w < nc && nc > 2048) {
        uint32_t w2 = 32;
        while (w2 < w) w2 <<= 1;
        const size_t smem = (size_t)((nc + 1) & ~1u) * 4 + (size_t)w2 * 8;
        if (smem <= 200 * 1024) {
            set_max_smem((const void*)topw_radix_kernel, (size_t)((int)smem));
            topw_radix_kernel<<<(unsigned)nq, TW_THREADS, smem, s>>>(D, nc, w, w2, out_idx, out_dist);
            PQRR_LAUNCH_CHECK();
            count_launch();
            return;
        }
    }
    uint32_t n2 = 1;
    while (n2 < nc) n2 <<= 1;
    size_t smem = (size_t)n2 * sizeof(u64);
    if (smem > 200 * 1024) throw ArgError("coarse quantizer too large for device top-w (c > 16384)");
    static size_t attr = 0;
    if (smem > attr) {
        set_max_smem((const void*)topw_kernel, (size_t)(200 * 1024));
        attr = 200 * 1024;
    }
    topw_kernel<<<(unsigned)nq, 512, smem, s>>>(D, nc, n2, w, out_idx, out_dist);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
