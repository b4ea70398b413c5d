// k_bound.cu — certified lower bound of a probed pair's sum of LUT minima on
// the tensor cores (two-phase LUT pass, far probes).
//
// For query x and probed list l with residual r = x - C_l, every ADC distance
// of the list is >= sum_j m_j with m_j = min_c l2_sq(r_j, B_j[c]) (fp32
// addition is monotone; see "Live pairs" in DESIGN.md).  A far pair whose sum
// of minima exceeds the query's threshold tau has no candidate, and its exact
// LUT (98,304 FP32 operations) need not be built.  This kernel bounds m_j
// from below without building it:
//     L~_jc = |r_j|^2 + |B_jc|^2 - 2 <r_j, B_jc>,
// the dot products on the tensor cores (mma.sync m16n8k8 TF32, fp32
// accumulation: 16 pairs x 8 codes x 16 dims per sub-space and code tile).
// Both operands round to TF32 (relative 2^-11 each); with
// sum_t |r_t b_t| <= (|r_j|^2 + |B_jc|^2) / 2 every error term of L~ (operand
// rounding, fp32 accumulation, the norms, the epilogue) and of the reference's
// own fp32 l2_sq (< 40 u) is below 2^-9 (|r_j|^2 + |B_jc|^2) (the bound used
// by K1-TC, k_coarse_tc.cu); the kernel subtracts 2^-8 of it:
//     lb_jc = (|r_j|^2 + |B_jc|^2) (1 - 2^-8) - 2 <r_j, B_jc>~  <=  l2_sq(r_j, B_jc).
// The pair's bound is sum_j max(0, min_c lb_jc) (1 - 2^-16) <= sum_j m_j.
// A pair with bound > tau is dead; the others get the exact LUT pass, whose
// sum of minima then decides exactly.  The bound only selects work: the
// exact path decides every result.
#include <float.h>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int BW = 8;      // warps per CTA: one 16-pair tile each
constexpr int RLD = 144;   // residual tile row stride (floats): conflict-free fragment loads
constexpr int M = 8, KS = 256, DS = 16, D = 128;

__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Lane (g, tig) of a k-step pair (the 16 dims of a sub-space) carries dims
// 4 tig .. 4 tig + 3 of its A row and B column: k-step 0 puts dim 4 tig at
// k = tig and 4 tig + 2 at k = tig + 4, k-step 1 dims 4 tig + 1 and 4 tig + 3
// — the same permutation for A and B, so the dot products are unchanged and
// each operand is one LDS.128.
__global__ __launch_bounds__(BW * 32, 1) void far_bound_kernel(
    const float* __restrict__ xq, const float* __restrict__ coarse, const float* __restrict__ books,
    const uint32_t* __restrict__ probes, size_t nq, uint32_t w, uint32_t R1,
    float* __restrict__ pair_bound) {
    extern __shared__ float4 bsm[];
    uint4* bk = reinterpret_cast<uint4*>(bsm);                          // [M][KS][4] tf32 bits
    float* bn2 = reinterpret_cast<float*>(bsm + M * KS * 4);            // [M][KS] |B_jc|^2 (1 - 2^-8)
    float* tiles = bn2 + M * KS;                                        // [BW][16][RLD]
    float* rn2s = tiles + BW * 16 * RLD;                                // [BW][16][M]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float shrink = 0.99609375f;  // 1 - 2^-8
    for (uint32_t i = threadIdx.x; i < M * KS * 4; i += blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(books) + i);
        bk[i] = make_uint4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
    }
    for (uint32_t rc = threadIdx.x; rc < M * KS; rc += blockDim.x) {
        const float* b = books + (size_t)rc * DS;
        float s = 0.f;
#pragma unroll
        for (int t = 0; t < DS; ++t) s = __fmaf_rn(b[t], b[t], s);
        bn2[rc] = __fmul_rn(s, shrink);
    }
    __syncthreads();

    const uint32_t wf = w - R1;
    const size_t nfar = nq * (size_t)wf;
    const size_t ntiles = (nfar + 15) / 16;
    float* tile = tiles + warp * 16 * RLD;
    float* rn2 = rn2s + warp * 16 * M;
    const int g = lane >> 2, tig = lane & 3;
    for (size_t tl = (size_t)blockIdx.x * BW + warp; tl < ntiles; tl += (size_t)gridDim.x * BW) {
        // residuals r = x - C_l of the tile's 16 far pairs (rows past the end: 0)
        for (int i = lane; i < 16 * (D / 4); i += 32) {
            const int row = i / (D / 4), c4 = i % (D / 4);
            const size_t k = tl * 16 + row;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k < nfar) {
                const size_t q = k / wf;
                const uint32_t l = probes[q * w + R1 + (uint32_t)(k % wf)];
                const float4 x = __ldg(reinterpret_cast<const float4*>(xq + q * D) + c4);
                const float4 cc = __ldg(reinterpret_cast<const float4*>(coarse + (size_t)l * D) + c4);
                v = make_float4(__fsub_rn(x.x, cc.x), __fsub_rn(x.y, cc.y), __fsub_rn(x.z, cc.z),
                                __fsub_rn(x.w, cc.w));
            }
            *reinterpret_cast<float4*>(tile + row * RLD + 4 * c4) = v;
        }
        __syncwarp();
        // |r_j|^2 (1 - 2^-8) per (pair, sub-space)
        for (int i = lane; i < 16 * M; i += 32) {
            const int row = i / M, j = i % M;
            const float* r = tile + row * RLD + j * DS;
            float s = 0.f;
#pragma unroll
            for (int t = 0; t < DS; ++t) s = __fmaf_rn(r[t], r[t], s);
            rn2[row * M + j] = __fmul_rn(s, shrink);
        }
        __syncwarp();
        float sum0 = 0.f, sum1 = 0.f;  // rows g and g + 8
#pragma unroll 1
        for (int j = 0; j < M; ++j) {
            const float4 ra = *reinterpret_cast<const float4*>(tile + g * RLD + j * DS + 4 * tig);
            const float4 rb = *reinterpret_cast<const float4*>(tile + (g + 8) * RLD + j * DS + 4 * tig);
            const uint32_t a00 = to_tf32(ra.x), a01 = to_tf32(rb.x), a02 = to_tf32(ra.z), a03 = to_tf32(rb.z);
            const uint32_t a10 = to_tf32(ra.y), a11 = to_tf32(rb.y), a12 = to_tf32(ra.w), a13 = to_tf32(rb.w);
            const float r0 = rn2[g * M + j], r1 = rn2[(g + 8) * M + j];
            float mn0 = FLT_MAX, mn1 = FLT_MAX;
#pragma unroll 4
            for (int nt = 0; nt < KS / 8; ++nt) {
                const uint4 bv = bk[(j * KS + nt * 8 + g) * 4 + tig];
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                // k-step 0: dims 4 tig + {0, 2}; k-step 1: 4 tig + {1, 3}
                mma_tf32(c, a00, a01, a02, a03, bv.x, bv.z);
                mma_tf32(c, a10, a11, a12, a13, bv.y, bv.w);
                const float2 bb = *reinterpret_cast<const float2*>(bn2 + j * KS + nt * 8 + 2 * tig);
                mn0 = fminf(mn0, fminf(__fmaf_rn(-2.f, c[0], __fadd_rn(r0, bb.x)),
                                       __fmaf_rn(-2.f, c[1], __fadd_rn(r0, bb.y))));
                mn1 = fminf(mn1, fminf(__fmaf_rn(-2.f, c[2], __fadd_rn(r1, bb.x)),
                                       __fmaf_rn(-2.f, c[3], __fadd_rn(r1, bb.y))));
            }
            mn0 = fminf(mn0, __shfl_xor_sync(0xffffffffu, mn0, 1));
            mn0 = fminf(mn0, __shfl_xor_sync(0xffffffffu, mn0, 2));
            mn1 = fminf(mn1, __shfl_xor_sync(0xffffffffu, mn1, 1));
            mn1 = fminf(mn1, __shfl_xor_sync(0xffffffffu, mn1, 2));
            sum0 = __fadd_rd(sum0, fmaxf(mn0, 0.f));
            sum1 = __fadd_rd(sum1, fmaxf(mn1, 0.f));
        }
        if (tig == 0) {
            const float keep = 0.9999847412109375f;  // 1 - 2^-16
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const size_t k = tl * 16 + g + 8 * h;
                if (k < nfar) {
                    const size_t q = k / wf;
                    pair_bound[q * w + R1 + (uint32_t)(k % wf)] = __fmul_rd(h ? sum1 : sum0, keep);
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace

bool far_bound_supported(uint32_t d, uint32_t m, uint32_t ks) { return d == D && m == M && ks == KS; }

void launch_far_bound(const float* xq, const float* coarse, const float* books, const uint32_t* probes,
                      size_t nq, uint32_t w, uint32_t R1, float* pair_bound, cudaStream_t s) {
    if (nq == 0 || w <= R1) return;
    const size_t smem = (size_t)M * KS * DS * 4 + (size_t)M * KS * 4 + (size_t)BW * 16 * RLD * 4 +
                        (size_t)BW * 16 * M * 4;
    set_max_smem((const void*)far_bound_kernel, (size_t)((int)smem));
    far_bound_kernel<<<sm_count(), BW * 32, smem, s>>>(xq, coarse, books, probes, nq, w, R1, pair_bound);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
