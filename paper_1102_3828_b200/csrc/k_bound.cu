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
// the dot products on the 5th-generation tensor cores (tcgen05.mma kind::f16,
// fp32 accumulation in TMEM: 128 pairs x 256 codes x the 16 dims of a
// sub-space per instruction).  Both operands round to fp16 (relative 2^-11
// each, like TF32 with round-to-nearest); with
// sum_t |r_t b_t| <= (|r_j|^2 + |B_jc|^2) / 2 every error term of L~ (operand
// rounding, fp32 accumulation, the norms, the epilogue) and of the reference's
// own fp32 l2_sq (< 40 u) is below 2^-9 (|r_j|^2 + |B_jc|^2) (the bound used
// by K1-TC, k_coarse_tc.cu); the kernel subtracts 2^-8 of it:
//     lb_jc = (|r_j|^2 + |B_jc|^2) (1 - 2^-8) - 2 <r_j, B_jc>~  <=  l2_sq(r_j, B_jc).
// The pair's bound is sum_j max(0, min_c lb_jc) (1 - 2^-16) <= sum_j m_j.
// A pair with bound > tau is dead; the others get the exact LUT pass, whose
// sum of minima then decides exactly.  The bound only selects work: the
// exact path decides every result.
#include <cuda_fp16.h>
#include <float.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int M = 8, KS = 256, DS = 16, D = 128;
constexpr int TM = 128;                  // far pairs per tile (TMEM lanes)
constexpr int FB_THREADS = 384;          // warp 1 MMA, 2-3 residuals, 4-11 epilogue (two per TMEM quadrant)
constexpr uint32_t A_BYTES = TM * D * 2;     // 32 KiB: residual rows, fp16, K-major 128-byte swizzle
constexpr uint32_t B_BYTES = KS * D * 2;     // 64 KiB: the code-major book [code][128 dims], fp16
constexpr uint32_t SMEM_BYTES = 1024 + 2 * A_BYTES + B_BYTES + M * KS * 4 + 3 * TM * M * 4 + 16 * 8 + 16;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned a, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned a) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned a, unsigned parity) {
    unsigned done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(unsigned addr) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16, D f32, A / B f16 K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(KS >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
__device__ __forceinline__ void mma_f16(unsigned dtmem, uint64_t ad, uint64_t bd) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
        ::"r"(dtmem), "l"(ad), "l"(bd), "r"(kIdesc));
}
__device__ __forceinline__ void mma_commit(unsigned bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
// byte offset of element (row, k) in a K-major, 128-byte-swizzled fp16 tile
// of `rows` rows (two K halves of rows x 64 elements)
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t k, uint32_t rows) {
    return (k >> 6) * rows * 128 + (row >> 3) * 1024 + (row & 7) * 128 + ((((k & 63) >> 3) ^ (row & 7)) << 4) +
           (k & 7) * 2;
}

// Far-pair bound on the 5th-generation tensor cores.  Rows = 128 far pairs,
// K = the 16 dims of one sub-space, N = the 256 codes: sub-space j is ONE
// tcgen05.mma (M = 128, N = 256, K = 16) of the residual tile against the
// code-major book at K step j, into one of two TMEM accumulators (256 columns
// each), so the epilogue of sub-space j overlaps the MMA of j + 1.  Operands
// round to fp16 (relative 2^-11 each, as TF32 with round-to-nearest; plus an
// absolute 2^-25 per subnormal element, covered by subtracting 2^-10); the
// bound arithmetic is the mma.sync version's:
//     lb_jc = (|r_j|^2 + |B_jc|^2)(1 - 2^-8) - 2 <r_j, B_jc>~ - 2^-10,
//     bound = sum_j max(0, min_c lb_jc), summed rounding down, x (1 - 2^-16).
__global__ void __launch_bounds__(FB_THREADS, 1) far_bound_tc_kernel(
    const float* __restrict__ xq, const float* __restrict__ coarse, const float* __restrict__ books,
    const uint32_t* __restrict__ probes, size_t nq, uint32_t w, uint32_t R1, float* __restrict__ pair_bound) {
    extern __shared__ uint8_t fb_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>(((uintptr_t)fb_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* As = sm;                                                  // [2][A_BYTES]
    uint8_t* Bs = sm + 2 * A_BYTES;                                    // [B_BYTES]
    float* bn2 = reinterpret_cast<float*>(Bs + B_BYTES);               // [M][KS] |B_jc|^2 (1 - 2^-8)
    float* rn2 = bn2 + M * KS;                                         // [2][TM][M] |r_j|^2 (1 - 2^-8)
    float* xmin = rn2 + 2 * TM * M;                                    // [TM][M] upper-half minima
    uint64_t* bars = reinterpret_cast<uint64_t*>(xmin + TM * M);       // a_full[2] a_empty[2] t_full[2] t_empty[2]
    const unsigned bar0 = su32(bars);
    auto BAR = [&](int kind, int i) { return bar0 + 8u * (2 * kind + i); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float shrink = 0.99609375f;  // 1 - 2^-8
    const uint32_t wf = w - R1;
    const size_t nfar = nq * (size_t)wf;
    const size_t ntiles = (nfar + TM - 1) / TM;

    // the code-major book (fp16, swizzled) and |B_jc|^2, once per CTA
    for (uint32_t i = threadIdx.x; i < (uint32_t)(KS * D / 4); i += blockDim.x) {
        const uint32_t c = i / (D / 4), k = 4 * (i % (D / 4)), j = k / DS;
        const float4 v = __ldg(reinterpret_cast<const float4*>(books + ((size_t)j * KS + c) * DS + (k % DS)));
        const __half2 lo = __floats2half2_rn(v.x, v.y), hi = __floats2half2_rn(v.z, v.w);
        uint2 pk;
        pk.x = *reinterpret_cast<const uint32_t*>(&lo);
        pk.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(Bs + sw128_off(c, k, KS)) = pk;
    }
    for (uint32_t rc = threadIdx.x; rc < M * KS; rc += blockDim.x) {
        const float* b = books + (size_t)rc * DS;
        float s2 = 0.f;
#pragma unroll
        for (int t = 0; t < DS; ++t) s2 = __fmaf_rn(b[t], b[t], s2);
        bn2[rc] = __fmul_rn(s2, shrink);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            bar_init(BAR(0, i), 64);   // a_full: the residual warps
            bar_init(BAR(1, i), 1);    // a_empty: MMA commit
            bar_init(BAR(2, i), 1);    // t_full: MMA commit
            bar_init(BAR(3, i), 256);  // t_empty: epilogue threads
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t g = 0, i = 0;
            const unsigned bbase = su32(Bs);
            for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
                const uint32_t a = i & 1u;
                bar_wait(BAR(0, a), (i >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned abase = su32(As + a * A_BYTES);
                for (int j = 0; j < M; ++j, ++g) {
                    const uint32_t acc = g & 1u, use = g >> 1;
                    if (use) bar_wait(BAR(3, acc), (use - 1) & 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const unsigned ka = (unsigned)(j >> 2) * (TM * 128) + (unsigned)(j & 3) * 32u;
                    const unsigned kb = (unsigned)(j >> 2) * (KS * 128) + (unsigned)(j & 3) * 32u;
                    mma_f16(tmem + acc * KS, sw128_desc(abase + ka), sw128_desc(bbase + kb));
                    mma_commit(BAR(2, acc));
                }
                mma_commit(BAR(1, a));
            }
        }
    } else if (warp == 2 || warp == 3) {
        // ------------------------------------------------ residual rows
        const int cw = warp - 2;
        uint32_t i = 0;
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const uint32_t a = i & 1u;
            if (i >= 2) bar_wait(BAR(1, a), ((i >> 1) - 1) & 1u);
            uint8_t* A = As + a * A_BYTES;
            // this warp's 64 rows r = cw + 2 i: the list ids first (lane i holds
            // rows i and i + 32), then 4 rows at a time with all loads in flight
            uint32_t lid[2], qid[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const size_t k = t * TM + cw + 2 * (lane + 32 * h);
                lid[h] = 0;
                qid[h] = 0xffffffffu;
                if (k < nfar) {
                    qid[h] = (uint32_t)(k / wf);
                    lid[h] = probes[(size_t)qid[h] * w + R1 + (uint32_t)(k % wf)];
                }
            }
#pragma unroll 1
            for (int i0 = 0; i0 < TM / 2; i0 += 4) {
                float4 xv[4], cv[4];
                uint32_t qq[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u, h = i >> 5;
                    qq[u] = __shfl_sync(0xffffffffu, h ? qid[1] : qid[0], i & 31);
                    const uint32_t l = __shfl_sync(0xffffffffu, h ? lid[1] : lid[0], i & 31);
                    xv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                    cv[u] = xv[u];
                    if (qq[u] != 0xffffffffu) {
                        xv[u] = __ldg(reinterpret_cast<const float4*>(xq + (size_t)qq[u] * D) + lane);
                        cv[u] = __ldg(reinterpret_cast<const float4*>(coarse + (size_t)l * D) + lane);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int r = cw + 2 * (i0 + u);
                    const float4 v = make_float4(__fsub_rn(xv[u].x, cv[u].x), __fsub_rn(xv[u].y, cv[u].y),
                                                 __fsub_rn(xv[u].z, cv[u].z), __fsub_rn(xv[u].w, cv[u].w));
                    const __half2 lo = __floats2half2_rn(v.x, v.y), hi = __floats2half2_rn(v.z, v.w);
                    uint2 pk;
                    pk.x = *reinterpret_cast<const uint32_t*>(&lo);
                    pk.y = *reinterpret_cast<const uint32_t*>(&hi);
                    *reinterpret_cast<uint2*>(A + sw128_off(r, 4 * lane, TM)) = pk;
                    // |r_j|^2 of the fp32 residual: lanes 4j .. 4j + 3 hold sub-space j
                    float s2 = __fmaf_rn(v.x, v.x, __fmaf_rn(v.y, v.y, __fmaf_rn(v.z, v.z, __fmul_rn(v.w, v.w))));
                    s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
                    s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
                    if ((lane & 3) == 0) rn2[(a * TM + r) * M + (lane >> 2)] = __fmul_rn(s2, shrink);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bar_arrive(BAR(0, a));
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue: min over codes, sum over j
        // warps 4 + qd and 8 + qd share TMEM lanes 32 qd .. + 31 (rows) and
        // take code columns 0..127 / 128..255; the upper half's minima meet
        // the lower half's in shared memory at the end of the tile
        const int ew = warp - 4, qd = ew & 3, hf = ew >> 2;
        const int r = 32 * qd + lane;
        const unsigned lane_off = (unsigned)(32 * qd) << 16;
        uint32_t g = 0, i = 0;
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const uint32_t a = i & 1u;
            bar_wait(BAR(0, a), (i >> 1) & 1u);  // rn2 of this tile is written
            // read now: the residual warps refill this buffer (tile i + 2) once
            // the tile's last MMA retired, while sub-spaces 6-7 still drain
            float rjs[M], mns[M];
#pragma unroll
            for (int j = 0; j < M; ++j) rjs[j] = rn2[(a * TM + r) * M + j];
#pragma unroll
            for (int j = 0; j < M; ++j, ++g) {
                const uint32_t acc = g & 1u;
                bar_wait(BAR(2, acc), (g >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const float rj = rjs[j];
                float mn = FLT_MAX;
#pragma unroll 1
                for (int c32 = 0; c32 < KS / 64; ++c32) {
                    const int col = 128 * hf + 32 * c32;
                    uint32_t u[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
                          "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
                          "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
                          "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
                          "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
                        : "r"(tmem + lane_off + acc * KS + col));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (c32 == KS / 64 - 1) {
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        bar_arrive(BAR(3, acc));
                    }
                    const float4* b4 = reinterpret_cast<const float4*>(bn2 + j * KS + col);
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4) {
                        const float4 bb = b4[q4];
                        mn = fminf(mn, fminf(fminf(__fmaf_rn(-2.f, __uint_as_float(u[4 * q4]), __fadd_rn(rj, bb.x)),
                                                   __fmaf_rn(-2.f, __uint_as_float(u[4 * q4 + 1]), __fadd_rn(rj, bb.y))),
                                             fminf(__fmaf_rn(-2.f, __uint_as_float(u[4 * q4 + 2]), __fadd_rn(rj, bb.z)),
                                                   __fmaf_rn(-2.f, __uint_as_float(u[4 * q4 + 3]), __fadd_rn(rj, bb.w)))));
                    }
                }
                mns[j] = mn;
            }
            if (hf) {
#pragma unroll
                for (int j = 0; j < M; ++j) xmin[r * M + j] = mns[j];
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 epilogue warps
            if (!hf) {
                float sum = 0.f;
#pragma unroll
                for (int j = 0; j < M; ++j)
                    sum = __fadd_rd(sum, fmaxf(__fsub_rd(fminf(mns[j], xmin[r * M + j]), 0x1p-10f), 0.f));
                const size_t k = t * TM + r;
                if (k < nfar) {
                    const size_t q = k / wf;
                    pair_bound[q * w + R1 + (uint32_t)(k % wf)] = __fmul_rd(sum, 0.9999847412109375f);  // 1 - 2^-16
                }
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");  // xmin is free for the next tile
        }
    }
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace

bool far_bound_supported(uint32_t d, uint32_t m, uint32_t ks) { return d == D && m == M && ks == KS; }

void launch_far_bound(const float* xq, const float* coarse, const float* books, const uint32_t* probes,
                      size_t nq, uint32_t w, uint32_t R1, float* pair_bound, cudaStream_t s) {
    if (nq == 0 || w <= R1) return;
    set_max_smem((const void*)far_bound_tc_kernel, SMEM_BYTES);
    const size_t nfar = nq * (size_t)(w - R1);
    const unsigned grid = (unsigned)std::min<size_t>((nfar + TM - 1) / TM, (size_t)sm_count());
    far_bound_tc_kernel<<<grid, FB_THREADS, SMEM_BYTES, s>>>(xq, coarse, books, probes, nq, w, R1, pair_bound);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
