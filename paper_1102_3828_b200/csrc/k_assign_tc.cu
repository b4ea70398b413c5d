// k_assign_tc.cu — add-path coarse assignment on the 5th-generation tensor
// cores (tcgen05.mma, accumulators in TMEM, centroid tiles by TMA), certified
// to return exactly the reference's assignment:
//     a(y) = argmin_k l2_sq(y, C_k), strict < in ascending k
// (kernels.cpp:21-39 assign_batch, ivf_index.hpp:54-56).
//
// Rows y are u8 (exact in fp16).  Each centroid is split c = c_hi + c_lo into
// two fp16 values (|c - c_hi - c_lo| <= 2^-22 |c| + 2^-25), so two
// kind::f16 MMAs per K step give <y, c> with products exact and fp32
// accumulation.  Per (row, centroid) the estimate
//     D~ = |y|^2 + |c|^2 - 2 <y, c>~
// differs from the reference's fp32 l2_sq by at most
//     delta = 2^-13 (|y|^2 + max_k |c_k|^2)
// (operand split 2^-22, tensor-core accumulation of 256 terms <= 2^-16,
// epilogue roundings <= 2^-16, the reference's own sequential fp32 sum
// <= 2^-18, each relative to |y|^2 + |c|^2 >= 2 |<y, c>|).  The true argmin
// therefore has D~ <= min D~ + 2 delta.  The epilogue keeps each row's four
// smallest D~; a row whose second-smallest is above min + 2 delta is certified
// outright, a row with 2-3 candidates recomputes them exactly in the
// reference order (l2_sq, distance.hpp:16-33) and takes the lowest index among
// equal distances, and a row whose fourth-smallest is still inside the window
// goes to an overflow list that a warp-per-row exact kernel settles.
//
// Roles (256 threads, one CTA per SM, persistent over 128-row tiles):
//   warp 0     TMA producer: 128-centroid blocks of C_hi and C_lo (K-major,
//              128-byte swizzle) into a 2-stage ring (full / empty mbarriers);
//   warp 1     TMEM allocation + the single-thread MMA issuer: per block 8
//              K steps x {hi, lo} of M = 128, N = 128, K = 16 into one of two
//              TMEM accumulators (128 columns each);
//   warps 2-3  convert the next tile's u8 rows to fp16 in the swizzled
//              K-major layout and compute |y|^2 (exact integers);
//   warps 4-7  epilogue: tcgen05.ld of the accumulator (row = TMEM lane),
//              D~ and the running 4 smallest per row.
#include <cuda.h>
#include <cuda_fp16.h>

#include <vector>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int AT_M = 128, AT_N = 128, AT_D = 128;
constexpr int AT_THREADS = 256;
constexpr uint32_t A_BYTES = AT_M * AT_D * 2;       // 32 KiB: two K halves of 16 KiB
constexpr uint32_t B_BYTES = 2 * AT_N * AT_D * 2;   // 64 KiB: hi halves, lo halves
constexpr uint32_t CN_SMEM = 8192;  // centroids whose |c|^2 are staged in shared memory
constexpr uint32_t SMEM_BASE = 1024 + 2 * A_BYTES + 2 * B_BYTES + 2 * AT_M * 4 + 16 * 8 + 16;
constexpr uint32_t SMEM_BYTES = SMEM_BASE + CN_SMEM * 4;

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
__device__ __forceinline__ void tma_2d(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
// K-major operand, 128-byte swizzle: 8-row core groups 1024 B apart (SBO);
// the K offset inside a swizzle atom is added to the start address.
__device__ __forceinline__ uint64_t sw128_desc(unsigned addr) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16: D f32, A / B f16, both K-major, M = 128, N = 128
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(AT_N >> 3) << 17) | ((uint32_t)(AT_M >> 4) << 24);

__device__ __forceinline__ void mma_f16(unsigned dtmem, uint64_t ad, uint64_t bd, uint32_t acc) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
        ::"r"(dtmem), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(unsigned bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

// Exact l2_sq(y, C_k) in the reference order (distance.hpp:16-33) for a u8 row.
__device__ float exact_row_dist(const uint8_t* __restrict__ y, const float* __restrict__ c) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 4
    for (int t = 0; t < AT_D; t += 4) {
        const uint32_t yv = *reinterpret_cast<const uint32_t*>(y + t);
        const float4 cv = __ldg(reinterpret_cast<const float4*>(c + t));
        const float d0 = __fsub_rn((float)(yv & 0xff), cv.x), d1 = __fsub_rn((float)((yv >> 8) & 0xff), cv.y);
        const float d2 = __fsub_rn((float)((yv >> 16) & 0xff), cv.z), d3 = __fsub_rn((float)(yv >> 24), cv.w);
        s0 = __fadd_rn(s0, __fmul_rn(d0, d0));
        s1 = __fadd_rn(s1, __fmul_rn(d1, d1));
        s2 = __fadd_rn(s2, __fmul_rn(d2, d2));
        s3 = __fadd_rn(s3, __fmul_rn(d3, d3));
    }
    return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
}

__global__ void __launch_bounds__(AT_THREADS, 1) assign_tc_kernel(
    const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
    const uint8_t* __restrict__ y, size_t n, const float* __restrict__ coarse,
    const float* __restrict__ cnorm, uint32_t nc, float cmax, uint32_t* __restrict__ out,
    uint32_t* __restrict__ ovf_rows, uint32_t* __restrict__ ovf_cnt) {
    extern __shared__ uint8_t at_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>(((uintptr_t)at_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* As = sm;                       // [2][A_BYTES]
    uint8_t* Bs = sm + 2 * A_BYTES;         // [2][B_BYTES]
    float* nx = reinterpret_cast<float*>(Bs + 2 * B_BYTES);  // [2][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(nx + 2 * AT_M);
    // a_full[2] a_empty[2] b_full[2] b_empty[2] t_full[2] t_empty[2]
    const unsigned bar0 = su32(bars);
    auto BAR = [&](int kind, int i) { return bar0 + 8u * (2 * kind + i); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nblocks = nc / AT_N;
    const size_t ntiles = (n + AT_M - 1) / AT_M;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            bar_init(BAR(0, i), 64);   // a_full: the converter threads
            bar_init(BAR(1, i), 1);    // a_empty: MMA commit
            bar_init(BAR(2, i), 1);    // b_full: producer + TMA bytes
            bar_init(BAR(3, i), 1);    // b_empty: MMA commit
            bar_init(BAR(4, i), 1);    // t_full: MMA commit
            bar_init(BAR(5, i), 128);  // t_empty: epilogue threads
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    // |c|^2 of every centroid in shared memory (the epilogue reads 128 per
    // block as broadcast LDS instead of global loads)
    const float* cns = cnorm;
    if (nc <= CN_SMEM) {
        float* dst = reinterpret_cast<float*>(tmem_slot + 4);
        for (uint32_t k = threadIdx.x; k < nc; k += blockDim.x) dst[k] = __ldg(cnorm + k);
        __syncthreads();
        cns = dst;
    }

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_hi) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_lo) : "memory");
            uint32_t g = 0;
            for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x)
                for (uint32_t b = 0; b < nblocks; ++b, ++g) {
                    const uint32_t st = g & 1u, use = g >> 1;
                    if (use) bar_wait(BAR(3, st), (use - 1) & 1u);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(BAR(2, st)),
                                 "r"(B_BYTES) : "memory");
                    const unsigned dst = su32(Bs + st * B_BYTES);
                    const int row = (int)(b * AT_N);
                    tma_2d(dst, &map_hi, 0, row, BAR(2, st));
                    tma_2d(dst + 16384, &map_hi, 64, row, BAR(2, st));
                    tma_2d(dst + 32768, &map_lo, 0, row, BAR(2, st));
                    tma_2d(dst + 49152, &map_lo, 64, row, BAR(2, st));
                }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t g = 0, i = 0;
            for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
                const uint32_t a = i & 1u;
                bar_wait(BAR(0, a), (i >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned abase = su32(As + a * A_BYTES);
                for (uint32_t b = 0; b < nblocks; ++b, ++g) {
                    const uint32_t st = g & 1u, acc = g & 1u, use = g >> 1;
                    bar_wait(BAR(2, st), use & 1u);                  // centroid block landed
                    if (use) bar_wait(BAR(5, acc), (use - 1) & 1u);  // epilogue drained the accumulator
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const unsigned bbase = su32(Bs + st * B_BYTES);
                    const unsigned d = tmem + acc * AT_N;
#pragma unroll
                    for (int kk = 0; kk < AT_D / 16; ++kk) {
                        const unsigned off = (unsigned)(kk >> 2) * 16384u + (unsigned)(kk & 3) * 32u;
                        const uint64_t ad = sw128_desc(abase + off);
                        mma_f16(d, ad, sw128_desc(bbase + off), kk > 0 ? 1u : 0u);
                        mma_f16(d, ad, sw128_desc(bbase + 32768u + off), 1u);
                    }
                    mma_commit(BAR(3, st));  // smem stage free once these MMAs retire
                    mma_commit(BAR(4, acc)); // accumulator ready
                }
                mma_commit(BAR(1, a));  // the tile's rows are no longer read
            }
        }
    } else if (warp < 4) {
        // ------------------------------------------------ row converters
        const int cw = warp - 2;  // 0..1
        uint32_t i = 0;
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const uint32_t a = i & 1u;
            if (i >= 2) bar_wait(BAR(1, a), ((i >> 1) - 1) & 1u);
            uint8_t* A = As + a * A_BYTES;
            uint32_t pre[4];
#pragma unroll 1
            for (int r0 = cw; r0 < AT_M; r0 += 8) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // 4 rows' loads in flight
                const size_t rr = t * AT_M + r0 + 2 * u;
                pre[u] = rr < n ? __ldg(reinterpret_cast<const uint32_t*>(y + rr * AT_D) + lane) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = r0 + 2 * u;
                const uint32_t v = pre[u];
                // dims 4 lane .. 4 lane + 3: chunk (k & 63) / 8 of K half k / 64, swizzled by row
                const int k = 4 * lane, h = k >> 6, ch = ((k & 63) >> 3) ^ (r & 7);
                const __half2 lo = __halves2half2(__uint2half_rn(v & 0xff), __uint2half_rn((v >> 8) & 0xff));
                const __half2 hi = __halves2half2(__uint2half_rn((v >> 16) & 0xff), __uint2half_rn(v >> 24));
                uint2 pk;
                pk.x = *reinterpret_cast<const uint32_t*>(&lo);
                pk.y = *reinterpret_cast<const uint32_t*>(&hi);
                *reinterpret_cast<uint2*>(A + h * 16384 + (r >> 3) * 1024 + (r & 7) * 128 + ch * 16 + (k & 7) * 2) = pk;
                uint32_t s = (v & 0xff) * (v & 0xff) + ((v >> 8) & 0xff) * ((v >> 8) & 0xff) +
                             ((v >> 16) & 0xff) * ((v >> 16) & 0xff) + (v >> 24) * (v >> 24);
#pragma unroll
                for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) nx[a * AT_M + r] = (float)s;  // exact: < 2^24
            }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bar_arrive(BAR(0, a));
        }
    } else {
        // ------------------------------------------------ epilogue
        const int ew = warp - 4;  // TMEM lanes 32 ew .. 32 ew + 31
        const int r = 32 * ew + lane;
        const unsigned lane_off = (unsigned)(32 * ew) << 16;
        uint32_t g = 0, i = 0;
        for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const uint32_t a = i & 1u;
            bar_wait(BAR(0, a), (i >> 1) & 1u);
            const float xn = nx[a * AT_M + r];
            float v0 = __int_as_float(0x7f800000), v1 = v0, v2 = v0, v3 = v0;
            uint32_t i0 = 0, i1 = 0, i2 = 0;
            for (uint32_t b = 0; b < nblocks; ++b, ++g) {
                const uint32_t acc = g & 1u;
                bar_wait(BAR(4, acc), (g >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
                for (int c4 = 0; c4 < AT_N / 32; ++c4) {
                    uint32_t u[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
                          "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
                          "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
                          "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
                          "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
                        : "r"(tmem + lane_off + acc * AT_N + 32 * c4));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (c4 == AT_N / 32 - 1) {
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        bar_arrive(BAR(5, acc));
                    }
                    const uint32_t k0 = b * AT_N + 32 * c4;
                    const float4* cn4 = reinterpret_cast<const float4*>(cns + k0);
                    // the chunk's 32 estimates (independent ops), then the
                    // insertion only when one of them beats the 4th smallest
                    float dts[32];
                    float cmin = __int_as_float(0x7f800000);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 cn = cn4[q];
                        dts[4 * q + 0] = __fmaf_rn(-2.f, __uint_as_float(u[4 * q + 0]), __fadd_rn(xn, cn.x));
                        dts[4 * q + 1] = __fmaf_rn(-2.f, __uint_as_float(u[4 * q + 1]), __fadd_rn(xn, cn.y));
                        dts[4 * q + 2] = __fmaf_rn(-2.f, __uint_as_float(u[4 * q + 2]), __fadd_rn(xn, cn.z));
                        dts[4 * q + 3] = __fmaf_rn(-2.f, __uint_as_float(u[4 * q + 3]), __fadd_rn(xn, cn.w));
                        cmin = fminf(cmin, fminf(fminf(dts[4 * q], dts[4 * q + 1]), fminf(dts[4 * q + 2], dts[4 * q + 3])));
                    }
                    if (cmin < v3) {
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const float dt = dts[e];
                            if (dt < v3) {
                                const uint32_t k = k0 + e;
                                if (dt < v2) {
                                    v3 = v2;
                                    if (dt < v1) {
                                        v2 = v1, i2 = i1;
                                        if (dt < v0) v1 = v0, i1 = i0, v0 = dt, i0 = k;
                                        else v1 = dt, i1 = k;
                                    } else {
                                        v2 = dt, i2 = k;
                                    }
                                } else {
                                    v3 = dt;
                                }
                            }
                        }
                    }
                }
            }
            const size_t row = t * AT_M + r;
            if (row >= n) continue;
            // certification window: every centroid within 2 delta of the smallest D~
            const float thr = __fadd_rn(v0, 2.f * ldexpf(__fadd_rn(xn, cmax), -13));
            uint32_t best = i0;
            if (v3 <= thr) {
                const uint32_t slot = atomicAdd(ovf_cnt, 1u);
                ovf_rows[slot] = (uint32_t)row;
                best = 0xffffffffu;
            } else if (v1 <= thr) {
                const uint8_t* yr = y + row * AT_D;
                float bd = exact_row_dist(yr, coarse + (size_t)i0 * AT_D);
                const float d1 = exact_row_dist(yr, coarse + (size_t)i1 * AT_D);
                if (d1 < bd || (d1 == bd && i1 < best)) bd = d1, best = i1;
                if (v2 <= thr) {
                    const float d2 = exact_row_dist(yr, coarse + (size_t)i2 * AT_D);
                    if (d2 < bd || (d2 == bd && i2 < best)) bd = d2, best = i2;
                }
            }
            out[row] = best;
        }
    }
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// Search-side coarse distances on the same machinery: rows
// are queries already widened to f32 whose components are u8 integers (exact
// in fp16); the epilogue writes D~[q][c] = |x|^2 + |c|^2 - 2 <x, c>~ row-major
// for the certified top-w selection (k_coarse_tc.cu) and the per-row minimum
// and maximum as the certify kernel's order-preserving keys, so it skips its
// first pass over the row.
__device__ __forceinline__ uint32_t signed_key(float v) {
    const uint32_t u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(AT_THREADS, 1) dtilde_tc_kernel(
    const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
    const float* __restrict__ x, size_t n, const float* __restrict__ cnorm, uint32_t nc,
    float* __restrict__ Dt, uint32_t* __restrict__ kmm, uint32_t nsplit) {
    extern __shared__ uint8_t at_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>(((uintptr_t)at_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* As = sm;
    uint8_t* Bs = sm + 2 * A_BYTES;
    float* nx = reinterpret_cast<float*>(Bs + 2 * B_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(nx + 2 * AT_M);
    const unsigned bar0 = su32(bars);
    auto BAR = [&](int kind, int i) { return bar0 + 8u * (2 * kind + i); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // work unit = (128-query tile, a 1/nsplit range of the centroid blocks):
    // small batches spread one tile's centroids over several SMs
    const uint32_t nblocks_all = nc / AT_N;
    const size_t ntiles = (n + AT_M - 1) / AT_M;
    const size_t nunits = ntiles * nsplit;
    auto unit = [&](size_t u, size_t& t, uint32_t& b0, uint32_t& b1) {
        t = u / nsplit;
        const uint32_t sp = (uint32_t)(u % nsplit);
        b0 = (uint32_t)((uint64_t)nblocks_all * sp / nsplit);
        b1 = (uint32_t)((uint64_t)nblocks_all * (sp + 1) / nsplit);
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            bar_init(BAR(0, i), 64);
            bar_init(BAR(1, i), 1);
            bar_init(BAR(2, i), 1);
            bar_init(BAR(3, i), 1);
            bar_init(BAR(4, i), 1);
            bar_init(BAR(5, i), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    // |c|^2 of every centroid in shared memory (the epilogue reads 128 per
    // block as broadcast LDS instead of global loads)
    const float* cns = cnorm;
    if (nc <= CN_SMEM && nsplit == 1) {  // split small batches read their few blocks' |c|^2 directly
        float* dst = reinterpret_cast<float*>(tmem_slot + 4);
        for (uint32_t k = threadIdx.x; k < nc; k += blockDim.x) dst[k] = __ldg(cnorm + k);
        __syncthreads();
        cns = dst;
    }

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_hi) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_lo) : "memory");
            uint32_t g = 0;
            for (size_t u = blockIdx.x; u < nunits; u += gridDim.x) {
                size_t t;
                uint32_t bb0, bb1;
                unit(u, t, bb0, bb1);
                for (uint32_t b = bb0; b < bb1; ++b, ++g) {
                    const uint32_t st = g & 1u, use = g >> 1;
                    if (use) bar_wait(BAR(3, st), (use - 1) & 1u);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(BAR(2, st)),
                                 "r"(B_BYTES) : "memory");
                    const unsigned dst = su32(Bs + st * B_BYTES);
                    const int row = (int)(b * AT_N);
                    tma_2d(dst, &map_hi, 0, row, BAR(2, st));
                    tma_2d(dst + 16384, &map_hi, 64, row, BAR(2, st));
                    tma_2d(dst + 32768, &map_lo, 0, row, BAR(2, st));
                    tma_2d(dst + 49152, &map_lo, 64, row, BAR(2, st));
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            uint32_t g = 0, i = 0;
            for (size_t u = blockIdx.x; u < nunits; u += gridDim.x, ++i) {
                size_t t;
                uint32_t bb0, bb1;
                unit(u, t, bb0, bb1);
                const uint32_t a = i & 1u;
                bar_wait(BAR(0, a), (i >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned abase = su32(As + a * A_BYTES);
                for (uint32_t b = bb0; b < bb1; ++b, ++g) {
                    const uint32_t st = g & 1u, acc = g & 1u, use = g >> 1;
                    bar_wait(BAR(2, st), use & 1u);
                    if (use) bar_wait(BAR(5, acc), (use - 1) & 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const unsigned bbase = su32(Bs + st * B_BYTES);
                    const unsigned d = tmem + acc * AT_N;
#pragma unroll
                    for (int kk = 0; kk < AT_D / 16; ++kk) {
                        const unsigned off = (unsigned)(kk >> 2) * 16384u + (unsigned)(kk & 3) * 32u;
                        const uint64_t ad = sw128_desc(abase + off);
                        mma_f16(d, ad, sw128_desc(bbase + off), kk > 0 ? 1u : 0u);
                        mma_f16(d, ad, sw128_desc(bbase + 32768u + off), 1u);
                    }
                    mma_commit(BAR(3, st));
                    mma_commit(BAR(4, acc));
                }
                mma_commit(BAR(1, a));
            }
        }
    } else if (warp < 4) {
        const int cw = warp - 2;
        uint32_t i = 0;
        for (size_t u = blockIdx.x; u < nunits; u += gridDim.x, ++i) {
            const size_t t = u / nsplit;
            const uint32_t a = i & 1u;
            if (i >= 2) bar_wait(BAR(1, a), ((i >> 1) - 1) & 1u);
            uint8_t* A = As + a * A_BYTES;
            float4 pre[4];
#pragma unroll 1
            for (int r0 = cw; r0 < AT_M; r0 += 8) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // 4 rows' loads in flight
                const size_t rr = t * AT_M + r0 + 2 * u;
                pre[u] = rr < n ? __ldg(reinterpret_cast<const float4*>(x + rr * AT_D) + lane)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = r0 + 2 * u;
                const float4 v = pre[u];
                const int k = 4 * lane, h = k >> 6, ch = ((k & 63) >> 3) ^ (r & 7);
                const __half2 lo = __floats2half2_rn(v.x, v.y);  // u8 integers: exact
                const __half2 hi = __floats2half2_rn(v.z, v.w);
                uint2 pk;
                pk.x = *reinterpret_cast<const uint32_t*>(&lo);
                pk.y = *reinterpret_cast<const uint32_t*>(&hi);
                *reinterpret_cast<uint2*>(A + h * 16384 + (r >> 3) * 1024 + (r & 7) * 128 + ch * 16 + (k & 7) * 2) = pk;
                float s2 = __fmaf_rn(v.x, v.x, __fmaf_rn(v.y, v.y, __fmaf_rn(v.z, v.z, v.w * v.w)));
#pragma unroll
                for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
                if (lane == 0) nx[a * AT_M + r] = s2;  // exact: integer sum < 2^24
            }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bar_arrive(BAR(0, a));
        }
    } else {
        const int ew = warp - 4;
        const int r = 32 * ew + lane;
        const unsigned lane_off = (unsigned)(32 * ew) << 16;
        uint32_t g = 0, i = 0;
        for (size_t u = blockIdx.x; u < nunits; u += gridDim.x, ++i) {
            size_t t;
            uint32_t bb0, bb1;
            unit(u, t, bb0, bb1);
            const uint32_t a = i & 1u;
            bar_wait(BAR(0, a), (i >> 1) & 1u);
            const float xn = nx[a * AT_M + r];
            const size_t row = t * AT_M + r;
            const bool live = row < n;
            float* out = Dt + (live ? row : 0) * (size_t)nc;
            uint32_t kmin = 0xffffffffu, kmax = 0u;
            for (uint32_t b = bb0; b < bb1; ++b, ++g) {
                const uint32_t acc = g & 1u;
                bar_wait(BAR(4, acc), (g >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
                for (int c4 = 0; c4 < AT_N / 32; ++c4) {
                    uint32_t u[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
                          "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
                          "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
                          "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
                          "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
                        : "r"(tmem + lane_off + acc * AT_N + 32 * c4));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (c4 == AT_N / 32 - 1) {
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        bar_arrive(BAR(5, acc));
                    }
                    const uint32_t k0 = b * AT_N + 32 * c4;
                    const float4* cn4 = reinterpret_cast<const float4*>(cns + k0);
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4) {
                        const float4 cn = cn4[q4];
                        float4 dv;
                        dv.x = __fmaf_rn(-2.f, __uint_as_float(u[4 * q4 + 0]), __fadd_rn(xn, cn.x));
                        dv.y = __fmaf_rn(-2.f, __uint_as_float(u[4 * q4 + 1]), __fadd_rn(xn, cn.y));
                        dv.z = __fmaf_rn(-2.f, __uint_as_float(u[4 * q4 + 2]), __fadd_rn(xn, cn.z));
                        dv.w = __fmaf_rn(-2.f, __uint_as_float(u[4 * q4 + 3]), __fadd_rn(xn, cn.w));
                        kmin = min(kmin, min(min(signed_key(dv.x), signed_key(dv.y)),
                                             min(signed_key(dv.z), signed_key(dv.w))));
                        kmax = max(kmax, max(max(signed_key(dv.x), signed_key(dv.y)),
                                             max(signed_key(dv.z), signed_key(dv.w))));
                        if (live) __stcs(reinterpret_cast<float4*>(out + k0) + q4, dv);
                    }
                }
            }
            if (live) {  // kmm = [min keys n][max keys n], combined over the splits
                if (nsplit == 1) {
                    kmm[row] = kmin;
                    kmm[n + row] = kmax;
                } else {
                    atomicMin(kmm + row, kmin);
                    atomicMax(kmm + n + row, kmax);
                }
            }
        }
    }
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// Rows whose certification window held 4+ centroids: exact argmin, one warp
// per row, strict < in ascending index (kernels.cpp:29-35).
__global__ void assign_overflow_kernel(const uint8_t* __restrict__ y, const float* __restrict__ coarse,
                                       uint32_t nc, const uint32_t* __restrict__ rows,
                                       const uint32_t* __restrict__ cnt, uint32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint32_t nrows = *cnt;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nrows;
         w += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t row = rows[w];
        float bd = __int_as_float(0x7f800000);
        uint32_t bi = 0xffffffffu;
        for (uint32_t k = lane; k < nc; k += 32) {
            const float dk = exact_row_dist(y + (size_t)row * AT_D, coarse + (size_t)k * AT_D);
            if (dk < bd) bd = dk, bi = k;  // ascending k per lane
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const float od = __shfl_xor_sync(0xffffffffu, bd, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (od < bd || (od == bd && oi < bi)) bd = od, bi = oi;
        }
        if (lane == 0) out[row] = bi;
    }
}

__global__ void split_centroids_kernel(const float* __restrict__ c, size_t total, __half* __restrict__ hi,
                                       __half* __restrict__ lo) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const float v = c[i];
        const __half h = __float2half_rn(v);
        hi[i] = h;
        lo[i] = __float2half_rn(__fsub_rn(v, __half2float(h)));  // exact difference
    }
}

__global__ void centroid_norms_kernel(const float* __restrict__ c, uint32_t nc, float* __restrict__ out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nc) return;
    float s = 0.f;
    for (int t = 0; t < AT_D; ++t) s = __fmaf_rn(c[(size_t)k * AT_D + t], c[(size_t)k * AT_D + t], s);
    out[k] = s;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        PQRR_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

CUtensorMap make_map(const __half* base, uint32_t rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {AT_D, rows};
    const cuuint64_t strides[1] = {AT_D * sizeof(__half)};
    const cuuint32_t box[2] = {64, AT_N};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed");
    return m;
}

}  // namespace

bool assign_tc_supported(uint32_t d, uint32_t nc) { return d == AT_D && nc >= AT_N && nc % AT_N == 0; }

void AssignTc::dtilde(const float* x, size_t n, float* Dt, uint32_t* kmm, cudaStream_t s) {
    if (n == 0) return;
    const CUtensorMap mh = make_map(static_cast<const __half*>(hi), nc);
    const CUtensorMap ml = make_map(static_cast<const __half*>(lo), nc);
    set_max_smem((const void*)dtilde_tc_kernel, SMEM_BYTES);
    const size_t ntiles = (n + AT_M - 1) / AT_M;
    const uint32_t nblocks = nc / AT_N, sms = (uint32_t)sm_count();
    // fewer tiles than SMs: split each tile's centroid blocks over the idle SMs
    const uint32_t nsplit = ntiles >= sms ? 1u : std::min<uint32_t>(nblocks, (uint32_t)(sms / ntiles));
    if (nsplit > 1) {
        PQRR_CUDA(cudaMemsetAsync(kmm, 0xff, n * sizeof(uint32_t), s));
        PQRR_CUDA(cudaMemsetAsync(kmm + n, 0, n * sizeof(uint32_t), s));
    }
    const unsigned grid = (unsigned)std::min<size_t>(ntiles * nsplit, (size_t)sms);
    dtilde_tc_kernel<<<grid, AT_THREADS, SMEM_BYTES, s>>>(mh, ml, x, n, cn, nc, Dt, kmm, nsplit);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

AssignTc::~AssignTc() {
    if (hi) cudaFree(hi);
    if (lo) cudaFree(lo);
    if (cn) cudaFree(cn);
}

// One-time preparation per coarse quantizer: the fp16 split, |c|^2 and their
// maximum.  Returns false (exact path) when a centroid is not finite or too
// large for fp16.
bool AssignTc::prepare(const float* coarse, uint32_t nc_, cudaStream_t s) {
    if (ready) return usable;
    ready = true;
    nc = nc_;
    std::vector<float> h((size_t)nc * AT_D);
    PQRR_CUDA(cudaMemcpyAsync(h.data(), coarse, h.size() * 4, cudaMemcpyDeviceToHost, s));
    PQRR_CUDA(cudaStreamSynchronize(s));
    double mx = 0.0;
    for (size_t k = 0; k < nc; ++k) {
        double sq = 0.0;
        for (int t = 0; t < AT_D; ++t) {
            const float v = h[k * AT_D + t];
            if (!(v > -60000.f && v < 60000.f)) return usable = false;
            sq += (double)v * v;
        }
        mx = sq > mx ? sq : mx;
    }
    cmax = (float)(mx * (1.0 + 1.0 / 1024));
    const size_t total = (size_t)nc * AT_D;
    PQRR_CUDA(cudaMalloc(&hi, total * 2));
    PQRR_CUDA(cudaMalloc(&lo, total * 2));
    PQRR_CUDA(cudaMalloc(&cn, (size_t)nc * 4));
    split_centroids_kernel<<<256, 256, 0, s>>>(coarse, total, static_cast<__half*>(hi), static_cast<__half*>(lo));
    PQRR_LAUNCH_CHECK();
    centroid_norms_kernel<<<(nc + 127) / 128, 128, 0, s>>>(coarse, nc, cn);
    PQRR_LAUNCH_CHECK();
    count_launch(2);
    return usable = true;
}

void AssignTc::assign(const uint8_t* y, size_t n, const float* coarse, uint32_t* out, cudaStream_t s) {
    if (n == 0) return;
    const CUtensorMap mh = make_map(static_cast<const __half*>(hi), nc);
    const CUtensorMap ml = make_map(static_cast<const __half*>(lo), nc);
    uint32_t* ovf = nullptr;
    PQRR_CUDA(cudaMallocAsync(&ovf, (n + 1) * sizeof(uint32_t), s));
    PQRR_CUDA(cudaMemsetAsync(ovf + n, 0, sizeof(uint32_t), s));
    set_max_smem((const void*)assign_tc_kernel, (size_t)((int)SMEM_BYTES));
    const size_t ntiles = (n + AT_M - 1) / AT_M;
    const unsigned grid = (unsigned)std::min<size_t>(ntiles, (size_t)sm_count());
    assign_tc_kernel<<<grid, AT_THREADS, SMEM_BYTES, s>>>(mh, ml, y, n, coarse, cn, nc, cmax, out, ovf, ovf + n);
    PQRR_LAUNCH_CHECK();
    assign_overflow_kernel<<<sm_count(), 256, 0, s>>>(y, coarse, nc, ovf, ovf + n, out);
    PQRR_LAUNCH_CHECK();
    count_launch(2);
    PQRR_CUDA(cudaFreeAsync(ovf, s));
}

}  // namespace pqrr_b200
