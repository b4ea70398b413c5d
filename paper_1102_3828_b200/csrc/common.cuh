// common.cuh — shared device helpers for the pqrr B200 kernels (sm_100a).
//
// Exact arithmetic: every distance follows the reference l2_sq order
// (distance.hpp:16-33): t = a - b, s[j mod 4] += t*t, remainder into s0..s2,
// result (s0 + s1) + (s2 + s3), with SEPARATE multiply and add roundings.
// nvcc contracts a*b+c into FFMA by default, and ptxas 12.9 even contracts
// explicit `mul.rn.f32x2` + `add.rn.f32x2` into FFMA2 (verified in SASS, with
// and without --fmad=false).  So packed products are computed as
// fma(t, t, nz) where nz = -0.0 arrives as a kernel parameter that ptxas cannot
// see through: t*t + (-0) rounds once, i.e. equals the rounded product exactly
// (and +0 stays +0), and the following FADD2 cannot fuse with an FFMA2.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pqrr_b200 {

typedef unsigned long long u64;

// ------------------------------------------------------------ packed f32x2
__device__ __forceinline__ u64 pk2(float lo, float hi) {
    return (u64)__float_as_uint(lo) | ((u64)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float lo2(u64 v) { return __uint_as_float((unsigned)(v & 0xffffffffull)); }
__device__ __forceinline__ float hi2(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }

__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// Exact rounded square of each lane: fma(t, t, nz) with nz = {-0,-0} opaque.
__device__ __forceinline__ u64 sq2(u64 t, u64 nz) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(t), "l"(nz));
    return r;
}
// s += t*t for both lanes, exact order.
__device__ __forceinline__ u64 acc_sq2(u64 s, u64 a, u64 b, u64 nz) {
    return add2(s, sq2(sub2(a, b), nz));
}

static const u64 kNegZero2 = 0x8000000080000000ull;

// ------------------------------------------------------------ scalar exact
// Generic l2_sq in the reference order (any d, any alignment).
__device__ __forceinline__ float l2sq_scalar(const float* a, const float* b, int d) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int j = 0;
    for (; j + 4 <= d; j += 4) {
        float t0 = __fsub_rn(a[j], b[j]);
        float t1 = __fsub_rn(a[j + 1], b[j + 1]);
        float t2 = __fsub_rn(a[j + 2], b[j + 2]);
        float t3 = __fsub_rn(a[j + 3], b[j + 3]);
        s0 = __fadd_rn(s0, __fmul_rn(t0, t0));
        s1 = __fadd_rn(s1, __fmul_rn(t1, t1));
        s2 = __fadd_rn(s2, __fmul_rn(t2, t2));
        s3 = __fadd_rn(s3, __fmul_rn(t3, t3));
    }
    if (j < d) { float t = __fsub_rn(a[j], b[j]); s0 = __fadd_rn(s0, __fmul_rn(t, t)); ++j; }
    if (j < d) { float t = __fsub_rn(a[j], b[j]); s1 = __fadd_rn(s1, __fmul_rn(t, t)); ++j; }
    if (j < d) { float t = __fsub_rn(a[j], b[j]); s2 = __fadd_rn(s2, __fmul_rn(t, t)); ++j; }
    return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
}

// Packed l2_sq for d % 4 == 0 with both operands 16-byte aligned.
// s01 holds (s0, s1), s23 holds (s2, s3).
template <int D>
__device__ __forceinline__ float l2sq_packed(const float* __restrict__ a,
                                             const float* __restrict__ b, u64 nz) {
    static_assert(D % 4 == 0, "packed l2_sq needs d % 4 == 0");
    u64 s01 = 0, s23 = 0;
#pragma unroll
    for (int j = 0; j < D; j += 4) {
        const float4 x = *reinterpret_cast<const float4*>(a + j);
        const float4 y = *reinterpret_cast<const float4*>(b + j);
        s01 = acc_sq2(s01, pk2(x.x, x.y), pk2(y.x, y.y), nz);
        s23 = acc_sq2(s23, pk2(x.z, x.w), pk2(y.z, y.w), nz);
    }
    return __fadd_rn(__fadd_rn(lo2(s01), hi2(s01)), __fadd_rn(lo2(s23), hi2(s23)));
}

// Total order of types.hpp:47-50 on (dist, id) as one 64-bit key.  Distances
// are non-negative (sums of squares starting at +0), so the IEEE bit pattern
// orders like the value.
__device__ __forceinline__ u64 nb_key(float dist, uint32_t id) {
    return ((u64)__float_as_uint(dist) << 32) | (u64)id;
}
__device__ __forceinline__ float key_dist(u64 k) { return __uint_as_float((unsigned)(k >> 32)); }
__device__ __forceinline__ uint32_t key_id(u64 k) { return (uint32_t)(k & 0xffffffffull); }

// A pair can have a candidate (dist <= tau) only if sum_m <= tau (within the
// roundings slot_params covers); the same test as slot_params' dead case.
__device__ __forceinline__ bool pair_live(float tau, float summ) {
    const float e_up = 1.000003814697265625f, e_dn = 0.999996185302734375f;  // 1 +- 2^-18
    if (!(tau < __int_as_float(0x7f800000))) return true;
    return __fsub_rn(__fmul_rn(tau, e_up), __fmul_rn(summ, e_dn)) >= 0.f;
}

// Position of threshold sample si at stride st in a list of len entries.  The
// list order pairs entries by code parity (pair_perm_kernel), so an even
// stride alone would only ever sample one side of the pairs (a biased
// sample: measured as frequent under-full retries at even strides).  A
// Thue-Morse jitter popc(si) & 1 balances both sides on every sub-grid
// si = k 2^s that the per-lane tiers of the LUT pass take.  At stride 1 every
// entry is sampled exactly once (the exact case the retry ladder ends in), so
// no jitter applies there; at stride >= 2 the jittered positions stay distinct.
__device__ __forceinline__ uint32_t sample_pos(uint32_t si, uint32_t st, uint32_t len) {
    const uint32_t jit = st > 1u ? ((uint32_t)__popc(si) & 1u) : 0u;
    return min(si * st + jit, len - 1u);
}

// 8-bit LUT block of a LUT-pass item (K2 -> K4f): LANE-major, 16 query lanes
// x (M * KS) row bytes, so K4f can copy any lane's 2 KiB column with
// coalesced 16-byte loads.  r0..r3 hold rows 4 rq .. 4 rq + 3, each the bytes
// of lanes 4 g .. 4 g + 3; a 4 x 4 byte transpose gives each lane's 4 rows.
__device__ __forceinline__ void q8_put_rows(uint32_t* __restrict__ block, int g, int rq, uint32_t r0,
                                            uint32_t r1, uint32_t r2, uint32_t r3) {
    constexpr int LANE_WORDS = 8 * 256 / 4;  // one lane's column (M = 8, KS = 256)
    const uint32_t lo01 = __byte_perm(r0, r1, 0x5140), hi01 = __byte_perm(r0, r1, 0x7362);
    const uint32_t lo23 = __byte_perm(r2, r3, 0x5140), hi23 = __byte_perm(r2, r3, 0x7362);
    block[(4 * g + 0) * LANE_WORDS + rq] = __byte_perm(lo01, lo23, 0x5410);
    block[(4 * g + 1) * LANE_WORDS + rq] = __byte_perm(lo01, lo23, 0x7632);
    block[(4 * g + 2) * LANE_WORDS + rq] = __byte_perm(hi01, hi23, 0x5410);
    block[(4 * g + 3) * LANE_WORDS + rq] = __byte_perm(hi01, hi23, 0x7632);
}

// Ascending bitonic sort of a[0, n2) in shared memory by the whole CTA (n2 a
// power of two >= 32, blockDim.x a multiple of 32).  Element i lives with
// thread i % blockDim.x, so partners at distance < 32 sit in one warp: those
// steps run in registers through shuffles, and only the steps at distance
// >= 32 go through shared memory and a block barrier (n2 = 1024: 21 barriers
// instead of 55 — single-CTA sorts of small batches are barrier bound).
template <class T>
__device__ __forceinline__ void cta_bitonic_sort(T* a, uint32_t n2) {
    for (uint32_t k = 2; k <= n2; k <<= 1) {
        uint32_t j = k >> 1;
        if (k <= 32) {
            if (k != 2) continue;  // k = 2..32 are done together below
        } else {
            for (; j >= 32; j >>= 1) {
                for (uint32_t i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                    const uint32_t lo = 2 * i - (i & (j - 1)), hi = lo + j;
                    const bool up = (lo & k) == 0;
                    const T x = a[lo], y = a[hi];
                    if ((x > y) == up) {
                        a[lo] = y;
                        a[hi] = x;
                    }
                }
                __syncthreads();
            }
        }
        for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
            T v = a[i];
            if (k == 2) {
#pragma unroll
                for (uint32_t kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
                    for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
                        const T o = __shfl_xor_sync(0xffffffffu, v, jj);
                        const bool keep_min = ((i & jj) == 0) == ((i & kk) == 0);
                        v = (keep_min == (v < o)) ? v : o;
                    }
            } else {
#pragma unroll
                for (uint32_t jj = 16; jj > 0; jj >>= 1) {
                    const T o = __shfl_xor_sync(0xffffffffu, v, jj);
                    const bool keep_min = ((i & jj) == 0) == ((i & k) == 0);
                    v = (keep_min == (v < o)) ? v : o;
                }
            }
            a[i] = v;
        }
        __syncthreads();
    }
}

// Upper bound of the R-th smallest value a CTA holds, without atomics: every
// thread passes the minimum of the values it read (all threads must have read
// at least one); the R-th smallest of those minima has at least R values at or
// below it.  A histogram-based select then only counts the values <= the
// bound — the low tail — instead of serialising its shared-memory atomics on
// the few bins that hold nearly every value.  blockDim.x must be a power of
// two >= 32, R <= blockDim.x; s_mins holds blockDim.x words.  All threads call.
__device__ __forceinline__ uint32_t cta_tail_bound(uint32_t my_min, uint32_t R, uint32_t* s_mins) {
    s_mins[threadIdx.x] = my_min;
    __syncthreads();
    cta_bitonic_sort(s_mins, blockDim.x);
    return s_mins[R - 1];
}

}  // namespace pqrr_b200
