// k_encode.cu — K6: the add/encode path (ivf_build + ivf_refine_encode,
// ivf_index.hpp:54-56 / :72-73) and the plain PQ codec of the kernel seam
// (kernels::encode_batch / decode_batch, kernels.cpp:41-53).
//
// Layout: a CTA owns 32 vectors; warp w handles sub-quantizers w, w+8, ...,
// lane v handles vector v, so every lane of a warp reads the same centroid of
// the same sub-codebook (a broadcast load) and the per-lane residual lives in
// registers.  Each argmin is a strict-< scan in ascending centroid index
// (lowest index wins ties) over l2_sq in the reference order.
// Residual conventions: r0 = y - C_a, rec1 = C_a + p
// computed first, r1 = y - rec1.
#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int EV = 32;      // vectors per CTA
constexpr int EW = 8;       // warps per CTA

// argmin_i l2_sq(r, book[i]) with r in registers (DS known at compile time).
template <int DS>
__device__ __forceinline__ uint32_t nearest_code(const float (&r)[DS], const float* __restrict__ book,
                                                 uint32_t ks, u64 nz) {
    uint32_t best = 0;
    float bd = __int_as_float(0x7f800000);
    for (uint32_t i = 0; i < ks; ++i) {
        const float* b = book + (size_t)i * DS;
        float dd;
        if constexpr (DS % 4 == 0) {
            u64 s01 = 0, s23 = 0;
#pragma unroll
            for (int t = 0; t < DS; t += 4) {
                const float4 c = __ldg(reinterpret_cast<const float4*>(b + t));
                s01 = acc_sq2(s01, pk2(r[t], r[t + 1]), pk2(c.x, c.y), nz);
                s23 = acc_sq2(s23, pk2(r[t + 2], r[t + 3]), pk2(c.z, c.w), nz);
            }
            dd = __fadd_rn(__fadd_rn(lo2(s01), hi2(s01)), __fadd_rn(lo2(s23), hi2(s23)));
        } else {
            float bb[DS];
#pragma unroll
            for (int t = 0; t < DS; ++t) bb[t] = __ldg(b + t);
            dd = l2sq_scalar(r, bb, DS);
        }
        if (i == 0 || dd < bd) {
            bd = dd;
            best = i;
        }
    }
    return best;
}

// Runtime-dimension fallback (any dsub <= 64).
__device__ uint32_t nearest_code_rt(const float* r, int ds, const float* __restrict__ book,
                                    uint32_t ks) {
    uint32_t best = 0;
    float bd = 0.f;
    for (uint32_t i = 0; i < ks; ++i) {
        float dd = l2sq_scalar(r, book + (size_t)i * ds, ds);
        if (i == 0 || dd < bd) {
            bd = dd;
            best = i;
        }
    }
    return best;
}

template <int DS>
__device__ __forceinline__ uint32_t encode_sub(const float* __restrict__ ys, int yld,
                                               const float* __restrict__ crow, int t0,
                                               const float* __restrict__ book, uint32_t ks, u64 nz,
                                               int ds_rt) {
    if constexpr (DS > 0) {
        float r[DS];
#pragma unroll
        for (int t = 0; t < DS; ++t)
            r[t] = crow ? __fsub_rn(ys[t0 + t], __ldg(crow + t0 + t)) : ys[t0 + t];
        return nearest_code<DS>(r, book, ks, nz);
    } else {
        float r[64];
        for (int t = 0; t < ds_rt; ++t)
            r[t] = crow ? __fsub_rn(ys[t0 + t], __ldg(crow + t0 + t)) : ys[t0 + t];
        return nearest_code_rt(r, ds_rt, book, ks);
    }
    (void)yld;
}

// r1[t] = y[t] - (C_a[t] + p[t]) with p the first-stage decode (ivf_index.hpp:66-67).
__device__ __forceinline__ float refine_residual(const float* y, const float* __restrict__ crow,
                                                 const float* __restrict__ books,
                                                 const uint8_t* code, uint32_t ks, int ds, int t) {
    const int jj = t / ds;
    const float p = __ldg(books + ((size_t)jj * ks + code[jj]) * ds + (t - jj * ds));
    const float rec1 = __fadd_rn(__ldg(crow + t), p);
    return __fsub_rn(y[t], rec1);
}

template <int DS, int DSR>
__global__ __launch_bounds__(256) void ivf_encode_kernel(
    const float* __restrict__ xf, const uint8_t* __restrict__ xu, size_t n, uint32_t d,
    const uint32_t* __restrict__ assign, const float* __restrict__ coarse,
    const float* __restrict__ books, uint32_t m, const float* __restrict__ rbooks, uint32_t mprime,
    uint32_t ks, uint8_t* __restrict__ codes, uint8_t* __restrict__ rcodes, u64 nz) {
    extern __shared__ float ys_all[];
    const int yld = (int)d + 1;
    float* ys = ys_all;                                       // [EV][d+1]
    uint8_t* cs = reinterpret_cast<uint8_t*>(ys + EV * yld);  // [EV][m]
    uint8_t* rs = cs + EV * m;                                // [EV][mprime]
    __shared__ uint32_t as[EV];
    const size_t v0 = (size_t)blockIdx.x * EV;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t idx = threadIdx.x; idx < EV * d; idx += blockDim.x) {
        uint32_t v = idx / d, t = idx % d;
        float val = 0.f;
        if (v0 + v < n) val = xf ? xf[(v0 + v) * d + t] : (float)xu[(v0 + v) * d + t];
        ys[v * yld + t] = val;
    }
    if (threadIdx.x < EV) as[threadIdx.x] = (v0 + threadIdx.x < n) ? assign[v0 + threadIdx.x] : 0u;
    __syncthreads();
    const float* y = ys + lane * yld;
    const float* crow = coarse + (size_t)as[lane] * d;
    const int ds = (int)(d / m), dsr = mprime ? (int)(d / mprime) : 0;
    // phase 1: first-stage codes of r0 = y - C_a
    for (uint32_t j = warp; j < m; j += EW) {
        uint32_t code = encode_sub<DS>(y, yld, crow, (int)j * ds,
                                       books + (size_t)j * ks * ds, ks, nz, ds);
        cs[lane * m + j] = (uint8_t)code;
    }
    __syncthreads();
    // phase 2: refine codes of r1 = y - (C_a + p)
    if (mprime) {
        for (uint32_t j = warp; j < mprime; j += EW) {
            const int t0 = (int)j * dsr;
            uint32_t code;
            if constexpr (DSR > 0) {
                float r[DSR];
#pragma unroll
                for (int tt = 0; tt < DSR; ++tt) r[tt] = refine_residual(y, crow, books, cs + lane * m, ks, ds, t0 + tt);
                code = nearest_code<DSR>(r, rbooks + (size_t)j * ks * dsr, ks, nz);
            } else {
                float r[64];
                for (int tt = 0; tt < dsr; ++tt) r[tt] = refine_residual(y, crow, books, cs + lane * m, ks, ds, t0 + tt);
                code = nearest_code_rt(r, dsr, rbooks + (size_t)j * ks * dsr, ks);
            }
            rs[lane * mprime + j] = (uint8_t)code;
        }
    }
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < EV * m; idx += blockDim.x) {
        uint32_t v = idx / m;
        if (v0 + v < n) codes[v0 * m + idx] = cs[idx];
    }
    if (mprime)
        for (uint32_t idx = threadIdx.x; idx < EV * mprime; idx += blockDim.x) {
            uint32_t v = idx / mprime;
            if (v0 + v < n) rcodes[v0 * mprime + idx] = rs[idx];
        }
}

// Plain PQ encode (no coarse residual).
template <int DS>
__global__ __launch_bounds__(256) void pq_encode_kernel(const float* __restrict__ x, size_t n,
                                                        uint32_t d, const float* __restrict__ books,
                                                        uint32_t m, uint32_t ks,
                                                        uint8_t* __restrict__ codes, u64 nz) {
    extern __shared__ float ys_all[];
    const int yld = (int)d + 1;
    float* ys = ys_all;
    const size_t v0 = (size_t)blockIdx.x * EV;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t idx = threadIdx.x; idx < EV * d; idx += blockDim.x) {
        uint32_t v = idx / d, t = idx % d;
        ys[v * yld + t] = (v0 + v < n) ? x[(v0 + v) * d + t] : 0.f;
    }
    __syncthreads();
    const int ds = (int)(d / m);
    for (uint32_t j = warp; j < m; j += EW) {
        uint32_t code = encode_sub<DS>(ys + lane * yld, yld, nullptr, (int)j * ds,
                                       books + (size_t)j * ks * ds, ks, nz, ds);
        if (v0 + lane < n) codes[(v0 + lane) * m + j] = (uint8_t)code;
    }
}

__global__ void pq_decode_kernel(const uint8_t* __restrict__ codes, size_t n, uint32_t d,
                                 const float* __restrict__ books, uint32_t m, uint32_t ks,
                                 float* __restrict__ out) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * d) return;
    size_t v = idx / d;
    uint32_t t = (uint32_t)(idx % d);
    uint32_t ds = d / m, j = t / ds;
    out[idx] = books[((size_t)j * ks + codes[v * m + j]) * ds + (t - j * ds)];
}

template <int DS, int DSR>
void ivf_encode_t(const float* xf, const uint8_t* xu, size_t n, uint32_t d, const uint32_t* assign,
                  const float* coarse, const float* books, uint32_t m, const float* rbooks,
                  uint32_t mprime, uint32_t ks, uint8_t* codes, uint8_t* rcodes, cudaStream_t s) {
    size_t smem = (size_t)EV * (d + 1) * sizeof(float) + EV * (m + mprime);
    smem = (smem + 15) & ~size_t(15);
    set_max_smem((const void*)ivf_encode_kernel<DS, DSR>, (size_t)((int)smem));
    ivf_encode_kernel<DS, DSR><<<(unsigned)((n + EV - 1) / EV), EV * EW, smem, s>>>(
        xf, xu, n, d, assign, coarse, books, m, rbooks, mprime, ks, codes, rcodes, kNegZero2);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

template <int DS>
void ivf_encode_r(int dsr, const float* xf, const uint8_t* xu, size_t n, uint32_t d,
                  const uint32_t* assign, const float* coarse, const float* books, uint32_t m,
                  const float* rbooks, uint32_t mprime, uint32_t ks, uint8_t* codes,
                  uint8_t* rcodes, cudaStream_t s) {
    switch (dsr) {
        case 16: return ivf_encode_t<DS, 16>(xf, xu, n, d, assign, coarse, books, m, rbooks, mprime, ks, codes, rcodes, s);
        case 8: return ivf_encode_t<DS, 8>(xf, xu, n, d, assign, coarse, books, m, rbooks, mprime, ks, codes, rcodes, s);
        case 4: return ivf_encode_t<DS, 4>(xf, xu, n, d, assign, coarse, books, m, rbooks, mprime, ks, codes, rcodes, s);
        default: return ivf_encode_t<DS, 0>(xf, xu, n, d, assign, coarse, books, m, rbooks, mprime, ks, codes, rcodes, s);
    }
}

}  // namespace

void launch_ivf_encode(const float* x_f32, const uint8_t* x_u8, size_t n, uint32_t d,
                       const uint32_t* assign, const float* coarse, const float* books, uint32_t m,
                       const float* rbooks, uint32_t mprime, uint32_t ks, uint8_t* codes,
                       uint8_t* rcodes, cudaStream_t s) {
    if (n == 0) return;
    if (d / m > 64 || (mprime && d / mprime > 64))
        throw ArgError("sub-vector dimension above 64 is not supported on the device");
    const int ds = (int)(d / m), dsr = mprime ? (int)(d / mprime) : 0;
    switch (ds) {
        case 16: return ivf_encode_r<16>(dsr, x_f32, x_u8, n, d, assign, coarse, books, m, rbooks, mprime, ks, codes, rcodes, s);
        case 8: return ivf_encode_r<8>(dsr, x_f32, x_u8, n, d, assign, coarse, books, m, rbooks, mprime, ks, codes, rcodes, s);
        case 4: return ivf_encode_r<4>(dsr, x_f32, x_u8, n, d, assign, coarse, books, m, rbooks, mprime, ks, codes, rcodes, s);
        default: return ivf_encode_r<0>(dsr, x_f32, x_u8, n, d, assign, coarse, books, m, rbooks, mprime, ks, codes, rcodes, s);
    }
}

void launch_pq_encode(const float* data, size_t n, uint32_t d, const float* books, uint32_t m,
                      uint32_t ks, uint8_t* codes, cudaStream_t s) {
    if (n == 0) return;
    if (d / m > 64) throw ArgError("sub-vector dimension above 64 is not supported on the device");
    size_t smem = (size_t)EV * (d + 1) * sizeof(float);
    const unsigned grid = (unsigned)((n + EV - 1) / EV);
#define PQE(DS)                                                                                  \
    do {                                                                                         \
        set_max_smem((const void*)pq_encode_kernel<DS>, smem);                                  \
        pq_encode_kernel<DS><<<grid, EV * EW, smem, s>>>(data, n, d, books, m, ks, codes,         \
                                                         kNegZero2);                             \
    } while (0)
    switch (d / m) {
        case 16: PQE(16); break;
        case 8: PQE(8); break;
        case 4: PQE(4); break;
        default: PQE(0); break;
    }
#undef PQE
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_pq_decode(const uint8_t* codes, size_t n, uint32_t d, const float* books, uint32_t m,
                      uint32_t ks, float* out, cudaStream_t s) {
    if (n == 0) return;
    size_t total = n * d;
    pq_decode_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(codes, n, d, books, m, ks, out);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
