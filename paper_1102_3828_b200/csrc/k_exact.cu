// k_exact.cu — exact k-nearest-neighbour ground truth for u8 vectors
// (compute_groundtruth / exact_search, eval.hpp:13-19) on the integer tensor
// cores.
//
// For u8 vectors every squared distance is an integer
//     |x - y|^2 = |x|^2 + |y|^2 - 2 <x, y>  <=  128 * 255^2 < 2^24,
// so int32 arithmetic (mma.sync m16n8k32 u8 x u8 -> s32) gives it exactly, and
// so does its float value: the reference accumulates in double, and every
// summation order gives the same integer.  A CTA computes a 64-query x
// 128-vector tile of distances for a chunk of the base; per chunk the k
// smallest (dist, id) of every query are selected (launch_select_topk) and
// merged with the running result (launch_merge_topk), ties by id
// (types.hpp:47-50).
#include <algorithm>
#include <functional>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int EQ = 64, EB = 128, ED = 128;  // queries x base vectors per CTA, dims
constexpr int ELD = ED + 16;                // smem row stride (bytes): conflict-free fragment loads

__device__ __forceinline__ void mma_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void u8_norms_kernel(const uint8_t* __restrict__ v, size_t n, int* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4* r = reinterpret_cast<const uint4*>(v + i * ED);
    int s = 0;
#pragma unroll
    for (int c = 0; c < ED / 16; ++c) {
        const uint4 u = r[c];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int t = (w[k] >> (8 * b)) & 0xff;
                s += t * t;
            }
    }
    out[i] = s;
}

// D[q][i] = |x_q|^2 + |y_i|^2 - 2 <x_q, y_i> for a chunk of nb base rows.
// 8 warps: 4 (16 queries) x 2 (64 vectors = 8 n-tiles); K = 128 = 4 k-steps.
__global__ __launch_bounds__(256) void exact_dist_kernel(const uint8_t* __restrict__ xq, const int* __restrict__ qn,
                                                        size_t nq, const uint8_t* __restrict__ yb,
                                                        const int* __restrict__ bn, uint32_t nb,
                                                        float* __restrict__ D, unsigned long long* __restrict__ best,
                                                        uint64_t id_base) {
    __shared__ __align__(16) uint8_t sq[EQ * ELD], sb[EB * ELD];
    const size_t q0 = (size_t)blockIdx.y * EQ;
    const uint32_t b0 = blockIdx.x * EB;
    for (int i = threadIdx.x; i < EQ * (ED / 16); i += blockDim.x) {
        const int r = i / (ED / 16), c = i % (ED / 16);
        uint4 v = make_uint4(0, 0, 0, 0);
        if (q0 + r < nq) v = *reinterpret_cast<const uint4*>(xq + (q0 + r) * ED + 16 * c);
        *reinterpret_cast<uint4*>(sq + r * ELD + 16 * c) = v;
    }
    for (int i = threadIdx.x; i < EB * (ED / 16); i += blockDim.x) {
        const int r = i / (ED / 16), c = i % (ED / 16);
        uint4 v = make_uint4(0, 0, 0, 0);
        if (b0 + r < nb) v = *reinterpret_cast<const uint4*>(yb + ((size_t)b0 + r) * ED + 16 * c);
        *reinterpret_cast<uint4*>(sb + r * ELD + 16 * c) = v;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int wq = (warp & 3) * 16, wb = (warp >> 2) * 64;
    int acc[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[nt][e] = 0;
#pragma unroll
    for (int ks = 0; ks < ED / 32; ++ks) {
        const uint8_t* ar = sq + (wq + g) * ELD + ks * 32 + 4 * tig;
        const uint32_t a0 = *reinterpret_cast<const uint32_t*>(ar);
        const uint32_t a1 = *reinterpret_cast<const uint32_t*>(ar + 8 * ELD);
        const uint32_t a2 = *reinterpret_cast<const uint32_t*>(ar + 16);
        const uint32_t a3 = *reinterpret_cast<const uint32_t*>(ar + 8 * ELD + 16);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            const uint8_t* br = sb + (wb + nt * 8 + g) * ELD + ks * 32 + 4 * tig;
            mma_u8(acc[nt], a0, a1, a2, a3, *reinterpret_cast<const uint32_t*>(br),
                   *reinterpret_cast<const uint32_t*>(br + 16));
        }
    }
    if (best) {  // k = 1: fused argmin under (dist, id), no distance matrix
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const size_t q = q0 + wq + g + 8 * h;
            const int xn = q < nq ? qn[q] : 0;
            unsigned long long m = ~0ull;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t i = b0 + wb + nt * 8 + 2 * tig + e;
                    if (i < nb) {
                        const float dd = (float)(xn + bn[i] - 2 * acc[nt][2 * h + e]);
                        m = min(m, ((unsigned long long)__float_as_uint(dd) << 32) | (uint32_t)(id_base + i));
                    }
                }
            m = min(m, __shfl_xor_sync(0xffffffffu, m, 1));
            m = min(m, __shfl_xor_sync(0xffffffffu, m, 2));
            if (tig == 0 && q < nq && m != ~0ull) atomicMin(best + q, m);
        }
        return;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const size_t q = q0 + wq + g + 8 * h;
        if (q >= nq) continue;
        const int xn = qn[q];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t i = b0 + wb + nt * 8 + 2 * tig + e;
                if (i < nb) D[q * nb + i] = (float)(xn + bn[i] - 2 * acc[nt][2 * h + e]);
            }
    }
}

__global__ void chunk_pos_kernel(uint32_t* __restrict__ pos, uint32_t* __restrict__ ids,
                                 uint32_t* __restrict__ cnt, size_t nq, uint32_t nb, uint64_t base) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nq * nb) pos[i] = (uint32_t)(i % nb);
    if (i < nb) ids[i] = (uint32_t)(base + i);
    if (i < nq) cnt[i] = nb;
}

__global__ void best_out_kernel(const unsigned long long* __restrict__ best, size_t nq,
                                uint32_t* __restrict__ ids, float* __restrict__ d, uint32_t* __restrict__ cnt) {
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const unsigned long long m = best[q];
    ids[q] = (uint32_t)m;
    d[q] = __uint_as_float((uint32_t)(m >> 32));
    cnt[q] = m != ~0ull ? 1u : 0u;
}

__global__ void put_part_kernel(const uint32_t* __restrict__ ids, const float* __restrict__ d,
                                const uint32_t* __restrict__ c, size_t nq, uint32_t k,
                                uint32_t* __restrict__ pi, float* __restrict__ pd, uint32_t* __restrict__ pc) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nq * k) {
        pi[i] = ids[i];
        pd[i] = d[i];
    }
    if (i < nq) pc[i] = c[i];
}

}  // namespace

bool exact_knn_supported(uint32_t d) { return d == ED; }

// Queries resident on the device (nq x 128 u8); the base arrives in chunks
// through `fetch(row0, n, dst)` (host copy or device generator).  Result:
// per query the min(k, n) nearest (dist, id), ascending.
void exact_knn_u8(const uint8_t* d_queries, size_t nq, size_t n, uint64_t id_base, uint32_t k,
                  const std::function<void(uint64_t, uint32_t, uint8_t*)>& fetch, uint32_t* out_ids,
                  float* out_dists, uint32_t* out_cnt, cudaStream_t s) {
    // chunk: distances + positions of nq x chunk within ~2 GiB
    const size_t chunk = std::max<size_t>(8192, std::min<size_t>(std::min<size_t>(n, 1u << 22),
                                                                 ((size_t)1 << 28) / std::max<size_t>(nq, 1)));
    std::vector<void*> bufs;
    auto alloc = [&](size_t bytes) {
        void* p = nullptr;
        PQRR_CUDA(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), s));
        bufs.push_back(p);
        return p;
    };
    int* qn = (int*)alloc(nq * 4);
    u8_norms_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, s>>>(d_queries, nq, qn);
    PQRR_LAUNCH_CHECK();
    if (k == 1) {  // nearest neighbour only (recall@R ground truth): fused argmin
        const size_t ch1 = std::min<size_t>(n, 1u << 22);
        uint8_t* yb1 = (uint8_t*)alloc(ch1 * ED);
        int* bn1 = (int*)alloc(ch1 * 4);
        unsigned long long* best = (unsigned long long*)alloc(nq * 8);
        PQRR_CUDA(cudaMemsetAsync(best, 0xff, nq * 8, s));
        int launches = 2;
        for (uint64_t r0 = 0; r0 < n; r0 += ch1) {
            const uint32_t nb = (uint32_t)std::min<uint64_t>(ch1, n - r0);
            fetch(r0, nb, yb1);
            u8_norms_kernel<<<(nb + 255) / 256, 256, 0, s>>>(yb1, nb, bn1);
            const dim3 grid((nb + EB - 1) / EB, (unsigned)((nq + EQ - 1) / EQ));
            exact_dist_kernel<<<grid, 256, 0, s>>>(d_queries, qn, nq, yb1, bn1, nb, nullptr, best, id_base + r0);
            PQRR_LAUNCH_CHECK();
            launches += 2;
        }
        uint32_t* oi = (uint32_t*)alloc(nq * 4);
        float* od = (float*)alloc(nq * 4);
        uint32_t* oc = (uint32_t*)alloc(nq * 4);
        best_out_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, s>>>(best, nq, oi, od, oc);
        PQRR_LAUNCH_CHECK();
        count_launch(launches);
        PQRR_CUDA(cudaMemcpyAsync(out_ids, oi, nq * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaMemcpyAsync(out_dists, od, nq * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaMemcpyAsync(out_cnt, oc, nq * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaStreamSynchronize(s));
        for (void* p : bufs) cudaFreeAsync(p, s);
        return;
    }
    uint8_t* yb = (uint8_t*)alloc(chunk * ED);
    int* bn = (int*)alloc(chunk * 4);
    float* D = (float*)alloc(nq * chunk * 4);
    uint32_t* pos = (uint32_t*)alloc(nq * chunk * 4);
    uint32_t* cids = (uint32_t*)alloc(chunk * 4);
    uint32_t* ccnt = (uint32_t*)alloc(nq * 4);
    uint64_t* skey = (uint64_t*)alloc(nq * (size_t)k * 8);
    uint32_t* spos = (uint32_t*)alloc(nq * (size_t)k * 4);
    uint32_t* scnt = (uint32_t*)alloc(nq * 4);
    // running result = part 0, this chunk's top-k = part 1 of the K7 merge input
    uint32_t* mi = (uint32_t*)alloc(2 * nq * (size_t)k * 4);
    float* md = (float*)alloc(2 * nq * (size_t)k * 4);
    uint32_t* mc = (uint32_t*)alloc(2 * nq * 4);
    PQRR_CUDA(cudaMemsetAsync(mc, 0, 2 * nq * 4, s));
    uint32_t* ti = (uint32_t*)alloc(nq * (size_t)k * 4);
    float* td = (float*)alloc(nq * (size_t)k * 4);
    const size_t nqk = nq * (size_t)k;
    int launches = 1;
    for (uint64_t r0 = 0; r0 < n; r0 += chunk) {
        const uint32_t nb = (uint32_t)std::min<uint64_t>(chunk, n - r0);
        fetch(r0, nb, yb);
        u8_norms_kernel<<<(nb + 255) / 256, 256, 0, s>>>(yb, nb, bn);
        const dim3 grid((nb + EB - 1) / EB, (unsigned)((nq + EQ - 1) / EQ));
        exact_dist_kernel<<<grid, 256, 0, s>>>(d_queries, qn, nq, yb, bn, nb, D, nullptr, 0);
        chunk_pos_kernel<<<(unsigned)((nq * nb + 255) / 256), 256, 0, s>>>(pos, cids, ccnt, nq, nb,
                                                                           id_base + r0);
        PQRR_LAUNCH_CHECK();
        launches += 3;
        launch_select_topk(D, pos, ccnt, nb, nb, nq, cids, k, true, skey, spos, scnt, s);
        launch_unpack_keys(skey, scnt, nq, k, ti, td, s);
        put_part_kernel<<<(unsigned)((nqk + 255) / 256), 256, 0, s>>>(ti, td, scnt, nq, k, mi + nqk, md + nqk,
                                                                      mc + nq);
        PQRR_LAUNCH_CHECK();
        launch_merge_topk(mi, md, mc, nq, 2, k, k, ti, td, scnt, s);
        put_part_kernel<<<(unsigned)((nqk + 255) / 256), 256, 0, s>>>(ti, td, scnt, nq, k, mi, md, mc);
        PQRR_LAUNCH_CHECK();
        launches += 2;
    }
    count_launch(launches);
    PQRR_CUDA(cudaMemcpyAsync(out_ids, mi, nqk * 4, cudaMemcpyDeviceToHost, s));
    PQRR_CUDA(cudaMemcpyAsync(out_dists, md, nqk * 4, cudaMemcpyDeviceToHost, s));
    PQRR_CUDA(cudaMemcpyAsync(out_cnt, mc, nq * 4, cudaMemcpyDeviceToHost, s));
    PQRR_CUDA(cudaStreamSynchronize(s));
    for (void* p : bufs) cudaFreeAsync(p, s);
}

}  // namespace pqrr_b200
