// train.cu — device k-means and the PQ / IVF trainers (kmeans.hpp:21-38,
// product_quantizer.hpp:37-40, ivf_index.hpp:48-52, :66-70).  Training is
// offline but the bench must build codebooks for 10M-1B
// vector indexes, so the O(n k d) assignment runs on the exact argmin tile
// kernel while the policy decisions stay on the host, identical to the serial
// reference policy:
//  * init: partial Fisher-Yates with bounded_u32 on mt19937(uint32(seed + r))
//    (rng.hpp:15-21) picks k distinct rows;
//  * objective: fp64 sum of f32 distances in id order (host);
//  * update: id-order fp64 sums per (cluster, component) on the device
//    (k_kmeans.cu), same addition sequence as the serial loop;
//  * empty cluster c (ascending), unless the objective is exactly zero: copy
//    the most populated cluster b (lowest index on ties), jitter each component
//    by (uniform01 - 0.5) * 2^-9 * (|x| + 1) in f32 (uniform01: rng.hpp:24-26),
//    move half of b's count to c;
//  * final_mse from a final assignment; best of `redo` restarts (strict <).
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "../../include/pqrr_dev.h"
#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {

extern thread_local std::string g_last_error;

namespace {

inline uint32_t bounded_u32(std::mt19937& g, uint32_t bound) {
    const uint32_t threshold = (-bound) % bound;
    for (;;) {
        uint32_t x = g();
        if (x >= threshold) return x % bound;
    }
}
inline float uniform01(std::mt19937& g) { return float(g() >> 8) * (1.0f / 16777216.0f); }

struct Scratch {
    cudaStream_t s;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t st) : s(st) {}
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
    }
    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        PQRR_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
};

int bits_of(uint32_t n) {
    int b = 1;
    while ((1ull << b) < n) ++b;
    return b;
}

__global__ void extract_cols(const float* __restrict__ x, size_t n, uint32_t d, uint32_t c0,
                             uint32_t w, float* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * w) return;
    out[i] = x[(i / w) * d + c0 + i % w];
}

__global__ void coarse_residual_kernel(const float* __restrict__ y, size_t n, uint32_t d,
                                       const uint32_t* __restrict__ assign,
                                       const float* __restrict__ coarse, float* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * d) return;
    out[i] = __fsub_rn(y[i], coarse[(size_t)assign[i / d] * d + i % d]);
}

// r1 = y - (C_a + p), p = decode(code) (ivf_index.hpp:66-67).
__global__ void refine_residual_kernel(const float* __restrict__ y, size_t n, uint32_t d,
                                       const uint32_t* __restrict__ assign,
                                       const float* __restrict__ coarse, const uint8_t* __restrict__ codes,
                                       const float* __restrict__ books, uint32_t m, uint32_t ks,
                                       float* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * d) return;
    const size_t v = i / d;
    const uint32_t t = (uint32_t)(i % d), ds = d / m, jj = t / ds;
    const float rec1 = __fadd_rn(coarse[(size_t)assign[v] * d + t],
                                 books[((size_t)jj * ks + codes[v * m + jj]) * ds + (t - jj * ds)]);
    out[i] = __fsub_rn(y[i], rec1);
}

inline unsigned nb(size_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

void kmeans_device(const float* d_points, size_t n, uint32_t dim, uint32_t k, uint32_t iterations,
                   uint64_t seed, uint32_t redo, float* h_centroids, double* out_mse,
                   double* out_trace, cudaStream_t s) {
    if (k == 0) throw ArgError("k must be positive");
    if (n < k || n == 0) throw ArgError("insufficient training data");
    Scratch ws(s);
    float* C = ws.alloc<float>((size_t)k * dim);
    uint32_t* assign = ws.alloc<uint32_t>(n);
    float* dist = ws.alloc<float>(n);
    uint32_t* cnt = ws.alloc<uint32_t>(k + 1);
    uint32_t* off = ws.alloc<uint32_t>(k + 1);
    uint32_t* iota = ws.alloc<uint32_t>(n);
    uint32_t* skeys = ws.alloc<uint32_t>(n);
    uint32_t* sids = ws.alloc<uint32_t>(n);
    uint32_t* rows = ws.alloc<uint32_t>(k);
    launch_iota(iota, n, s);
    std::vector<float> h_dist(n), hC((size_t)k * dim), best;
    std::vector<uint32_t> h_cnt(k);
    std::vector<double> trace, best_trace;
    double best_mse = 0.0;
    bool have = false;
    for (uint32_t r = 0; r < std::max<uint32_t>(redo, 1); ++r) {
        std::mt19937 g(uint32_t(seed + r));
        std::vector<uint32_t> perm(n);
        for (size_t i = 0; i < n; ++i) perm[i] = uint32_t(i);
        for (uint32_t i = 0; i < k; ++i) {
            uint32_t j = i + bounded_u32(g, uint32_t(n - i));
            std::swap(perm[i], perm[j]);
        }
        PQRR_CUDA(cudaMemcpyAsync(rows, perm.data(), k * 4, cudaMemcpyHostToDevice, s));
        launch_gather_rows(d_points, dim, rows, k, C, s);
        trace.clear();
        for (uint32_t it = 0; it < iterations; ++it) {
            launch_argmin(d_points, n, C, k, dim, assign, dist, s);
            PQRR_CUDA(cudaMemcpyAsync(h_dist.data(), dist, n * 4, cudaMemcpyDeviceToHost, s));
            PQRR_CUDA(cudaMemsetAsync(cnt, 0, (k + 1) * 4, s));
            launch_histogram(assign, n, k, cnt, s);
            exclusive_scan_u32(cnt, off, k + 1, s);
            sort_pairs(assign, skeys, iota, sids, n, bits_of(k), s);
            launch_centroid_update(d_points, dim, sids, off, k, C, s);
            PQRR_CUDA(cudaMemcpyAsync(h_cnt.data(), cnt, k * 4, cudaMemcpyDeviceToHost, s));
            PQRR_CUDA(cudaStreamSynchronize(s));
            double obj = 0.0;
            for (size_t i = 0; i < n; ++i) obj += double(h_dist[i]);
            trace.push_back(obj);
            bool empty = false;
            for (uint32_t c = 0; c < k; ++c) empty |= h_cnt[c] == 0;
            if (empty && obj != 0.0) {
                std::vector<size_t> counts(h_cnt.begin(), h_cnt.end());
                PQRR_CUDA(cudaMemcpyAsync(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost, s));
                PQRR_CUDA(cudaStreamSynchronize(s));
                for (uint32_t c = 0; c < k; ++c) {
                    if (counts[c] != 0) continue;
                    uint32_t b = 0;
                    for (uint32_t q = 1; q < k; ++q)
                        if (counts[q] > counts[b]) b = q;
                    for (uint32_t t = 0; t < dim; ++t) {
                        float x = hC[size_t(b) * dim + t];
                        float jit = (uniform01(g) - 0.5f) * (1.0f / 512.0f) * (std::fabs(x) + 1.0f);
                        hC[size_t(c) * dim + t] = x + jit;
                    }
                    counts[c] = counts[b] / 2;
                    counts[b] -= counts[c];
                }
                PQRR_CUDA(cudaMemcpyAsync(C, hC.data(), hC.size() * 4, cudaMemcpyHostToDevice, s));
            }
        }
        launch_argmin(d_points, n, C, k, dim, assign, dist, s);
        PQRR_CUDA(cudaMemcpyAsync(h_dist.data(), dist, n * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaMemcpyAsync(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaStreamSynchronize(s));
        double obj = 0.0;
        for (size_t i = 0; i < n; ++i) obj += double(h_dist[i]);
        const double mse = obj / double(n);
        if (!have || mse < best_mse) {
            best = hC;
            best_mse = mse;
            best_trace = trace;
            have = true;
        }
    }
    std::memcpy(h_centroids, best.data(), best.size() * 4);
    if (out_mse) *out_mse = best_mse;
    if (out_trace)
        for (size_t i = 0; i < best_trace.size(); ++i) out_trace[i] = best_trace[i];
}

// pq_train on device-resident training rows (n x d) -> host books.
void pq_train_device(const float* d_x, size_t n, uint32_t d, uint32_t m, uint32_t ks,
                     uint32_t iterations, uint64_t seed, uint32_t redo, float* h_books,
                     cudaStream_t s) {
    if (m == 0 || d % m) throw ArgError("dimension not divisible");
    if (ks == 0 || ks > 256) throw ArgError("ks must be in [1, 256]");
    const uint32_t ds = d / m;
    Scratch ws(s);
    float* sub = ws.alloc<float>(n * ds);
    for (uint32_t j = 0; j < m; ++j) {
        extract_cols<<<nb(n * ds), 256, 0, s>>>(d_x, n, d, j * ds, ds, sub);
        PQRR_LAUNCH_CHECK();
        count_launch();
        kmeans_device(sub, n, ds, ks, iterations, seed + j, redo, h_books + (size_t)j * ks * ds,
                      nullptr, nullptr, s);
    }
}

}  // namespace pqrr_b200

using namespace pqrr_b200;

namespace {

template <class F>
int guarded_train(F&& f) {
    try {
        f();
        return PQRR_OK;
    } catch (const ArgError& e) {
        g_last_error = e.what();
        return PQRR_EINVAL;
    } catch (const CudaError& e) {
        g_last_error = e.what();
        return PQRR_ECUDA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return PQRR_EINTERNAL;
    }
}

struct TrainSession {
    int prev = 0;
    cudaStream_t s = nullptr;
    explicit TrainSession(int dev) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            throw std::runtime_error("no CUDA device available (the B200 path has no CPU fallback)");
        }
        if (dev < 0 || dev >= n) throw ArgError("device ordinal out of range");
        PQRR_CUDA(cudaGetDevice(&prev));
        PQRR_CUDA(cudaSetDevice(dev));
        PQRR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    ~TrainSession() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
        cudaSetDevice(prev);
    }
};

void check_finite(const float* x, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(x[i])) throw ArgError("VectorSet: non-finite value");
}

}  // namespace

extern "C" {

int pqrr_dev_pq_train(int device, const float* training, size_t n, uint32_t d, uint32_t m,
                      uint32_t ks, uint32_t iterations, uint64_t seed, uint32_t redo,
                      float* out_books) {
    return guarded_train([&] {
        if (m == 0 || d % m) throw ArgError("dimension not divisible");
        if (n < ks) throw ArgError("insufficient training data");
        check_finite(training, n * d);
        TrainSession se(device);
        Scratch ws(se.s);
        float* x = ws.alloc<float>(n * d);
        PQRR_CUDA(cudaMemcpyAsync(x, training, n * d * 4, cudaMemcpyHostToDevice, se.s));
        pq_train_device(x, n, d, m, ks, iterations, seed, redo, out_books, se.s);
    });
}

int pqrr_dev_ivf_train(int device, const float* training, size_t n, uint32_t d, uint32_t c,
                       uint32_t m, uint32_t ks, uint32_t iterations, uint64_t seed,
                       float* out_coarse, float* out_books) {
    return guarded_train([&] {
        if (m == 0 || d % m) throw ArgError("dimension not divisible");
        if (n < c || n < ks) throw ArgError("insufficient training data");
        check_finite(training, n * d);
        TrainSession se(device);
        Scratch ws(se.s);
        float* x = ws.alloc<float>(n * d);
        PQRR_CUDA(cudaMemcpyAsync(x, training, n * d * 4, cudaMemcpyHostToDevice, se.s));
        kmeans_device(x, n, d, c, iterations, seed, 1, out_coarse, nullptr, nullptr, se.s);
        float* C = ws.alloc<float>((size_t)c * d);
        PQRR_CUDA(cudaMemcpyAsync(C, out_coarse, (size_t)c * d * 4, cudaMemcpyHostToDevice, se.s));
        uint32_t* a = ws.alloc<uint32_t>(n);
        launch_argmin(x, n, C, c, d, a, nullptr, se.s);
        float* r = ws.alloc<float>(n * d);
        coarse_residual_kernel<<<nb(n * d), 256, 0, se.s>>>(x, n, d, a, C, r);
        PQRR_LAUNCH_CHECK();
        count_launch();
        pq_train_device(r, n, d, m, ks, iterations, seed, 1, out_books, se.s);
    });
}

int pqrr_dev_ivf_refine_train(int device, const float* coarse, uint32_t c, const float* books,
                              uint32_t d, uint32_t m, uint32_t ks, const float* training,
                              size_t n, uint32_t mprime, uint32_t iterations, uint64_t seed,
                              float* out_rbooks) {
    return guarded_train([&] {
        if (m == 0 || d % m || mprime == 0 || d % mprime) throw ArgError("dimension not divisible");
        if (n < ks) throw ArgError("insufficient training data");
        check_finite(training, n * d);
        TrainSession se(device);
        Scratch ws(se.s);
        float* x = ws.alloc<float>(n * d);
        PQRR_CUDA(cudaMemcpyAsync(x, training, n * d * 4, cudaMemcpyHostToDevice, se.s));
        float* C = ws.alloc<float>((size_t)c * d);
        PQRR_CUDA(cudaMemcpyAsync(C, coarse, (size_t)c * d * 4, cudaMemcpyHostToDevice, se.s));
        float* B = ws.alloc<float>((size_t)ks * d);
        PQRR_CUDA(cudaMemcpyAsync(B, books, (size_t)ks * d * 4, cudaMemcpyHostToDevice, se.s));
        uint32_t* a = ws.alloc<uint32_t>(n);
        launch_argmin(x, n, C, c, d, a, nullptr, se.s);
        float* r0 = ws.alloc<float>(n * d);
        coarse_residual_kernel<<<nb(n * d), 256, 0, se.s>>>(x, n, d, a, C, r0);
        PQRR_LAUNCH_CHECK();
        count_launch();
        uint8_t* codes = ws.alloc<uint8_t>(n * m);
        launch_pq_encode(r0, n, d, B, m, ks, codes, se.s);
        float* r1 = ws.alloc<float>(n * d);
        refine_residual_kernel<<<nb(n * d), 256, 0, se.s>>>(x, n, d, a, C, codes, B, m, ks, r1);
        PQRR_LAUNCH_CHECK();
        count_launch();
        pq_train_device(r1, n, d, mprime, ks, iterations, seed, 1, out_rbooks, se.s);
    });
}

}  // extern "C"
