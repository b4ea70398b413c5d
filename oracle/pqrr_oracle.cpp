// pqrr_oracle.cpp — CPU oracle for the IVFADC+R search path (arXiv 1102.3828).
//
// TEST INFRASTRUCTURE ONLY (see pqrr_oracle.h).  This file is a plain C++20
// restatement of the arithmetic contract in the reference headers under
// /root/reference/proj/include/pqrr/, plus definitions of the bodies the
// reference only declares.  The parity contract it fixes is
// SURVEY.md §8a items 1-10; each function cites the reference line it follows.
// Build flags mirror the reference (CMakeLists.txt:11-13): -O3, no -ffast-math,
// no -march=native, plus -ffp-contract=off so no multiply-add is ever fused.
#include "pqrr_oracle.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(const std::string& msg) {
    g_err = msg;
    return -1;
}

// ---------------------------------------------------------------- L0
// distance.hpp:16-33 — four partial sums over lanes j mod 4, remainder into
// s0..s2, reduced as (s0 + s1) + (s2 + s3).  Separate mul and add roundings.
inline float l2_sq(const float* a, const float* b, std::size_t d) {
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
    std::size_t j = 0;
    for (; j + 4 <= d; j += 4) {
        float t0 = a[j] - b[j];
        float t1 = a[j + 1] - b[j + 1];
        float t2 = a[j + 2] - b[j + 2];
        float t3 = a[j + 3] - b[j + 3];
        s0 += t0 * t0;
        s1 += t1 * t1;
        s2 += t2 * t2;
        s3 += t3 * t3;
    }
    if (j < d) { float t = a[j] - b[j]; s0 += t * t; ++j; }
    if (j < d) { float t = a[j] - b[j]; s1 += t * t; ++j; }
    if (j < d) { float t = a[j] - b[j]; s2 += t * t; ++j; }
    return (s0 + s1) + (s2 + s3);
}

// distance.hpp:36-53 — fp64 twin used by the exact-search oracle.
inline double l2_sq_d(const float* a, const float* b, std::size_t d) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    std::size_t j = 0;
    for (; j + 4 <= d; j += 4) {
        double t0 = double(a[j]) - double(b[j]);
        double t1 = double(a[j + 1]) - double(b[j + 1]);
        double t2 = double(a[j + 2]) - double(b[j + 2]);
        double t3 = double(a[j + 3]) - double(b[j + 3]);
        s0 += t0 * t0;
        s1 += t1 * t1;
        s2 += t2 * t2;
        s3 += t3 * t3;
    }
    if (j < d) { double t = double(a[j]) - double(b[j]); s0 += t * t; ++j; }
    if (j < d) { double t = double(a[j]) - double(b[j]); s1 += t * t; ++j; }
    if (j < d) { double t = double(a[j]) - double(b[j]); s2 += t * t; ++j; }
    return (s0 + s1) + (s2 + s3);
}

// types.hpp:40-50 — (dist asc, id asc) total order.
struct Nb {
    uint32_t id;
    float dist;
};
inline bool nb_less(const Nb& a, const Nb& b) {
    if (a.dist != b.dist) return a.dist < b.dist;
    return a.id < b.id;
}

// topk.hpp:14-52 — bounded max-heap under nb_less.
class TopK {
  public:
    explicit TopK(std::size_t k) : cap_(k) { heap_.reserve(k); }
    void push(uint32_t id, float dist) {
        Nb c{id, dist};
        if (heap_.size() < cap_) {
            heap_.push_back(c);
            std::push_heap(heap_.begin(), heap_.end(), nb_less);
            return;
        }
        if (cap_ == 0 || !nb_less(c, heap_.front())) return;
        std::pop_heap(heap_.begin(), heap_.end(), nb_less);
        heap_.back() = c;
        std::push_heap(heap_.begin(), heap_.end(), nb_less);
    }
    std::vector<Nb> take_sorted() {
        std::sort_heap(heap_.begin(), heap_.end(), nb_less);
        return std::move(heap_);
    }

  private:
    std::size_t cap_;
    std::vector<Nb> heap_;
};

// ---------------------------------------------------------------- L1
struct PQ {
    uint32_t d, m, ks;
    const float* books;  // m * ks * dsub
    uint32_t dsub() const { return d / m; }
    const float* centroid(uint32_t j, uint32_t i) const {
        return books + (std::size_t(j) * ks + i) * dsub();
    }
};

// product_quantizer.hpp:42 (pq_encode_into; body missing in the reference).
// Per sub-space argmin of l2_sq over the ks centroids, strict < so the lowest
// index wins ties (kernels.cpp:29-35 argmin pattern).
void pq_encode_into(const PQ& pq, const float* y, uint8_t* code) {
    const uint32_t ds = pq.dsub();
    for (uint32_t j = 0; j < pq.m; ++j) {
        const float* yj = y + std::size_t(j) * ds;
        uint32_t best = 0;
        float bd = l2_sq(yj, pq.centroid(j, 0), ds);
        for (uint32_t i = 1; i < pq.ks; ++i) {
            float dd = l2_sq(yj, pq.centroid(j, i), ds);
            if (dd < bd) {
                bd = dd;
                best = i;
            }
        }
        code[j] = uint8_t(best);
    }
}

// product_quantizer.hpp:45 (pq_decode_into) — concatenation of centroids.
void pq_decode_into(const PQ& pq, const uint8_t* code, float* out) {
    const uint32_t ds = pq.dsub();
    for (uint32_t j = 0; j < pq.m; ++j)
        std::memcpy(out + std::size_t(j) * ds, pq.centroid(j, code[j]), ds * sizeof(float));
}

// product_quantizer.hpp:48-49 (build_lut) — entry (j,i) = l2_sq(x^j, B_j[i]).
void build_lut(const PQ& pq, const float* x, float* lut) {
    const uint32_t ds = pq.dsub();
    for (uint32_t j = 0; j < pq.m; ++j)
        for (uint32_t i = 0; i < pq.ks; ++i)
            lut[std::size_t(j) * pq.ks + i] = l2_sq(x + std::size_t(j) * ds, pq.centroid(j, i), ds);
}

// product_quantizer.hpp:53-57 — j-ascending float sum.
inline float adc_distance(const float* lut, uint32_t m, uint32_t ks, const uint8_t* code) {
    float acc = 0.0f;
    for (uint32_t j = 0; j < m; ++j) acc += lut[std::size_t(j) * ks + code[j]];
    return acc;
}

// kernels.cpp:21-39 — per-point argmin, strict <, lowest index on ties.
void assign_batch(const float* points, std::size_t n, uint32_t dim, const float* centroids,
                  uint32_t k, uint32_t* out_assign, float* out_dist) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i) {
        const float* p = points + std::size_t(i) * dim;
        uint32_t best = 0;
        float bd = l2_sq(p, centroids, dim);
        for (uint32_t c = 1; c < k; ++c) {
            float dd = l2_sq(p, centroids + std::size_t(c) * dim, dim);
            if (dd < bd) {
                bd = dd;
                best = c;
            }
        }
        out_assign[i] = best;
        if (out_dist) out_dist[i] = bd;
    }
}

// ---------------------------------------------------------------- RNG (rng.hpp)
// rng.hpp:15-21
inline uint32_t bounded_u32(std::mt19937& g, uint32_t bound) {
    const uint32_t threshold = (-bound) % bound;
    for (;;) {
        uint32_t x = g();
        if (x >= threshold) return x % bound;
    }
}
// rng.hpp:24-26
inline float uniform01(std::mt19937& g) { return float(g() >> 8) * (1.0f / 16777216.0f); }

// ---------------------------------------------------------------- k-means
// kmeans.hpp:30-38 + SPEC.md:121-127.  Policies (the oracle's decisions, also
// implemented identically by the product trainer):
//  * init: partial Fisher-Yates with bounded_u32 on mt19937(uint32(seed+r))
//    picks k distinct training rows;
//  * each iteration: pure assignment (assign_batch), objective = fp64 sum of
//    the f32 distances in id order, centroid = fp64 id-order sum / count,
//    rounded to f32;
//  * empty cluster c (ascending), unless the objective is exactly zero: split
//    the most populated cluster b (lowest index on ties): copy its centroid,
//    jitter each component by (uniform01 - 0.5) * 2^-9 * (|x| + 1) in f32, and
//    hand half of b's count to c;
//  * final_mse = fp64 id-order objective of a final assignment / n;
//  * restarts r = 0..redo-1, best final_mse (strict <) wins.
struct KmeansOut {
    std::vector<float> centroids;
    double final_mse = 0.0;
    std::vector<double> trace;
};

KmeansOut kmeans_train(const float* pts, std::size_t n, uint32_t dim, uint32_t k,
                       uint32_t iterations, uint64_t seed, uint32_t redo) {
    if (k == 0) throw std::invalid_argument("k must be positive");
    if (n < k || n == 0) throw std::invalid_argument("insufficient training data");
    for (std::size_t i = 0; i < n * dim; ++i)
        if (!std::isfinite(pts[i])) throw std::invalid_argument("VectorSet: non-finite value");
    KmeansOut best;
    bool have = false;
    std::vector<uint32_t> assign(n);
    std::vector<float> dist(n);
    for (uint32_t r = 0; r < std::max<uint32_t>(redo, 1); ++r) {
        std::mt19937 g(uint32_t(seed + r));
        std::vector<uint32_t> perm(n);
        for (std::size_t i = 0; i < n; ++i) perm[i] = uint32_t(i);
        for (uint32_t i = 0; i < k; ++i) {
            uint32_t j = i + bounded_u32(g, uint32_t(n - i));
            std::swap(perm[i], perm[j]);
        }
        std::vector<float> C(std::size_t(k) * dim);
        for (uint32_t c = 0; c < k; ++c)
            std::memcpy(&C[std::size_t(c) * dim], pts + std::size_t(perm[c]) * dim,
                        dim * sizeof(float));
        std::vector<double> trace;
        std::vector<double> sums(std::size_t(k) * dim);
        std::vector<std::size_t> counts(k);
        for (uint32_t it = 0; it < iterations; ++it) {
            assign_batch(pts, n, dim, C.data(), k, assign.data(), dist.data());
            double obj = 0.0;
            for (std::size_t i = 0; i < n; ++i) obj += double(dist[i]);
            trace.push_back(obj);
            std::fill(sums.begin(), sums.end(), 0.0);
            std::fill(counts.begin(), counts.end(), 0);
            for (std::size_t i = 0; i < n; ++i) {
                const uint32_t a = assign[i];
                ++counts[a];
                double* s = &sums[std::size_t(a) * dim];
                const float* p = pts + i * dim;
                for (uint32_t t = 0; t < dim; ++t) s[t] += double(p[t]);
            }
            for (uint32_t c = 0; c < k; ++c) {
                if (counts[c] == 0) continue;
                for (uint32_t t = 0; t < dim; ++t)
                    C[std::size_t(c) * dim + t] =
                        float(sums[std::size_t(c) * dim + t] / double(counts[c]));
            }
            if (obj != 0.0) {
                for (uint32_t c = 0; c < k; ++c) {
                    if (counts[c] != 0) continue;
                    uint32_t b = 0;
                    for (uint32_t q = 1; q < k; ++q)
                        if (counts[q] > counts[b]) b = q;
                    for (uint32_t t = 0; t < dim; ++t) {
                        float x = C[std::size_t(b) * dim + t];
                        float jit = (uniform01(g) - 0.5f) * (1.0f / 512.0f) * (std::fabs(x) + 1.0f);
                        C[std::size_t(c) * dim + t] = x + jit;
                    }
                    counts[c] = counts[b] / 2;
                    counts[b] -= counts[c];
                }
            }
        }
        assign_batch(pts, n, dim, C.data(), k, assign.data(), dist.data());
        double obj = 0.0;
        for (std::size_t i = 0; i < n; ++i) obj += double(dist[i]);
        double mse = obj / double(n);
        if (!have || mse < best.final_mse) {
            best.centroids = std::move(C);
            best.final_mse = mse;
            best.trace = std::move(trace);
            have = true;
        }
    }
    return best;
}

// product_quantizer.hpp:37-40 — sub-book j trained on slice j, seed + j.
std::vector<float> pq_train(const float* tr, std::size_t n, uint32_t d, uint32_t m, uint32_t ks,
                            uint32_t iterations, uint64_t seed, uint32_t redo) {
    if (m == 0 || d % m != 0) throw std::invalid_argument("dimension not divisible");
    if (ks == 0 || ks > 256) throw std::invalid_argument("ks must be in [1, 256]");
    const uint32_t ds = d / m;
    std::vector<float> books(std::size_t(m) * ks * ds);
    std::vector<float> sub(n * ds);
    for (uint32_t j = 0; j < m; ++j) {
        for (std::size_t i = 0; i < n; ++i)
            std::memcpy(&sub[i * ds], tr + i * d + std::size_t(j) * ds, ds * sizeof(float));
        KmeansOut o = kmeans_train(sub.data(), n, ds, ks, iterations, seed + j, redo);
        std::memcpy(&books[std::size_t(j) * ks * ds], o.centroids.data(),
                    std::size_t(ks) * ds * sizeof(float));
    }
    return books;
}

}  // namespace

// ================================================================= IVF index
// ivf_index.hpp:15-41: per-list (ids ascending, codes), id -> (list, pos).
struct orc_ivf {
    uint32_t d = 0, c = 0, m = 0, ks = 0;
    std::vector<float> coarse;  // c * d
    std::vector<float> books;   // m * ks * d/m
    std::vector<std::vector<uint32_t>> ids;
    std::vector<std::vector<uint8_t>> codes;
    std::size_t n = 0;
    std::vector<uint32_t> list_of_id, pos_of_id;
    // refinement (refine.hpp:13-28), id-aligned
    uint32_t mprime = 0;
    std::vector<float> rbooks;
    std::vector<uint8_t> rcodes;

    PQ pq() const { return PQ{d, m, ks, books.data()}; }
    PQ rq() const { return PQ{d, mprime, ks, rbooks.data()}; }
    const uint8_t* code_of_id(uint32_t id) const {
        return codes[list_of_id[id]].data() + std::size_t(pos_of_id[id]) * m;
    }
    // ivf_index.hpp:75-77 three-term estimate; refine residual convention of
    // ivf_index.hpp:66-67 / SPEC.md:344: rec1 = C_a + decode(code) first, then
    // yhat = rec1 + decode_r(rcode).
    void reconstruct(uint32_t id, float* out) const {
        const uint32_t a = list_of_id[id];
        std::vector<float> p(d), r(d);
        pq_decode_into(pq(), code_of_id(id), p.data());
        const float* C = coarse.data() + std::size_t(a) * d;
        for (uint32_t t = 0; t < d; ++t) out[t] = C[t] + p[t];
        if (mprime) {
            pq_decode_into(rq(), rcodes.data() + std::size_t(id) * mprime, r.data());
            for (uint32_t t = 0; t < d; ++t) out[t] = out[t] + r[t];
        }
    }
};

namespace {

// Coarse probe selection inside ivf_search (ivf_index.hpp:58-61, SPEC.md:321;
// ties to the lowest list index): the v smallest (l2_sq, k).
void coarse_probe(const float* C, uint32_t c, uint32_t d, const float* x, uint32_t v,
                  uint32_t* lists, float* dists) {
    std::vector<Nb> all(c);
    for (uint32_t k = 0; k < c; ++k) all[k] = Nb{k, l2_sq(x, C + std::size_t(k) * d, d)};
    std::partial_sort(all.begin(), all.begin() + v, all.end(), nb_less);
    for (uint32_t i = 0; i < v; ++i) {
        lists[i] = all[i].id;
        if (dists) dists[i] = all[i].dist;
    }
}

// ivf_search (ivf_index.hpp:58-61): probe v lists; per list a LUT on the
// residual query x - C_l; min(kprime, #candidates) smallest.
std::vector<Nb> ivf_search(const orc_ivf& ix, const float* x, uint32_t v, std::size_t kprime) {
    std::vector<uint32_t> probes(v);
    coarse_probe(ix.coarse.data(), ix.c, ix.d, x, v, probes.data(), nullptr);
    std::vector<float> xr(ix.d), lut(std::size_t(ix.m) * ix.ks);
    TopK heap(kprime);
    const PQ pq = ix.pq();
    for (uint32_t l : probes) {
        const float* C = ix.coarse.data() + std::size_t(l) * ix.d;
        for (uint32_t t = 0; t < ix.d; ++t) xr[t] = x[t] - C[t];
        build_lut(pq, xr.data(), lut.data());
        const auto& ids = ix.ids[l];
        const uint8_t* codes = ix.codes[l].data();
        for (std::size_t i = 0; i < ids.size(); ++i)
            heap.push(ids[i], adc_distance(lut.data(), ix.m, ix.ks, codes + i * ix.m));
    }
    return heap.take_sorted();
}

}  // namespace

// ================================================================= C ABI
extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_set_threads(int t) {
    omp_set_num_threads(t <= 0 ? omp_get_num_procs() : t);
    return omp_get_max_threads();
}

float orc_l2_sq(const float* a, const float* b, size_t d) { return l2_sq(a, b, d); }
double orc_l2_sq_d(const float* a, const float* b, size_t d) { return l2_sq_d(a, b, d); }

size_t orc_topk(const uint32_t* ids, const float* dists, size_t n, size_t k, uint32_t* out_ids,
                float* out_dists) {
    TopK h(k);
    for (size_t i = 0; i < n; ++i) h.push(ids[i], dists[i]);
    auto r = h.take_sorted();
    for (size_t i = 0; i < r.size(); ++i) {
        out_ids[i] = r[i].id;
        out_dists[i] = r[i].dist;
    }
    return r.size();
}

int orc_assign_batch(const float* points, size_t n, uint32_t dim, const float* centroids,
                     uint32_t k, uint32_t* out_assign, float* out_dist) {
    if (k == 0) return fail("k must be positive");
    assign_batch(points, n, dim, centroids, k, out_assign, out_dist);
    return 0;
}

int orc_encode_batch(const float* books, uint32_t d, uint32_t m, uint32_t ks, const float* data,
                     size_t n, uint8_t* out_codes) {
    if (m == 0 || d % m) return fail("dimension not divisible");
    PQ pq{d, m, ks, books};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i)
        pq_encode_into(pq, data + size_t(i) * d, out_codes + size_t(i) * m);
    return 0;
}

int orc_decode_batch(const float* books, uint32_t d, uint32_t m, uint32_t ks,
                     const uint8_t* codes, size_t n, float* out_data) {
    if (m == 0 || d % m) return fail("dimension not divisible");
    PQ pq{d, m, ks, books};
    for (size_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < m; ++j)
            if (codes[i * m + j] >= ks) return fail("code index out of range");
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i)
        pq_decode_into(pq, codes + size_t(i) * m, out_data + size_t(i) * d);
    return 0;
}

int orc_build_lut(const float* books, uint32_t d, uint32_t m, uint32_t ks, const float* x,
                  float* out_lut) {
    if (m == 0 || d % m) return fail("dimension not divisible");
    build_lut(PQ{d, m, ks, books}, x, out_lut);
    return 0;
}

float orc_adc_distance(const float* lut, uint32_t m, uint32_t ks, const uint8_t* code) {
    return adc_distance(lut, m, ks, code);
}

size_t orc_scan_topk(const float* lut, uint32_t m, uint32_t ks, const uint8_t* codes, size_t n,
                     size_t kprime, uint32_t id_base, uint32_t* out_ids, float* out_dists) {
    TopK h(kprime);
    for (size_t i = 0; i < n; ++i) h.push(id_base + uint32_t(i), adc_distance(lut, m, ks, codes + i * m));
    auto r = h.take_sorted();
    for (size_t i = 0; i < r.size(); ++i) {
        out_ids[i] = r[i].id;
        out_dists[i] = r[i].dist;
    }
    return r.size();
}

int orc_kmeans_train(const float* points, size_t n, uint32_t dim, uint32_t k, uint32_t iterations,
                     uint64_t seed, uint32_t redo, float* out_centroids, double* out_final_mse,
                     double* out_trace) {
    try {
        KmeansOut o = kmeans_train(points, n, dim, k, iterations, seed, redo);
        std::memcpy(out_centroids, o.centroids.data(), o.centroids.size() * sizeof(float));
        if (out_final_mse) *out_final_mse = o.final_mse;
        if (out_trace)
            for (size_t i = 0; i < o.trace.size(); ++i) out_trace[i] = o.trace[i];
        return 0;
    } catch (const std::exception& e) {
        return fail(e.what());
    }
}

int orc_pq_train(const float* training, size_t n, uint32_t d, uint32_t m, uint32_t ks,
                 uint32_t iterations, uint64_t seed, uint32_t redo, float* out_books) {
    try {
        auto b = pq_train(training, n, d, m, ks, iterations, seed, redo);
        std::memcpy(out_books, b.data(), b.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e.what());
    }
}

// ivf_index.hpp:48-52 — coarse on raw vectors, PQ on coarse residuals.
int orc_ivf_train(const float* training, size_t n, uint32_t d, uint32_t c, uint32_t m,
                  uint32_t ks, uint32_t iterations, uint64_t seed, float* out_coarse,
                  float* out_books) {
    try {
        KmeansOut co = kmeans_train(training, n, d, c, iterations, seed, 1);
        std::vector<uint32_t> a(n);
        assign_batch(training, n, d, co.centroids.data(), c, a.data(), nullptr);
        std::vector<float> res(n * d);
        for (size_t i = 0; i < n; ++i)
            for (uint32_t t = 0; t < d; ++t)
                res[i * d + t] = training[i * d + t] - co.centroids[size_t(a[i]) * d + t];
        auto b = pq_train(res.data(), n, d, m, ks, iterations, seed, 1);
        std::memcpy(out_coarse, co.centroids.data(), co.centroids.size() * sizeof(float));
        std::memcpy(out_books, b.data(), b.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e.what());
    }
}

// ivf_index.hpp:66-70 — residuals against coarse + PQ decode of the training set.
int orc_ivf_refine_train(const float* coarse, uint32_t c, const float* books, uint32_t d,
                         uint32_t m, uint32_t ks, const float* training, size_t n,
                         uint32_t mprime, uint32_t iterations, uint64_t seed,
                         float* out_rbooks) {
    try {
        if (m == 0 || d % m) throw std::invalid_argument("dimension not divisible");
        std::vector<uint32_t> a(n);
        assign_batch(training, n, d, coarse, c, a.data(), nullptr);
        PQ pq{d, m, ks, books};
        std::vector<float> res(n * d);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < int64_t(n); ++i) {
            std::vector<float> r0(d), p(d);
            const float* y = training + size_t(i) * d;
            const float* C = coarse + size_t(a[i]) * d;
            for (uint32_t t = 0; t < d; ++t) r0[t] = y[t] - C[t];
            uint8_t code[256];
            pq_encode_into(pq, r0.data(), code);
            pq_decode_into(pq, code, p.data());
            for (uint32_t t = 0; t < d; ++t) {
                float rec1 = C[t] + p[t];
                res[size_t(i) * d + t] = y[t] - rec1;
            }
        }
        auto b = pq_train(res.data(), n, d, mprime, ks, iterations, seed, 1);
        std::memcpy(out_rbooks, b.data(), b.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e.what());
    }
}

// ivf_index.hpp:54-56 — append each base vector to its nearest list with the
// code of y - C_a; lists id-ascending (stable over id order).
orc_ivf* orc_ivf_build(const float* coarse, uint32_t c, const float* books, uint32_t d,
                       uint32_t m, uint32_t ks, const float* base, size_t n) {
    if (c == 0 || m == 0 || d % m) {
        fail("dimension not divisible");
        return nullptr;
    }
    auto* ix = new orc_ivf;
    ix->d = d;
    ix->c = c;
    ix->m = m;
    ix->ks = ks;
    ix->coarse.assign(coarse, coarse + size_t(c) * d);
    ix->books.assign(books, books + size_t(m) * ks * (d / m));
    ix->n = n;
    std::vector<uint32_t> a(n);
    assign_batch(base, n, d, coarse, c, a.data(), nullptr);
    std::vector<uint8_t> codes(n * m);
    const PQ pq = ix->pq();
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i) {
        std::vector<float> r(d);
        const float* y = base + size_t(i) * d;
        const float* C = coarse + size_t(a[i]) * d;
        for (uint32_t t = 0; t < d; ++t) r[t] = y[t] - C[t];
        pq_encode_into(pq, r.data(), codes.data() + size_t(i) * m);
    }
    ix->ids.assign(c, {});
    ix->codes.assign(c, {});
    ix->list_of_id.resize(n);
    ix->pos_of_id.resize(n);
    for (size_t i = 0; i < n; ++i) {
        const uint32_t l = a[i];
        ix->list_of_id[i] = l;
        ix->pos_of_id[i] = uint32_t(ix->ids[l].size());
        ix->ids[l].push_back(uint32_t(i));
        ix->codes[l].insert(ix->codes[l].end(), codes.begin() + i * m, codes.begin() + (i + 1) * m);
    }
    return ix;
}

void orc_ivf_free(orc_ivf* ix) { delete ix; }

size_t orc_ivf_list_size(const orc_ivf* ix, uint32_t list) { return ix->ids[list].size(); }

int orc_ivf_list_get(const orc_ivf* ix, uint32_t list, uint32_t* ids, uint8_t* codes) {
    if (list >= ix->c) return fail("list out of range");
    std::memcpy(ids, ix->ids[list].data(), ix->ids[list].size() * sizeof(uint32_t));
    std::memcpy(codes, ix->codes[list].data(), ix->codes[list].size());
    return 0;
}

int orc_ivf_assignments(const orc_ivf* ix, uint32_t* list_of_id, uint32_t* pos_of_id) {
    std::memcpy(list_of_id, ix->list_of_id.data(), ix->n * sizeof(uint32_t));
    std::memcpy(pos_of_id, ix->pos_of_id.data(), ix->n * sizeof(uint32_t));
    return 0;
}

// ivf_index.hpp:72-73 + refine.hpp:38-40: rcode_i = encode_r(y_i - (C_a + p_i)).
int orc_ivf_refine_encode(orc_ivf* ix, const float* rbooks, uint32_t mprime, const float* base,
                          size_t n, uint8_t* out_rcodes) {
    if (n != ix->n) return fail("count mismatch");
    if (mprime == 0 || ix->d % mprime) return fail("dimension not divisible");
    const uint32_t d = ix->d;
    ix->mprime = mprime;
    ix->rbooks.assign(rbooks, rbooks + size_t(mprime) * ix->ks * (d / mprime));
    ix->rcodes.assign(n * mprime, 0);
    const PQ pq = ix->pq(), rq = ix->rq();
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i) {
        std::vector<float> p(d), r1(d);
        const float* y = base + size_t(i) * d;
        const float* C = ix->coarse.data() + size_t(ix->list_of_id[i]) * d;
        pq_decode_into(pq, ix->code_of_id(uint32_t(i)), p.data());
        for (uint32_t t = 0; t < d; ++t) {
            float rec1 = C[t] + p[t];
            r1[t] = y[t] - rec1;
        }
        pq_encode_into(rq, r1.data(), ix->rcodes.data() + size_t(i) * mprime);
    }
    if (out_rcodes) std::memcpy(out_rcodes, ix->rcodes.data(), ix->rcodes.size());
    return 0;
}

int orc_ivf_search_batch(const orc_ivf* ix, const float* queries, size_t nq, uint32_t v,
                         size_t kprime, uint32_t* out_ids, float* out_dists, uint32_t* counts) {
    if (v < 1 || v > ix->c) return fail("v must satisfy 1 <= v <= c");
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < int64_t(nq); ++q) {
        auto r = ivf_search(*ix, queries + size_t(q) * ix->d, v, kprime);
        for (size_t i = 0; i < r.size(); ++i) {
            out_ids[size_t(q) * kprime + i] = r[i].id;
            out_dists[size_t(q) * kprime + i] = r[i].dist;
        }
        counts[q] = uint32_t(r.size());
    }
    return 0;
}

int orc_ivf_reconstruct(const orc_ivf* ix, uint32_t id, float* out) {
    if (id >= ix->n) return fail("id out of range");
    ix->reconstruct(id, out);
    return 0;
}

// ivf_index.hpp:79-81: distances recomputed as l2_sq(x, yhat)
// (estimator path, distance.hpp:15), k smallest under (dist,id).
int orc_ivf_rerank_batch(const orc_ivf* ix, const float* queries, size_t nq,
                         const uint32_t* sl_ids, const uint32_t* sl_counts, size_t sl_stride,
                         size_t k, uint32_t* out_ids, float* out_dists) {
    for (size_t q = 0; q < nq; ++q)
        if (k > sl_counts[q]) return fail("shortlist too small");
    const uint32_t d = ix->d;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < int64_t(nq); ++q) {
        const float* x = queries + size_t(q) * d;
        std::vector<float> yh(d);
        TopK h(k);
        for (uint32_t i = 0; i < sl_counts[q]; ++i) {
            const uint32_t id = sl_ids[size_t(q) * sl_stride + i];
            ix->reconstruct(id, yh.data());
            h.push(id, l2_sq(x, yh.data(), d));
        }
        auto r = h.take_sorted();
        for (size_t i = 0; i < r.size(); ++i) {
            out_ids[size_t(q) * k + i] = r[i].id;
            out_dists[size_t(q) * k + i] = r[i].dist;
        }
    }
    return 0;
}

// ================================================================= ADC / ADC+R
// adc_index.hpp:13-31 and refine.hpp:30-53 restated directly (no coarse
// quantizer): codes are pq_encode(y) in id order; adc_search builds ONE LUT on
// x and returns the min(kprime, n) smallest adc_distance under (dist, id)
// (SPEC.md:165-172); refine residual r = y - pq_decode(pq_encode(y))
// (refine.hpp:30-31); reconstruct = decode_c + decode_r (refine.hpp:42-45);
// rerank = l2_sq(x, reconstruct) -> k smallest (refine.hpp:47-53).

int orc_adc_encode(const float* books, uint32_t d, uint32_t m, uint32_t ks, const float* base,
                   size_t n, uint8_t* out_codes) {
    if (m == 0 || d % m) return fail("dimension not divisible");
    const PQ pq{d, m, ks, books};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i)
        pq_encode_into(pq, base + size_t(i) * d, out_codes + size_t(i) * m);
    return 0;
}

int orc_adc_search_batch(const float* books, uint32_t d, uint32_t m, uint32_t ks,
                         const uint8_t* codes, size_t n, const float* queries, size_t nq,
                         size_t kprime, uint32_t* out_ids, float* out_dists, uint32_t* counts) {
    const PQ pq{d, m, ks, books};
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < int64_t(nq); ++q) {
        std::vector<float> lut(size_t(m) * ks);
        build_lut(pq, queries + size_t(q) * d, lut.data());
        TopK heap(kprime);
        for (size_t i = 0; i < n; ++i)
            heap.push(uint32_t(i), adc_distance(lut.data(), m, ks, codes + i * m));
        auto r = heap.take_sorted();
        for (size_t i = 0; i < r.size(); ++i) {
            out_ids[size_t(q) * kprime + i] = r[i].id;
            out_dists[size_t(q) * kprime + i] = r[i].dist;
        }
        counts[q] = uint32_t(r.size());
    }
    return 0;
}

// refine.hpp:30-31 residual of each row; used by refine_train and refine_encode
static void adc_residuals(const PQ& pq, const float* y, size_t n, float* res) {
    const uint32_t d = pq.d;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i) {
        std::vector<float> p(d);
        uint8_t code[256];
        pq_encode_into(pq, y + size_t(i) * d, code);
        pq_decode_into(pq, code, p.data());
        for (uint32_t t = 0; t < d; ++t) res[size_t(i) * d + t] = y[size_t(i) * d + t] - p[t];
    }
}

// refine.hpp:33-36: pq_train on the residual set, 8 bits per sub-quantizer.
int orc_refine_train(const float* books, uint32_t d, uint32_t m, uint32_t ks, const float* training,
                     size_t n, uint32_t mprime, uint32_t iterations, uint64_t seed,
                     float* out_rbooks) {
    try {
        if (m == 0 || d % m || mprime == 0 || d % mprime)
            throw std::invalid_argument("dimension not divisible");
        std::vector<float> res(n * d);
        adc_residuals(PQ{d, m, ks, books}, training, n, res.data());
        auto b = pq_train(res.data(), n, d, mprime, ks, iterations, seed, 1);
        std::memcpy(out_rbooks, b.data(), b.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e.what());
    }
}

// refine.hpp:38-40: id-aligned encode_r(y - decode(encode(y))).
int orc_adc_refine_encode(const float* books, uint32_t d, uint32_t m, const float* rbooks,
                          uint32_t mprime, uint32_t ks, const float* base, size_t n,
                          uint8_t* out_rcodes) {
    if (mprime == 0 || d % mprime) return fail("dimension not divisible");
    std::vector<float> res(n * d);
    adc_residuals(PQ{d, m, ks, books}, base, n, res.data());
    const PQ rq{d, mprime, ks, rbooks};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i)
        pq_encode_into(rq, res.data() + size_t(i) * d, out_rcodes + size_t(i) * mprime);
    return 0;
}

// refine.hpp:42-45
int orc_adc_reconstruct(const float* books, uint32_t d, uint32_t m, const float* rbooks,
                        uint32_t mprime, uint32_t ks, const uint8_t* code, const uint8_t* rcode,
                        float* out) {
    std::vector<float> p(d), r(d);
    pq_decode_into(PQ{d, m, ks, books}, code, p.data());
    pq_decode_into(PQ{d, mprime, ks, rbooks}, rcode, r.data());
    for (uint32_t t = 0; t < d; ++t) out[t] = p[t] + r[t];
    return 0;
}

// refine.hpp:47-53 ("shortlist too small" when k exceeds the shortlist).
int orc_adc_rerank_batch(const float* books, uint32_t d, uint32_t m, const float* rbooks,
                         uint32_t mprime, uint32_t ks, const uint8_t* codes, const uint8_t* rcodes,
                         const float* queries, size_t nq, const uint32_t* sl_ids,
                         const uint32_t* sl_counts, size_t sl_stride, size_t k, uint32_t* out_ids,
                         float* out_dists) {
    for (size_t q = 0; q < nq; ++q)
        if (k > sl_counts[q]) return fail("shortlist too small");
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < int64_t(nq); ++q) {
        const float* x = queries + size_t(q) * d;
        std::vector<float> yh(d);
        TopK h(k);
        for (uint32_t i = 0; i < sl_counts[q]; ++i) {
            const uint32_t id = sl_ids[size_t(q) * sl_stride + i];
            orc_adc_reconstruct(books, d, m, rbooks, mprime, ks, codes + size_t(id) * m,
                                rcodes + size_t(id) * mprime, yh.data());
            h.push(id, l2_sq(x, yh.data(), d));
        }
        auto r = h.take_sorted();
        for (size_t i = 0; i < r.size(); ++i) {
            out_ids[size_t(q) * k + i] = r[i].id;
            out_dists[size_t(q) * k + i] = r[i].dist;
        }
    }
    return 0;
}

int orc_coarse_probe(const float* coarse, uint32_t c, uint32_t d, const float* queries, size_t nq,
                     uint32_t v, uint32_t* out_lists, float* out_dists) {
    if (v < 1 || v > c) return fail("v must satisfy 1 <= v <= c");
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < int64_t(nq); ++q)
        coarse_probe(coarse, c, d, queries + size_t(q) * d, v, out_lists + size_t(q) * v,
                     out_dists ? out_dists + size_t(q) * v : nullptr);
    return 0;
}

// eval.hpp:13-15 — fp64 exact distances; nearest = lowest id among exact ties
// (SPEC.md:463).
int orc_exact_nearest(const float* base, size_t n, uint32_t d, const float* queries, size_t nq,
                      uint32_t* out_ids, double* out_dists) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t q = 0; q < int64_t(nq); ++q) {
        const float* x = queries + size_t(q) * d;
        uint32_t best = 0;
        double bd = INFINITY;
        for (size_t i = 0; i < n; ++i) {
            double dd = l2_sq_d(x, base + i * d, d);
            if (dd < bd) {
                bd = dd;
                best = uint32_t(i);
            }
        }
        out_ids[q] = best;
        if (out_dists) out_dists[q] = bd;
    }
    return 0;
}

// eval.hpp:21-24 — fraction of queries whose GT nearest is in the first
// min(r, |result|) entries.
double orc_recall_at_r(const uint32_t* res_ids, const uint32_t* res_counts, size_t stride,
                       size_t nq, const uint32_t* gt_nearest, size_t r) {
    if (nq == 0) return 0.0;
    size_t hit = 0;
    for (size_t q = 0; q < nq; ++q) {
        size_t lim = std::min<size_t>(r, res_counts[q]);
        for (size_t i = 0; i < lim; ++i)
            if (res_ids[q * stride + i] == gt_nearest[q]) {
                ++hit;
                break;
            }
    }
    return double(hit) / double(nq);
}

// ================================================================= generator
// BASELINE.json configs + SURVEY.md §8d.  SplitMix64 exactly as rng.hpp:30-45;
// one counter stream per (seed, set, row) so any row range is generated
// independently.  ln / sin / cos are spelled out with IEEE + - * / only so a
// device implementation with _rn intrinsics is bit-identical (libm and
// libdevice differ in the last ulp).
namespace {
inline uint64_t fmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
inline uint64_t sm_next(uint64_t& s) {
    s += 0x9e3779b97f4a7c15ULL;
    return fmix64(s);
}
inline double sm_open01(uint64_t& s) {
    return double((sm_next(s) >> 11) + 1) * (1.0 / 9007199254740992.0);
}
inline double my_ln(double u) {
    uint64_t b;
    std::memcpy(&b, &u, 8);
    int e = int((b >> 52) & 0x7ff) - 1023;
    uint64_t fb = (b & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
    double f;
    std::memcpy(&f, &fb, 8);
    if (f > 0x1.6a09e667f3bcdp+0) {
        f = f * 0.5;
        e += 1;
    }
    double s = (f - 1.0) / (f + 1.0);
    double z = s * s;
    double p = 0x1.8618618618618p-5;  // 1/21
    p = p * z + 0x1.af286bca1af28p-5;
    p = p * z + 0x1.e1e1e1e1e1e1ep-5;
    p = p * z + 0x1.1111111111111p-4;
    p = p * z + 0x1.3b13b13b13b14p-4;
    p = p * z + 0x1.745d1745d1746p-4;
    p = p * z + 0x1.c71c71c71c71cp-4;
    p = p * z + 0x1.2492492492492p-3;
    p = p * z + 0x1.999999999999ap-3;
    p = p * z + 0x1.5555555555555p-2;
    p = p * z + 1.0;
    double lnf = (2.0 * s) * p;
    return double(e) * 0x1.62e42fefa39efp-1 + lnf;
}
inline void my_sincos_2pi(double u, double& sn, double& cs) {
    double t = u * 4.0;
    double q = std::floor(t);
    double r = t - q;
    double ph = r * 0x1.921fb54442d18p+0;
    double z = ph * ph;
    double ps = -0x1.761b41316381ap-75;
    ps = ps * z + 0x1.71b8ef6dcf572p-66;
    ps = ps * z + -0x1.2f49b46814157p-57;
    ps = ps * z + 0x1.952c77030ad4ap-49;
    ps = ps * z + -0x1.ae7f3e733b81fp-41;
    ps = ps * z + 0x1.6124613a86d09p-33;
    ps = ps * z + -0x1.ae64567f544e4p-26;
    ps = ps * z + 0x1.71de3a556c734p-19;
    ps = ps * z + -0x1.a01a01a01a01ap-13;
    ps = ps * z + 0x1.1111111111111p-7;
    ps = ps * z + -0x1.5555555555555p-3;
    ps = ps * z + 1.0;
    double s = ph * ps;
    double pc = -0x1.0ce396db7f853p-70;
    pc = pc * z + 0x1.e542ba4020225p-62;
    pc = pc * z + -0x1.6827863b97d97p-53;
    pc = pc * z + 0x1.ae7f3e733b81fp-45;
    pc = pc * z + -0x1.93974a8c07c9dp-37;
    pc = pc * z + 0x1.1eed8eff8d898p-29;
    pc = pc * z + -0x1.27e4fb7789f5cp-22;
    pc = pc * z + 0x1.a01a01a01a01ap-16;
    pc = pc * z + -0x1.6c16c16c16c17p-10;
    pc = pc * z + 0x1.5555555555555p-5;
    pc = pc * z + -0x1.0000000000000p-1;
    pc = pc * z + 1.0;
    double c = pc;
    int qi = int(q) & 3;
    switch (qi) {
        case 0: sn = s; cs = c; break;
        case 1: sn = c; cs = -s; break;
        case 2: sn = -s; cs = -c; break;
        default: sn = -c; cs = s; break;
    }
}
inline uint8_t quantize(double v) {
    if (!(v > 0.0)) v = 0.0;
    if (v > 255.0) v = 255.0;
    double r = std::nearbyint(v);  // round half to even (default FE_TONEAREST)
    int iv = int(r);
    return iv < 4 ? 0 : uint8_t(iv);
}
}  // namespace

uint64_t orc_splitmix_stream_state(uint64_t seed, uint32_t set, uint64_t row) {
    return fmix64(fmix64(seed ^ (uint64_t(set + 1) * 0xD1B54A32D192ED03ULL)) + row);
}
uint64_t orc_splitmix_next(uint64_t* state) { return sm_next(*state); }
void orc_bounded_u32(uint32_t seed, uint32_t bound, size_t n, uint32_t* out) {
    std::mt19937 g(seed);
    for (size_t i = 0; i < n; ++i) out[i] = bounded_u32(g, bound);
}
void orc_uniform01(uint32_t seed, size_t n, float* out) {
    std::mt19937 g(seed);
    for (size_t i = 0; i < n; ++i) out[i] = uniform01(g);
}
double orc_ln(double u) { return my_ln(u); }
void orc_sincos_2pi(double u, double* s, double* c) { my_sincos_2pi(u, *s, *c); }

// Mixture centres: mu[k][t] = -20 ln(U), U in (0,1] (Exp with mean 20).
int orc_synth_centers(uint64_t seed, uint32_t clusters, uint32_t d, double* out) {
    for (uint32_t k = 0; k < clusters; ++k) {
        uint64_t s = orc_splitmix_stream_state(seed, ORC_SET_CENTERS, k);
        for (uint32_t t = 0; t < d; ++t) out[size_t(k) * d + t] = -20.0 * my_ln(sm_open01(s));
    }
    return 0;
}

// Row = mu[comp] + 10 * N(0,1) per dim (Box-Muller pairs), clamped to
// [0,255], rounded half-to-even, values < 4 zeroed; comp = mulhi(next, K).
int orc_synth_rows(uint64_t seed, uint32_t set, uint64_t row0, size_t n, uint32_t d,
                   const double* centers, uint32_t clusters, uint8_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i) {
        uint64_t s = orc_splitmix_stream_state(seed, set, row0 + uint64_t(i));
        uint64_t comp = uint64_t((unsigned __int128)sm_next(s) * clusters >> 64);
        const double* mu = centers + comp * d;
        uint8_t* o = out + size_t(i) * d;
        for (uint32_t t = 0; t < d; t += 2) {
            double u1 = sm_open01(s);
            double u2 = sm_open01(s);
            double r = std::sqrt(-2.0 * my_ln(u1));
            double sn, cs;
            my_sincos_2pi(u2, sn, cs);
            o[t] = quantize(mu[t] + 10.0 * (r * cs));
            if (t + 1 < d) o[t + 1] = quantize(mu[t + 1] + 10.0 * (r * sn));
        }
    }
    return 0;
}

}  // extern "C"
