// ref_shim.cpp — links the reference's OWN hot-kernel code into a testable
// library (oracle/_ref/libpqrr_ref.so).  TEST INFRASTRUCTURE ONLY.
//
// Built by oracle/Makefile together with /root/reference/proj/src/kernels.cpp,
// compiled in place (never copied) against /root/reference/proj/include with
// the reference's FP flags (CMakeLists.txt:11-13).  Everything computed here
// runs through the reference's real code: l2_sq (distance.hpp:16-33),
// adc_distance (product_quantizer.hpp:53-57), TopK (topk.hpp:14-52),
// neighbor_less (types.hpp:47-50), SplitMix64 / bounded_u32 / uniform01
// (rng.hpp), and kernels::assign_batch / encode_batch / decode_batch /
// scan_topk (kernels.cpp:21-96).  The reference declares but never defines
// pq_encode_into / pq_decode_into / build_lut (product_quantizer.hpp:42-49);
// the minimal bodies below are the parity contract of SURVEY.md §8a written
// against the reference's own types, so kernels.cpp links.
#include <omp.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "pqrr/distance.hpp"
#include "pqrr/kernels.hpp"
#include "pqrr/product_quantizer.hpp"
#include "pqrr/rng.hpp"
#include "pqrr/topk.hpp"
#include "pqrr/types.hpp"

namespace pqrr {

void pq_encode_into(const ProductQuantizer& pq, const float* y, std::uint8_t* code) {
    const std::uint32_t ds = pq.dsub();
    for (std::uint32_t j = 0; j < pq.m; ++j) {
        const Codebook& b = pq.books[j];
        std::uint32_t best = 0;
        float bd = l2_sq(y + std::size_t(j) * ds, b.centroid(0), ds);
        for (std::uint32_t i = 1; i < b.k; ++i) {
            float d = l2_sq(y + std::size_t(j) * ds, b.centroid(i), ds);
            if (d < bd) {
                bd = d;
                best = i;
            }
        }
        code[j] = std::uint8_t(best);
    }
}

void pq_decode_into(const ProductQuantizer& pq, const std::uint8_t* code, float* out) {
    const std::uint32_t ds = pq.dsub();
    for (std::uint32_t j = 0; j < pq.m; ++j)
        std::memcpy(out + std::size_t(j) * ds, pq.books[j].centroid(code[j]), ds * sizeof(float));
}

LookupTable build_lut(const ProductQuantizer& pq, std::span<const float> x) {
    LookupTable t;
    t.m = pq.m;
    t.ks = pq.ks;
    t.values.resize(std::size_t(pq.m) * pq.ks);
    const std::uint32_t ds = pq.dsub();
    for (std::uint32_t j = 0; j < pq.m; ++j)
        for (std::uint32_t i = 0; i < pq.ks; ++i)
            t.values[std::size_t(j) * pq.ks + i] =
                l2_sq(x.data() + std::size_t(j) * ds, pq.books[j].centroid(i), ds);
    return t;
}

}  // namespace pqrr

namespace {

pqrr::ProductQuantizer make_pq(const float* books, std::uint32_t d, std::uint32_t m,
                               std::uint32_t ks) {
    pqrr::ProductQuantizer pq;
    pq.d = d;
    pq.m = m;
    pq.ks = ks;
    const std::uint32_t ds = d / m;
    pq.books.resize(m);
    for (std::uint32_t j = 0; j < m; ++j) {
        pq.books[j].k = ks;
        pq.books[j].dim = ds;
        pq.books[j].centroids.assign(books + std::size_t(j) * ks * ds,
                                     books + std::size_t(j + 1) * ks * ds);
    }
    return pq;
}

}  // namespace

extern "C" {

void ref_set_threads(int t) { pqrr::kernels::set_threads(t); }
int ref_max_threads(void) { return pqrr::kernels::max_threads(); }

float ref_l2_sq(const float* a, const float* b, std::size_t d) { return pqrr::l2_sq(a, b, d); }
double ref_l2_sq_d(const float* a, const float* b, std::size_t d) { return pqrr::l2_sq_d(a, b, d); }

void ref_assign_batch(const float* points, std::size_t n, std::uint32_t dim,
                      const float* centroids, std::uint32_t k, std::uint32_t* out_assign,
                      float* out_dist) {
    pqrr::kernels::assign_batch(points, n, dim, centroids, k, out_assign, out_dist);
}

void ref_encode_batch(const float* books, std::uint32_t d, std::uint32_t m, std::uint32_t ks,
                      const float* data, std::size_t n, std::uint8_t* out) {
    auto pq = make_pq(books, d, m, ks);
    pqrr::kernels::encode_batch(pq, data, n, out);
}

void ref_decode_batch(const float* books, std::uint32_t d, std::uint32_t m, std::uint32_t ks,
                      const std::uint8_t* codes, std::size_t n, float* out) {
    auto pq = make_pq(books, d, m, ks);
    pqrr::kernels::decode_batch(pq, codes, n, out);
}

void ref_build_lut(const float* books, std::uint32_t d, std::uint32_t m, std::uint32_t ks,
                   const float* x, float* out) {
    auto pq = make_pq(books, d, m, ks);
    auto t = pqrr::build_lut(pq, std::span<const float>(x, d));
    std::memcpy(out, t.values.data(), t.values.size() * sizeof(float));
}

float ref_adc_distance(const float* lut, std::uint32_t m, std::uint32_t ks,
                       const std::uint8_t* code) {
    pqrr::LookupTable t;
    t.m = m;
    t.ks = ks;
    t.values.assign(lut, lut + std::size_t(m) * ks);
    return pqrr::adc_distance(t, code);
}

std::size_t ref_scan_topk(const float* lut, std::uint32_t m, std::uint32_t ks,
                          const std::uint8_t* codes, std::size_t n, std::size_t kprime,
                          std::uint32_t id_base, std::uint32_t* out_ids, float* out_dists) {
    pqrr::LookupTable t;
    t.m = m;
    t.ks = ks;
    t.values.assign(lut, lut + std::size_t(m) * ks);
    auto r = pqrr::kernels::scan_topk(t, codes, n, kprime, id_base);
    for (std::size_t i = 0; i < r.size(); ++i) {
        out_ids[i] = r[i].id;
        out_dists[i] = r[i].dist;
    }
    return r.size();
}

std::size_t ref_topk(const std::uint32_t* ids, const float* dists, std::size_t n, std::size_t k,
                     std::uint32_t* out_ids, float* out_dists) {
    pqrr::TopK h(k);
    for (std::size_t i = 0; i < n; ++i) h.push(ids[i], dists[i]);
    auto r = h.take_sorted();
    for (std::size_t i = 0; i < r.size(); ++i) {
        out_ids[i] = r[i].id;
        out_dists[i] = r[i].dist;
    }
    return r.size();
}

void ref_splitmix(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
    pqrr::SplitMix64 s(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = s.next();
}

void ref_bounded_u32(std::uint32_t seed, std::uint32_t bound, std::size_t n, std::uint32_t* out) {
    std::mt19937 g(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = pqrr::bounded_u32(g, bound);
}

void ref_uniform01(std::uint32_t seed, std::size_t n, float* out) {
    std::mt19937 g(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = pqrr::uniform01(g);
}

// The reference's ivf_search (ivf_index.hpp:58-64) has no body.  This is the
// closest reference-backed form: coarse probe with the reference l2_sq, one
// reference LUT per probed list on x - C_l, and the reference's own
// kernels::scan_topk over each list's codes (its positions map to list ids
// monotonically because lists are id-ascending, ivf_index.hpp:15-16), merged
// under the reference neighbor_less.  Lists are passed flattened:
// offsets[c+1], ids[n], codes[n*m] in list order.
void ref_ivf_search_batch(const float* coarse, std::uint32_t c, const float* books,
                          std::uint32_t d, std::uint32_t m, std::uint32_t ks,
                          const std::uint64_t* offsets, const std::uint32_t* ids,
                          const std::uint8_t* codes, const float* queries, std::size_t nq,
                          std::uint32_t v, std::size_t kprime, std::uint32_t* out_ids,
                          float* out_dists, std::uint32_t* counts) {
    auto pq = make_pq(books, d, m, ks);
#pragma omp parallel for schedule(dynamic, 1)
    for (std::int64_t q = 0; q < std::int64_t(nq); ++q) {
        const float* x = queries + std::size_t(q) * d;
        std::vector<pqrr::Neighbor> cd(c);
        for (std::uint32_t k = 0; k < c; ++k)
            cd[k] = pqrr::Neighbor{k, pqrr::l2_sq(x, coarse + std::size_t(k) * d, d)};
        std::partial_sort(cd.begin(), cd.begin() + v, cd.end(), pqrr::neighbor_less);
        std::vector<float> xr(d);
        pqrr::TopK heap(kprime);
        for (std::uint32_t p = 0; p < v; ++p) {
            const std::uint32_t l = cd[p].id;
            const float* C = coarse + std::size_t(l) * d;
            for (std::uint32_t t = 0; t < d; ++t) xr[t] = x[t] - C[t];
            auto lut = pqrr::build_lut(pq, std::span<const float>(xr.data(), d));
            const std::uint64_t lo = offsets[l], hi = offsets[l + 1];
            auto part = pqrr::kernels::scan_topk(lut, codes + lo * m, hi - lo, kprime, 0);
            for (const auto& e : part.entries) heap.push(ids[lo + e.id], e.dist);
        }
        auto r = heap.take_sorted();
        for (std::size_t i = 0; i < r.size(); ++i) {
            out_ids[std::size_t(q) * kprime + i] = r[i].id;
            out_dists[std::size_t(q) * kprime + i] = r[i].dist;
        }
        counts[q] = std::uint32_t(r.size());
    }
}

// ivf_rerank (ivf_index.hpp:79-81) through reference helpers: ŷ = (C_a + p) + r
// decoded with kernels::decode-equivalent pq_decode_into, distance pqrr::l2_sq,
// selection pqrr::TopK.  list_of_id / code lookups come flattened.
int ref_ivf_rerank_batch(const float* coarse, const float* books, const float* rbooks,
                         std::uint32_t d, std::uint32_t m, std::uint32_t mprime,
                         std::uint32_t ks, const std::uint32_t* list_of_id,
                         const std::uint8_t* codes_by_id, const std::uint8_t* rcodes_by_id,
                         const float* queries, std::size_t nq, const std::uint32_t* sl_ids,
                         const std::uint32_t* sl_counts, std::size_t sl_stride, std::size_t k,
                         std::uint32_t* out_ids, float* out_dists) {
    for (std::size_t q = 0; q < nq; ++q)
        if (k > sl_counts[q]) return -1;  // "shortlist too small"
    auto pq = make_pq(books, d, m, ks);
    auto rq = make_pq(rbooks, d, mprime, ks);
#pragma omp parallel for schedule(dynamic, 1)
    for (std::int64_t q = 0; q < std::int64_t(nq); ++q) {
        const float* x = queries + std::size_t(q) * d;
        std::vector<float> p(d), r(d), yh(d);
        pqrr::TopK h(k);
        for (std::uint32_t i = 0; i < sl_counts[q]; ++i) {
            const std::uint32_t id = sl_ids[std::size_t(q) * sl_stride + i];
            const float* C = coarse + std::size_t(list_of_id[id]) * d;
            pqrr::pq_decode_into(pq, codes_by_id + std::size_t(id) * m, p.data());
            pqrr::pq_decode_into(rq, rcodes_by_id + std::size_t(id) * mprime, r.data());
            for (std::uint32_t t = 0; t < d; ++t) {
                float rec1 = C[t] + p[t];
                yh[t] = rec1 + r[t];
            }
            h.push(id, pqrr::l2_sq(x, yh.data(), d));
        }
        auto res = h.take_sorted();
        for (std::size_t i = 0; i < res.size(); ++i) {
            out_ids[std::size_t(q) * k + i] = res[i].id;
            out_dists[std::size_t(q) * k + i] = res[i].dist;
        }
    }
    return 0;
}

}  // extern "C"
