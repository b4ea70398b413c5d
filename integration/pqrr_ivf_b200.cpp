// pqrr_ivf_b200.cpp — reference-side drop-in for the IVFADC+R path.
//
// Compiled against the reference's own headers (proj/include/pqrr/), this
// translation unit DEFINES the functions the reference declares for the path
// (ivf_index.hpp:48-81, kmeans.hpp:38, product_quantizer.hpp:39-49) and the
// link-time hot-kernel seam (kernels.hpp:13-43, replacing src/kernels.cpp) on
// top of the C ABI in include/pqrr_dev.h.  A maintainer adds this file and
// libpqrr_b200.so to the reference build; callers keep using pqrr::ivf_*.
//
// The device index behind a host IvfIndex is created lazily and cached.  A
// cache entry is found by the addresses of the IvfIndex's list storage (and
// the RefineCodes buffer when re-ranking) and is only reused when its content
// signature still matches: n, every list length, the coarse / PQ / refine
// code books in full, the first and last (id, code) of every list, a strided
// sample of all entries and of the refinement codes.  A new IvfIndex that
// reuses a freed address therefore gets a fresh device index.  The cache is
// LRU-bounded (PQRR_INDEX_CACHE entries, default 2); evicted device indexes
// are destroyed once no call still uses them, and
// pqrr::b200::release_device_indexes() drops them all.
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pqrr/ivf_index.hpp"
#include "pqrr/kernels.hpp"
#include "pqrr/kmeans.hpp"
#include "pqrr/product_quantizer.hpp"
#include "pqrr/refine.hpp"
#include "pqrr_dev.h"

namespace pqrr {
namespace {

void check(int rc) {
    if (rc == PQRR_OK) return;
    const std::string msg = pqrr_dev_last_error();
    if (rc == PQRR_EINVAL || rc == PQRR_ESHORTLIST) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

int device() {
    const char* e = std::getenv("PQRR_DEVICE");
    return e ? std::atoi(e) : 0;
}

std::vector<float> flat_books(const ProductQuantizer& pq) {
    std::vector<float> out;
    out.reserve(std::size_t(pq.ks) * pq.d);
    for (const Codebook& b : pq.books) out.insert(out.end(), b.centroids.begin(), b.centroids.end());
    return out;
}

ProductQuantizer make_pq(std::uint32_t d, std::uint32_t m, std::uint32_t ks, const float* books) {
    ProductQuantizer pq;
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

using Handle = std::shared_ptr<pqrr_dev_index>;

Handle own(pqrr_dev_index* h) {
    return Handle(h, [](pqrr_dev_index* p) { pqrr_dev_index_destroy(p); });
}

// FNV-1a over byte ranges
struct Fnv {
    std::uint64_t h = 1469598103934665603ull;
    void add(const void* p, std::size_t n) {
        const auto* b = static_cast<const std::uint8_t*>(p);
        for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    }
    template <class T>
    void pod(const T& v) { add(&v, sizeof(T)); }
};

struct Signature {
    std::uint64_t n = 0, books = 0, entries = 0, refine = 0;
    std::vector<std::uint64_t> lens;
    bool operator==(const Signature&) const = default;
};

Signature signature(const IvfIndex& ix, const RefineQuantizer* rq, const RefineCodes* codes) {
    Signature s;
    s.n = ix.n;
    s.lens.reserve(ix.c());
    Fnv b, e;
    b.add(ix.coarse.centroids.data(), ix.coarse.centroids.size() * 4);
    for (const Codebook& cb : ix.pq.books) b.add(cb.centroids.data(), cb.centroids.size() * 4);
    const std::uint32_t m = ix.pq.m;
    std::uint64_t total = 0;
    for (const IvfList& L : ix.lists) {
        s.lens.push_back(L.ids.size());
        total += L.ids.size();
        if (!L.ids.empty()) {
            e.pod(L.ids.front());
            e.pod(L.ids.back());
            e.add(L.codes.data(), m);
            e.add(L.codes.data() + (L.ids.size() - 1) * m, m);
        }
    }
    const std::uint64_t stride = std::max<std::uint64_t>(1, total / 65536);
    std::uint64_t base = 0;
    for (const IvfList& L : ix.lists) {  // every stride-th entry of the list-order concatenation
        for (std::uint64_t g = (base + stride - 1) / stride * stride; g < base + L.ids.size(); g += stride) {
            e.pod(L.ids[g - base]);
            e.add(L.codes.data() + (g - base) * m, m);
        }
        base += L.ids.size();
    }
    s.books = b.h;
    s.entries = e.h;
    if (rq && codes) {
        Fnv r;
        for (const Codebook& cb : rq->pq.books) r.add(cb.centroids.data(), cb.centroids.size() * 4);
        r.pod(codes->m);
        const std::size_t nb = codes->bytes.size();
        r.pod(nb);
        const std::size_t st = std::max<std::size_t>(1, nb / 65536);
        for (std::size_t i = 0; i < nb; i += st) r.pod(codes->bytes[i]);
        if (nb) r.pod(codes->bytes[nb - 1]);
        s.refine = r.h;
    }
    return s;
}

struct Entry {
    std::pair<const void*, const void*> key;
    Signature sig;
    Handle h;
};

struct Cache {
    std::mutex mu;
    std::list<Entry> lru;  // most recently used first
    std::size_t cap() const {
        const char* e = std::getenv("PQRR_INDEX_CACHE");
        const long v = e ? std::atol(e) : 2;
        return v > 0 ? std::size_t(v) : 1;
    }
    void put(Entry en) {  // caller holds mu
        for (auto it = lru.begin(); it != lru.end(); ++it)
            if (it->key == en.key) {
                lru.erase(it);
                break;
            }
        lru.push_front(std::move(en));
        while (lru.size() > cap()) lru.pop_back();
    }
};
Cache& cache() {
    static Cache c;
    return c;
}

std::pair<const void*, const void*> cache_key(const IvfIndex& ix, const RefineCodes* codes) {
    return {static_cast<const void*>(ix.lists.data()),
            static_cast<const void*>(codes ? codes->bytes.data() : nullptr)};
}

// Device index for (index[, refinement]); built from the host lists on a
// cache miss or a signature mismatch.
Handle device_index(const IvfIndex& ix, const RefineQuantizer* rq, const RefineCodes* codes) {
    const auto key = cache_key(ix, codes);
    Signature sig = signature(ix, rq, codes);
    auto& c = cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto it = c.lru.begin(); it != c.lru.end(); ++it)
            if (it->key == key) {
                if (it->sig == sig) {
                    c.lru.splice(c.lru.begin(), c.lru, it);
                    return it->h;
                }
                c.lru.erase(it);  // a different index now lives at this address
                break;
            }
    }
    const std::uint32_t mp = rq ? rq->pq.m : 0;
    auto books = flat_books(ix.pq);
    std::vector<float> rbooks;
    if (rq) rbooks = flat_books(rq->pq);
    pqrr_dev_index* raw = nullptr;
    check(pqrr_dev_index_create(device(), ix.pq.d, ix.c(), ix.coarse.centroids.data(), ix.pq.m,
                                books.data(), mp, rq ? rbooks.data() : nullptr, ix.pq.ks, &raw));
    Handle h = own(raw);
    std::vector<std::uint64_t> off(ix.c() + 1, 0);
    for (std::uint32_t l = 0; l < ix.c(); ++l) off[l + 1] = off[l] + ix.lists[l].size();
    std::vector<std::uint32_t> ids(off.back());
    std::vector<std::uint8_t> cds(off.back() * ix.pq.m), rcs(off.back() * std::max<std::uint32_t>(mp, 1));
    for (std::uint32_t l = 0; l < ix.c(); ++l) {
        const IvfList& L = ix.lists[l];
        std::memcpy(ids.data() + off[l], L.ids.data(), L.ids.size() * 4);
        std::memcpy(cds.data() + off[l] * ix.pq.m, L.codes.data(), L.codes.size());
        if (mp)
            for (std::size_t i = 0; i < L.ids.size(); ++i)
                std::memcpy(rcs.data() + (off[l] + i) * mp, codes->code(L.ids[i]), mp);
    }
    check(pqrr_dev_load_lists(h.get(), off.data(), ids.data(), cds.data(), mp ? rcs.data() : nullptr));
    std::lock_guard<std::mutex> lk(c.mu);
    c.put(Entry{key, std::move(sig), h});
    return h;
}

SearchResult to_result(const std::uint32_t* ids, const float* d, std::uint32_t n) {
    SearchResult r;
    r.entries.resize(n);
    for (std::uint32_t i = 0; i < n; ++i) r.entries[i] = Neighbor{ids[i], d[i]};
    return r;
}

}  // namespace

// ------------------------------------------------------------------ training
Codebook kmeans_train(const VectorSet& points, std::uint32_t k, const TrainParams& params) {
    points.validate();
    Codebook cb;
    cb.k = k;
    cb.dim = points.d;
    cb.centroids.resize(std::size_t(k) * points.d);
    std::vector<double> trace(std::max<std::uint32_t>(params.iterations, 1));
    check(pqrr_dev_kmeans_train(device(), points.data.data(), points.n(), points.d, k,
                                params.iterations, params.seed, params.redo, cb.centroids.data(),
                                &cb.final_mse, trace.data()));
    if (params.trace) params.trace->assign(trace.begin(), trace.begin() + params.iterations);
    return cb;
}

ProductQuantizer pq_train(const VectorSet& training, std::uint32_t m, std::uint32_t ks,
                          const TrainParams& params) {
    if (m == 0 || training.d % m) throw std::invalid_argument("dimension not divisible");
    std::vector<float> books(std::size_t(ks) * training.d);
    check(pqrr_dev_pq_train(device(), training.data.data(), training.n(), training.d, m, ks,
                            params.iterations, params.seed, params.redo, books.data()));
    return make_pq(training.d, m, ks, books.data());
}

std::pair<Codebook, ProductQuantizer> ivf_train(const VectorSet& training, std::uint32_t c,
                                                std::uint32_t m, std::uint32_t ks,
                                                const TrainParams& params) {
    if (m == 0 || training.d % m) throw std::invalid_argument("dimension not divisible");
    Codebook coarse;
    coarse.k = c;
    coarse.dim = training.d;
    coarse.centroids.resize(std::size_t(c) * training.d);
    std::vector<float> books(std::size_t(ks) * training.d);
    check(pqrr_dev_ivf_train(device(), training.data.data(), training.n(), training.d, c, m, ks,
                             params.iterations, params.seed, coarse.centroids.data(), books.data()));
    return {std::move(coarse), make_pq(training.d, m, ks, books.data())};
}

RefineQuantizer ivf_refine_train(const Codebook& coarse, const ProductQuantizer& pq,
                                 const VectorSet& training, std::uint32_t mprime,
                                 const TrainParams& params) {
    if (mprime == 0 || training.d % mprime) throw std::invalid_argument("dimension not divisible");
    auto books = flat_books(pq);
    std::vector<float> rb(std::size_t(pq.ks) * training.d);
    check(pqrr_dev_ivf_refine_train(device(), coarse.centroids.data(), coarse.k, books.data(), pq.d,
                                    pq.m, pq.ks, training.data.data(), training.n(), mprime,
                                    params.iterations, params.seed, rb.data()));
    RefineQuantizer rq;
    rq.pq = make_pq(training.d, mprime, pq.ks, rb.data());
    return rq;
}

// ------------------------------------------------------------------ PQ codec (product_quantizer.hpp:42-49)
void pq_encode_into(const ProductQuantizer& pq, const float* y, std::uint8_t* code) {
    kernels::encode_batch(pq, y, 1, code);
}
std::vector<std::uint8_t> pq_encode(const ProductQuantizer& pq, std::span<const float> y) {
    if (y.size() != pq.d) throw std::invalid_argument("length mismatch");
    std::vector<std::uint8_t> c(pq.m);
    pq_encode_into(pq, y.data(), c.data());
    return c;
}
void pq_decode_into(const ProductQuantizer& pq, const std::uint8_t* code, float* out) {
    kernels::decode_batch(pq, code, 1, out);
}
std::vector<float> pq_decode(const ProductQuantizer& pq, std::span<const std::uint8_t> code) {
    std::vector<float> out(pq.d);
    pq_decode_into(pq, code.data(), out.data());
    return out;
}
LookupTable build_lut(const ProductQuantizer& pq, std::span<const float> x) {
    if (x.size() != pq.d) throw std::invalid_argument("length mismatch");
    LookupTable t;
    t.m = pq.m;
    t.ks = pq.ks;
    t.values.resize(std::size_t(pq.m) * pq.ks);
    auto books = flat_books(pq);
    check(pqrr_dev_build_lut(device(), books.data(), pq.d, pq.m, pq.ks, x.data(), 1, t.values.data()));
    return t;
}

// ------------------------------------------------------------------ IVF index (ivf_index.hpp:54-81)
IvfIndex ivf_build(Codebook coarse, ProductQuantizer pq, const VectorSet& base) {
    base.validate();
    if (base.d != pq.d) throw std::invalid_argument("dimension mismatch");
    auto books = flat_books(pq);
    pqrr_dev_index* h = nullptr;
    check(pqrr_dev_index_create(device(), pq.d, coarse.k, coarse.centroids.data(), pq.m, books.data(), 0,
                                nullptr, pq.ks, &h));
    check(pqrr_dev_add_f32(h, base.data.data(), base.n(), 0));
    IvfIndex ix;
    ix.coarse = std::move(coarse);
    ix.pq = std::move(pq);
    ix.n = base.n();
    std::vector<std::uint64_t> off(ix.c() + 1);
    std::vector<std::uint32_t> ids(ix.n);
    std::vector<std::uint8_t> cds(ix.n * ix.pq.m);
    check(pqrr_dev_export_lists(h, off.data(), ids.data(), cds.data(), nullptr));
    ix.lists.resize(ix.c());
    ix.list_of_id.resize(ix.n);
    ix.pos_of_id.resize(ix.n);
    for (std::uint32_t l = 0; l < ix.c(); ++l) {
        IvfList& L = ix.lists[l];
        L.ids.assign(ids.begin() + off[l], ids.begin() + off[l + 1]);
        L.codes.assign(cds.begin() + off[l] * ix.pq.m, cds.begin() + off[l + 1] * ix.pq.m);
        for (std::size_t i = 0; i < L.ids.size(); ++i) {
            ix.list_of_id[L.ids[i]] = l;
            ix.pos_of_id[L.ids[i]] = std::uint32_t(i);
        }
    }
    auto& c = cache();
    Entry en{cache_key(ix, nullptr), signature(ix, nullptr, nullptr), own(h)};
    std::lock_guard<std::mutex> lk(c.mu);
    c.put(std::move(en));
    return ix;
}

std::vector<SearchResult> ivf_search_batch(const IvfIndex& index, const VectorSet& queries,
                                           const IvfSearchParams& params) {
    if (queries.d != index.pq.d) throw std::invalid_argument("dimension mismatch");
    Handle h = device_index(index, nullptr, nullptr);
    const std::size_t nq = queries.n(), kp = params.kprime;
    std::vector<std::uint32_t> ids(nq * kp), cnt(nq);
    std::vector<float> d(nq * kp);
    check(pqrr_dev_search_f32(h.get(), queries.data.data(), nq, params.v, kp, 0, ids.data(), d.data(),
                              cnt.data()));
    std::vector<SearchResult> out(nq);
    for (std::size_t q = 0; q < nq; ++q) out[q] = to_result(&ids[q * kp], &d[q * kp], cnt[q]);
    return out;
}

SearchResult ivf_search(const IvfIndex& index, std::span<const float> x, const IvfSearchParams& params) {
    VectorSet q(index.pq.d, 1);
    if (x.size() != index.pq.d) throw std::invalid_argument("dimension mismatch");
    std::memcpy(q.data.data(), x.data(), x.size() * 4);
    return ivf_search_batch(index, q, params)[0];
}

RefineCodes ivf_refine_encode(const IvfIndex& index, const RefineQuantizer& rq, const VectorSet& base) {
    if (base.n() != index.n) throw std::invalid_argument("count mismatch");
    auto books = flat_books(index.pq), rb = flat_books(rq.pq);
    pqrr_dev_index* h = nullptr;
    check(pqrr_dev_index_create(device(), index.pq.d, index.c(), index.coarse.centroids.data(),
                                index.pq.m, books.data(), rq.pq.m, rb.data(), index.pq.ks, &h));
    check(pqrr_dev_add_f32(h, base.data.data(), base.n(), 0));
    std::vector<std::uint64_t> off(index.c() + 1);
    std::vector<std::uint32_t> ids(index.n);
    std::vector<std::uint8_t> rc(index.n * rq.pq.m);
    check(pqrr_dev_export_lists(h, off.data(), ids.data(), nullptr, rc.data()));
    check(pqrr_dev_index_destroy(h));
    RefineCodes codes;
    codes.m = rq.pq.m;
    codes.bytes.resize(index.n * rq.pq.m);
    for (std::size_t i = 0; i < index.n; ++i)
        std::memcpy(codes.bytes.data() + std::size_t(ids[i]) * codes.m, rc.data() + i * codes.m, codes.m);
    return codes;
}

std::vector<float> ivf_reconstruct(const IvfIndex& index, const RefineQuantizer& rq, std::uint32_t id,
                                   const RefineCodes& codes) {
    Handle h = device_index(index, &rq, &codes);
    std::vector<float> out(index.pq.d);
    check(pqrr_dev_reconstruct(h.get(), &id, 1, out.data()));
    return out;
}

SearchResult ivf_rerank(std::span<const float> x, const SearchResult& shortlist, const IvfIndex& index,
                        const RefineQuantizer& rq, const RefineCodes& codes, std::size_t k) {
    if (k > shortlist.size()) throw std::invalid_argument("shortlist too small");
    Handle h = device_index(index, &rq, &codes);
    std::vector<std::uint32_t> sl(shortlist.size());
    for (std::size_t i = 0; i < sl.size(); ++i) sl[i] = shortlist[i].id;
    const std::uint32_t cnt = std::uint32_t(sl.size());
    std::vector<std::uint32_t> ids(std::max<std::size_t>(k, 1));
    std::vector<float> d(std::max<std::size_t>(k, 1));
    check(pqrr_dev_rerank_f32(h.get(), x.data(), 1, sl.data(), &cnt, std::max<std::size_t>(sl.size(), 1), k,
                              ids.data(), d.data()));
    return to_result(ids.data(), d.data(), std::uint32_t(k));
}

// Drops every cached device index (each is destroyed once no call uses it).
namespace b200 {
void release_device_indexes() {
    auto& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.lru.clear();
}
}  // namespace b200

// ------------------------------------------------------------------ kernel seam (kernels.hpp:13-43)
namespace kernels {

void set_threads(int) {}
int max_threads() { return 1; }

void assign_batch(const float* points, std::size_t n, std::uint32_t dim, const float* centroids,
                  std::uint32_t k, std::uint32_t* out_assign, float* out_dist) {
    check(pqrr_dev_assign_batch(device(), points, n, dim, centroids, k, out_assign, out_dist));
}

void encode_batch(const ProductQuantizer& pq, const float* data, std::size_t n, std::uint8_t* out_codes) {
    auto books = flat_books(pq);
    check(pqrr_dev_encode_batch(device(), books.data(), pq.d, pq.m, pq.ks, data, n, out_codes));
}

void decode_batch(const ProductQuantizer& pq, const std::uint8_t* codes, std::size_t n, float* out) {
    auto books = flat_books(pq);
    check(pqrr_dev_decode_batch(device(), books.data(), pq.d, pq.m, pq.ks, codes, n, out));
}

SearchResult scan_topk(const LookupTable& lut, const std::uint8_t* codes, std::size_t n,
                       std::size_t kprime, std::uint32_t id_base) {
    std::vector<std::uint32_t> ids(std::max<std::size_t>(kprime, 1));
    std::vector<float> d(std::max<std::size_t>(kprime, 1));
    std::size_t cnt = 0;
    check(pqrr_dev_scan_topk(device(), lut.values.data(), lut.m, lut.ks, codes, n, kprime, id_base,
                             ids.data(), d.data(), &cnt));
    return to_result(ids.data(), d.data(), std::uint32_t(cnt));
}

}  // namespace kernels
}  // namespace pqrr
