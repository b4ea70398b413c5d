// test_shim.cpp — exercises the reference-side drop-in exactly as a reference
// caller would (pqrr::ivf_train / ivf_build / ivf_search_batch / ivf_rerank /
// ivf_reconstruct / kernels::scan_topk, declared in the reference headers) and
// checks every output bit-for-bit against the CPU oracle (test infrastructure,
// oracle/pqrr_oracle.h).  Prints "SHIM OK <checks>" and exits 0 on success.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../oracle/pqrr_oracle.h"
#include "pqrr/ivf_index.hpp"
#include "pqrr/kernels.hpp"
#include "pqrr_dev.h"

using namespace pqrr;

namespace pqrr::b200 {
void release_device_indexes();  // integration/pqrr_ivf_b200.cpp
}

static int checks = 0, failures = 0;
#define EXPECT(cond, what)                                      \
    do {                                                        \
        ++checks;                                               \
        if (!(cond)) {                                          \
            ++failures;                                         \
            std::fprintf(stderr, "FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
        }                                                       \
    } while (0)

static bool same_bits(const float* a, const float* b, size_t n) { return std::memcmp(a, b, n * 4) == 0; }

int main() {
    const uint32_t d = 128, c = 32, m = 8, mp = 16, ks = 256;
    const size_t n = 6000, nt = 3000, nq = 16;
    std::vector<double> centers(64 * d);
    orc_synth_centers(7, 64, d, centers.data());
    auto gen = [&](uint32_t set, size_t rows) {
        std::vector<uint8_t> u(rows * d);
        orc_synth_rows(7, set, 0, rows, d, centers.data(), 64, u.data());
        VectorSet v(d, rows);
        for (size_t i = 0; i < u.size(); ++i) v.data[i] = float(u[i]);
        return v;
    };
    VectorSet base = gen(2, n), train = gen(1, nt), queries = gen(3, nq);
    TrainParams tp;
    tp.iterations = 5;
    tp.seed = 3;
    auto [coarse, pq] = ivf_train(train, c, m, ks, tp);
    std::vector<float> oc(c * d), ob(ks * d);
    orc_ivf_train(train.data.data(), nt, d, c, m, ks, 5, 3, oc.data(), ob.data());
    EXPECT(same_bits(coarse.centroids.data(), oc.data(), oc.size()), "ivf_train coarse");
    std::vector<float> books;
    for (auto& b : pq.books) books.insert(books.end(), b.centroids.begin(), b.centroids.end());
    EXPECT(same_bits(books.data(), ob.data(), ob.size()), "ivf_train pq");
    RefineQuantizer rq = ivf_refine_train(coarse, pq, train, mp, tp);
    std::vector<float> orb(ks * d), rb;
    orc_ivf_refine_train(oc.data(), c, ob.data(), d, m, ks, train.data.data(), nt, mp, 5, 3, orb.data());
    for (auto& b : rq.pq.books) rb.insert(rb.end(), b.centroids.begin(), b.centroids.end());
    EXPECT(same_bits(rb.data(), orb.data(), orb.size()), "ivf_refine_train");

    IvfIndex ix = ivf_build(coarse, pq, base);
    orc_ivf* ox = orc_ivf_build(oc.data(), c, ob.data(), d, m, ks, base.data.data(), n);
    for (uint32_t l = 0; l < c; ++l) {
        size_t len = orc_ivf_list_size(ox, l);
        std::vector<uint32_t> ids(len);
        std::vector<uint8_t> cds(len * m);
        orc_ivf_list_get(ox, l, ids.data(), cds.data());
        EXPECT(ix.lists[l].ids == ids && ix.lists[l].codes == cds, "ivf_build lists");
    }
    RefineCodes rc = ivf_refine_encode(ix, rq, base);
    std::vector<uint8_t> orc(n * mp);
    orc_ivf_refine_encode(ox, orb.data(), mp, base.data.data(), n, orc.data());
    EXPECT(rc.bytes == orc, "ivf_refine_encode");

    IvfSearchParams prm;
    prm.v = 6;
    prm.kprime = 300;
    auto res = ivf_search_batch(ix, queries, prm);
    std::vector<uint32_t> oi(nq * prm.kprime), ocnt(nq);
    std::vector<float> od(nq * prm.kprime);
    orc_ivf_search_batch(ox, queries.data.data(), nq, prm.v, prm.kprime, oi.data(), od.data(), ocnt.data());
    for (size_t q = 0; q < nq; ++q) {
        bool ok = res[q].size() == ocnt[q];
        for (size_t i = 0; ok && i < res[q].size(); ++i)
            ok = res[q][i].id == oi[q * prm.kprime + i] &&
                 std::memcmp(&res[q][i].dist, &od[q * prm.kprime + i], 4) == 0;
        EXPECT(ok, "ivf_search_batch");
        SearchResult one = ivf_search(ix, queries.vec(q), prm);
        EXPECT(one.size() == res[q].size() && one[0].id == res[q][0].id, "ivf_search == batch");
        SearchResult rr = ivf_rerank(queries.vec(q), res[q], ix, rq, rc, 20);
        std::vector<uint32_t> ri(20);
        std::vector<float> rd(20);
        orc_ivf_rerank_batch(ox, queries.row(q), 1, &oi[q * prm.kprime], &ocnt[q], prm.kprime, 20,
                             ri.data(), rd.data());
        bool ok2 = rr.size() == 20;
        for (size_t i = 0; ok2 && i < 20; ++i)
            ok2 = rr[i].id == ri[i] && std::memcmp(&rr[i].dist, &rd[i], 4) == 0;
        EXPECT(ok2, "ivf_rerank");
    }
    std::vector<float> yo(d);
    for (uint32_t id : {0u, 17u, 5999u}) {
        auto yh = ivf_reconstruct(ix, rq, id, rc);
        orc_ivf_reconstruct(ox, id, yo.data());
        EXPECT(same_bits(yh.data(), yo.data(), d), "ivf_reconstruct");
    }
    bool threw = false;
    try {
        ivf_rerank(queries.vec(0), SearchResult{}, ix, rq, rc, 5);
    } catch (const std::invalid_argument& e) {
        threw = std::strcmp(e.what(), "shortlist too small") == 0;
    }
    EXPECT(threw, "shortlist too small");

    // device-index cache: a different index in the SAME list storage (what a
    // new IvfIndex at a freed address looks like) must not reuse the cached
    // device index of the old one
    {
        std::vector<uint8_t> u(n * d);
        orc_synth_rows(8, 2, 0, n, d, centers.data(), 64, u.data());
        VectorSet base2(d, n);
        for (size_t i = 0; i < u.size(); ++i) base2.data[i] = float(u[i]);
        IvfIndex ix2 = ivf_build(coarse, pq, base2);
        const void* storage = ix.lists.data();
        for (uint32_t l = 0; l < c; ++l) ix.lists[l] = ix2.lists[l];
        ix.list_of_id = ix2.list_of_id;
        ix.pos_of_id = ix2.pos_of_id;
        EXPECT(ix.lists.data() == storage, "same list storage");
        orc_ivf* ox2 = orc_ivf_build(oc.data(), c, ob.data(), d, m, ks, base2.data.data(), n);
        auto res2 = ivf_search_batch(ix, queries, prm);
        orc_ivf_search_batch(ox2, queries.data.data(), nq, prm.v, prm.kprime, oi.data(), od.data(),
                             ocnt.data());
        bool ok = true;
        for (size_t q = 0; q < nq; ++q) {
            ok = ok && res2[q].size() == ocnt[q];
            for (size_t i = 0; ok && i < res2[q].size(); ++i)
                ok = res2[q][i].id == oi[q * prm.kprime + i] &&
                     std::memcmp(&res2[q][i].dist, &od[q * prm.kprime + i], 4) == 0;
        }
        EXPECT(ok, "cache: index replaced in the same storage");
        orc_ivf_free(ox2);
        b200::release_device_indexes();
    }

    // multi-GPU group API (C ABI, one process): 2 and 3 id-range shards on
    // device 0 (device-copy all-gathers), exact mode == one index bit for bit
    {
        std::vector<uint8_t> qu(nq * d);
        for (size_t i = 0; i < qu.size(); ++i) qu[i] = uint8_t(queries.data[i]);
        const uint32_t kp = 300, kk = 20;
        std::vector<uint32_t> oi(nq * kp), ocnt(nq), ri(nq * kk);
        std::vector<float> od(nq * kp), rd(nq * kk);
        orc_ivf_search_batch(ox, queries.data.data(), nq, 6, kp, oi.data(), od.data(), ocnt.data());
        orc_ivf_rerank_batch(ox, queries.data.data(), nq, oi.data(), ocnt.data(), kp, kk, ri.data(), rd.data());
        for (uint32_t G : {2u, 3u}) {
            std::vector<pqrr_dev_index*> sh(G);
            for (uint32_t r = 0; r < G; ++r) {
                const size_t lo = n * r / G, hi = n * (r + 1) / G;
                pqrr_dev_index_create(0, d, c, oc.data(), m, ob.data(), mp, orb.data(), ks, &sh[r]);
                pqrr_dev_add_f32(sh[r], base.row(lo), hi - lo, uint32_t(lo));
            }
            pqrr_dev_group* grp = nullptr;
            EXPECT(pqrr_dev_group_create(G, sh.data(), &grp) == PQRR_OK, "group_create");
            std::vector<uint32_t> gi(nq * kk), gc(nq);
            std::vector<float> gd(nq * kk);
            const int grc = pqrr_dev_group_search_u8(grp, qu.data(), nq, 6, kp, kk, PQRR_GROUP_EXACT, gi.data(),
                                                     gd.data(), gc.data());
            if (grc != PQRR_OK) std::fprintf(stderr, "group_search(G=%u): %s\n", G, pqrr_dev_last_error());
            EXPECT(grc == PQRR_OK, "group_search");
            EXPECT(gi == ri && std::memcmp(gd.data(), rd.data(), rd.size() * 4) == 0, "group exact == one index");
            pqrr_dev_group_destroy(grp);
            for (auto h : sh) pqrr_dev_index_destroy(h);
        }
    }

    // kernel seam: scan_topk against the serial oracle
    std::mt19937 g(5);
    LookupTable lut;
    lut.m = m;
    lut.ks = ks;
    lut.values.resize(m * ks);
    for (auto& v : lut.values) v = float(g() % 1000);
    std::vector<uint8_t> codes(20000 * m);
    for (auto& b : codes) b = uint8_t(g());
    SearchResult st = kernels::scan_topk(lut, codes.data(), 20000, 100, 3);
    std::vector<uint32_t> si(100);
    std::vector<float> sd(100);
    orc_scan_topk(lut.values.data(), m, ks, codes.data(), 20000, 100, 3, si.data(), sd.data());
    bool ok3 = st.size() == 100;
    for (size_t i = 0; ok3 && i < 100; ++i) ok3 = st[i].id == si[i] && st[i].dist == sd[i];
    EXPECT(ok3, "kernels::scan_topk");
    orc_ivf_free(ox);
    if (failures) {
        std::printf("SHIM FAILED %d/%d\n", failures, checks);
        return 1;
    }
    std::printf("SHIM OK %d\n", checks);
    return 0;
}
