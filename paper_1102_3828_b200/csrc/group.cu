// group.cu — multi-GPU search in ONE process:
// pqrr_dev_group_create / pqrr_dev_group_search_u8 / pqrr_dev_group_destroy.
//
// The database is sharded by id range (each shard an index handle on its own
// device holding all coarse cells over its ids).  Queries are broadcast; each
// shard searches locally; per merge ONE all-gather of every shard's packed
// rows [ids | dists | counts] (pqrr_dev_merge_packed_device) feeds the K7
// merge under (dist, id) (types.hpp:47-50) — the partition-invariant merge of
// kernels.cpp:70-95.
//   exact mode (default): each shard's IVFADC top-k' -> all-gather -> global
//     top-k' on every device -> each shard re-ranks the global-shortlist
//     entries it holds -> all-gather -> top-k: bit-identical to one index
//     (ivf_search_batch + ivf_rerank, ivf_index.hpp:58-64,79-81);
//   local mode: each shard's fused search to top-k -> all-gather -> top-k.
// With every shard on its own device the all-gathers are NCCL collectives
// (ncclCommInitAll over the group's devices, one ncclAllGather per rank inside
// ncclGroupStart / ncclGroupEnd).  NCCL is loaded on first use with dlopen, so
// the library has no link-time NCCL dependency (and a process that already
// loaded torch's NCCL shares that copy).  Shards that share a device (the
// one-GPU parity test of the sharded flow) gather with device copies instead.
// Written against the public C ABI only, like storage.cu.
#include <dlfcn.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pqrr_dev.h"
#include "internal.h"

namespace pqrr_b200 {

struct ShortlistGroupError : std::runtime_error {
    ShortlistGroupError() : std::runtime_error("shortlist too small") {}
};

namespace {

// ---- the slice of the NCCL API the group uses (nccl.h, resolved at run time)
typedef struct ncclComm* ncclComm_t;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclInt32 = 2 } ncclDataType_t;
struct Nccl {
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL not found: ") + dlerror();
            return;
        }
        n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(dlsym(h, "ncclAllGather"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(h, "ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!n.CommInitAll || !n.AllGather || !n.GroupStart || !n.GroupEnd)
        throw CudaError(err.empty() ? "NCCL symbols missing" : err);
    return n;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw CudaError(std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error"));
}

void ck(int rc) {
    if (rc == PQRR_ESHORTLIST) throw ShortlistGroupError();
    if (rc != PQRR_OK) throw std::runtime_error(pqrr_dev_last_error());
}

struct DevBuf {
    int dev = 0;
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(int d, size_t b) {
        if (p && bytes >= b) return;
        release();
        dev = d;
        int cur;
        PQRR_CUDA(cudaGetDevice(&cur));
        PQRR_CUDA(cudaSetDevice(d));
        PQRR_CUDA(cudaMalloc(&p, b));
        PQRR_CUDA(cudaSetDevice(cur));
        bytes = b;
    }
    void release() {
        if (p) {
            int cur;
            cudaGetDevice(&cur);
            cudaSetDevice(dev);
            cudaFree(p);
            cudaSetDevice(cur);
        }
        p = nullptr;
        bytes = 0;
    }
    ~DevBuf() { release(); }
    template <class T>
    T* as(size_t off_bytes = 0) const {
        return reinterpret_cast<T*>(static_cast<char*>(p) + off_bytes);
    }
};

struct Shard {
    pqrr_dev_index* ix = nullptr;
    int dev = 0;
    cudaStream_t s = nullptr;
    DevBuf q, own, all, sl, out;  // queries, packed rows, gathered rows, merged shortlist, final rows
};

}  // namespace
}  // namespace pqrr_b200

using namespace pqrr_b200;

struct pqrr_dev_group {
    std::vector<Shard> sh;
    bool use_nccl = false;
    std::vector<ncclComm_t> comms;
    std::mutex mu;
};

namespace pqrr_b200 {
namespace {

// Every device's [G x packed] buffer receives every shard's packed rows.
void all_gather(pqrr_dev_group& g, size_t words, bool stage2) {
    const size_t bytes = words * 4;
    const size_t G = g.sh.size();
    if (g.use_nccl) {
        const Nccl& n = nccl();
        nck(n.GroupStart(), "ncclGroupStart");
        for (size_t r = 0; r < G; ++r) {
            Shard& s = g.sh[r];
            PQRR_CUDA(cudaSetDevice(s.dev));
            nck(n.AllGather(s.own.p, s.all.p, words, ncclInt32, g.comms[r], s.s), "ncclAllGather");
        }
        nck(n.GroupEnd(), "ncclGroupEnd");
        return;
    }
    // shards sharing devices: copy every shard's rows into every gather buffer
    // (only the first shard's buffer is read after the final merge)
    std::vector<cudaEvent_t> done(G);
    for (size_t r = 0; r < G; ++r) {
        PQRR_CUDA(cudaSetDevice(g.sh[r].dev));
        PQRR_CUDA(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
        PQRR_CUDA(cudaEventRecord(done[r], g.sh[r].s));
    }
    const size_t targets = stage2 ? 1 : G;
    for (size_t t = 0; t < targets; ++t) {
        Shard& dst = g.sh[t];
        PQRR_CUDA(cudaSetDevice(dst.dev));
        for (size_t r = 0; r < G; ++r) {
            PQRR_CUDA(cudaStreamWaitEvent(dst.s, done[r], 0));
            PQRR_CUDA(cudaMemcpyPeerAsync(dst.all.as<char>(r * bytes), dst.dev, g.sh[r].own.p, g.sh[r].dev, bytes,
                                          dst.s));
        }
    }
    // the sources' next writes into their own rows wait for these copies
    std::vector<cudaEvent_t> copied(targets);
    for (size_t t = 0; t < targets; ++t) {
        PQRR_CUDA(cudaSetDevice(g.sh[t].dev));
        PQRR_CUDA(cudaEventCreateWithFlags(&copied[t], cudaEventDisableTiming));
        PQRR_CUDA(cudaEventRecord(copied[t], g.sh[t].s));
    }
    for (size_t r = 0; r < G; ++r) {
        PQRR_CUDA(cudaSetDevice(g.sh[r].dev));
        for (size_t t = 0; t < targets; ++t) PQRR_CUDA(cudaStreamWaitEvent(g.sh[r].s, copied[t], 0));
    }
    for (auto e : done) cudaEventDestroy(e);
    for (auto e : copied) cudaEventDestroy(e);
}

template <class F>
void each_shard(pqrr_dev_group& g, F&& f) {
    // one host thread per shard: a shard's search synchronises its own stream
    std::vector<std::thread> th;
    std::vector<std::string> err(g.sh.size());
    std::vector<int> shortlist(g.sh.size(), 0);
    for (size_t r = 0; r < g.sh.size(); ++r)
        th.emplace_back([&, r] {
            try {
                PQRR_CUDA(cudaSetDevice(g.sh[r].dev));
                f(r, g.sh[r]);
            } catch (const ShortlistGroupError&) {
                shortlist[r] = 1;
            } catch (const std::exception& e) {
                err[r] = e.what();
            }
        });
    for (auto& t : th) t.join();
    for (size_t r = 0; r < g.sh.size(); ++r)
        if (!err[r].empty()) throw std::runtime_error("shard " + std::to_string(r) + ": " + err[r]);
    for (int v : shortlist)
        if (v) throw ShortlistGroupError();
}

int status(const std::function<void()>& f) {
    try {
        f();
        return PQRR_OK;
    } catch (const ShortlistGroupError& e) {
        return report_error(PQRR_ESHORTLIST, e.what());
    } catch (const ArgError& e) {
        return report_error(PQRR_EINVAL, e.what());
    } catch (const CudaError& e) {
        return report_error(PQRR_ECUDA, e.what());
    } catch (const std::exception& e) {
        return report_error(PQRR_EINTERNAL, e.what());
    }
}

}  // namespace
}  // namespace pqrr_b200

extern "C" {

int pqrr_dev_group_create(uint32_t G, pqrr_dev_index* const* shards, pqrr_dev_group** out) {
    *out = nullptr;
    return status([&] {
        if (G == 0) throw ArgError("a group needs at least one shard");
        auto g = std::make_unique<pqrr_dev_group>();
        g->sh.resize(G);
        std::vector<int> devs(G);
        pqrr_dev_index_info i0{};
        for (uint32_t r = 0; r < G; ++r) {
            Shard& s = g->sh[r];
            s.ix = shards[r];
            ck(pqrr_dev_index_device(s.ix, &s.dev));
            pqrr_dev_index_info in{};
            ck(pqrr_dev_index_get_info(s.ix, &in));
            if (r == 0) i0 = in;
            if (in.d != i0.d || in.c != i0.c || in.m != i0.m || in.mprime != i0.mprime || in.ks != i0.ks)
                throw ArgError("group shards must share d, c, m, mprime and ks");
            devs[r] = s.dev;
            PQRR_CUDA(cudaSetDevice(s.dev));
            PQRR_CUDA(cudaStreamCreateWithFlags(&s.s, cudaStreamNonBlocking));
        }
        bool distinct = true;
        for (uint32_t a = 0; a < G; ++a)
            for (uint32_t b = a + 1; b < G; ++b) distinct = distinct && devs[a] != devs[b];
        g->use_nccl = distinct && G > 1;
        if (g->use_nccl) {
            g->comms.resize(G);
            nck(nccl().CommInitAll(g->comms.data(), (int)G, devs.data()), "ncclCommInitAll");
        }
        *out = g.release();
    });
}

int pqrr_dev_group_search_u8(pqrr_dev_group* g, const uint8_t* queries, size_t nq, uint32_t w, size_t kprime,
                             size_t k, int mode, uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    return status([&] {
        if (mode != PQRR_GROUP_EXACT && mode != PQRR_GROUP_LOCAL) throw ArgError("unknown group mode");
        if (k > kprime) throw ShortlistGroupError();
        if (nq == 0) return;
        std::lock_guard<std::mutex> lk(g->mu);
        const size_t G = g->sh.size();
        pqrr_dev_index_info in{};
        ck(pqrr_dev_index_get_info(g->sh[0].ix, &in));
        const uint32_t d = in.d;
        const bool exact = mode == PQRR_GROUP_EXACT && k > 0;
        const size_t width1 = exact ? kprime : (k ? k : kprime);
        const size_t words1 = 2 * nq * width1 + nq;
        const size_t kw = k ? k : kprime;
        const size_t words2 = 2 * nq * kw + nq;
        // queries broadcast: one H2D per device; every shard's packed rows
        each_shard(*g, [&](size_t, Shard& s) {
            s.q.ensure(s.dev, nq * d);
            s.own.ensure(s.dev, std::max(words1, words2) * 4);
            s.all.ensure(s.dev, G * std::max(words1, words2) * 4);
            PQRR_CUDA(cudaMemcpyAsync(s.q.p, queries, nq * d, cudaMemcpyHostToDevice, s.s));
            uint32_t* base = s.own.as<uint32_t>();
            ck(pqrr_dev_search_u8_device(s.ix, s.q.as<uint8_t>(), nq, w, kprime, exact ? 0 : k, base,
                                         reinterpret_cast<float*>(base + nq * width1), base + 2 * nq * width1,
                                         s.s));
        });
        all_gather(*g, words1, !exact);
        if (exact) {
            // global top-k' on every device, then each shard re-ranks what it holds
            each_shard(*g, [&](size_t, Shard& s) {
                s.sl.ensure(s.dev, (2 * nq * kprime + nq) * 4);
                uint32_t* sl = s.sl.as<uint32_t>();
                ck(pqrr_dev_merge_packed_device(s.dev, s.all.p, nq, (uint32_t)G, (uint32_t)kprime,
                                                (uint32_t)kprime, sl, reinterpret_cast<float*>(sl + nq * kprime),
                                                sl + 2 * nq * kprime, s.s));
                uint32_t* base = s.own.as<uint32_t>();
                ck(pqrr_dev_rerank_owned_u8_device(s.ix, s.q.as<uint8_t>(), nq, sl, sl + 2 * nq * kprime, kprime,
                                                   k, base, reinterpret_cast<float*>(base + nq * k),
                                                   base + 2 * nq * k, s.s));
            });
            all_gather(*g, words2, true);
        }
        Shard& s0 = g->sh[0];
        PQRR_CUDA(cudaSetDevice(s0.dev));
        s0.out.ensure(s0.dev, words2 * 4);
        uint32_t* o = s0.out.as<uint32_t>();
        ck(pqrr_dev_merge_packed_device(s0.dev, s0.all.p, nq, (uint32_t)G, (uint32_t)(exact ? k : width1),
                                        (uint32_t)kw, o, reinterpret_cast<float*>(o + nq * kw), o + 2 * nq * kw,
                                        s0.s));
        PQRR_CUDA(cudaMemcpyAsync(out_ids, o, nq * kw * 4, cudaMemcpyDeviceToHost, s0.s));
        PQRR_CUDA(cudaMemcpyAsync(out_dists, o + nq * kw, nq * kw * 4, cudaMemcpyDeviceToHost, s0.s));
        PQRR_CUDA(cudaMemcpyAsync(out_counts, o + 2 * nq * kw, nq * 4, cudaMemcpyDeviceToHost, s0.s));
        std::vector<uint32_t> slc;
        if (exact) {  // "shortlist too small" exactly when one index would
            slc.resize(nq);
            PQRR_CUDA(cudaMemcpyAsync(slc.data(), s0.sl.as<uint32_t>() + 2 * nq * kprime, nq * 4,
                                      cudaMemcpyDeviceToHost, s0.s));
        }
        PQRR_CUDA(cudaStreamSynchronize(s0.s));
        for (uint32_t c : slc)
            if (c < k) throw ShortlistGroupError();
    });
}

int pqrr_dev_group_size(pqrr_dev_group* g, uint32_t* shards, int* uses_nccl) {
    return status([&] {
        if (shards) *shards = (uint32_t)g->sh.size();
        if (uses_nccl) *uses_nccl = g->use_nccl ? 1 : 0;
    });
}

int pqrr_dev_group_destroy(pqrr_dev_group* g) {
    if (!g) return PQRR_OK;
    return status([&] {
        for (auto c : g->comms)
            if (c && nccl().CommDestroy) nccl().CommDestroy(c);
        for (auto& s : g->sh) {
            if (s.s) {
                cudaSetDevice(s.dev);
                cudaStreamSynchronize(s.s);
                cudaStreamDestroy(s.s);
            }
        }
        delete g;
    });
}

}  // extern "C"
