// pqrr_dev.cu — host orchestration behind the C ABI of include/pqrr_dev.h:
// the device-resident IVF index (ivf_index.hpp:27-41 + refine.hpp:15-28),
// its add path (ivf_build / ivf_refine_encode), and the fused batched search
// (ivf_search_batch + ivf_rerank).  One CUDA stream per index; calls on one
// index are serialised by a mutex (SPEC.md:346 allows concurrent searches —
// they queue on the device in order).
#include <cuda_runtime.h>

#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pqrr_dev.h"
#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {

thread_local std::string g_last_error;

int report_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

struct ShortlistError : std::runtime_error {
    ShortlistError() : std::runtime_error("shortlist too small") {}
};
struct UnsupportedError : std::runtime_error {
    explicit UnsupportedError(const std::string& s) : std::runtime_error(s) {}
};
struct NoDevice : std::runtime_error {
    explicit NoDevice(const std::string& s) : std::runtime_error(s) {}
};

// ------------------------------------------------------------------ helpers
class DeviceGuard {
  public:
    explicit DeviceGuard(int dev) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            throw NoDevice("no CUDA device available (the B200 path has no CPU fallback)");
        }
        if (dev < 0 || dev >= n) throw ArgError("device ordinal out of range");
        PQRR_CUDA(cudaGetDevice(&prev_));
        PQRR_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev_); }

  private:
    int prev_ = 0;
};

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) PQRR_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void swap(DBuf& o) {
        std::swap(p, o.p);
        std::swap(n, o.n);
    }
    size_t bytes() const { return n * sizeof(T); }
};

// Stream-ordered scratch: everything is freed (stream-ordered) at scope exit.
class Workspace {
  public:
    explicit Workspace(cudaStream_t s) : s_(s) {}
    ~Workspace() {
        for (void* p : ptrs_) cudaFreeAsync(p, s_);
    }
    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        PQRR_CUDA(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), s_));
        ptrs_.push_back(p);
        return static_cast<T*>(p);
    }
    template <class T>
    T* zeros(size_t count) {
        T* p = alloc<T>(count);
        PQRR_CUDA(cudaMemsetAsync(p, 0, std::max<size_t>(count, 1) * sizeof(T), s_));
        return p;
    }

  private:
    cudaStream_t s_;
    std::vector<void*> ptrs_;
};

int bits_for(uint32_t n) {
    int b = 1;
    while ((1ull << b) < n) ++b;
    return b;
}

// ------------------------------------------------------------------ small kernels
namespace {

__global__ void iota_base_kernel(uint32_t* out, size_t n, uint32_t base) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = base + (uint32_t)i;
}

// Status word of an enqueue-only search (no host round trip inside the batch):
// a set bit means the batch must be redone on the synchronising path.
constexpr uint32_t kStatusCoarseOverflow = 1u;  // a certified coarse candidate set overflowed
constexpr uint32_t kStatusThreshold = 2u;       // a query's sampled threshold failed its exactness check

// le (optional): per query, how many candidates have an exact distance <= tau
// (the filter path keeps a superset of those in the buffer).
__global__ void check_fail_kernel(const uint8_t* __restrict__ sampled, const uint32_t* __restrict__ cnt,
                                  const uint32_t* __restrict__ le, size_t nq, uint32_t kprime,
                                  uint32_t cap, uint8_t* __restrict__ fail, unsigned* __restrict__ max_n,
                                  unsigned long long* __restrict__ total,
                                  unsigned long long* __restrict__ total_le,
                                  const uint32_t* __restrict__ coarse_ovf, uint32_t* __restrict__ status) {
    size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    // enqueue-only search: the host reads one status word after the batch
    if (status && q == 0 && coarse_ovf && *coarse_ovf) atomicOr(status, kStatusCoarseOverflow);
    atomicMax(max_n, min(cnt[q], cap));
    atomicAdd(total, (unsigned long long)cnt[q]);
    if (le) atomicAdd(total_le, (unsigned long long)le[q]);
    uint8_t f = 0;
    if (cnt[q] > cap) {
        f = 2;  // buffer overflow: candidates were dropped
    } else if (sampled[q]) {
        const uint32_t exact = le ? le[q] : cnt[q];
        if (exact < kprime) f = 1;  // threshold too tight: shortlist may be incomplete
    }
    fail[q] = f;
    if (status && f) atomicOr(status, kStatusThreshold);
}

__global__ void gather_rows_f32(const float* __restrict__ x, uint32_t d, const uint32_t* __restrict__ rows,
                                size_t nr, float* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr * d) return;
    out[i] = x[(size_t)rows[i / d] * d + i % d];
}

__global__ void scatter_shortlist(const u64* __restrict__ skey, const uint32_t* __restrict__ spos,
                                  const uint32_t* __restrict__ scnt, const uint32_t* __restrict__ rows,
                                  size_t nr, uint32_t kprime, u64* __restrict__ key,
                                  uint32_t* __restrict__ pos, uint32_t* __restrict__ cnt) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr * kprime) return;
    size_t r = i / kprime, j = i % kprime;
    size_t q = rows[r];
    key[q * kprime + j] = skey[i];
    pos[q * kprime + j] = spos[i];
    if (j == 0) cnt[q] = scnt[r];
}

// flag[0]: some row holds fewer than k entries ("shortlist too small");
// flag[2..3]: the total shortlist entries (u64), the re-ranker's candidates
__global__ void min_count_kernel(const uint32_t* __restrict__ cnt, size_t nq, uint32_t k,
                                 unsigned* __restrict__ flag) {
    size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < nq && cnt[q] < k) atomicOr(flag, 1u);
    const unsigned long long c = q < nq ? cnt[q] : 0ull;
    unsigned long long v = c;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(reinterpret_cast<unsigned long long*>(flag + 2), v);
}

// code_of_id (ivf_index.hpp:33-40) + RefineCodes::code (refine.hpp:27): per id
// its list, first-stage code and refinement code (list = UINT32_MAX if absent)
__global__ void lookup_ids_kernel(const uint32_t* __restrict__ ids, size_t n, uint32_t id_lo,
                                  uint32_t map_n, const uint32_t* __restrict__ map,
                                  const uint64_t* __restrict__ off, uint32_t nlists,
                                  const uint8_t* __restrict__ codes, uint32_t m,
                                  const uint8_t* __restrict__ rcodes, uint32_t mprime,
                                  uint32_t* __restrict__ o_list, uint8_t* __restrict__ o_codes,
                                  uint8_t* __restrict__ o_rcodes) {
    const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint32_t id = ids[v];
    const uint32_t p = (id >= id_lo && id - id_lo < map_n) ? map[id - id_lo] : 0xffffffffu;
    if (p == 0xffffffffu) {
        if (o_list) o_list[v] = 0xffffffffu;
        if (o_codes) for (uint32_t j = 0; j < m; ++j) o_codes[v * m + j] = 0;
        if (o_rcodes) for (uint32_t j = 0; j < mprime; ++j) o_rcodes[v * mprime + j] = 0;
        return;
    }
    uint32_t lo = 0, hi = nlists;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (off[mid] <= p) lo = mid;
        else hi = mid;
    }
    if (o_list) o_list[v] = lo;
    if (o_codes) for (uint32_t j = 0; j < m; ++j) o_codes[v * m + j] = codes[(size_t)p * m + j];
    if (o_rcodes) for (uint32_t j = 0; j < mprime; ++j) o_rcodes[v * mprime + j] = rcodes[(size_t)p * mprime + j];
}

__global__ void id_to_pos_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                 const uint32_t* __restrict__ ids, uint32_t id_lo,
                                 uint32_t* __restrict__ map) {
    const uint32_t l = blockIdx.x;
    const uint64_t o = off[l];
    for (uint32_t r = threadIdx.x; r < len[l]; r += blockDim.x) map[ids[o + r] - id_lo] = (uint32_t)(o + r);
}

__global__ void ids_to_shortlist(const uint32_t* __restrict__ sl_ids, const uint32_t* __restrict__ map,
                                 size_t total, u64* __restrict__ key, uint32_t* __restrict__ pos,
                                 unsigned* __restrict__ bad, uint32_t id_lo, uint32_t nmap) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const uint32_t id = sl_ids[i];
    uint32_t p = 0xffffffffu;
    if (id >= id_lo && id - id_lo < nmap) p = map[id - id_lo];
    if (p == 0xffffffffu) {
        atomicOr(bad, 1u);
        p = 0;
    }
    key[i] = (u64)id;
    pos[i] = p;
}

// Exact multi-shard mode: keep, per query row of a GLOBAL shortlist, the ids
// this shard holds (id map hit), compacted in row order; one warp per query.
__global__ void owned_shortlist_kernel(const uint32_t* __restrict__ sl_ids,
                                       const uint32_t* __restrict__ sl_cnt, size_t nq, uint32_t stride,
                                       const uint32_t* __restrict__ map, uint32_t id_lo, uint32_t nmap,
                                       u64* __restrict__ key, uint32_t* __restrict__ pos,
                                       uint32_t* __restrict__ cnt) {
    const size_t q = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (q >= nq) return;
    const uint32_t n = sl_cnt[q];
    uint32_t o = 0;
    for (uint32_t b = 0; b < n; b += 32) {
        const uint32_t i = b + lane;
        uint32_t p = 0xffffffffu, id = 0;
        if (i < n) {
            id = sl_ids[q * stride + i];
            if (id >= id_lo && id - id_lo < nmap) p = map[id - id_lo];
        }
        const bool own = p != 0xffffffffu;
        const unsigned bal = __ballot_sync(0xffffffffu, own);
        if (own) {
            const uint32_t j = o + __popc(bal & ((1u << lane) - 1u));
            key[q * stride + j] = (u64)id;
            pos[q * stride + j] = p;
        }
        o += __popc(bal);
    }
    if (lane == 0) cnt[q] = o;
}

// refine.hpp:42-45: yhat = decode_c(code) + decode_r(rcode) (ADC+R estimate).
__global__ void reconstruct_codes_kernel(const uint8_t* __restrict__ codes,
                                         const uint8_t* __restrict__ rcodes, size_t n, uint32_t d,
                                         const float* __restrict__ books, uint32_t m,
                                         const float* __restrict__ rbooks, uint32_t mprime,
                                         uint32_t ks, float* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * d) return;
    const size_t v = i / d;
    const uint32_t t = (uint32_t)(i % d);
    const uint32_t ds = d / m, j = t / ds, dsr = d / mprime, jr = t / dsr;
    const float p = books[((size_t)j * ks + codes[v * m + j]) * ds + (t - j * ds)];
    const float r = rbooks[((size_t)jr * ks + rcodes[v * mprime + jr]) * dsr + (t - jr * dsr)];
    out[i] = __fadd_rn(p, r);
}

// refine.hpp:30-31: r = y - decode(code), code = encode(y).
__global__ void pq_residual_kernel(const float* __restrict__ y, const uint8_t* __restrict__ codes,
                                   size_t n, uint32_t d, const float* __restrict__ books, uint32_t m,
                                   uint32_t ks, float* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * d) return;
    const size_t v = i / d;
    const uint32_t t = (uint32_t)(i % d);
    const uint32_t ds = d / m, j = t / ds;
    out[i] = __fsub_rn(y[i], books[((size_t)j * ks + codes[v * m + j]) * ds + (t - j * ds)]);
}

__global__ void reconstruct_kernel(const uint32_t* __restrict__ ids, size_t n, uint32_t id_lo,
                                   const uint32_t* __restrict__ map,
                                   const uint64_t* __restrict__ off, uint32_t nlists, uint32_t d,
                                   const float* __restrict__ coarse, const uint8_t* __restrict__ codes,
                                   const float* __restrict__ books, uint32_t m,
                                   const uint8_t* __restrict__ rcodes, const float* __restrict__ rbooks,
                                   uint32_t mprime, uint32_t ks, float* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * d) return;
    const size_t v = i / d;
    const uint32_t t = (uint32_t)(i % d);
    const uint32_t p = map[ids[v] - id_lo];
    if (p == 0xffffffffu) {
        out[i] = __int_as_float(0x7fc00000);  // id never added
        return;
    }
    uint32_t lo = 0, hi = nlists;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (off[mid] <= p) lo = mid;
        else hi = mid;
    }
    const uint32_t ds = d / m, jj = t / ds;
    float y = __fadd_rn(coarse[(size_t)lo * d + t],
                        books[((size_t)jj * ks + codes[(size_t)p * m + jj]) * ds + (t - jj * ds)]);
    if (mprime) {
        const uint32_t dsr = d / mprime, jr = t / dsr;
        y = __fadd_rn(y, rbooks[((size_t)jr * ks + rcodes[(size_t)p * mprime + jr]) * dsr + (t - jr * dsr)]);
    }
    out[i] = y;
}

__global__ void compact_lists_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                     const uint64_t* __restrict__ uoff, const uint32_t* __restrict__ ids,
                                     const uint8_t* __restrict__ codes, const uint8_t* __restrict__ rcodes,
                                     uint32_t m, uint32_t mprime, uint32_t* __restrict__ o_ids,
                                     uint8_t* __restrict__ o_codes, uint8_t* __restrict__ o_rcodes) {
    const uint32_t l = blockIdx.x;
    const uint64_t o = off[l], u = uoff[l];
    for (uint32_t r = threadIdx.x; r < len[l]; r += blockDim.x) {
        o_ids[u + r] = ids[o + r];
        for (uint32_t j = 0; j < m; ++j) o_codes[(u + r) * m + j] = codes[(o + r) * m + j];
        for (uint32_t j = 0; j < mprime; ++j) o_rcodes[(u + r) * mprime + j] = rcodes[(o + r) * mprime + j];
    }
}

__global__ void lut_keys_kernel(const float* __restrict__ dist, size_t n, uint32_t id_base,
                                u64* __restrict__ keys) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = nb_key(dist[i], id_base + (uint32_t)i);
}

inline unsigned nblk(size_t n, unsigned t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

// ------------------------------------------------------------------ index
struct DevIndex {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    uint32_t d = 0, c = 0, m = 0, mprime = 0, ks = 0;
    DBuf<float> coarse, books, rbooks;
    // list-major layout
    uint64_t n = 0, slots = 0;
    DBuf<uint64_t> list_off;
    DBuf<uint32_t> list_len;
    std::vector<uint64_t> h_off;
    std::vector<uint32_t> h_len;
    std::vector<uint32_t> h_len_desc;  // list lengths, longest first (bounds of the enqueue-only search)
    uint64_t h_len_desc_n = ~0ull;
    DBuf<uint8_t> codes, rcodes;
    DBuf<uint32_t> ids;
    DBuf<uint16_t> block_list;  // list of each 16-entry block of positions
    DBuf<float> cnorm;          // |C_l|^2 (tensor-core K1), cnorm_max their maximum
    float cnorm_max = 0.f;
    AssignTc atc;               // tcgen05 coarse distances (add path; u8 queries)
    bool q_u8 = false;          // the search in flight has u8-valued queries
    bool keys_need_ids = true;  // the shortlist keys must carry ids (see search_device)
    DBuf<uint8_t> q8_cache;     // per LUT-pass item 8-bit LUT (32 KiB) for the K4f filter
    DBuf<float> q8_param;       // per LUT-pass item and query lane: (scale, sum of minima)
    uint64_t next_id = 0;
    uint64_t id_lo = ~0ull;  // smallest id held (id-range shards start above 0)
    // id -> position (lazy)
    DBuf<uint32_t> id_map;
    bool id_map_valid = false;
    // staging (id order)
    uint64_t st_n = 0, st_cap = 0;
    DBuf<uint32_t> st_assign, st_ids;
    DBuf<uint8_t> st_codes, st_rcodes;
    pqrr_dev_search_stats stats{};
    cudaEvent_t ev[13] = {};
    // enqueue-only search: cached graphs, the device status block
    // ([0..3] min_count flag, [4] status bits) and its pinned host copy,
    // staging buffers with stable addresses for the host-buffer API
    struct SearchGraph {
        const void* xq = nullptr;
        size_t nq = 0, kprime = 0, k = 0;
        uint32_t w = 0;
        const void *oi = nullptr, *od = nullptr, *oc = nullptr;
        const void* h_in = nullptr;  // host-staged variant (copies inside the graph)
        bool q_u8 = false;
        uint64_t sig = 0;
        cudaGraphExec_t exec = nullptr;
        uint32_t kernels = 0;
        uint64_t used = 0;
        double bytes = 0;  // scratch its memory nodes reserve (bounds)
    };
    std::vector<SearchGraph> graphs;
    uint64_t graph_clock = 0;
    bool graph_enabled = true;  // pqrr_dev_index_set_graph
    DBuf<uint32_t> d_stat;
    uint32_t* h_stat = nullptr;
    DBuf<uint8_t> sg_qu8;
    DBuf<float> sg_xq;
    DBuf<uint32_t> sg_out;  // [ids | dists | counts] of the host-buffer API
    // pinned host staging of small batches: the graph copies queries in and
    // results out itself, the API call only memcpy's on the CPU
    void* h_in = nullptr;
    void* h_out = nullptr;
    size_t h_in_bytes = 0, h_out_bytes = 0;
    cudaEvent_t ev_fast[2] = {};
    // the enqueued search pqrr_dev_search_finish completes
    struct Pending {
        bool on = false;
        const uint8_t* d_queries = nullptr;
        size_t nq = 0, kprime = 0, k = 0;
        uint32_t w = 0;
        uint32_t* oi = nullptr;
        float* od = nullptr;
        uint32_t* oc = nullptr;
        cudaStream_t user = nullptr;
    } pending;

    void drop_graphs() {
        for (auto& g : graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        if (!graphs.empty()) cudaDeviceGraphMemTrim(device);
        graphs.clear();
    }

    ~DevIndex() {
        drop_graphs();
        if (h_stat) cudaFreeHost(h_stat);
        if (h_in) cudaFreeHost(h_in);
        if (h_out) cudaFreeHost(h_out);
        for (auto& e : ev_fast)
            if (e) cudaEventDestroy(e);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }
    uint32_t max_len() const {
        uint32_t mx = 0;
        for (uint32_t v : h_len) mx = std::max(mx, v);
        return mx;
    }
};

namespace {

void check_shape(uint32_t d, uint32_t m, uint32_t ks) {
    if (d == 0) throw ArgError("d must be positive");
    if (m == 0 || d % m != 0) throw ArgError("dimension not divisible");
    if (ks == 0 || ks > 256) throw ArgError("ks must be in [1, 256]");
}

void grow_staging(DevIndex& ix, uint64_t need) {
    if (need <= ix.st_cap) return;
    uint64_t cap = std::max<uint64_t>(need, ix.st_cap * 2);
    DBuf<uint32_t> a, i;
    DBuf<uint8_t> c, r;
    a.alloc(cap);
    i.alloc(cap);
    c.alloc(cap * ix.m);
    if (ix.mprime) r.alloc(cap * ix.mprime);
    if (ix.st_n) {
        PQRR_CUDA(cudaMemcpyAsync(a.p, ix.st_assign.p, ix.st_n * 4, cudaMemcpyDeviceToDevice, ix.stream));
        PQRR_CUDA(cudaMemcpyAsync(i.p, ix.st_ids.p, ix.st_n * 4, cudaMemcpyDeviceToDevice, ix.stream));
        PQRR_CUDA(cudaMemcpyAsync(c.p, ix.st_codes.p, ix.st_n * ix.m, cudaMemcpyDeviceToDevice, ix.stream));
        if (ix.mprime)
            PQRR_CUDA(cudaMemcpyAsync(r.p, ix.st_rcodes.p, ix.st_n * ix.mprime, cudaMemcpyDeviceToDevice,
                                      ix.stream));
        PQRR_CUDA(cudaStreamSynchronize(ix.stream));
    }
    ix.st_assign.swap(a);
    ix.st_ids.swap(i);
    ix.st_codes.swap(c);
    ix.st_rcodes.swap(r);
    ix.st_cap = cap;
}

// Encode a device-resident chunk (f32 or u8) into the staging arrays.
void stage_chunk(DevIndex& ix, const float* xf, const uint8_t* xu, size_t n, uint32_t id_base) {
    if (n == 0) return;
    if ((uint64_t)id_base < ix.next_id)
        throw ArgError("ids must be added in ascending order (id_base below the next free id)");
    if ((uint64_t)id_base + n > 0xffffffffull) throw ArgError("ids exceed the 32-bit id space");
    cudaStream_t s = ix.stream;
    grow_staging(ix, ix.st_n + n);
    Workspace ws(s);
    const float* x = xf;
    if (!x) {
        float* tmp = ws.alloc<float>(n * ix.d);
        launch_widen_u8(xu, tmp, n * ix.d, s);
        x = tmp;
    }
    uint32_t* a = ix.st_assign.p + ix.st_n;
    // u8 rows: certified tensor-core assignment (k_assign_tc.cu); float rows
    // (not exact in fp16) keep the exact CUDA-core argmin
    if (xu && assign_tc_supported(ix.d, ix.c) && ix.atc.prepare(ix.coarse.p, ix.c, s))
        ix.atc.assign(xu, n, ix.coarse.p, a, s);
    else
        launch_argmin(x, n, ix.coarse.p, ix.c, ix.d, a, nullptr, s);
    launch_ivf_encode(x, nullptr, n, ix.d, a, ix.coarse.p, ix.books.p, ix.m, ix.rbooks.p, ix.mprime,
                      ix.ks, ix.st_codes.p + ix.st_n * ix.m,
                      ix.mprime ? ix.st_rcodes.p + ix.st_n * ix.mprime : nullptr, s);
    iota_base_kernel<<<nblk(n), 256, 0, s>>>(ix.st_ids.p + ix.st_n, n, id_base);
    PQRR_LAUNCH_CHECK();
    count_launch();
    ix.st_n += n;
    ix.id_lo = std::min<uint64_t>(ix.id_lo, id_base);
    ix.next_id = (uint64_t)id_base + n;
}

void finalize(DevIndex& ix) {
    if (ix.st_n == 0) return;
    cudaStream_t s = ix.stream;
    const uint32_t c = ix.c;
    const size_t n = ix.st_n;
    Workspace ws(s);
    uint32_t* cnt = ws.alloc<uint32_t>(c + 1);
    PQRR_CUDA(cudaMemsetAsync(cnt, 0, (c + 1) * sizeof(uint32_t), s));
    launch_histogram(ix.st_assign.p, n, c, cnt, s);
    uint32_t* stage_off = ws.alloc<uint32_t>(c + 1);
    exclusive_scan_u32(cnt, stage_off, c + 1, s);
    uint32_t* iota = ws.alloc<uint32_t>(n);
    launch_iota(iota, n, s);
    uint32_t* skeys = ws.alloc<uint32_t>(n);
    uint32_t* sidx = ws.alloc<uint32_t>(n);
    sort_pairs(ix.st_assign.p, skeys, iota, sidx, n, bits_for(c), s);
    std::vector<uint32_t> h_cnt(c);
    PQRR_CUDA(cudaMemcpyAsync(h_cnt.data(), cnt, c * 4, cudaMemcpyDeviceToHost, s));
    PQRR_CUDA(cudaStreamSynchronize(s));
    std::vector<uint32_t> old_len = ix.h_len;
    if (old_len.empty()) old_len.assign(c, 0);
    std::vector<uint32_t> new_len(c);
    std::vector<uint64_t> new_off(c + 1);
    uint64_t acc = 0;
    for (uint32_t l = 0; l < c; ++l) {
        new_len[l] = old_len[l] + h_cnt[l];
        new_off[l] = acc;
        acc += (uint64_t(new_len[l]) + 15) & ~uint64_t(15);
    }
    new_off[c] = acc;
    if (acc > 0xffffffffull) throw UnsupportedError("more than 2^32 entries on one device");
    DBuf<uint64_t> d_off;
    DBuf<uint32_t> d_len, d_oldlen;
    d_off.alloc(c + 1);
    d_len.alloc(c);
    d_oldlen.alloc(c);
    PQRR_CUDA(cudaMemcpyAsync(d_off.p, new_off.data(), (c + 1) * 8, cudaMemcpyHostToDevice, s));
    PQRR_CUDA(cudaMemcpyAsync(d_len.p, new_len.data(), c * 4, cudaMemcpyHostToDevice, s));
    PQRR_CUDA(cudaMemcpyAsync(d_oldlen.p, old_len.data(), c * 4, cudaMemcpyHostToDevice, s));
    DBuf<uint8_t> codes, rcodes;
    DBuf<uint32_t> ids;
    codes.alloc(acc * ix.m + 16);
    ids.alloc(acc + 1);
    if (ix.mprime) rcodes.alloc(acc * ix.mprime + 16);
    if (ix.n) {
        uint32_t mx = 0;
        for (uint32_t v : ix.h_len) mx = std::max(mx, v);
        launch_layout_copy_old(ix.list_off.p, ix.list_len.p, c, d_off.p, ix.codes.p, ix.ids.p,
                               ix.rcodes.p, ix.m, ix.mprime, codes.p, ids.p, rcodes.p, mx, s);
    }
    launch_layout_place_new(skeys, sidx, n, stage_off, d_off.p, d_oldlen.p, ix.st_codes.p,
                            ix.st_rcodes.p, ix.st_ids.p, ix.m, ix.mprime, codes.p, ids.p, rcodes.p, s);
    // Staging (and the previous layout) are dead once placed: release them
    // before the pairing copy so a 1B-entry build peaks near 2.5x the index.
    PQRR_CUDA(cudaStreamSynchronize(s));
    ix.st_assign.release();
    ix.st_ids.release();
    ix.st_codes.release();
    ix.st_rcodes.release();
    ix.st_cap = 0;
    ix.codes.release();
    ix.ids.release();
    ix.rcodes.release();
    if (ix.m == 8) {
        // parity-balanced order inside every list (bank-conflict-free LUT gathers)
        std::vector<uint64_t> h_end(c);
        for (uint32_t l = 0; l < c; ++l) h_end[l] = new_off[l] + new_len[l];
        uint64_t* d_end = ws.alloc<uint64_t>(c);
        PQRR_CUDA(cudaMemcpyAsync(d_end, h_end.data(), c * 8, cudaMemcpyHostToDevice, s));
        uint32_t* pk = ws.alloc<uint32_t>(acc);
        uint32_t* pv = ws.alloc<uint32_t>(acc);
        uint32_t* spk = ws.alloc<uint32_t>(acc);
        uint32_t* spv = ws.alloc<uint32_t>(acc);
        uint32_t* perm = ws.alloc<uint32_t>(acc);
        launch_parity_keys(d_off.p, d_len.p, c, codes.p, pk, pv, s);
        segmented_sort_pairs(pk, spk, pv, spv, acc, c, d_off.p, d_end, 8, s);
        launch_pair_perm(d_off.p, d_len.p, c, spk, spv, perm, s);
        DBuf<uint8_t> codes2, rcodes2;
        DBuf<uint32_t> ids2;
        codes2.alloc(acc * ix.m + 16);
        ids2.alloc(acc + 1);
        if (ix.mprime) rcodes2.alloc(acc * ix.mprime + 16);
        launch_gather_layout(d_off.p, d_len.p, c, perm, codes.p, ids.p, rcodes.p, ix.m, ix.mprime,
                             codes2.p, ids2.p, rcodes2.p, s);
        PQRR_CUDA(cudaStreamSynchronize(s));
        codes.swap(codes2);
        ids.swap(ids2);
        rcodes.swap(rcodes2);
    }
    PQRR_CUDA(cudaStreamSynchronize(s));
    ix.codes.swap(codes);
    ix.rcodes.swap(rcodes);
    ix.ids.swap(ids);
    ix.list_off.swap(d_off);
    ix.block_list.alloc(acc / 16 + 1);
    launch_block_list(ix.list_off.p, c, ix.block_list.p, s);
    ix.list_len.swap(d_len);
    ix.h_off = new_off;
    ix.h_len = new_len;
    ix.n += n;
    ix.slots = acc;
    ix.st_n = 0;
    ix.id_map_valid = false;
}


uint64_t id_lo_of(const DevIndex& ix) { return ix.id_lo == ~0ull ? 0 : ix.id_lo; }

void ensure_id_map(DevIndex& ix) {
    finalize(ix);
    if (ix.id_map_valid) return;
    ix.id_map.alloc(std::max<uint64_t>(ix.next_id - id_lo_of(ix), 1));
    PQRR_CUDA(cudaMemsetAsync(ix.id_map.p, 0xff, ix.id_map.bytes(), ix.stream));
    if (ix.c)
        id_to_pos_kernel<<<ix.c, 256, 0, ix.stream>>>(ix.list_off.p, ix.list_len.p, ix.ids.p,
                                                      (uint32_t)id_lo_of(ix), ix.id_map.p);
    PQRR_LAUNCH_CHECK();
    count_launch();
    ix.id_map_valid = true;
}

struct ShortlistDev {
    u64* key;
    uint32_t* pos;
    uint32_t* cnt;
};

// Work items of one pair set (see k_scan.cu): pairs (list, pair id = q*w+r)
// sorted by list, grouped by <= 16 queries, scheduled longest first.
struct ItemSet {
    uint32_t* pair_sorted = nullptr;
    uint32_t* list_cnt = nullptr;
    uint32_t* list_first = nullptr;
    uint32_t* item_off = nullptr;
    uint32_t n_items = 0, c = 0, qt = 0, chunk = 1u << 30;
    uint32_t *item_list = nullptr, *item_start = nullptr, *item_nq = nullptr;
    uint32_t *item_e0 = nullptr, *item_e1 = nullptr, *item_order = nullptr;
    void apply(ScanArgs& a) const {
        a.item_list = item_list;
        a.item_start = item_start;
        a.item_nq = item_nq;
        a.item_e0 = item_e0;
        a.item_e1 = item_e1;
        a.item_order = item_order;
        a.num_items = item_off + c;
        a.pair_sorted = pair_sorted;
    }
};

// Pairs (list, pair id) sorted by list, per-list pair counts / first pair, and
// the per-list item counts + offsets for items of <= qt queries.  `share`
// reuses another set's sorted pairs (same pairs, different qt).
// Sort key of a pair (q, l): (list, coarse-distance gap d(q, l) - d(q, l_0)
// to the query's nearest probe, top 16 bits of its float pattern).  Within a
// list the pairs are ordered by that gap, so the pairs likely to reach the
// query's threshold (small gap) fill the first 16-query blocks and the others
// the last ones: K4f then skips whole dead blocks (ivf_filter_kernel).  The
// order affects only speed (every ranking is by (dist, id)).  D holds the
// coarse distances (approximate on the tensor-core path: fine for a sort).
__global__ void pair_key_kernel(const uint32_t* __restrict__ lists, const uint32_t* __restrict__ pair_ids,
                                size_t np, uint32_t w, const float* __restrict__ D, uint32_t c,
                                const uint32_t* __restrict__ probes, uint32_t* __restrict__ key) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const uint32_t p = pair_ids[i];
    const size_t q = p / w;
    const float gap = fmaxf(__fsub_rn(D[q * c + lists[i]], D[q * c + probes[q * w]]), 0.f);
    // the sampling tier of the probe rank first (a 16-query block then shares
    // one sampling stride in the LUT pass), then the gap (bits 30..19 of a
    // non-negative float: exponent + 4 mantissa bits, monotone): 14 key bits
    // below the list, so Kc = 1024 sorts in 3 radix passes
    const uint32_t tier = sample_tier(p % w, w, 1);
    key[i] = (lists[i] << 14) | (tier << 12) | (__float_as_uint(gap) >> 19);
}

// Two-phase LUT pass: pairs of probe rank r < R1 (near) and r >= R1 (far).
__global__ void split_pairs_kernel(const uint32_t* __restrict__ probes, size_t nq, uint32_t w, uint32_t R1,
                                   uint32_t* __restrict__ near_lists, uint32_t* __restrict__ near_ids,
                                   uint32_t* __restrict__ far_lists, uint32_t* __restrict__ far_ids) {
    const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nq * w) return;
    const size_t q = p / w;
    const uint32_t r = (uint32_t)(p % w);
    if (r < R1) {
        const size_t k = q * R1 + r;
        near_lists[k] = probes[p];
        near_ids[k] = (uint32_t)p;
    } else {
        const size_t k = q * (w - R1) + (r - R1);
        far_lists[k] = probes[p];
        far_ids[k] = (uint32_t)p;
    }
}

ItemSet items_phase1(Workspace& ws, const uint32_t* lists, const uint32_t* pair_ids, size_t np,
                     uint32_t c, const uint32_t* list_len, uint32_t qt, cudaStream_t s,
                     const ItemSet* share = nullptr, uint32_t chunk = 1u << 30, uint32_t w = 1,
                     const float* D = nullptr, const uint32_t* probes = nullptr, bool counts_only = false) {
    ItemSet it;
    it.c = c;
    it.qt = qt;
    it.chunk = chunk;
    if (share) {
        it.pair_sorted = share->pair_sorted;
        it.list_cnt = share->list_cnt;
        it.list_first = share->list_first;
    } else if (counts_only) {  // per-list pair counts / first pair only (two-phase K4f bases)
        it.list_cnt = ws.zeros<uint32_t>(c + 1);
        launch_histogram(lists, np, c, it.list_cnt, s);
        it.list_first = ws.alloc<uint32_t>(c + 1);
        exclusive_scan_u32(it.list_cnt, it.list_first, c + 1, s);
    } else {
        uint32_t* sorted_keys = ws.alloc<uint32_t>(np);
        it.pair_sorted = ws.alloc<uint32_t>(np);
        if (D && bits_for(c) <= 18) {
            uint32_t* key = ws.alloc<uint32_t>(np);
            pair_key_kernel<<<nblk(np), 256, 0, s>>>(lists, pair_ids, np, w, D, c, probes ? probes : lists, key);
            PQRR_LAUNCH_CHECK();
            count_launch();
            sort_pairs(key, sorted_keys, pair_ids, it.pair_sorted, np, 14 + bits_for(c), s);
        } else {
            sort_pairs(lists, sorted_keys, pair_ids, it.pair_sorted, np, bits_for(c), s);
        }
        it.list_cnt = ws.zeros<uint32_t>(c + 1);
        launch_histogram(lists, np, c, it.list_cnt, s);
        it.list_first = ws.alloc<uint32_t>(c + 1);
        exclusive_scan_u32(it.list_cnt, it.list_first, c + 1, s);
    }
    uint32_t* items = ws.alloc<uint32_t>(c + 1);
    launch_items_per_list(it.list_cnt, list_len, c, items, qt, s, chunk);
    it.item_off = ws.alloc<uint32_t>(c + 1);
    exclusive_scan_u32(items, it.item_off, c + 1, s);
    return it;
}

// n_items may be an upper bound (enqueue-only search, `padded`): the slots
// past the real count keep an all-ones sort key, so they sort last and no
// kernel reaches them (every kernel reads the real count from item_off[c]).
// identity_order: items keep their build order (chunked K4f items of a small
// batch are all one chunk long but for list tails: the longest-first sort
// would only cost its launches).
void items_phase2(Workspace& ws, ItemSet& it, uint32_t c, const uint32_t* list_len, cudaStream_t s,
                  bool padded = false, bool identity_order = false) {
    const uint32_t n = it.n_items;
    it.item_list = ws.alloc<uint32_t>(n);
    it.item_start = ws.alloc<uint32_t>(n);
    it.item_nq = ws.alloc<uint32_t>(n);
    it.item_e0 = ws.alloc<uint32_t>(n);
    it.item_e1 = ws.alloc<uint32_t>(n);
    uint32_t* key = ws.alloc<uint32_t>(n);
    uint32_t* key2 = ws.alloc<uint32_t>(n);
    uint32_t* iota = ws.alloc<uint32_t>(n);
    it.item_order = ws.alloc<uint32_t>(n);
    if (padded) PQRR_CUDA(cudaMemsetAsync(key, 0xff, (size_t)std::max<uint32_t>(n, 1) * 4, s));
    launch_items_build(it.list_cnt, it.list_first, list_len, c, it.item_off, it.item_list,
                       it.item_start, it.item_nq, it.item_e0, it.item_e1, key, it.qt, s, it.chunk, n);
    if (identity_order) {
        launch_iota(it.item_order, n, s);
        return;
    }
    launch_iota(iota, n, s);
    sort_pairs(key, key2, iota, it.item_order, n, 32, s);
}

// Threshold target (alpha k' entries) and samples expected below it, tuned
// per regime (tuning hooks PQRR_ALPHA / PQRR_SAMPLES, read per search):
//   k' >= 4096 (C4): 1.5 / 128 — fewer survivors to recheck and select
//     (44.1 -> 40.7 ms at C4);
//   512 <= k' < 4096 and w < 32 (C2): 1.8 / 96 (5.63 -> 5.50 ms, no retries);
//   otherwise 2.0 / 64 (small k' would sample every entry; w >= 32 takes
//     tau from the near probes only).
double default_alpha(uint32_t kprime, uint32_t w) {
    const char* e = getenv("PQRR_ALPHA");
    if (e) return std::max(1.05, atof(e));
    return kprime >= 4096 ? 1.5 : (kprime >= 512 && w < 32 ? 1.8 : 2.0);
}
double default_spq(uint32_t kprime, uint32_t w) {
    const char* e = getenv("PQRR_SAMPLES");
    if (e) return std::max(1.0, atof(e));
    return kprime >= 4096 ? 128.0 : (kprime >= 512 && w < 32 ? 96.0 : 64.0);
}

// ---- enqueue-only search (no host round trip inside the batch) ----
// The synchronising path reads four kinds of counts back before it sizes its
// buffers: work items per item set, threshold samples, the coarse overflow
// flag and the per-query exactness check.  The enqueue-only path replaces the
// counts by host-side upper bounds (from the list lengths the host holds) and
// folds the two flags into one device status word that the caller reads with
// the results; a set bit sends the batch to the synchronising path.  Every
// kernel takes its real counts from device memory, so both paths run the same
// kernels on the same data and return the same bits.
struct FastBounds {
    bool two_phase = false;
    uint32_t R1 = 0, fchunk = 1u << 30;
    uint32_t items_all = 0, items_f64 = 0, items_near = 0, items_far = 0;
    uint64_t samples = 0;
    size_t q8_items = 0;
    double bytes = 0;  // scratch the bounds ask for
};

uint32_t items_bound(size_t np, uint32_t c, uint32_t qt) {
    // sum over lists of ceil(cnt / qt) with sum cnt = np
    const size_t lists = std::min<size_t>(np, c);
    return (uint32_t)std::min<size_t>(np, lists + np / qt);
}

const std::vector<uint32_t>& lens_desc(DevIndex& ix) {
    if (ix.h_len_desc_n != ix.n || ix.h_len_desc.size() != ix.h_len.size()) {
        ix.h_len_desc = ix.h_len;
        std::sort(ix.h_len_desc.begin(), ix.h_len_desc.end(), std::greater<uint32_t>());
        ix.h_len_desc_n = ix.n;
    }
    return ix.h_len_desc;
}

// Builds the exact top-kprime shortlist of every query into `out` (device,
// [nq][kprime]).  alpha scales the sampled threshold rank (expected
// candidates ~ alpha * kprime).
// Lazy state of the tensor-core coarse stage (|C_l|^2 and their maximum, the
// fp16 hi/lo centroid split); synchronises on first use, so the enqueue-only
// path calls it before it starts capturing.
AssignTc* prepare_coarse_tc(DevIndex& ix, uint32_t w) {
    const uint32_t c = ix.c;
    cudaStream_t s = ix.stream;
    if (!(c >= 1024u && coarse_tc_supported(ix.d, w))) return nullptr;
    if (!ix.cnorm.p) {
        ix.cnorm.alloc(c);
        launch_coarse_norms(ix.coarse.p, c, ix.d, ix.cnorm.p, s);
        std::vector<float> h(c);
        PQRR_CUDA(cudaMemcpyAsync(h.data(), ix.cnorm.p, c * sizeof(float), cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaStreamSynchronize(s));
        ix.cnorm_max = *std::max_element(h.begin(), h.end());
    }
    // u8 queries (exact in fp16): D~ on tcgen05 with the add path's
    // centroid split; float queries: mma.sync TF32
    return (ix.q_u8 && assign_tc_supported(ix.d, c) && ix.atc.prepare(ix.coarse.p, c, s)) ? &ix.atc : nullptr;
}

// Shape decisions of one shortlist batch (shared by the synchronising and the
// enqueue-only path).
struct Plan {
    bool filter_ok, coarse_tc, two_phase;
    uint32_t cap, stride, R1, fchunk;
    int tiered;
};

Plan make_plan(const DevIndex& ix, size_t nq, uint32_t w, uint32_t kprime, double alpha,
               uint32_t stride_div, uint32_t cap_shift, bool exact_coarse) {
    Plan pl{};
    const size_t P = nq * (size_t)w;
    // K4f (filter + exact recheck) unless disabled or out of its envelope:
    // m = 8, ks = 256, w*d residuals in shared memory, and an 8-bit LUT cache
    // of 32 KiB per item (index-owned: a per-search allocation of GBs was
    // measured to pay first-touch costs on every batch)
    static const bool exact_env = [] {
        const char* e = getenv("PQRR_SCAN");
        return e && std::string(e) == "exact";
    }();
    pl.filter_ok = !exact_env && ix.m == 8 && ix.ks == 256 && recheck_supported(ix.d, ix.m, w);
    // candidate buffer per query: the sampled threshold targets ~2k' entries;
    // >= 4k' for the exact scan, >= 8k' for the filter's superset; beyond
    // 8192 the selector streams candidates from global memory
    const uint32_t cap_mul = pl.filter_ok ? 8 : 4;
    pl.cap = std::max<uint32_t>(8192, ((cap_mul * kprime + 1023) / 1024) * 1024) << cap_shift;
    // sample density: ~64 samples expected below the alpha*k'-th distance
    // tuning hook (read per search): expected samples below the target rank
    const double spq = default_spq(kprime, w);  // samples expected below the target rank
    uint32_t stride = (uint32_t)std::max(1.0, std::floor(alpha * kprime / spq));
    pl.stride = std::max<uint32_t>(1, stride / std::max<uint32_t>(1, stride_div));
    // (up to 256 queries the exact CUDA-core distances cost a few 64-row tile
    // passes over the centroids and need no certification, while the
    // warp-per-query certify kernel would run on a handful of warps: C5 batch 1
    // coarse stage 0.11 -> 0.03 ms, batch 256 0.11 -> 0.06 ms)
    pl.coarse_tc = !exact_coarse && nq > 256 && ix.c >= 1024u && coarse_tc_supported(ix.d, w);
    // Two-phase LUT pass (w >= 32): the near probes (rank < w/8, the sampling
    // tier 0, where the shortlist lives at C3-C5) get the full LUT pass with
    // sampling, which fixes tau; the far probes get a bound pass (exact LUTs,
    // only their per-lane sum of minima), and a second full pass builds the
    // 8-bit blocks of the far items that have a live lane.  tau comes from
    // the near samples only: a quantile over a subset of the entries, so at
    // least as large as the full one (never under-full; exactness is still
    // checked) and equal to it when the near probes hold the entries below it.
    // far probes are bounded on the tensor cores (k_bound.cu): pays from w = 32
    constexpr uint32_t kTwoPhaseW = 32u, kR1Div = 8u;
    // (large batches only: for a few hundred pairs the extra item sets and
    // launches cost more than the LUT builds they save)
    pl.two_phase = pl.filter_ok && w >= kTwoPhaseW && P >= (size_t)64 * sm_count() &&
                   lut_pass_supported(ix.d, ix.m, ix.ks);
    pl.R1 = pl.two_phase ? (w + kR1Div - 1) / kR1Div : w;
    // small batches (few query-list pairs per SM): K4f items split long lists
    // into chunks so one list does not serialise on one SM
    pl.fchunk = P < (size_t)64 * sm_count() ? 16384u : (1u << 30);
    // importance-weighted sampling needs the warp-specialised LUT pass
    pl.tiered = (w >= 8 && lut_pass_supported(ix.d, ix.m, ix.ks)) ? 1 : 0;
    return pl;
}

FastBounds fast_bounds(DevIndex& ix, const Plan& pl, size_t nq, uint32_t w, uint32_t kprime) {
    FastBounds b;
    const size_t P = nq * (size_t)w;
    const uint32_t c = ix.c;
    b.two_phase = pl.two_phase;
    b.R1 = pl.R1;
    b.fchunk = pl.fchunk;
    const auto& ld = lens_desc(ix);
    const uint32_t max_len = ld.empty() ? 0u : ld[0];
    b.items_all = items_bound(P, c, kQT);
    const uint32_t chunks = std::max<uint32_t>(1, (uint32_t)(((uint64_t)max_len + pl.fchunk - 1) / pl.fchunk));
    b.items_f64 = items_bound(P, c, kFQ) * chunks;
    if (pl.two_phase) {
        b.items_near = items_bound(nq * (size_t)pl.R1, c, kQT);
        b.items_far = items_bound(nq * (size_t)(w - pl.R1), c, kQT);
    }
    // threshold samples of one query: its probes' lists sampled at the stride
    // of their rank tier; the longest lists at the densest tiers bound any probe set
    uint64_t per_q = 0;
    for (uint32_t r = 0; r < pl.R1 && r < ld.size(); ++r) {
        const uint64_t st = (uint64_t)pl.stride << tier_shift(sample_tier(r, w, pl.tiered), w);
        per_q += (ld[r] + st - 1) / st;
    }
    b.samples = per_q * nq;
    b.q8_items = pl.filter_ok ? (size_t)(pl.two_phase ? b.items_near + b.items_far : b.items_all) : 0;
    const double items = (double)b.items_all + b.items_f64 + b.items_near + b.items_far;
    b.bytes = (double)b.samples * 4.0 + (double)b.q8_items * (8.0 * 256 * kQT + kQT * 8.0) + items * 40.0 +
              (double)nq * ((double)pl.cap * 16.0 + c * 4.0 + (double)kprime * 16.0) + (double)P * 64.0;
    return b;
}

void shortlist_core(DevIndex& ix, const float* xq, size_t nq, uint32_t w, uint32_t kprime,
                    bool sorted, double alpha, uint32_t stride_div, ShortlistDev out, int depth,
                    bool timed, uint32_t cap_shift = 0, bool exact_coarse = false,
                    uint32_t* fast_status = nullptr) {
    cudaStream_t s = ix.stream;
    auto& st = ix.stats;
    const uint32_t c = ix.c;
    const size_t P = nq * (size_t)w;
    const Plan pl = make_plan(ix, nq, w, kprime, alpha, stride_div, cap_shift, exact_coarse);
    const bool filter_ok = pl.filter_ok;
    const uint32_t cap = pl.cap, stride = pl.stride;
    // enqueue-only: host-side bounds stand in for the counts read back below
    const bool fast = fast_status != nullptr;
    FastBounds fb;
    if (fast) fb = fast_bounds(ix, pl, nq, w, kprime);
    Workspace ws(s);

    if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[0], s));
    // ---- K1: coarse distances + top-w probes.  Kc >= 1024: tensor-core
    // distances with a certified candidate set recomputed exactly
    // (k_coarse_tc.cu); a query whose candidate set overflows restarts the
    // batch on the exact CUDA-core path (checked at the first readback below)
    float* D = ws.alloc<float>(nq * (size_t)c);
    uint32_t* probes = ws.alloc<uint32_t>(P);
    const bool coarse_tc = pl.coarse_tc;
    uint32_t* coarse_ovf = ws.zeros<uint32_t>(1);
    if (coarse_tc) {
        AssignTc* atc = prepare_coarse_tc(ix, w);
        launch_coarse_tc(xq, nq, ix.coarse.p, c, ix.cnorm.p, ix.cnorm_max, w, D, probes, coarse_ovf, s, atc);
    } else {
        launch_pair_dists(xq, nq, ix.coarse.p, c, ix.d, D, s);
        launch_topw(D, nq, c, w, probes, nullptr, s);
    }
    if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[1], s));

    // ---- invert probes into list-major work items: 16-query items for the
    // LUT pass (and the exact scan), 64-query items for the K4f filter
    // (small batches: the whole inversion in one single-CTA launch, k_invert.cu;
    // its buffers are sized by host-side bounds in both search modes)
    const bool small_inv = !pl.two_phase && invert_small_supported(P, c);
    if (small_inv && !fast) fb = fast_bounds(ix, pl, nq, w, kprime);
    // room for the 8-bit LUT blocks of n_items LUT-pass items (index-owned cache)
    auto ensure_q8 = [&](uint32_t n_items) {
        const size_t need = (size_t)n_items * 8 * 256 * kQT;
        // (enqueue-only: ensure_fast sized the cache to the bound before the capture)
        if (fast && ix.q8_cache.bytes() < need) throw std::runtime_error("enqueue-only search: LUT cache not prepared");
        if (ix.q8_cache.bytes() < need) {
            size_t free_b = 0, total_b = 0;
            PQRR_CUDA(cudaMemGetInfo(&free_b, &total_b));
            if (need - ix.q8_cache.bytes() < free_b / 2) {
                PQRR_CUDA(cudaStreamSynchronize(s));  // (the stream may still read the old cache)
                ix.q8_cache.alloc(need);
                ix.q8_param.alloc((size_t)n_items * kQT * 2);
            }
        }
        return ix.q8_cache.bytes() >= need;
    };
    bool use_filter = filter_ok;
    uint32_t* pair_ids = ws.alloc<uint32_t>(P);
    if (!small_inv) launch_iota(pair_ids, P, s);
    // two-phase LUT pass: see make_plan
    const bool two_phase = pl.two_phase;
    const uint32_t R1 = pl.R1;
    // all pairs: the single-phase LUT pass items, or (two-phase) only the
    // per-list counts that place the K4f live pairs
    const uint32_t fchunk = pl.fchunk;
    ItemSet im, if64;
    if (small_inv) {
        im.c = if64.c = c;
        im.qt = kQT;
        if64.qt = kFQ;
        if64.chunk = fchunk;
        im.pair_sorted = if64.pair_sorted = ws.alloc<uint32_t>(P);
        im.list_cnt = if64.list_cnt = ws.alloc<uint32_t>(c + 1);
        im.list_first = if64.list_first = ws.alloc<uint32_t>(c + 1);
        im.item_off = ws.alloc<uint32_t>(c + 1);
        if64.item_off = ws.alloc<uint32_t>(c + 1);
        im.n_items = fb.items_all;
        if64.n_items = fb.items_f64;
        if (use_filter) use_filter = ensure_q8(im.n_items);
        // item sets within the shared-memory sort are finished in the same
        // launch; a larger one (long lists cut into many chunks) goes through
        // items_phase2 with its bound
        auto prep = [&](ItemSet& it, bool wanted) {
            SmallItems o{it.item_off, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, it.qt, it.chunk, 0u};
            if (!wanted || it.n_items > kInvertSmallMaxItems) return o;
            const uint32_t n = std::max<uint32_t>(it.n_items, 1);
            o.item_list = it.item_list = ws.alloc<uint32_t>(n);
            o.item_start = it.item_start = ws.alloc<uint32_t>(n);
            o.item_nq = it.item_nq = ws.alloc<uint32_t>(n);
            o.item_e0 = it.item_e0 = ws.alloc<uint32_t>(n);
            o.item_e1 = it.item_e1 = ws.alloc<uint32_t>(n);
            o.item_order = it.item_order = ws.alloc<uint32_t>(n);
            o.bound = n;
            return o;
        };
        const SmallItems sa = prep(im, true), sb = prep(if64, use_filter);
        launch_invert_small(probes, (uint32_t)P, w, D, c, ix.list_len.p, im.pair_sorted, im.list_cnt,
                            im.list_first, sa, sb, s);
    } else {
        im = items_phase1(ws, probes, pair_ids, P, c, ix.list_len.p, kQT, s, nullptr, 1u << 30, w, D, probes,
                          two_phase);
        if64 = items_phase1(ws, probes, pair_ids, P, c, ix.list_len.p, kFQ, s, &im, fchunk);
    }
    ItemSet im_near, im_far;
    if (two_phase) {
        const size_t pn = nq * (size_t)R1, pf = nq * (size_t)(w - R1);
        uint32_t* nl = ws.alloc<uint32_t>(pn);
        uint32_t* ni = ws.alloc<uint32_t>(pn);
        uint32_t* fl = ws.alloc<uint32_t>(pf);
        uint32_t* fi = ws.alloc<uint32_t>(pf);
        split_pairs_kernel<<<nblk(P), 256, 0, s>>>(probes, nq, w, R1, nl, ni, fl, fi);
        PQRR_LAUNCH_CHECK();
        count_launch();
        im_near = items_phase1(ws, nl, ni, pn, c, ix.list_len.p, kQT, s, nullptr, 1u << 30, w, D, probes);
        im_far = items_phase1(ws, fl, fi, pf, c, ix.list_len.p, kQT, s, nullptr, 1u << 30, w, D, probes);
    }
    uint64_t* n_entries = ws.alloc<uint64_t>(nq);
    uint8_t* sampled = ws.alloc<uint8_t>(nq);
    uint64_t* grand = ws.zeros<uint64_t>(2);
    const int tiered = pl.tiered;
    uint64_t* sample_off = ws.alloc<uint64_t>(P + 1);
    if (!launch_query_sizes_small(probes, nq, w, ix.list_len.p, stride, tiered, cap, n_entries, sampled,
                                  sample_off, grand, s, R1)) {
        uint64_t* pair_samples = ws.zeros<uint64_t>(P + 1);
        launch_query_sizes(probes, nq, w, ix.list_len.p, stride, tiered, cap, n_entries, sampled,
                           pair_samples, grand, s, R1);
        exclusive_scan_u64(pair_samples, sample_off, P + 1, s);
    }
    uint64_t total_samples = 0, h_grand[2] = {0, 0};
    uint32_t h_ovf = 0;
    if (fast) {
        // bounds instead of the readback; the kernels read the real counts on
        // the device, the coarse overflow flag joins the status word
        total_samples = fb.samples;
        h_grand[1] = 8192;  // the threshold kernel's staging capacity
        im.n_items = fb.items_all;
        if64.n_items = fb.items_f64;
        im_near.n_items = fb.items_near;
        im_far.n_items = fb.items_far;
    } else {
        PQRR_CUDA(cudaMemcpyAsync(h_grand, grand, 16, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaMemcpyAsync(&total_samples, sample_off + P, 8, cudaMemcpyDeviceToHost, s));
        if (!small_inv) {
            PQRR_CUDA(cudaMemcpyAsync(&im.n_items, im.item_off + c, 4, cudaMemcpyDeviceToHost, s));
            PQRR_CUDA(cudaMemcpyAsync(&if64.n_items, if64.item_off + c, 4, cudaMemcpyDeviceToHost, s));
        }
        if (two_phase) {
            PQRR_CUDA(cudaMemcpyAsync(&im_near.n_items, im_near.item_off + c, 4, cudaMemcpyDeviceToHost, s));
            PQRR_CUDA(cudaMemcpyAsync(&im_far.n_items, im_far.item_off + c, 4, cudaMemcpyDeviceToHost, s));
        }
        if (coarse_tc) PQRR_CUDA(cudaMemcpyAsync(&h_ovf, coarse_ovf, 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaStreamSynchronize(s));
    }
    if (h_ovf) {  // rare: a certified candidate set did not fit; redo on the exact path
        shortlist_core(ix, xq, nq, w, kprime, sorted, alpha, stride_div, out, depth, timed, cap_shift, true);
        return;
    }
    const uint32_t n_items = two_phase ? im_near.n_items + im_far.n_items : im.n_items;

    if (use_filter && !small_inv) use_filter = ensure_q8(n_items);
    if (two_phase && !use_filter && fast) throw std::runtime_error("enqueue-only search: LUT cache not prepared");
    if (two_phase && !use_filter) {
        // rare (no room for the 8-bit LUT cache): the exact scan needs the
        // sorted all-pairs items after all
        im = items_phase1(ws, probes, pair_ids, P, c, ix.list_len.p, kQT, s, nullptr, 1u << 30, w, D);
        PQRR_CUDA(cudaMemcpyAsync(&im.n_items, im.item_off + c, 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaStreamSynchronize(s));
    }
    // (small_inv: the sets finished by invert_small_kernel have their items;
    // their counts are bounds, so a set finished here is padded)
    if ((!two_phase || !use_filter) && !im.item_order) items_phase2(ws, im, c, ix.list_len.p, s, fast || small_inv);
    if (use_filter && !if64.item_order)
        items_phase2(ws, if64, c, ix.list_len.p, s, fast || small_inv, small_inv && fchunk < (1u << 30));
    if (two_phase) {
        items_phase2(ws, im_near, c, ix.list_len.p, s, fast);
        items_phase2(ws, im_far, c, ix.list_len.p, s, fast);
    }
    if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[2], s));

    ScanArgs a{};
    a.codes = ix.codes.p;
    a.list_off = ix.list_off.p;
    a.list_len = ix.list_len.p;
    a.coarse = ix.coarse.p;
    a.books = ix.books.p;
    a.xq = xq;
    a.d = ix.d;
    a.m = ix.m;
    a.ks = ix.ks;
    a.w = w;
    a.cap = cap;
    a.query_sampled = sampled;
    uint32_t* counter = ws.zeros<uint32_t>(2);

    // ---- K2 LUT pass: per item the exact LUT -> sampled distances (threshold
    // estimation) and, for the filter, the 8-bit LUT block
    float* tau = ws.alloc<float>(nq);
    float* sample_dist = ws.alloc<float>(total_samples);
    if (total_samples || use_filter) {
        (two_phase ? im_near : im).apply(a);
        a.pass = 1;
        a.q8_cache = use_filter ? ix.q8_cache.p : nullptr;
        a.q8_param = use_filter ? ix.q8_param.p : nullptr;
        a.stride = stride;
        a.tiered = tiered;
        a.sample_off = sample_off;
        a.sample_dist = total_samples ? sample_dist : nullptr;
        a.tau = tau;  // unused in the LUT pass
        a.item_counter = counter;
        // (no more pairs than lists: about one probing query per item, where
        // the 16-lane pass spends its time on dead lanes and its code-book ring)
        // (two-phase: this is the near pass, nq * R1 pairs)
        const size_t p_first = two_phase ? nq * (size_t)R1 : P;
        if (p_first <= (size_t)c && lut_pass_narrow_supported(ix.d, ix.m, ix.ks)) launch_lut_pass_narrow(a, s, p_first);
        else if (lut_pass_supported(ix.d, ix.m, ix.ks)) launch_lut_pass(a, s);
        else launch_ivf_scan(a, s);
    }
    if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[3], s));
    launch_sample_threshold(sample_dist, sample_off, w, nq, sampled, (float)(alpha * kprime), stride,
                            tiered, (uint32_t)h_grand[1], tau, s);
    if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[4], s));
    float* pair_bound = (two_phase && use_filter && far_bound_supported(ix.d, ix.m, ix.ks))
                            ? ws.alloc<float>(P) : nullptr;
    if (two_phase && use_filter && im_far.n_items) {
        // far probes: bound pass (per-lane sum of minima), then the 8-bit
        // blocks of the far items with a lane that can reach tau
        ScanArgs b = a;
        im_far.apply(b);
        b.pass = 1;
        b.q8_cache = ix.q8_cache.p + (size_t)im_near.n_items * 8 * 256 * kQT;
        b.q8_param = ix.q8_param.p + (size_t)im_near.n_items * kQT * 2;
        b.sample_dist = nullptr;
        b.tau = tau;
        uint32_t* cnt2 = ws.zeros<uint32_t>(2);
        if (pair_bound) {
            // tensor-core lower bound of every far pair's sum of minima
            launch_far_bound(xq, ix.coarse.p, ix.books.p, probes, nq, w, R1, pair_bound, s);
            b.pair_bound = pair_bound;
        } else {
            b.item_counter = cnt2;
            b.q8_mode = 1;  // exact bound pass (sum of minima from the FMA LUT build)
            b.skip_dead = 0;
            launch_lut_pass(b, s);
        }
        b.item_counter = cnt2 + 1;
        b.q8_mode = 0;
        b.skip_dead = 1;
        launch_lut_pass(b, s);
    }
    if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[11], s));

    // ---- K4 main scan: candidates (d <= tau, or the filter's superset)
    // exactness-check readback: [0..1] max count / fail, [2..5] u64 candidate
    // totals, [6..7] u64 (live pair, entry) lookups of K4f
    unsigned* maxn = ws.zeros<unsigned>(8);
    float* cand_dist = ws.alloc<float>(nq * (size_t)cap);
    uint32_t* cand_pos = ws.alloc<uint32_t>(nq * (size_t)cap);
    uint32_t* cand_cnt = ws.zeros<uint32_t>(nq);
    uint32_t* cand_le = nullptr;
    uint32_t* cand_mm = nullptr;
    if (use_filter) {
        FilterArgs f{};
        f.codes = ix.codes.p;
        f.list_off = ix.list_off.p;
        f.list_len = ix.list_len.p;
        f.item_list = if64.item_list;
        f.item_start = if64.item_start;
        f.item_nq = if64.item_nq;
        f.item_e0 = if64.item_e0;
        f.item_e1 = if64.item_e1;
        f.item_order = if64.item_order;
        f.num_items = if64.item_off + c;
        f.item_counter = counter + 1;
        f.list_first = im.list_first;
        f.sub_item_off = im.item_off;
        f.pair_sorted = im.pair_sorted;
        f.w = w;
        f.tau = tau;
        f.q8_cache = ix.q8_cache.p;
        f.q8_param = ix.q8_param.p;
        f.cand_aux = reinterpret_cast<uint32_t*>(cand_dist);
        f.cand_pos = cand_pos;
        f.cand_cnt = cand_cnt;
        f.cap = cap;
        // candidates' codes next to them (K4r then reads no random DRAM sectors)
        uint64_t* cand_code = ws.alloc<uint64_t>(nq * (size_t)cap);
        f.cand_code = cand_code;
        uint32_t* cand_used = ws.zeros<uint32_t>(nq * 8);
        f.cand_used = w <= 256 ? cand_used : nullptr;
        static const bool pass_all = getenv("PQRR_FILTER_ALL") != nullptr;  // debug hook
        f.pass_all = pass_all ? 1 : 0;
        const char* bd_env = getenv("PQRR_BANDDIV");  // tuning hook (read per search)
        // 100: measured flat at C2 (80..120) and better than 80 at C4 (k' = 1e4);
        // >= 160 saturates the 5-bit values and overflows candidate buffers
        const float band_div = bd_env ? (float)atof(bd_env) : 100.f;
        f.band_div = band_div;
        {
            uint32_t* live_slot = ws.alloc<uint32_t>(P);
            uint32_t* live_pair = ws.alloc<uint32_t>(P);
            uint32_t* live_cnt = ws.alloc<uint32_t>(c);
            f.live_slot = live_slot;
            f.live_pair = live_pair;
            const ItemSet& s0 = two_phase ? im_near : im;
            PairSet p0{s0.pair_sorted, s0.list_cnt, s0.list_first, s0.item_off, 0u, nullptr};
            PairSet p1{nullptr, nullptr, nullptr, nullptr, 0u, nullptr};
            if (two_phase) p1 = PairSet{im_far.pair_sorted, im_far.list_cnt, im_far.list_first, im_far.item_off,
                                        im_near.n_items, pair_bound};
            launch_live_pairs(f, p0, p1, im.list_first, im.list_cnt, c, live_slot, live_pair, live_cnt,
                              if64.item_off, if64.item_start, if64.item_nq, if64.chunk, s,
                              reinterpret_cast<unsigned long long*>(maxn + 6));
        }
        launch_ivf_filter(f, s);
        if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[9], s));
        cand_le = ws.alloc<uint32_t>(nq);
        // exact distances' range per query (K4r smem variant; all-ones = unknown)
        cand_mm = ws.alloc<uint32_t>(2 * nq);
        PQRR_CUDA(cudaMemsetAsync(cand_mm, 0xff, 2 * nq * sizeof(uint32_t), s));
        launch_recheck(xq, ix.d, ix.m, ix.coarse.p, ix.books.p, probes, w, ix.codes.p, cand_cnt, cap,
                       cand_pos, cand_dist, tau, nq, cand_le, s, cand_mm, cand_code, f.cand_used);
    } else {
        im.apply(a);
        a.pass = 0;
        a.q8_cache = nullptr;
        a.q8_param = nullptr;
        a.stride = 1;
        a.sample_dist = nullptr;
        a.tau = tau;
        a.cand_dist = cand_dist;
        a.cand_pos = cand_pos;
        a.cand_cnt = cand_cnt;
        a.item_counter = counter + 1;
        launch_ivf_scan(a, s);
    }
    if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[5], s));

    // ---- exactness check of the threshold
    uint8_t* fail = ws.alloc<uint8_t>(nq);
    check_fail_kernel<<<nblk(nq), 256, 0, s>>>(sampled, cand_cnt, cand_le, nq, kprime, cap, fail,
                                                maxn, reinterpret_cast<unsigned long long*>(maxn + 2),
                                                reinterpret_cast<unsigned long long*>(maxn + 4),
                                                coarse_tc ? coarse_ovf : nullptr, fast_status);
    PQRR_LAUNCH_CHECK();
    count_launch();
    // the unsorted selection (a re-rank follows) needs no host-side count:
    // queue it before the readback so the GPU stays busy during the round
    // trip (rows that fail the check are redone and overwritten below)
    const bool early_select = !sorted;
    if (early_select) {
        launch_select_topk(cand_dist, cand_pos, cand_cnt, cap, cap, nq, ix.ids.p, kprime, sorted,
                           reinterpret_cast<uint64_t*>(out.key), out.pos, out.cnt, s, cand_mm,
                           ix.keys_need_ids);
        if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[6], s));
    }
    if (fast) {
        // no readback: failed rows are flagged in the status word (the caller
        // redoes the batch on the synchronising path); the sorted selection
        // sizes its staging by the buffer capacity instead of the largest count
        if (!early_select)
            launch_select_topk(cand_dist, cand_pos, cand_cnt, cap, cap, nq, ix.ids.p, kprime, sorted,
                               reinterpret_cast<uint64_t*>(out.key), out.pos, out.cnt, s);
        return;
    }
    std::vector<uint8_t> h_fail(nq);
    unsigned h_maxn[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    PQRR_CUDA(cudaMemcpyAsync(h_fail.data(), fail, nq, cudaMemcpyDeviceToHost, s));
    PQRR_CUDA(cudaMemcpyAsync(h_maxn, maxn, 32, cudaMemcpyDeviceToHost, s));
    PQRR_CUDA(cudaStreamSynchronize(s));
    static const bool force_retry = getenv("PQRR_FORCE_RETRY") != nullptr;  // test hook
    if (force_retry && depth == 0)
        for (size_t q = 0; q < nq; ++q) h_fail[q] = (uint8_t)(1 + (q & 1));
    uint64_t total_cand = 0, total_le = 0, live_entries = 0;
    std::memcpy(&total_cand, h_maxn + 2, 8);
    std::memcpy(&total_le, h_maxn + 4, 8);
    std::memcpy(&live_entries, h_maxn + 6, 8);

    // ---- exact top-k' selection (sorted: smem sized by the largest count)
    if (!early_select) {
        launch_select_topk(cand_dist, cand_pos, cand_cnt, cap, h_maxn[0], nq, ix.ids.p, kprime, sorted,
                           reinterpret_cast<uint64_t*>(out.key), out.pos, out.cnt, s);
        if (timed) PQRR_CUDA(cudaEventRecord(ix.ev[6], s));
        PQRR_CUDA(cudaStreamSynchronize(s));
    }
    if (timed) {
        st.candidates += total_cand;
        st.exact_candidates += use_filter ? total_le : total_cand;
        // stage times (accumulated over the chunks of a large batch)
        auto el = [&](int a, int b) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ix.ev[a], ix.ev[b]);
            return ms;
        };
        st.ms_coarse += el(0, 1);
        st.ms_invert += el(1, 2);
        // the far-probe LUT passes (two-phase) count as LUT-pass time
        st.ms_sample_scan += el(2, 3) + el(4, 11);
        st.ms_threshold += el(3, 4);
        st.ms_scan += el(11, 5);
        st.ms_select += el(5, 6);
        if (use_filter) {
            st.ms_filter += el(11, 9);
            st.ms_recheck += el(9, 5);
            st.filter_live_entries += live_entries;
        }
        st.work_items += n_items;
        st.sampled_entries += total_samples;
        st.scanned_entries += h_grand[0];
        st.stride = stride;
    }

    // ---- retry queries whose threshold failed (rare): under-full -> raise
    // alpha; overflow -> lower alpha and sample more densely.
    for (int kind = 1; kind <= 2; ++kind) {
        std::vector<uint32_t> rows;
        for (size_t q = 0; q < nq; ++q)
            if (h_fail[q] == kind) rows.push_back((uint32_t)q);
        if (rows.empty()) continue;
        if (depth >= 8) throw std::runtime_error("shortlist threshold did not converge");
        st.retries += (uint32_t)rows.size();
        Workspace ws2(s);
        uint32_t* d_rows = ws2.alloc<uint32_t>(rows.size());
        PQRR_CUDA(cudaMemcpyAsync(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, s));
        float* sx = ws2.alloc<float>(rows.size() * ix.d);
        gather_rows_f32<<<nblk(rows.size() * ix.d), 256, 0, s>>>(xq, ix.d, d_rows, rows.size(), sx);
        PQRR_LAUNCH_CHECK();
        ShortlistDev sub{ws2.alloc<u64>(rows.size() * kprime), ws2.alloc<uint32_t>(rows.size() * kprime),
                         ws2.alloc<uint32_t>(rows.size())};
        // under-full: widen the target; overflow: narrow it (never below the
        // k' it must cover) and sample twice as densely for a tighter estimate
        const double a2 = kind == 1 ? alpha * 2.0 : std::max(1.25, alpha / 1.5);
        // an overflow also doubles the candidate buffer (the filter's superset
        // of the entries <= tau, not tau itself, may be what does not fit)
        shortlist_core(ix, sx, rows.size(), w, kprime, sorted, a2, stride_div * 2, sub, depth + 1,
                       false, cap_shift + (kind == 2 ? 1u : 0u));
        scatter_shortlist<<<nblk(rows.size() * kprime), 256, 0, s>>>(
            sub.key, sub.pos, sub.cnt, d_rows, rows.size(), kprime, out.key, out.pos, out.cnt);
        PQRR_LAUNCH_CHECK();
        count_launch(2);
        PQRR_CUDA(cudaStreamSynchronize(s));
    }
}

// ---- enqueue-only search: one CUDA graph per (shape, buffers) ----
// Small batches are launch- and round-trip-bound (C5 batch 1: 37 kernels and
// three host synchronisations for 0.2 ms of device work), so the whole search
// is captured once per shape into a graph (host-side bounds instead of
// readbacks, see FastBounds) and replayed with one launch.  Larger batches
// stay on the synchronising path: their two round trips are noise against
// tens of milliseconds, and a failed threshold there retries only its row.
constexpr size_t kFastMaxQueries = 1024;

uint64_t index_signature(const DevIndex& ix) {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    auto mix = [&](uint64_t v) { h = (h ^ v) * 0xbf58476d1ce4e5b9ull; h ^= h >> 29; };
    for (const void* p : {(const void*)ix.codes.p, (const void*)ix.rcodes.p, (const void*)ix.ids.p,
                          (const void*)ix.list_off.p, (const void*)ix.list_len.p, (const void*)ix.coarse.p,
                          (const void*)ix.books.p, (const void*)ix.rbooks.p, (const void*)ix.block_list.p,
                          (const void*)ix.q8_cache.p, (const void*)ix.q8_param.p, (const void*)ix.cnorm.p,
                          (const void*)ix.atc.hi, (const void*)ix.d_stat.p})
        mix((uint64_t)(uintptr_t)p);
    mix(ix.n);
    mix(ix.slots);
    return h;
}

// Whether the batch may take the enqueue-only path; allocates what the
// capture must not (status block, LUT cache sized to the bounds, lazy coarse state).
bool ensure_fast(DevIndex& ix, size_t nq, uint32_t w, uint32_t kprime, uint32_t k, double* scratch_bytes = nullptr) {
    if (!ix.graph_enabled || nq == 0 || nq > kFastMaxQueries) return false;
    static size_t dev_total = 0;
    if (!dev_total) {
        size_t f = 0;
        PQRR_CUDA(cudaMemGetInfo(&f, &dev_total));
    }
    const Plan pl = make_plan(ix, nq, w, kprime, default_alpha(kprime, w), 1, 0, false);
    const FastBounds fb = fast_bounds(ix, pl, nq, w, kprime);
    if (fb.bytes > 0.125 * (double)dev_total) return false;
    if (scratch_bytes) *scratch_bytes = fb.bytes;
    if (!ix.d_stat.p) {
        ix.d_stat.alloc(8);
        PQRR_CUDA(cudaMallocHost(&ix.h_stat, 8 * sizeof(uint32_t)));
        for (auto& e : ix.ev_fast) PQRR_CUDA(cudaEventCreate(&e));
    }
    if (pl.filter_ok) {
        const size_t need = fb.q8_items * 8 * 256 * kQT;
        if (ix.q8_cache.bytes() < need) {
            // (the stream may still read the old cache)
            PQRR_CUDA(cudaStreamSynchronize(ix.stream));
            ix.q8_cache.alloc(need);
            ix.q8_param.alloc(fb.q8_items * kQT * 2);
        }
    }
    if (pl.coarse_tc) prepare_coarse_tc(ix, w);
    (void)k;
    return true;
}

void search_body_fast(DevIndex& ix, const float* xq, size_t nq, uint32_t w, uint32_t kprime, uint32_t k,
                      uint32_t* out_ids, float* out_dists, uint32_t* out_cnt) {
    cudaStream_t s = ix.stream;
    const bool pair = k > 0 && kprime >= 4096 && rerank_pair_supported(ix.d, ix.m, ix.ks, ix.mprime);
    ix.keys_need_ids = !pair;
    PQRR_CUDA(cudaMemsetAsync(ix.d_stat.p, 0, 8 * sizeof(uint32_t), s));
    Workspace ws(s);
    ShortlistDev sl{ws.alloc<u64>(nq * (size_t)kprime), ws.alloc<uint32_t>(nq * (size_t)kprime),
                    ws.alloc<uint32_t>(nq)};
    shortlist_core(ix, xq, nq, w, kprime, k == 0, default_alpha(kprime, w), 1, sl, 0, false, 0, false,
                   ix.d_stat.p + 4);
    min_count_kernel<<<nblk(nq), 256, 0, s>>>(sl.cnt, nq, k, ix.d_stat.p);
    PQRR_LAUNCH_CHECK();
    count_launch();
    if (k > 0) {
        launch_rerank(reinterpret_cast<uint64_t*>(sl.key), sl.pos, sl.cnt, kprime, nq, xq, ix.d,
                      ix.block_list.p, ix.coarse.p, ix.codes.p, ix.books.p, ix.m, ix.rcodes.p,
                      ix.rbooks.p, ix.mprime, ix.ks, k, out_ids, out_dists, out_cnt, s, nullptr,
                      pair ? ix.ids.p : nullptr);
    } else {
        launch_unpack_keys(reinterpret_cast<uint64_t*>(sl.key), sl.cnt, nq, kprime, out_ids, out_dists, s);
        PQRR_CUDA(cudaMemcpyAsync(out_cnt, sl.cnt, nq * 4, cudaMemcpyDeviceToDevice, s));
    }
    PQRR_CUDA(cudaMemcpyAsync(ix.h_stat, ix.d_stat.p, 8 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
}

// Host-staged small batch: the graph starts with the H2D copy of the queries
// from pinned staging and ends with one D2H copy of [ids | dists | counts].
struct HostStage {
    const void* h_in;
    void* d_in;
    size_t in_bytes;
    void* h_out;
    const void* d_out;
    size_t out_bytes;
};

// Enqueues the whole search on ix.stream without blocking the host (graph
// replay; the first call of a shape captures it).  `widen_from` (optional):
// u8 queries on the device, widened into xq inside the graph.  Returns false
// if the shape cannot take this path.
bool search_enqueue(DevIndex& ix, const uint8_t* widen_from, float* xq, size_t nq, uint32_t w,
                    uint32_t kprime, uint32_t k, uint32_t* out_ids, float* out_dists, uint32_t* out_cnt,
                    const HostStage* hs = nullptr) {
    double scratch = 0;
    if (!ensure_fast(ix, nq, w, kprime, k, &scratch)) return false;
    cudaStream_t s = ix.stream;
    const uint64_t sig = index_signature(ix);
    const void* qkey = widen_from ? (const void*)widen_from : (const void*)xq;
    DevIndex::SearchGraph* g = nullptr;
    for (auto& c : ix.graphs)
        if (c.xq == qkey && c.nq == nq && c.w == w && c.kprime == kprime && c.k == k && c.oi == out_ids &&
            c.od == out_dists && c.oc == out_cnt && c.q_u8 == ix.q_u8 && c.h_in == (hs ? hs->h_in : nullptr)) {
            g = &c;
            break;
        }
    if (g && g->sig != sig) {  // the index moved or grew under the graph
        if (g->exec) cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
    }
    if (g && !g->exec && g->sig == sig) return false;  // this shape failed to capture before
    bool captured_now = false;
    if (!g || !g->exec) {
        captured_now = true;
        if (!g) {
            // cached graphs keep the scratch of their memory nodes mapped:
            // at most 16 graphs and a quarter of the device, least recently
            // used evicted (and their memory trimmed) first
            static size_t dev_total = 0;
            if (!dev_total) {
                size_t f = 0;
                PQRR_CUDA(cudaMemGetInfo(&f, &dev_total));
            }
            auto held = [&] {
                double b = 0;
                for (auto& c : ix.graphs) b += c.exec ? c.bytes : 0.0;
                return b;
            };
            bool trimmed = false;
            while (!ix.graphs.empty() &&
                   (ix.graphs.size() >= 16 || held() + scratch > 0.25 * (double)dev_total)) {
                size_t lru = 0;
                for (size_t i = 1; i < ix.graphs.size(); ++i)
                    if (ix.graphs[i].used < ix.graphs[lru].used) lru = i;
                if (ix.graphs[lru].exec) cudaGraphExecDestroy(ix.graphs[lru].exec);
                ix.graphs.erase(ix.graphs.begin() + lru);
                trimmed = true;
            }
            if (trimmed) {
                PQRR_CUDA(cudaStreamSynchronize(s));
                cudaDeviceGraphMemTrim(ix.device);
            }
            ix.graphs.emplace_back();
            g = &ix.graphs.back();
            g->xq = qkey; g->nq = nq; g->w = w; g->kprime = kprime; g->k = k;
            g->oi = out_ids; g->od = out_dists; g->oc = out_cnt; g->q_u8 = ix.q_u8;
            g->h_in = hs ? hs->h_in : nullptr;
        }
        g->sig = sig;
        g->bytes = scratch;
        cudaGraph_t graph = nullptr;
        const unsigned long long l0 = launch_count();
        PQRR_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        bool ok = true;
        std::string why;
        try {
            if (hs) PQRR_CUDA(cudaMemcpyAsync(hs->d_in, hs->h_in, hs->in_bytes, cudaMemcpyHostToDevice, s));
            if (widen_from) launch_widen_u8(widen_from, xq, nq * ix.d, s);
            search_body_fast(ix, xq, nq, w, kprime, k, out_ids, out_dists, out_cnt);
            if (hs) PQRR_CUDA(cudaMemcpyAsync(hs->h_out, hs->d_out, hs->out_bytes, cudaMemcpyDeviceToHost, s));
        } catch (const std::exception& e) {
            ok = false;
            why = e.what();
        }
        const cudaError_t ce = cudaStreamEndCapture(s, &graph);
        if (ce != cudaSuccess || !graph) ok = false;
        if (ok && cudaGraphInstantiate(&g->exec, graph, 0) != cudaSuccess) {
            ok = false;
            g->exec = nullptr;
        }
        if (graph) cudaGraphDestroy(graph);
        if (!ok) {
            cudaGetLastError();  // clear a capture error; the shape stays on the synchronising path
            g->exec = nullptr;
            return false;
        }
        g->kernels = (uint32_t)(launch_count() - l0);
    }
    g->used = ++ix.graph_clock;
    // (launch accounting: the capture call counted its kernels as they were
    // recorded; a replay launches the same kernels)
    if (!captured_now) count_launch(g->kernels);
    PQRR_CUDA(cudaEventRecord(ix.ev_fast[0], s));
    PQRR_CUDA(cudaGraphLaunch(g->exec, s));
    PQRR_CUDA(cudaEventRecord(ix.ev_fast[1], s));
    ix.stats = pqrr_dev_search_stats{};
    ix.stats.nq = nq;
    ix.stats.kernels = g->kernels;
    return true;
}

// After the enqueued search finished: 0 = results valid, 1 = the batch must be
// redone on the synchronising path; throws "shortlist too small".
int search_fast_outcome(DevIndex& ix, uint32_t k) {
    static const bool force_retry = getenv("PQRR_FORCE_RETRY") != nullptr;  // test hook: take the fallback
    if (ix.h_stat[4] || force_retry) return 1;
    if (k > 0 && ix.h_stat[0]) throw ShortlistError();
    std::memcpy(&ix.stats.rerank_candidates, ix.h_stat + 2, 8);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ix.ev_fast[0], ix.ev_fast[1]);
    ix.stats.ms_total = ms;
    return 0;
}

// Target candidates per query = alpha * k' (the sampled threshold rank);
// tuning hook PQRR_ALPHA (read per search).
void search_sync(DevIndex& ix, const float* xq, size_t nq, uint32_t w, size_t kprime_sz, size_t k_sz,
                 uint32_t* out_ids, float* out_dists, uint32_t* out_cnt);

void validate_search(DevIndex& ix, uint32_t w, size_t kprime_sz, size_t k_sz) {
    if (w < 1 || w > ix.c) throw ArgError("v must satisfy 1 <= v <= c");
    if (kprime_sz < 1) throw ArgError("kprime must be positive");
    if (kprime_sz > 16384) throw UnsupportedError("kprime above 16384 is not supported on the device");
    if (k_sz > kprime_sz) throw ShortlistError();
    if (k_sz > 0 && ix.mprime == 0) throw ArgError("re-ranking needs refinement codes (mprime > 0)");
    finalize(ix);
}

// `widen_from` (optional): the queries as u8 on the device; xq is then the
// staging buffer they are widened into (inside the graph on the enqueue-only
// path).  Small batches replay a captured graph and synchronise once; a batch
// whose status word is set, and every large batch, runs the synchronising path.
// `hs` (optional, host-buffer API): queries wait in pinned staging; returns
// true if the graph also delivered the results to hs->h_out.
bool search_device(DevIndex& ix, float* xq, size_t nq, uint32_t w, size_t kprime_sz,
                   size_t k_sz, uint32_t* out_ids, float* out_dists, uint32_t* out_cnt,
                   const uint8_t* widen_from = nullptr, const HostStage* hs = nullptr) {
    validate_search(ix, w, kprime_sz, k_sz);
    const uint32_t kprime = (uint32_t)kprime_sz, k = (uint32_t)k_sz;
    cudaStream_t s = ix.stream;
    if (nq == 0) {
        ix.stats = pqrr_dev_search_stats{};
        return false;
    }
    if (search_enqueue(ix, widen_from, xq, nq, w, kprime, k, out_ids, out_dists, out_cnt, hs)) {
        PQRR_CUDA(cudaStreamSynchronize(s));
        if (search_fast_outcome(ix, k) == 0) return hs != nullptr;
        // redo the batch with per-row retries (xq is already widened)
    } else {
        if (hs) PQRR_CUDA(cudaMemcpyAsync(hs->d_in, hs->h_in, hs->in_bytes, cudaMemcpyHostToDevice, s));
        if (widen_from) launch_widen_u8(widen_from, xq, nq * ix.d, s);
    }
    search_sync(ix, xq, nq, w, kprime_sz, k_sz, out_ids, out_dists, out_cnt);
    return false;
}

// The synchronising path: counts read back, per-row threshold retries, stage times.
void search_sync(DevIndex& ix, const float* xq, size_t nq, uint32_t w, size_t kprime_sz, size_t k_sz,
                 uint32_t* out_ids, float* out_dists, uint32_t* out_cnt) {
    const uint32_t kprime = (uint32_t)kprime_sz, k = (uint32_t)k_sz;
    cudaStream_t s = ix.stream;
    const unsigned long long l0 = launch_count();
    ix.stats = pqrr_dev_search_stats{};
    ix.stats.nq = nq;
    for (auto& e : ix.ev)
        if (!e) PQRR_CUDA(cudaEventCreate(&e));
    PQRR_CUDA(cudaEventRecord(ix.ev[10], s));
    // large shortlists (k' >= 4096) ahead of the CTA-pair re-ranker: the keys
    // carry no ids, the selection gathers ids only for its boundary ties and
    // the re-ranker's rank 1 reads the ids of the entries it writes (C4:
    // selection 2.59 -> 1.41 ms, re-ranker +0.5 ms; at k' = 1000 the
    // selection's gathers are cheap and the re-ranker's extra load is not)
    const bool pair = k > 0 && kprime >= 4096 && rerank_pair_supported(ix.d, ix.m, ix.ks, ix.mprime);
    ix.keys_need_ids = !pair;
    Workspace ws(s);
    ShortlistDev sl{ws.alloc<u64>(nq * (size_t)kprime), ws.alloc<uint32_t>(nq * (size_t)kprime),
                    ws.alloc<uint32_t>(nq)};
    // Large batches run in chunks sized to the free device memory: per query
    // the sampled distances (~2 w avg_len / stride floats: uniform sampling of
    // the k'-quantile needs many samples when k' << N_q), the 8-bit LUT blocks,
    // the candidate buffers and the coarse distance row.
    {
        const double avg_len = ix.c ? (double)ix.n / ix.c : 0.0;
        const double stride = std::max(1.0, std::floor(default_alpha(kprime, w) * kprime /
                                                        default_spq(kprime, w)));
        const double per_q = 2.0 * w * avg_len / stride * 4.0 + (w / 16.0 + 1.0) * 32768.0 +
                             std::max(8192.0, 8.0 * kprime) * 8.0 + ix.c * 4.0 + w * 64.0;
        // cudaMemGetInfo costs ~1 ms with a large resident index: query it
        // only when the batch needs a sizeable share of the device
        static size_t dev_total = 0;
        if (!dev_total) {
            size_t f = 0;
            PQRR_CUDA(cudaMemGetInfo(&f, &dev_total));
        }
        size_t chunk = nq;
        if (per_q * (double)nq > 0.25 * (double)dev_total) {
            size_t free_b = 0, total_b = 0;
            PQRR_CUDA(cudaMemGetInfo(&free_b, &total_b));
            chunk = std::min(nq, std::max<size_t>(256, (size_t)(0.5 * (double)free_b / per_q)));
        }
        for (size_t c0 = 0; c0 < nq; c0 += chunk) {
            const size_t nc = std::min(chunk, nq - c0);
            ShortlistDev part{sl.key + c0 * kprime, sl.pos + c0 * kprime, sl.cnt + c0};
            shortlist_core(ix, xq + c0 * ix.d, nc, w, kprime, k == 0, default_alpha(kprime, w), 1, part, 0, true);
        }
    }
    // "shortlist too small" is checked after the re-rank, with the
    // final synchronisation: no host round trip between selection and re-rank
    // (a failing batch's outputs are not returned)
    unsigned h_flag[4] = {0, 0, 0, 0};
    if (k > 0) {
        unsigned* flag = ws.zeros<unsigned>(4);
        min_count_kernel<<<nblk(nq), 256, 0, s>>>(sl.cnt, nq, k, flag);
        PQRR_LAUNCH_CHECK();
        count_launch();
        PQRR_CUDA(cudaMemcpyAsync(h_flag, flag, 16, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaEventRecord(ix.ev[7], s));
        launch_rerank(reinterpret_cast<uint64_t*>(sl.key), sl.pos, sl.cnt, kprime, nq, xq, ix.d,
                      ix.block_list.p, ix.coarse.p, ix.codes.p, ix.books.p, ix.m, ix.rcodes.p,
                      ix.rbooks.p, ix.mprime, ix.ks, k, out_ids, out_dists, out_cnt, s, ix.ev[12],
                      pair ? ix.ids.p : nullptr);
    } else {
        PQRR_CUDA(cudaEventRecord(ix.ev[7], s));
        launch_unpack_keys(reinterpret_cast<uint64_t*>(sl.key), sl.cnt, nq, kprime, out_ids, out_dists, s);
        PQRR_CUDA(cudaMemcpyAsync(out_cnt, sl.cnt, nq * 4, cudaMemcpyDeviceToDevice, s));
    }
    PQRR_CUDA(cudaEventRecord(ix.ev[8], s));
    PQRR_CUDA(cudaEventSynchronize(ix.ev[8]));
    if (h_flag[0]) throw ShortlistError();
    std::memcpy(&ix.stats.rerank_candidates, h_flag + 2, 8);
    auto el = [&](int a, int b) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ix.ev[a], ix.ev[b]);
        return ms;
    };
    auto& st = ix.stats;
    st.ms_rerank = el(7, 8);
    if (k > 0) st.ms_rerank_dist = el(7, 12);
    st.ms_total = el(10, 8);
    st.kernels = (uint32_t)(launch_count() - l0);
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return PQRR_OK;
    } catch (const ShortlistError& e) {
        g_last_error = e.what();
        return PQRR_ESHORTLIST;
    } catch (const NoDevice& e) {
        g_last_error = e.what();
        return PQRR_ENODEV;
    } catch (const UnsupportedError& e) {
        g_last_error = e.what();
        return PQRR_EUNSUPPORTED;
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

// Temporary stream + guard for the stateless kernel-seam entry points.
struct Session {
    DeviceGuard g;
    cudaStream_t s = nullptr;
    explicit Session(int dev) : g(dev) { PQRR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Session() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
    template <class T>
    T* upload(Workspace& ws, const T* h, size_t n) {
        T* d = ws.alloc<T>(n);
        if (n) PQRR_CUDA(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
        return d;
    }
    template <class T>
    void download(T* h, const T* d, size_t n) {
        if (n) PQRR_CUDA(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    void sync() { PQRR_CUDA(cudaStreamSynchronize(s)); }
};

}  // namespace

// ------------------------------------------------------------------ training (train.cu)
void kmeans_device(const float* d_points, size_t n, uint32_t dim, uint32_t k, uint32_t iterations,
                   uint64_t seed, uint32_t redo, float* h_centroids, double* out_mse,
                   double* out_trace, cudaStream_t s);

}  // namespace pqrr_b200

// ====================================================================== C ABI
using namespace pqrr_b200;

struct pqrr_dev_index {
    DevIndex ix;
};

extern "C" {

const char* pqrr_dev_last_error(void) { return g_last_error.c_str(); }

int pqrr_dev_device_count(int* out) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (out) *out = n;
    return PQRR_OK;
}

uint64_t pqrr_dev_launch_count(void) { return launch_count(); }

int pqrr_dev_assign_batch(int device, const float* points, size_t n, uint32_t dim,
                          const float* centroids, uint32_t k, uint32_t* out_assign, float* out_dist) {
    return guarded([&] {
        if (k == 0) throw ArgError("k must be positive");
        if (n == 0) return;
        Session se(device);
        Workspace ws(se.s);
        const float* p = se.upload(ws, points, n * dim);
        const float* c = se.upload(ws, centroids, (size_t)k * dim);
        uint32_t* a = ws.alloc<uint32_t>(n);
        float* dd = ws.alloc<float>(n);
        launch_argmin(p, n, c, k, dim, a, dd, se.s);
        se.download(out_assign, a, n);
        if (out_dist) se.download(out_dist, dd, n);
        se.sync();
    });
}

int pqrr_dev_assign_u8(int device, const uint8_t* points, size_t n, uint32_t dim,
                       const float* centroids, uint32_t k, uint32_t* out_assign) {
    return guarded([&] {
        if (k == 0) throw ArgError("k must be positive");
        if (n == 0) return;
        Session se(device);
        Workspace ws(se.s);
        const uint8_t* p = se.upload(ws, points, n * dim);
        const float* c = se.upload(ws, centroids, (size_t)k * dim);
        uint32_t* a = ws.alloc<uint32_t>(n);
        AssignTc tc;
        if (assign_tc_supported(dim, k) && tc.prepare(c, k, se.s)) {
            tc.assign(p, n, c, a, se.s);
        } else {
            float* x = ws.alloc<float>(n * dim);
            launch_widen_u8(p, x, n * dim, se.s);
            launch_argmin(x, n, c, k, dim, a, nullptr, se.s);
        }
        se.download(out_assign, a, n);
        se.sync();
    });
}

int pqrr_dev_encode_batch(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                          const float* data, size_t n, uint8_t* out_codes) {
    return guarded([&] {
        check_shape(d, m, ks);
        if (n == 0) return;
        Session se(device);
        Workspace ws(se.s);
        const float* b = se.upload(ws, books, (size_t)ks * d);
        const float* x = se.upload(ws, data, n * d);
        uint8_t* c = ws.alloc<uint8_t>(n * m);
        launch_pq_encode(x, n, d, b, m, ks, c, se.s);
        se.download(out_codes, c, n * m);
        se.sync();
    });
}

int pqrr_dev_decode_batch(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                          const uint8_t* codes, size_t n, float* out_data) {
    return guarded([&] {
        check_shape(d, m, ks);
        for (size_t i = 0; i < n * m; ++i)
            if (codes[i] >= ks) throw ArgError("code index out of range");
        if (n == 0) return;
        Session se(device);
        Workspace ws(se.s);
        const float* b = se.upload(ws, books, (size_t)ks * d);
        const uint8_t* c = se.upload(ws, codes, n * m);
        float* o = ws.alloc<float>(n * d);
        launch_pq_decode(c, n, d, b, m, ks, o, se.s);
        se.download(out_data, o, n * d);
        se.sync();
    });
}

int pqrr_dev_build_lut(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                       const float* x, size_t nx, float* out_lut) {
    return guarded([&] {
        check_shape(d, m, ks);
        if (nx == 0) return;
        Session se(device);
        Workspace ws(se.s);
        const float* b = se.upload(ws, books, (size_t)ks * d);
        const float* xx = se.upload(ws, x, nx * d);
        float* o = ws.alloc<float>(nx * m * ks);
        launch_build_lut(xx, nx, d, b, m, ks, o, se.s);
        se.download(out_lut, o, nx * m * ks);
        se.sync();
    });
}

int pqrr_dev_scan_topk(int device, const float* lut, uint32_t m, uint32_t ks, const uint8_t* codes,
                       size_t n, size_t kprime, uint32_t id_base, uint32_t* out_ids,
                       float* out_dists, size_t* out_count) {
    return guarded([&] {
        if (out_count) *out_count = 0;
        if (kprime == 0 || n == 0) return;
        Session se(device);
        Workspace ws(se.s);
        const float* l = se.upload(ws, lut, (size_t)m * ks);
        const uint8_t* c = se.upload(ws, codes, n * m);
        float* dist = ws.alloc<float>(n);
        launch_lut_scan_all(l, m, ks, c, n, dist, se.s);
        u64* keys = ws.alloc<u64>(n);
        u64* sorted = ws.alloc<u64>(n);
        lut_keys_kernel<<<nblk(n), 256, 0, se.s>>>(dist, n, id_base, keys);
        PQRR_LAUNCH_CHECK();
        count_launch();
        size_t tmp = 0;
        PQRR_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys, sorted, (int64_t)n, 0, 64, se.s));
        void* t = ws.alloc<uint8_t>(tmp);
        PQRR_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, keys, sorted, (int64_t)n, 0, 64, se.s));
        count_launch(8);
        const size_t cnt = std::min(kprime, n);
        std::vector<u64> h(cnt);
        se.download(h.data(), sorted, cnt);
        se.sync();
        for (size_t i = 0; i < cnt; ++i) {
            out_ids[i] = (uint32_t)(h[i] & 0xffffffffull);
            uint32_t b = (uint32_t)(h[i] >> 32);
            std::memcpy(&out_dists[i], &b, 4);
        }
        if (out_count) *out_count = cnt;
    });
}

int pqrr_dev_kmeans_train(int device, const float* points, size_t n, uint32_t dim, uint32_t k,
                          uint32_t iterations, uint64_t seed, uint32_t redo, float* out_centroids,
                          double* out_final_mse, double* out_trace) {
    return guarded([&] {
        if (k == 0) throw ArgError("k must be positive");
        if (n < k || n == 0) throw ArgError("insufficient training data");
        for (size_t i = 0; i < n * dim; ++i)
            if (!std::isfinite(points[i])) throw ArgError("VectorSet: non-finite value");
        Session se(device);
        Workspace ws(se.s);
        const float* p = se.upload(ws, points, n * dim);
        kmeans_device(p, n, dim, k, iterations, seed, redo, out_centroids, out_final_mse, out_trace,
                      se.s);
    });
}

int pqrr_dev_synth(int device, uint64_t seed, uint32_t clusters, uint32_t d, uint32_t set,
                   uint64_t row0, size_t n, uint8_t* out) {
    return guarded([&] {
        if (clusters == 0 || d == 0) throw ArgError("clusters and d must be positive");
        if (n == 0) return;
        Session se(device);
        Workspace ws(se.s);
        double* centers = ws.alloc<double>((size_t)clusters * d);
        launch_synth_centers(seed, clusters, d, centers, se.s);
        uint8_t* o = ws.alloc<uint8_t>(n * d);
        if (set == 0) throw ArgError("set 0 holds the mixture centres, not rows");
        launch_synth_rows(seed, set, row0, n, d, centers, clusters, o, se.s);
        se.download(out, o, n * d);
        se.sync();
    });
}

int pqrr_dev_index_create(int device, uint32_t d, uint32_t c, const float* coarse, uint32_t m,
                          const float* books, uint32_t mprime, const float* rbooks, uint32_t ks,
                          pqrr_dev_index** out) {
    return guarded([&] {
        *out = nullptr;
        check_shape(d, m, ks);
        if (c == 0) throw ArgError("c must be positive");
        if (c > 65536) throw UnsupportedError("more than 65536 coarse centroids");
        if (mprime && d % mprime) throw ArgError("dimension not divisible");
        if (mprime && !rbooks) throw ArgError("rbooks required when mprime > 0");
        DeviceGuard g(device);
        auto h = std::make_unique<pqrr_dev_index>();
        DevIndex& ix = h->ix;
        ix.device = device;
        ix.d = d;
        ix.c = c;
        ix.m = m;
        ix.mprime = mprime;
        ix.ks = ks;
        PQRR_CUDA(cudaStreamCreateWithFlags(&ix.stream, cudaStreamNonBlocking));
        // the search's random gathers (codes, refinement codes, ids, block
        // table) use 4-32 B of each miss: fetch 32-B sectors, not wider lines
        PQRR_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32));
        cudaMemPool_t pool;
        PQRR_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        PQRR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        ix.coarse.alloc((size_t)c * d);
        ix.books.alloc((size_t)ks * d);
        PQRR_CUDA(cudaMemcpy(ix.coarse.p, coarse, ix.coarse.bytes(), cudaMemcpyHostToDevice));
        PQRR_CUDA(cudaMemcpy(ix.books.p, books, ix.books.bytes(), cudaMemcpyHostToDevice));
        if (mprime) {
            ix.rbooks.alloc((size_t)ks * d);
            PQRR_CUDA(cudaMemcpy(ix.rbooks.p, rbooks, ix.rbooks.bytes(), cudaMemcpyHostToDevice));
        }
        ix.h_len.assign(c, 0);
        ix.h_off.assign(c + 1, 0);
        ix.list_len.alloc(c);
        ix.list_off.alloc(c + 1);
        PQRR_CUDA(cudaMemset(ix.list_len.p, 0, c * 4));
        PQRR_CUDA(cudaMemset(ix.list_off.p, 0, (c + 1) * 8));
        *out = h.release();
    });
}

int pqrr_dev_index_destroy(pqrr_dev_index* h) {
    return guarded([&] {
        if (!h) return;
        DeviceGuard g(h->ix.device);
        delete h;
    });
}

int pqrr_dev_add_u8(pqrr_dev_index* h, const uint8_t* y, size_t n, uint32_t id_base) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        const size_t chunk = 1u << 20;
        for (size_t o = 0; o < n; o += chunk) {
            const size_t cn = std::min(chunk, n - o);
            Workspace ws(ix.stream);
            uint8_t* dy = ws.alloc<uint8_t>(cn * ix.d);
            PQRR_CUDA(cudaMemcpyAsync(dy, y + o * ix.d, cn * ix.d, cudaMemcpyHostToDevice, ix.stream));
            stage_chunk(ix, nullptr, dy, cn, id_base + (uint32_t)o);
        }
        PQRR_CUDA(cudaStreamSynchronize(ix.stream));
    });
}

int pqrr_dev_add_f32(pqrr_dev_index* h, const float* y, size_t n, uint32_t id_base) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        for (size_t i = 0; i < n * ix.d; ++i)
            if (!std::isfinite(y[i])) throw ArgError("VectorSet: non-finite value");
        const size_t chunk = 1u << 20;
        for (size_t o = 0; o < n; o += chunk) {
            const size_t cn = std::min(chunk, n - o);
            Workspace ws(ix.stream);
            float* dy = ws.alloc<float>(cn * ix.d);
            PQRR_CUDA(cudaMemcpyAsync(dy, y + o * ix.d, cn * ix.d * 4, cudaMemcpyHostToDevice, ix.stream));
            stage_chunk(ix, dy, nullptr, cn, id_base + (uint32_t)o);
        }
        PQRR_CUDA(cudaStreamSynchronize(ix.stream));
    });
}

int pqrr_dev_add_synthetic(pqrr_dev_index* h, uint64_t seed, uint32_t clusters, uint64_t row0,
                           size_t n, uint32_t id_base) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        Workspace wsc(ix.stream);
        double* centers = wsc.alloc<double>((size_t)clusters * ix.d);
        launch_synth_centers(seed, clusters, ix.d, centers, ix.stream);
        const size_t chunk = 1u << 21;
        for (size_t o = 0; o < n; o += chunk) {
            const size_t cn = std::min(chunk, n - o);
            Workspace ws(ix.stream);
            uint8_t* dy = ws.alloc<uint8_t>(cn * ix.d);
            launch_synth_rows(seed, 2, row0 + o, cn, ix.d, centers, clusters, dy, ix.stream);
            stage_chunk(ix, nullptr, dy, cn, id_base + (uint32_t)o);
        }
        PQRR_CUDA(cudaStreamSynchronize(ix.stream));
    });
}

int pqrr_dev_finalize(pqrr_dev_index* h) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        finalize(ix);
    });
}

int pqrr_dev_index_get_info(pqrr_dev_index* h, pqrr_dev_index_info* out) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        finalize(ix);
        out->n = ix.n;
        out->slots = ix.slots;
        out->d = ix.d;
        out->c = ix.c;
        out->m = ix.m;
        out->mprime = ix.mprime;
        out->ks = ix.ks;
        out->max_list_len = ix.max_len();
        out->device_bytes = ix.coarse.bytes() + ix.books.bytes() + ix.rbooks.bytes() +
                            ix.codes.bytes() + ix.rcodes.bytes() + ix.ids.bytes() +
                            ix.list_off.bytes() + ix.list_len.bytes() + ix.id_map.bytes();
    });
}

int pqrr_dev_export_lists(pqrr_dev_index* h, uint64_t* offsets, uint32_t* ids, uint8_t* codes,
                          uint8_t* rcodes) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        finalize(ix);
        std::vector<uint64_t> uoff(ix.c + 1, 0);
        for (uint32_t l = 0; l < ix.c; ++l) uoff[l + 1] = uoff[l] + ix.h_len[l];
        if (offsets) std::memcpy(offsets, uoff.data(), (ix.c + 1) * 8);
        if (ix.n == 0) return;
        Workspace ws(ix.stream);
        uint64_t* d_uoff = ws.alloc<uint64_t>(ix.c + 1);
        PQRR_CUDA(cudaMemcpyAsync(d_uoff, uoff.data(), (ix.c + 1) * 8, cudaMemcpyHostToDevice, ix.stream));
        // the device order inside a list is parity-balanced; the reference
        // layout is id-ascending (ivf_index.hpp:15-16): re-sort per list
        const size_t S = ix.slots;
        std::vector<uint64_t> h_end(ix.c);
        for (uint32_t l = 0; l < ix.c; ++l) h_end[l] = ix.h_off[l] + ix.h_len[l];
        uint64_t* d_end = ws.alloc<uint64_t>(ix.c);
        PQRR_CUDA(cudaMemcpyAsync(d_end, h_end.data(), ix.c * 8, cudaMemcpyHostToDevice, ix.stream));
        uint32_t* k0 = ws.alloc<uint32_t>(S);
        uint32_t* v0 = ws.alloc<uint32_t>(S);
        uint32_t* k1 = ws.alloc<uint32_t>(S);
        uint32_t* perm = ws.alloc<uint32_t>(S);
        launch_list_id_keys(ix.list_off.p, ix.list_len.p, ix.c, ix.ids.p, k0, v0, ix.stream);
        segmented_sort_pairs(k0, k1, v0, perm, S, ix.c, ix.list_off.p, d_end, 32, ix.stream);
        uint32_t* t_ids = ws.alloc<uint32_t>(S);
        uint8_t* t_codes = ws.alloc<uint8_t>(S * ix.m);
        uint8_t* t_rcodes = ws.alloc<uint8_t>(S * std::max<uint32_t>(ix.mprime, 1));
        launch_gather_layout(ix.list_off.p, ix.list_len.p, ix.c, perm, ix.codes.p, ix.ids.p,
                             ix.rcodes.p, ix.m, ix.mprime, t_codes, t_ids, t_rcodes, ix.stream);
        uint32_t* o_ids = ws.alloc<uint32_t>(ix.n);
        uint8_t* o_codes = ws.alloc<uint8_t>(ix.n * ix.m);
        uint8_t* o_rcodes = ws.alloc<uint8_t>(ix.n * std::max<uint32_t>(ix.mprime, 1));
        compact_lists_kernel<<<ix.c, 256, 0, ix.stream>>>(ix.list_off.p, ix.list_len.p, d_uoff, t_ids,
                                                         t_codes, t_rcodes, ix.m, ix.mprime,
                                                         o_ids, o_codes, o_rcodes);
        PQRR_LAUNCH_CHECK();
        count_launch();
        if (ids) PQRR_CUDA(cudaMemcpyAsync(ids, o_ids, ix.n * 4, cudaMemcpyDeviceToHost, ix.stream));
        if (codes) PQRR_CUDA(cudaMemcpyAsync(codes, o_codes, ix.n * ix.m, cudaMemcpyDeviceToHost, ix.stream));
        if (rcodes && ix.mprime)
            PQRR_CUDA(cudaMemcpyAsync(rcodes, o_rcodes, ix.n * ix.mprime, cudaMemcpyDeviceToHost, ix.stream));
        PQRR_CUDA(cudaStreamSynchronize(ix.stream));
    });
}

// Device-pointer API, small batches: the graph works on index-owned buffers
// (stable addresses: one graph per shape whatever pointers the caller passes,
// e.g. fresh torch tensors every call); queries are copied in and results out
// with device-to-device copies on the index stream around the replay.
struct DevStage {
    const uint8_t* dq;
    uint32_t* oi;
    float* od;
    uint32_t* oc;
    size_t width;
};
static DevStage stage_device_batch(DevIndex& ix, const uint8_t* d_queries, size_t nq, size_t kprime, size_t k) {
    cudaStream_t s = ix.stream;
    auto grow = [&](auto& b, size_t n) {
        if (b.n < n) {
            PQRR_CUDA(cudaStreamSynchronize(s));
            b.alloc(n + n / 2);
        }
    };
    const size_t width = k ? k : kprime;
    grow(ix.sg_xq, nq * ix.d);
    grow(ix.sg_qu8, nq * ix.d);
    grow(ix.sg_out, 2 * nq * width + nq);
    PQRR_CUDA(cudaMemcpyAsync(ix.sg_qu8.p, d_queries, nq * ix.d, cudaMemcpyDeviceToDevice, s));
    return DevStage{ix.sg_qu8.p, ix.sg_out.p, reinterpret_cast<float*>(ix.sg_out.p + nq * width),
                    ix.sg_out.p + 2 * nq * width, width};
}
static void unstage_device_batch(DevIndex& ix, const DevStage& st, size_t nq, uint32_t* d_ids, float* d_dists,
                                 uint32_t* d_counts) {
    cudaStream_t s = ix.stream;
    PQRR_CUDA(cudaMemcpyAsync(d_ids, st.oi, nq * st.width * 4, cudaMemcpyDeviceToDevice, s));
    PQRR_CUDA(cudaMemcpyAsync(d_dists, st.od, nq * st.width * 4, cudaMemcpyDeviceToDevice, s));
    PQRR_CUDA(cudaMemcpyAsync(d_counts, st.oc, nq * 4, cudaMemcpyDeviceToDevice, s));
}

static int search_host(pqrr_dev_index* h, const float* qf, const uint8_t* qu, size_t nq, uint32_t w,
                       size_t kprime, size_t k, uint32_t* out_ids, float* out_dists,
                       uint32_t* out_counts) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (nq == 0) return;
        cudaStream_t s = ix.stream;
        // index-owned staging with stable addresses (the captured graphs of
        // small batches bake them in); grows, never shrinks
        const size_t width = k ? k : kprime;
        auto grow = [&](auto& b, size_t n) {
            if (b.n < n) {
                PQRR_CUDA(cudaStreamSynchronize(s));
                b.alloc(n + n / 2);
            }
        };
        auto grow_pinned = [&](void*& p, size_t& have, size_t need) {
            if (have >= need) return;
            PQRR_CUDA(cudaStreamSynchronize(s));
            if (p) cudaFreeHost(p);
            p = nullptr;
            have = 0;
            PQRR_CUDA(cudaMallocHost(&p, need + need / 2));
            have = need + need / 2;
        };
        const size_t out_words = 2 * nq * width + nq;
        grow(ix.sg_xq, nq * ix.d);
        grow(ix.sg_out, out_words);
        if (!qf) grow(ix.sg_qu8, nq * ix.d);
        float* xq = ix.sg_xq.p;
        const uint8_t* dq = qf ? nullptr : ix.sg_qu8.p;
        uint32_t* oi = ix.sg_out.p;
        float* od = reinterpret_cast<float*>(ix.sg_out.p + nq * width);
        uint32_t* oc = ix.sg_out.p + 2 * nq * width;
        if (qf)
            for (size_t i = 0; i < nq * ix.d; ++i)
                if (!std::isfinite(qf[i])) throw ArgError("VectorSet: non-finite value");
        // small batches: queries and results pass through pinned staging and
        // the captured graph does both copies (one launch and one
        // synchronisation per search instead of four copies around it)
        const size_t in_bytes = nq * ix.d * (qf ? 4 : 1);
        const bool staged = ix.graph_enabled && nq <= kFastMaxQueries && out_words * 4 <= (256u << 10);
        HostStage hs{};
        if (staged) {
            grow_pinned(ix.h_in, ix.h_in_bytes, in_bytes);
            grow_pinned(ix.h_out, ix.h_out_bytes, out_words * 4);
            std::memcpy(ix.h_in, qf ? (const void*)qf : (const void*)qu, in_bytes);
            hs = HostStage{ix.h_in, qf ? (void*)xq : (void*)ix.sg_qu8.p, in_bytes, ix.h_out, ix.sg_out.p,
                           out_words * 4};
        } else {
            PQRR_CUDA(cudaMemcpyAsync(qf ? (void*)xq : (void*)ix.sg_qu8.p, qf ? (const void*)qf : (const void*)qu,
                                      in_bytes, cudaMemcpyHostToDevice, s));
        }
        ix.q_u8 = qf == nullptr;
        bool delivered = false;
        try {
            delivered = search_device(ix, xq, nq, w, kprime, k, oi, od, oc, dq, staged ? &hs : nullptr);
        } catch (...) {
            ix.q_u8 = false;
            throw;
        }
        ix.q_u8 = false;
        if (delivered) {
            const uint32_t* ho = static_cast<const uint32_t*>(ix.h_out);
            std::memcpy(out_ids, ho, nq * width * 4);
            std::memcpy(out_dists, ho + nq * width, nq * width * 4);
            std::memcpy(out_counts, ho + 2 * nq * width, nq * 4);
            return;
        }
        PQRR_CUDA(cudaMemcpyAsync(out_ids, oi, nq * width * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaMemcpyAsync(out_dists, od, nq * width * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaMemcpyAsync(out_counts, oc, nq * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaStreamSynchronize(s));
    });
}

int pqrr_dev_search_u8(pqrr_dev_index* h, const uint8_t* queries, size_t nq, uint32_t w,
                       size_t kprime, size_t k, uint32_t* out_ids, float* out_dists,
                       uint32_t* out_counts) {
    return search_host(h, nullptr, queries, nq, w, kprime, k, out_ids, out_dists, out_counts);
}

int pqrr_dev_search_f32(pqrr_dev_index* h, const float* queries, size_t nq, uint32_t w,
                        size_t kprime, size_t k, uint32_t* out_ids, float* out_dists,
                        uint32_t* out_counts) {
    return search_host(h, queries, nullptr, nq, w, kprime, k, out_ids, out_dists, out_counts);
}

static void stream_join(cudaStream_t from, cudaStream_t to) {
    cudaEvent_t e;
    PQRR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    PQRR_CUDA(cudaEventRecord(e, from));
    PQRR_CUDA(cudaStreamWaitEvent(to, e, 0));
    cudaEventDestroy(e);
}

int pqrr_dev_search_u8_device(pqrr_dev_index* h, const uint8_t* d_queries, size_t nq, uint32_t w,
                              size_t kprime, size_t k, uint32_t* d_out_ids, float* d_out_dists,
                              uint32_t* d_out_counts, void* stream) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (nq == 0) return;
        // NULL = the legacy default stream (torch's default stream has handle 0)
        cudaStream_t user = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
        cudaStream_t s = ix.stream;
        stream_join(user, s);
        const bool small = ix.graph_enabled && nq <= kFastMaxQueries;
        if (ix.sg_xq.n < nq * ix.d) {
            PQRR_CUDA(cudaStreamSynchronize(s));
            ix.sg_xq.alloc(nq * ix.d + nq * ix.d / 2);
        }
        ix.q_u8 = true;
        try {
            if (small) {
                validate_search(ix, w, kprime, k);  // before anything is staged
                const DevStage st = stage_device_batch(ix, d_queries, nq, kprime, k);
                search_device(ix, ix.sg_xq.p, nq, w, kprime, k, st.oi, st.od, st.oc, st.dq);
                unstage_device_batch(ix, st, nq, d_out_ids, d_out_dists, d_out_counts);
            } else {
                search_device(ix, ix.sg_xq.p, nq, w, kprime, k, d_out_ids, d_out_dists, d_out_counts, d_queries);
            }
        } catch (...) {
            ix.q_u8 = false;
            throw;
        }
        ix.q_u8 = false;
        stream_join(s, user);
    });
}


int pqrr_dev_search_u8_enqueue(pqrr_dev_index* h, const uint8_t* d_queries, size_t nq, uint32_t w,
                               size_t kprime, size_t k, uint32_t* d_out_ids, float* d_out_dists,
                               uint32_t* d_out_counts, void* stream) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (ix.pending.on) throw ArgError("an enqueued search is pending: call pqrr_dev_search_finish first");
        validate_search(ix, w, kprime, k);
        if (nq == 0) return;
        cudaStream_t user = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
        cudaStream_t s = ix.stream;
        if (!ix.graph_enabled || nq > kFastMaxQueries)
            throw UnsupportedError("batch shape outside the enqueue-only path: use pqrr_dev_search_u8_device");
        stream_join(user, s);
        ix.q_u8 = true;
        bool ok = false;
        try {
            const DevStage st = stage_device_batch(ix, d_queries, nq, kprime, k);
            ok = search_enqueue(ix, st.dq, ix.sg_xq.p, nq, w, (uint32_t)kprime, (uint32_t)k, st.oi, st.od, st.oc);
            if (ok) unstage_device_batch(ix, st, nq, d_out_ids, d_out_dists, d_out_counts);
        } catch (...) {
            ix.q_u8 = false;
            throw;
        }
        ix.q_u8 = false;
        if (!ok) throw UnsupportedError("batch shape outside the enqueue-only path: use pqrr_dev_search_u8_device");
        stream_join(s, user);
        ix.pending = DevIndex::Pending{true, d_queries, nq, kprime, k, w, d_out_ids, d_out_dists, d_out_counts, user};
    });
}

int pqrr_dev_index_set_graph(pqrr_dev_index* h, int enabled) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        if (ix.pending.on) throw ArgError("an enqueued search is pending: call pqrr_dev_search_finish first");
        ix.graph_enabled = enabled != 0;
        if (!ix.graph_enabled && !ix.graphs.empty()) {  // release the cached graphs and their scratch
            DeviceGuard g(ix.device);
            PQRR_CUDA(cudaStreamSynchronize(ix.stream));
            ix.drop_graphs();
        }
    });
}

int pqrr_dev_search_finish(pqrr_dev_index* h) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (!ix.pending.on) return;
        const DevIndex::Pending p = ix.pending;
        ix.pending.on = false;
        cudaStream_t s = ix.stream;
        PQRR_CUDA(cudaStreamSynchronize(s));
        if (search_fast_outcome(ix, (uint32_t)p.k) == 0) return;
        // rare: a threshold failed its exactness check (or a coarse candidate
        // set overflowed); redo the batch with per-row retries, ordered after
        // whatever the caller queued behind the first attempt
        stream_join(p.user, s);
        ix.q_u8 = true;
        try {
            launch_widen_u8(p.d_queries, ix.sg_xq.p, p.nq * ix.d, s);
            search_sync(ix, ix.sg_xq.p, p.nq, p.w, p.kprime, p.k, p.oi, p.od, p.oc);
        } catch (...) {
            ix.q_u8 = false;
            throw;
        }
        ix.q_u8 = false;
        stream_join(s, p.user);
    });
}

int pqrr_dev_rerank_owned_u8_device(pqrr_dev_index* h, const uint8_t* d_queries, size_t nq,
                                    const uint32_t* d_sl_ids, const uint32_t* d_sl_counts,
                                    size_t sl_stride, size_t k, uint32_t* d_out_ids,
                                    float* d_out_dists, uint32_t* d_out_counts, void* stream) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (ix.mprime == 0) throw ArgError("re-ranking needs refinement codes (mprime > 0)");
        if (nq == 0 || k == 0) return;
        if (sl_stride > 16384) throw UnsupportedError("shortlists above 16384 entries");
        ensure_id_map(ix);
        cudaStream_t user = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
        cudaStream_t s = ix.stream;
        stream_join(user, s);
        Workspace ws(s);
        float* xq = ws.alloc<float>(nq * ix.d);
        launch_widen_u8(d_queries, xq, nq * ix.d, s);
        u64* key = ws.alloc<u64>(nq * sl_stride);
        uint32_t* pos = ws.alloc<uint32_t>(nq * sl_stride);
        uint32_t* cnt = ws.alloc<uint32_t>(nq);
        owned_shortlist_kernel<<<nblk(nq * 32), 256, 0, s>>>(d_sl_ids, d_sl_counts, nq,
                                                             (uint32_t)sl_stride, ix.id_map.p,
                                                             (uint32_t)id_lo_of(ix),
                                                             (uint32_t)ix.id_map.n, key, pos, cnt);
        PQRR_LAUNCH_CHECK();
        count_launch();
        launch_rerank(reinterpret_cast<uint64_t*>(key), pos, cnt, (uint32_t)sl_stride, nq, xq, ix.d,
                      ix.block_list.p, ix.coarse.p, ix.codes.p, ix.books.p, ix.m, ix.rcodes.p,
                      ix.rbooks.p, ix.mprime, ix.ks, (uint32_t)k, d_out_ids, d_out_dists,
                      d_out_counts, s);
        stream_join(s, user);
    });
}

static int rerank_host(pqrr_dev_index* h, const float* qf, const uint8_t* qu, size_t nq,
                       const uint32_t* sl_ids, const uint32_t* sl_counts, size_t sl_stride, size_t k,
                       uint32_t* out_ids, float* out_dists) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (ix.mprime == 0) throw ArgError("re-ranking needs refinement codes (mprime > 0)");
        for (size_t q = 0; q < nq; ++q)
            if (k > sl_counts[q]) throw ShortlistError();
        if (nq == 0 || k == 0) return;
        if (sl_stride > 16384) throw UnsupportedError("shortlists above 16384 entries");
        ensure_id_map(ix);
        cudaStream_t s = ix.stream;
        Workspace ws(s);
        float* xq = ws.alloc<float>(nq * ix.d);
        if (qf) {
            PQRR_CUDA(cudaMemcpyAsync(xq, qf, nq * ix.d * 4, cudaMemcpyHostToDevice, s));
        } else {
            uint8_t* dq = ws.alloc<uint8_t>(nq * ix.d);
            PQRR_CUDA(cudaMemcpyAsync(dq, qu, nq * ix.d, cudaMemcpyHostToDevice, s));
            launch_widen_u8(dq, xq, nq * ix.d, s);
        }
        uint32_t* ids = ws.alloc<uint32_t>(nq * sl_stride);
        PQRR_CUDA(cudaMemcpyAsync(ids, sl_ids, nq * sl_stride * 4, cudaMemcpyHostToDevice, s));
        uint32_t* cnt = ws.alloc<uint32_t>(nq);
        PQRR_CUDA(cudaMemcpyAsync(cnt, sl_counts, nq * 4, cudaMemcpyHostToDevice, s));
        u64* key = ws.alloc<u64>(nq * sl_stride);
        uint32_t* pos = ws.alloc<uint32_t>(nq * sl_stride);
        unsigned* bad = ws.zeros<unsigned>(1);
        ids_to_shortlist<<<nblk(nq * sl_stride), 256, 0, s>>>(ids, ix.id_map.p, nq * sl_stride, key, pos,
                                                               bad, (uint32_t)id_lo_of(ix),
                                                               (uint32_t)ix.id_map.n);
        PQRR_LAUNCH_CHECK();
        count_launch();
        // unused tail entries of a row may hold junk ids: only the first cnt[q] are read
        uint32_t* oi = ws.alloc<uint32_t>(nq * k);
        float* od = ws.alloc<float>(nq * k);
        uint32_t* oc = ws.alloc<uint32_t>(nq);
        launch_rerank(reinterpret_cast<uint64_t*>(key), pos, cnt, (uint32_t)sl_stride, nq, xq, ix.d,
                      ix.block_list.p, ix.coarse.p, ix.codes.p, ix.books.p, ix.m, ix.rcodes.p,
                      ix.rbooks.p, ix.mprime, ix.ks, (uint32_t)k, oi, od, oc, s);
        PQRR_CUDA(cudaMemcpyAsync(out_ids, oi, nq * k * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaMemcpyAsync(out_dists, od, nq * k * 4, cudaMemcpyDeviceToHost, s));
        unsigned h_bad = 0;
        PQRR_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaStreamSynchronize(s));
        if (h_bad) throw ArgError("shortlist id not in the index");
    });
}

int pqrr_dev_rerank_u8(pqrr_dev_index* h, const uint8_t* queries, size_t nq, const uint32_t* sl_ids,
                       const uint32_t* sl_counts, size_t sl_stride, size_t k, uint32_t* out_ids,
                       float* out_dists) {
    return rerank_host(h, nullptr, queries, nq, sl_ids, sl_counts, sl_stride, k, out_ids, out_dists);
}

int pqrr_dev_rerank_f32(pqrr_dev_index* h, const float* queries, size_t nq, const uint32_t* sl_ids,
                        const uint32_t* sl_counts, size_t sl_stride, size_t k, uint32_t* out_ids,
                        float* out_dists) {
    return rerank_host(h, queries, nullptr, nq, sl_ids, sl_counts, sl_stride, k, out_ids, out_dists);
}

int pqrr_dev_lookup_ids(pqrr_dev_index* h, const uint32_t* ids, size_t n, uint32_t* out_list,
                        uint8_t* out_codes, uint8_t* out_rcodes) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (n == 0) return;
        ensure_id_map(ix);
        cudaStream_t s = ix.stream;
        Workspace ws(s);
        uint32_t* d_ids = ws.alloc<uint32_t>(n);
        PQRR_CUDA(cudaMemcpyAsync(d_ids, ids, n * 4, cudaMemcpyHostToDevice, s));
        uint32_t* o_l = out_list ? ws.alloc<uint32_t>(n) : nullptr;
        uint8_t* o_c = out_codes ? ws.alloc<uint8_t>(n * ix.m) : nullptr;
        uint8_t* o_r = (out_rcodes && ix.mprime) ? ws.alloc<uint8_t>(n * ix.mprime) : nullptr;
        lookup_ids_kernel<<<nblk(n), 256, 0, s>>>(d_ids, n, (uint32_t)id_lo_of(ix), (uint32_t)ix.id_map.n,
                                                  ix.id_map.p, ix.list_off.p, ix.c, ix.codes.p, ix.m,
                                                  ix.rcodes.p, ix.mprime, o_l, o_c, o_r);
        PQRR_LAUNCH_CHECK();
        count_launch();
        if (o_l) PQRR_CUDA(cudaMemcpyAsync(out_list, o_l, n * 4, cudaMemcpyDeviceToHost, s));
        if (o_c) PQRR_CUDA(cudaMemcpyAsync(out_codes, o_c, n * ix.m, cudaMemcpyDeviceToHost, s));
        if (o_r) PQRR_CUDA(cudaMemcpyAsync(out_rcodes, o_r, n * ix.mprime, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaStreamSynchronize(s));
    });
}

int pqrr_dev_reconstruct(pqrr_dev_index* h, const uint32_t* ids, size_t n, float* out) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (n == 0) return;
        ensure_id_map(ix);
        for (size_t i = 0; i < n; ++i)
            if (ids[i] >= ix.next_id || ids[i] < id_lo_of(ix)) throw ArgError("id out of range");
        cudaStream_t s = ix.stream;
        Workspace ws(s);
        uint32_t* d_ids = ws.alloc<uint32_t>(n);
        PQRR_CUDA(cudaMemcpyAsync(d_ids, ids, n * 4, cudaMemcpyHostToDevice, s));
        float* o = ws.alloc<float>(n * ix.d);
        reconstruct_kernel<<<nblk(n * ix.d), 256, 0, s>>>(d_ids, n, (uint32_t)id_lo_of(ix), ix.id_map.p, ix.list_off.p, ix.c, ix.d,
                                                           ix.coarse.p, ix.codes.p, ix.books.p, ix.m,
                                                           ix.rcodes.p, ix.rbooks.p, ix.mprime, ix.ks, o);
        PQRR_LAUNCH_CHECK();
        count_launch();
        PQRR_CUDA(cudaMemcpyAsync(out, o, n * ix.d * 4, cudaMemcpyDeviceToHost, s));
        PQRR_CUDA(cudaStreamSynchronize(s));
    });
}

int pqrr_dev_export_lists_subset(pqrr_dev_index* h, const uint32_t* lists, uint32_t nl,
                                 uint64_t* offsets, uint32_t* ids, uint8_t* codes,
                                 uint8_t* rcodes) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        finalize(ix);
        offsets[0] = 0;
        for (uint32_t i = 0; i < nl; ++i) {
            if (lists[i] >= ix.c) throw ArgError("list out of range");
            offsets[i + 1] = offsets[i] + ix.h_len[lists[i]];
        }
        if (!ids && !codes && !rcodes) return;
        const uint32_t m = ix.m, mp = ix.mprime;
        std::vector<uint32_t> t_ids, perm;
        std::vector<uint8_t> t_codes, t_rc;
        for (uint32_t i = 0; i < nl; ++i) {
            const uint32_t l = lists[i], len = ix.h_len[l];
            const uint64_t o = ix.h_off[l];
            if (!len) continue;
            t_ids.resize(len);
            t_codes.resize((size_t)len * m);
            t_rc.resize((size_t)len * mp);
            PQRR_CUDA(cudaMemcpy(t_ids.data(), ix.ids.p + o, (size_t)len * 4, cudaMemcpyDeviceToHost));
            PQRR_CUDA(cudaMemcpy(t_codes.data(), ix.codes.p + o * m, (size_t)len * m,
                                 cudaMemcpyDeviceToHost));
            if (mp && rcodes)
                PQRR_CUDA(cudaMemcpy(t_rc.data(), ix.rcodes.p + o * mp, (size_t)len * mp,
                                     cudaMemcpyDeviceToHost));
            // the device order inside a list is parity-paired: back to id order
            perm.resize(len);
            for (uint32_t r = 0; r < len; ++r) perm[r] = r;
            std::sort(perm.begin(), perm.end(), [&](uint32_t a, uint32_t b) { return t_ids[a] < t_ids[b]; });
            const uint64_t d0 = offsets[i];
            for (uint32_t r = 0; r < len; ++r) {
                const uint32_t sidx = perm[r];
                if (ids) ids[d0 + r] = t_ids[sidx];
                if (codes) std::memcpy(codes + (d0 + r) * m, &t_codes[(size_t)sidx * m], m);
                if (rcodes && mp) std::memcpy(rcodes + (d0 + r) * mp, &t_rc[(size_t)sidx * mp], mp);
            }
        }
    });
}

int pqrr_dev_export_codebooks(pqrr_dev_index* h, float* coarse, float* books, float* rbooks) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (coarse) PQRR_CUDA(cudaMemcpy(coarse, ix.coarse.p, ix.coarse.bytes(), cudaMemcpyDeviceToHost));
        if (books) PQRR_CUDA(cudaMemcpy(books, ix.books.p, ix.books.bytes(), cudaMemcpyDeviceToHost));
        if (rbooks && ix.mprime)
            PQRR_CUDA(cudaMemcpy(rbooks, ix.rbooks.p, ix.rbooks.bytes(), cudaMemcpyDeviceToHost));
    });
}

int pqrr_dev_load_lists(pqrr_dev_index* h, const uint64_t* offsets, const uint32_t* ids,
                        const uint8_t* codes, const uint8_t* rcodes) {
    return guarded([&] {
        DevIndex& ix = h->ix;
        std::lock_guard<std::mutex> lk(ix.mu);
        DeviceGuard g(ix.device);
        if (ix.n || ix.st_n) throw ArgError("load_lists needs an empty index");
        if (ix.mprime && !rcodes) throw ArgError("rcodes required when mprime > 0");
        const uint64_t n = offsets[ix.c];
        if (n == 0) return;
        if (n > 0xffffffffull) throw UnsupportedError("more than 2^32 entries on one device");
        std::vector<uint32_t> assign(n);
        uint64_t max_id = 0, min_id = ~0ull;
        for (uint32_t l = 0; l < ix.c; ++l) {
            if (offsets[l + 1] < offsets[l]) throw ArgError("corrupt file");
            for (uint64_t i = offsets[l]; i < offsets[l + 1]; ++i) {
                assign[i] = l;
                if (i > offsets[l] && ids[i] <= ids[i - 1]) throw ArgError("corrupt file");
                max_id = std::max<uint64_t>(max_id, ids[i]);
                min_id = std::min<uint64_t>(min_id, ids[i]);
            }
        }
        // every id once across all lists (the partition invariant of
        // ivf_index.hpp:27-36), code bytes inside the code books
        {
            std::vector<uint64_t> seen((max_id - min_id) / 64 + 1, 0);
            for (uint64_t i = 0; i < n; ++i) {
                const uint64_t b = ids[i] - min_id;
                if (seen[b >> 6] >> (b & 63) & 1) throw ArgError("corrupt file");
                seen[b >> 6] |= 1ull << (b & 63);
            }
        }
        if (ix.ks < 256) {
            for (uint64_t i = 0; i < n * ix.m; ++i)
                if (codes[i] >= ix.ks) throw ArgError("corrupt file");
            if (ix.mprime)
                for (uint64_t i = 0; i < n * ix.mprime; ++i)
                    if (rcodes[i] >= ix.ks) throw ArgError("corrupt file");
        }
        grow_staging(ix, n);
        cudaStream_t s = ix.stream;
        PQRR_CUDA(cudaMemcpyAsync(ix.st_assign.p, assign.data(), n * 4, cudaMemcpyHostToDevice, s));
        PQRR_CUDA(cudaMemcpyAsync(ix.st_ids.p, ids, n * 4, cudaMemcpyHostToDevice, s));
        PQRR_CUDA(cudaMemcpyAsync(ix.st_codes.p, codes, n * ix.m, cudaMemcpyHostToDevice, s));
        if (ix.mprime)
            PQRR_CUDA(cudaMemcpyAsync(ix.st_rcodes.p, rcodes, n * ix.mprime, cudaMemcpyHostToDevice, s));
        ix.st_n = n;
        ix.next_id = max_id + 1;
        ix.id_lo = min_id;
        finalize(ix);
    });
}

// Kernel seam of the two-phase LUT pass's tensor-core bound (k_bound.cu), for
// tests: lower bounds of sum_j min_c l2_sq(x_q - C_l, B_j[c]) of the pairs
// (q, probes[q w + r]) with r >= R1, into out[q w + r] (other slots untouched).
int pqrr_dev_pair_bounds(int device, const float* queries, size_t nq, uint32_t d, const float* coarse,
                         uint32_t c, const float* books, uint32_t m, uint32_t ks, const uint32_t* probes,
                         uint32_t w, uint32_t R1, float* out) {
    return guarded([&] {
        if (!far_bound_supported(d, m, ks)) throw UnsupportedError("pair bounds need d = 128, m = 8, ks = 256");
        if (R1 > w) throw ArgError("R1 must be <= w");
        for (size_t i = 0; i < nq * (size_t)w; ++i)
            if (probes[i] >= c) throw ArgError("probe out of range");
        if (nq == 0 || w == R1) return;
        Session se(device);
        Workspace ws(se.s);
        const float* dq = se.upload(ws, queries, nq * d);
        const float* dc = se.upload(ws, coarse, (size_t)c * d);
        const float* db = se.upload(ws, books, (size_t)ks * d);
        const uint32_t* dp = se.upload(ws, probes, nq * (size_t)w);
        float* o = ws.alloc<float>(nq * (size_t)w);
        PQRR_CUDA(cudaMemsetAsync(o, 0, nq * (size_t)w * 4, se.s));
        launch_far_bound(dq, dc, db, dp, nq, w, R1, o, se.s);
        se.download(out, o, nq * (size_t)w);
        se.sync();
    });
}

// compute_groundtruth / exact_search (eval.hpp:13-19) for u8 vectors: the
// exact k nearest base rows of every query under (dist, id), on the integer
// tensor cores (k_exact.cu).  Base rows from host memory, or generated on the
// device (the synthetic base set, rows [row0, row0 + n), ids = row index).
static int exact_knn_impl(int device, const uint8_t* base, uint64_t seed, uint32_t clusters, uint64_t row0,
                          size_t n, const uint8_t* queries, size_t nq, uint32_t d, uint32_t k,
                          uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    return guarded([&] {
        if (!exact_knn_supported(d)) throw UnsupportedError("exact k-NN on the device needs d = 128");
        if (k == 0 || k > 16384) throw UnsupportedError("exact k-NN supports 1 <= k <= 16384");
        if (n > 0xffffffffull || row0 + n > 0x100000000ull) throw ArgError("ids exceed the 32-bit id space");
        if (nq == 0) return;
        Session se(device);
        Workspace ws(se.s);
        const uint8_t* dq = se.upload(ws, queries, nq * d);
        double* centers = nullptr;
        if (!base) {
            if (clusters == 0) throw ArgError("clusters must be positive");
            centers = ws.alloc<double>((size_t)clusters * d);
            launch_synth_centers(seed, clusters, d, centers, se.s);
        }
        auto fetch = [&](uint64_t r0, uint32_t nb, uint8_t* dst) {
            if (base)
                PQRR_CUDA(cudaMemcpyAsync(dst, base + r0 * d, (size_t)nb * d, cudaMemcpyHostToDevice, se.s));
            else
                launch_synth_rows(seed, 2, row0 + r0, nb, d, centers, clusters, dst, se.s);
        };
        if (n == 0) {
            for (size_t q = 0; q < nq; ++q) out_counts[q] = 0;
            return;
        }
        exact_knn_u8(dq, nq, n, base ? 0 : row0, k, fetch, out_ids, out_dists, out_counts, se.s);
    });
}

int pqrr_dev_exact_knn_u8(int device, const uint8_t* base, size_t n, const uint8_t* queries, size_t nq,
                          uint32_t d, uint32_t k, uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    if (!base && n) return report_error(PQRR_EINVAL, "base is NULL");
    return exact_knn_impl(device, base, 0, 0, 0, n, queries, nq, d, k, out_ids, out_dists, out_counts);
}

int pqrr_dev_exact_knn_synthetic(int device, uint64_t seed, uint32_t clusters, uint64_t row0, size_t n,
                                 const uint8_t* queries, size_t nq, uint32_t k, uint32_t* out_ids,
                                 float* out_dists, uint32_t* out_counts) {
    return exact_knn_impl(device, nullptr, seed, clusters, row0, n, queries, nq, 128, k, out_ids, out_dists,
                          out_counts);
}

// ---------------------------------------------------------------- ADC / ADC+R
// The exhaustive index (adc_index.hpp:13-31) is the IVF machinery with ONE
// all-zero coarse centroid: y - 0 = y and x - 0 = x exactly in fp32, and
// (0 + p) + q_r = p + q_r, so codes, LUTs, ADC sums, refinement residuals and
// re-rank distances are the ADC / ADC+R ones bit for bit.
int pqrr_dev_adc_index_create(int device, uint32_t d, uint32_t m, const float* books,
                              uint32_t mprime, const float* rbooks, uint32_t ks,
                              pqrr_dev_index** out) {
    std::vector<float> zero(std::max<uint32_t>(d, 1), 0.f);
    return pqrr_dev_index_create(device, d, 1, zero.data(), m, books, mprime, rbooks, ks, out);
}

int pqrr_dev_refine_train(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                          const float* training, size_t n, uint32_t mprime, uint32_t iterations,
                          uint64_t seed, float* out_rbooks) {
    std::vector<float> zero(std::max<uint32_t>(d, 1), 0.f);
    return pqrr_dev_ivf_refine_train(device, zero.data(), 1, books, d, m, ks, training, n, mprime,
                                     iterations, seed, out_rbooks);
}

int pqrr_dev_residual(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                      const float* y, size_t n, float* out) {
    return guarded([&] {
        check_shape(d, m, ks);
        if (n == 0) return;
        Session se(device);
        Workspace ws(se.s);
        const float* b = se.upload(ws, books, (size_t)ks * d);
        const float* dy = se.upload(ws, y, n * d);
        uint8_t* c = ws.alloc<uint8_t>(n * m);
        launch_pq_encode(dy, n, d, b, m, ks, c, se.s);
        float* o = ws.alloc<float>(n * d);
        pq_residual_kernel<<<nblk(n * d), 256, 0, se.s>>>(dy, c, n, d, b, m, ks, o);
        PQRR_LAUNCH_CHECK();
        count_launch();
        se.download(out, o, n * d);
        se.sync();
    });
}

int pqrr_dev_reconstruct_codes(int device, const float* books, uint32_t d, uint32_t m,
                               const float* rbooks, uint32_t mprime, uint32_t ks,
                               const uint8_t* codes, const uint8_t* rcodes, size_t n, float* out) {
    return guarded([&] {
        check_shape(d, m, ks);
        if (mprime == 0 || d % mprime) throw ArgError("dimension not divisible");
        for (size_t i = 0; i < n * m; ++i)
            if (codes[i] >= ks) throw ArgError("code index out of range");
        for (size_t i = 0; i < n * mprime; ++i)
            if (rcodes[i] >= ks) throw ArgError("code index out of range");
        if (n == 0) return;
        Session se(device);
        Workspace ws(se.s);
        const float* b = se.upload(ws, books, (size_t)ks * d);
        const float* rb = se.upload(ws, rbooks, (size_t)ks * d);
        const uint8_t* c = se.upload(ws, codes, n * m);
        const uint8_t* rc = se.upload(ws, rcodes, n * mprime);
        float* o = ws.alloc<float>(n * d);
        reconstruct_codes_kernel<<<nblk(n * d), 256, 0, se.s>>>(c, rc, n, d, b, m, rb, mprime, ks, o);
        PQRR_LAUNCH_CHECK();
        count_launch();
        se.download(out, o, n * d);
        se.sync();
    });
}

static int merge_impl(int device, const uint32_t* ids, const float* dists, const uint32_t* counts,
                      size_t nq, uint32_t parts, uint32_t width, uint32_t k, uint32_t* out_ids,
                      float* out_dists, uint32_t* out_counts, bool on_device, void* stream) {
    return guarded([&] {
        if (nq == 0 || k == 0) return;
        if (parts == 0 || width == 0) throw ArgError("parts and width must be positive");
        DeviceGuard g(device);
        if (on_device) {
            launch_merge_topk(ids, dists, counts, nq, parts, width, k, out_ids, out_dists, out_counts,
                              static_cast<cudaStream_t>(stream));
            return;
        }
        Session se(device);
        Workspace ws(se.s);
        const size_t tot = (size_t)parts * nq * width;
        const uint32_t* di = se.upload(ws, ids, tot);
        const float* dd = se.upload(ws, dists, tot);
        const uint32_t* dc = se.upload(ws, counts, (size_t)parts * nq);
        uint32_t* oi = ws.alloc<uint32_t>(nq * k);
        float* od = ws.alloc<float>(nq * k);
        uint32_t* oc = ws.alloc<uint32_t>(nq);
        launch_merge_topk(di, dd, dc, nq, parts, width, k, oi, od, oc, se.s);
        se.download(out_ids, oi, nq * k);
        se.download(out_dists, od, nq * k);
        se.download(out_counts, oc, nq);
        se.sync();
    });
}

int pqrr_dev_merge_topk(int device, const uint32_t* ids, const float* dists, const uint32_t* counts,
                        size_t nq, uint32_t parts, uint32_t width, uint32_t k, uint32_t* out_ids,
                        float* out_dists, uint32_t* out_counts) {
    return merge_impl(device, ids, dists, counts, nq, parts, width, k, out_ids, out_dists, out_counts,
                      false, nullptr);
}

int pqrr_dev_merge_topk_device(int device, const uint32_t* ids, const float* dists,
                               const uint32_t* counts, size_t nq, uint32_t parts, uint32_t width,
                               uint32_t k, uint32_t* out_ids, float* out_dists, uint32_t* out_counts,
                               void* stream) {
    return merge_impl(device, ids, dists, counts, nq, parts, width, k, out_ids, out_dists, out_counts,
                      true, stream);
}

int pqrr_dev_index_device(pqrr_dev_index* h, int* device) {
    return guarded([&] { *device = h->ix.device; });
}

int pqrr_dev_merge_packed_device(int device, const void* packed, size_t nq, uint32_t parts,
                                 uint32_t width, uint32_t k, uint32_t* out_ids, float* out_dists,
                                 uint32_t* out_counts, void* stream) {
    return guarded([&] {
        if (nq == 0 || k == 0) return;
        if (parts == 0 || width == 0) throw ArgError("parts and width must be positive");
        DeviceGuard g(device);
        const uint32_t* base = static_cast<const uint32_t*>(packed);
        const size_t blk = 2 * nq * width + nq;
        launch_merge_topk(base, reinterpret_cast<const float*>(base + nq * width), base + 2 * nq * width,
                          nq, parts, width, k, out_ids, out_dists, out_counts,
                          static_cast<cudaStream_t>(stream), blk, blk);
    });
}

int pqrr_dev_last_search_stats(pqrr_dev_index* h, pqrr_dev_search_stats* out) {
    return guarded([&] {
        std::lock_guard<std::mutex> lk(h->ix.mu);
        *out = h->ix.stats;
    });
}

}  // extern "C"
