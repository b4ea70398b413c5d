// internal.h — host-side launchers shared between the .cu translation units of
// libpqrr_b200.so.  Nothing here is part of the public C ABI (include/pqrr_dev.h).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <functional>
#include <stdexcept>
#include <string>

namespace pqrr_b200 {

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};
struct ArgError : std::invalid_argument {
    explicit ArgError(const std::string& s) : std::invalid_argument(s) {}
};

#define PQRR_CUDA(call)                                                                     \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            throw ::pqrr_b200::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define PQRR_LAUNCH_CHECK() PQRR_CUDA(cudaGetLastError())

// Exact k-NN of u8 vectors (k_exact.cu): d = 128; the base arrives in chunks
// through fetch(row0, n, device dst); ids are id_base + row.
bool exact_knn_supported(uint32_t d);
void exact_knn_u8(const uint8_t* d_queries, size_t nq, size_t n, uint64_t id_base, uint32_t k,
                  const std::function<void(uint64_t, uint32_t, uint8_t*)>& fetch, uint32_t* out_ids,
                  float* out_dists, uint32_t* out_cnt, cudaStream_t s);

// Sets the calling thread's pqrr_dev_last_error() text; returns `code`.
int report_error(int code, const std::string& msg);

// Counts kernel launches issued by this library (gpu_launches evidence).
void count_launch(int n = 1);
unsigned long long launch_count();

// Number of SMs of the current device (cached).
int sm_count();

// Raises a kernel's dynamic shared-memory limit to at least `bytes` (never
// lowers it): the attribute is per function and process-wide, so a
// per-launch setting would race between host threads searching different
// indexes (a lowered limit fails the other thread's launch).
void set_max_smem(const void* kernel, size_t bytes);

// -------------------------------------------------------------- synth (k_synth.cu)
void launch_synth_centers(uint64_t seed, uint32_t clusters, uint32_t d, double* centers,
                          cudaStream_t s);
void launch_synth_rows(uint64_t seed, uint32_t set, uint64_t row0, size_t n, uint32_t d,
                       const double* centers, uint32_t clusters, uint8_t* out, cudaStream_t s);

// -------------------------------------------------------------- coarse (k_coarse.cu)
// u8 -> f32 exact widening.
void launch_widen_u8(const uint8_t* in, float* out, size_t count, cudaStream_t s);
// D[q][k] = l2_sq(x_q, C_k) for all pairs (exact reference order).
void launch_pair_dists(const float* x, size_t nx, const float* c, uint32_t nc, uint32_t d,
                       float* out, cudaStream_t s);
// argmin over centroids with ties to the lowest index (kernels.cpp:21-39).
void launch_argmin(const float* x, size_t nx, const float* c, uint32_t nc, uint32_t d,
                   uint32_t* out_idx, float* out_dist, cudaStream_t s);
// per row of D[nq][nc]: the w smallest (dist, idx), ascending.
void launch_topw(const float* D, size_t nq, uint32_t nc, uint32_t w, uint32_t* out_idx,
                 float* out_dist, cudaStream_t s);

// -------------------------------------------------------------- PQ codec (k_encode.cu)
// Plain PQ encode of vectors (kernels::encode_batch / pq_encode_into).
void launch_pq_encode(const float* data, size_t n, uint32_t d, const float* books, uint32_t m,
                      uint32_t ks, uint8_t* codes, cudaStream_t s);
void launch_pq_decode(const uint8_t* codes, size_t n, uint32_t d, const float* books, uint32_t m,
                      uint32_t ks, float* out, cudaStream_t s);
// IVF add path: codes of y - C_a and refine codes of y - (C_a + p).
// y given as f32 (x_f32 != null) or u8 (x_u8 != null).
void launch_ivf_encode(const float* x_f32, const uint8_t* x_u8, size_t n, uint32_t d,
                       const uint32_t* assign, const float* coarse, const float* books, uint32_t m,
                       const float* rbooks, uint32_t mprime, uint32_t ks, uint8_t* codes,
                       uint8_t* rcodes, cudaStream_t s);

// -------------------------------------------------------------- k-means (k_kmeans.cu)
void launch_gather_rows(const float* pts, uint32_t dim, const uint32_t* rows, uint32_t k,
                        float* out, cudaStream_t s);
// Deterministic id-order fp64 centroid update from (cluster-sorted ids).
void launch_centroid_update(const float* pts, uint32_t dim, const uint32_t* sorted_ids,
                            const uint32_t* cl_off, uint32_t k, float* centroids,
                            cudaStream_t s);

// -------------------------------------------------------------- misc (k_util.cu)
void launch_histogram(const uint32_t* keys, size_t n, uint32_t nbins, uint32_t* hist,
                      cudaStream_t s);
void launch_iota(uint32_t* out, size_t n, cudaStream_t s);
// Stable sort of (key, value) pairs by key (CUB radix sort, low `bits` bits).
void sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                uint32_t* vals_out, size_t n, int bits, cudaStream_t s);
void exclusive_scan_u64(const uint64_t* in, uint64_t* out, size_t n, cudaStream_t s);
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, cudaStream_t s);

// -------------------------------------------------------------- layout (k_layout.cu)
// Scatter an existing list-major layout into a new one (per-list prefix kept).
void launch_layout_copy_old(const uint64_t* old_off, const uint32_t* old_len, uint32_t nlists,
                            const uint64_t* new_off, const uint8_t* old_codes,
                            const uint32_t* old_ids, const uint8_t* old_rcodes, uint32_t m,
                            uint32_t mprime, uint8_t* codes, uint32_t* ids, uint8_t* rcodes,
                            uint32_t max_len, cudaStream_t s);
// Scatter staged (id-ordered) entries, sorted by list, behind the old entries.
void launch_layout_place_new(const uint32_t* sorted_list, const uint32_t* sorted_idx, size_t n,
                             const uint32_t* stage_off, const uint64_t* new_off,
                             const uint32_t* old_len, const uint8_t* st_codes,
                             const uint8_t* st_rcodes, const uint32_t* st_ids, uint32_t m,
                             uint32_t mprime, uint8_t* codes, uint32_t* ids, uint8_t* rcodes,
                             cudaStream_t s);

// position -> list table at 16-entry granularity (list starts are 16-aligned).
void launch_block_list(const uint64_t* off, uint32_t nlists, uint16_t* bl, cudaStream_t s);
// Parity-balanced list order (see k_layout.cu) and per-list re-sorting.
void launch_parity_keys(const uint64_t* off, const uint32_t* len, uint32_t nlists,
                        const uint8_t* codes, uint32_t* keys, uint32_t* vals, cudaStream_t s);
void launch_list_id_keys(const uint64_t* off, const uint32_t* len, uint32_t nlists,
                         const uint32_t* ids, uint32_t* keys, uint32_t* vals, cudaStream_t s);
void launch_pair_perm(const uint64_t* off, const uint32_t* len, uint32_t nlists,
                      const uint32_t* skeys, const uint32_t* svals, uint32_t* perm, cudaStream_t s);
void launch_gather_layout(const uint64_t* off, const uint32_t* len, uint32_t nlists,
                          const uint32_t* perm, const uint8_t* codes, const uint32_t* ids,
                          const uint8_t* rcodes, uint32_t m, uint32_t mprime, uint8_t* o_codes,
                          uint32_t* o_ids, uint8_t* o_rcodes, cudaStream_t s);
// Stable per-segment sort (CUB segmented radix sort).
void segmented_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                          uint32_t* vals_out, size_t n, uint32_t nseg, const uint64_t* seg_begin,
                          const uint64_t* seg_end, int bits, cudaStream_t s);

// -------------------------------------------------------------- search (k_scan.cu / k_select.cu)
// Importance-weighted threshold sampling: probe rank r (0 = nearest list) of
// w is sampled at stride << sample_tier(r, w): the nearest eighth of the
// probes at the base stride, then 2x, 4x and 8x for the farther quarter /
// half.  Each sample stands for its stride's worth of entries, so the
// threshold is a weighted quantile (unbiased); the near probes, which hold
// most entries below the threshold, keep the full density.  Tiers are
// contiguous ranges of r, i.e. of a query's sample slots.
__host__ __device__ inline uint32_t sample_tier(uint32_t r, uint32_t w, int tiered) {
    if (!tiered) return 0;
    const uint32_t r8 = 8 * r;
    return r8 < w ? 0u : (r8 < 2 * w ? 1u : (r8 < 4 * w ? 2u : 3u));
}
// Stride shift of tier t: x2 per tier, x4 per tier when w >= 16 (many far
// probes: at C3-C5 the shortlist lives in the first few probes, and the far
// half would otherwise hold most samples).
__host__ __device__ inline uint32_t tier_shift(uint32_t t, uint32_t w) { return w >= 16 ? 2 * t : t; }
static const int kQT = 16;        // queries per scan work item
static const int kScanThreads = 512;

struct ScanArgs {
    const uint8_t* codes;      // list-major, m bytes per entry (m == 8)
    const uint64_t* list_off;  // padded list starts, nlists + 1
    const uint32_t* list_len;  // nlists
    const float* coarse;       // nlists x d
    const float* books;        // m x ks x dsub
    const float* xq;           // nq x d
    uint32_t d, m, ks;
    // work items
    const uint32_t* item_list;
    const uint32_t* item_start;  // into pair_sorted
    const uint32_t* item_nq;
    const uint32_t* item_e0;     // entry range of the list covered by the item
    const uint32_t* item_e1;
    const uint32_t* item_order;  // items sorted longest first
    // pass 0 = exact main scan (LUT rebuilt, candidates <= tau emitted with
    // their exact distance); pass 1 = LUT pass: build each item's exact LUT,
    // write the sampled distances (sample_dist != null) and, when q8_cache is
    // set, the item's 8-bit LUT + per-query (scale, sum of minima) for K4f.
    int pass;
    uint8_t* q8_cache;           // [items][8][256][16] bytes
    float* q8_param;             // [items][16][2]: scale s, sum_j min_j
    const uint32_t* num_items;   // device scalar
    uint32_t* item_counter;      // device scalar, zeroed before launch
    const uint32_t* pair_sorted;  // pair index q * w + r, grouped by list
    uint32_t w;
    const float* tau;  // per query threshold
    // main mode
    float* cand_dist;
    uint32_t* cand_pos;
    uint32_t* cand_cnt;
    uint32_t cap;
    // sample mode (pass 1, sample_dist != null)
    uint32_t stride;             // base stride (probe-rank tier 0)
    int tiered;                  // importance-weighted strides (sample_tier)
    const uint64_t* sample_off;  // per pair
    float* sample_dist;
    const uint8_t* query_sampled;  // per query: 1 if the query is in sample mode
    // two-phase LUT pass (w >= 32, k_lutpass.cu): q8_mode 1 = bound pass
    // (per-lane scale and sum of minima only, no 8-bit block); skip_dead = skip
    // items none of whose lanes can reach tau (pair_live on a bound pass's
    // q8_param) and write the blocks of the others
    int q8_mode;
    int skip_dead;
    const float* pair_bound;  // skip_dead: per pair id, a lower bound of the sum of minima (k_bound.cu)
};
// Certified lower bound (tensor cores) of the sum of LUT minima of the far
// pairs (probe rank >= R1), per pair id into pair_bound (k_bound.cu).
bool far_bound_supported(uint32_t d, uint32_t m, uint32_t ks);
void launch_far_bound(const float* xq, const float* coarse, const float* books, const uint32_t* probes,
                      size_t nq, uint32_t w, uint32_t R1, float* pair_bound, cudaStream_t s);
void launch_ivf_scan(const ScanArgs& a, cudaStream_t s);
// K2 LUT pass (pass 1) as a warp-specialised kernel (k_lutpass.cu).
bool lut_pass_supported(uint32_t d, uint32_t m, uint32_t ks);
void launch_lut_pass(const ScanArgs& a, cudaStream_t s);
// The same pass for small batches (about one probing query per list): code
// book resident, two query lanes per LUT (k_lutnarrow.cu).  Single-phase only.
bool lut_pass_narrow_supported(uint32_t d, uint32_t m, uint32_t ks);
// max_items: an upper bound of the pass's items (no more than SMs: one item per CTA, undivided)
void launch_lut_pass_narrow(const ScanArgs& a, cudaStream_t s, size_t max_items);

// K4f: the main scan as a conservative 4-bit filter over 64-query items
// (k_filter.cu).  Candidates are emitted as (position, probe rank); K4r
// recomputes their exact distances.
static const int kFQ = 64;  // queries per filter item (4 LUT-pass items)
struct FilterArgs {
    const uint8_t* codes;
    const uint64_t* list_off;
    const uint32_t* item_list;   // 64-query items
    const uint32_t* item_start;
    const uint32_t* item_nq;
    const uint32_t* item_e0;     // entry range of the list covered by the item
    const uint32_t* item_e1;
    const uint32_t* item_order;
    const uint32_t* num_items;
    uint32_t* item_counter;
    const uint32_t* list_len;
    const uint32_t* list_first;  // first pair of each list in pair_sorted
    const uint32_t* sub_item_off;  // first 16-query item of each list
    const uint32_t* pair_sorted;
    const uint32_t* live_slot;   // per list from list_first[l]: q8 slot (block * 16 + lane) of each live pair
    const uint32_t* live_pair;   // ... and its pair id q * w + r
    uint32_t w;
    const float* tau;
    const uint8_t* q8_cache;
    const float* q8_param;
    uint32_t* cand_aux;  // probe rank of each candidate
    uint32_t* cand_pos;
    uint32_t* cand_cnt;
    uint32_t cap;
    // optional: each candidate's 8 code bytes next to its position, read from
    // the list K4f just streamed (L2) so K4r needs no random DRAM gather
    uint64_t* cand_code;
    // optional: per query a 256-bit mask of the probe ranks that got a
    // candidate (zeroed by the caller; K4r builds LUTs for exactly those)
    uint32_t* cand_used;
    int pass_all;  // debug: every probed entry is a candidate
    float band_div;  // Delta target = (tau - sum of minima) / band_div
};
void launch_ivf_filter(const FilterArgs& a, cudaStream_t s);
// Live-pair compaction before K4f: a pair (q, l) is live when its LUT's sum of
// sub-table minima can reach tau_q (no entry of l is at or below tau_q
// otherwise).  Writes, per list, the positions of its live pairs from
// list_first[l] on (live_pos) and rewrites the 64-query K4f items
// (item_start / item_nq) over the live pairs only.
// The pairs come from up to two LUT-pass item sets (near / far probes of the
// two-phase LUT pass); set k's blocks start at q8 block blk_base[k].
struct PairSet {
    const uint32_t* pair_sorted;
    const uint32_t* list_cnt;
    const uint32_t* list_first;
    const uint32_t* sub_item_off;
    uint32_t blk_base;
    const float* pair_bound;  // set: a pair is live only if its bound also admits it
};
void launch_live_pairs(const FilterArgs& a, PairSet s0, PairSet s1, const uint32_t* all_first,
                       const uint32_t* all_cnt, uint32_t nlists, uint32_t* live_slot,
                       uint32_t* live_pair, uint32_t* live_cnt, const uint32_t* item_off,
                       uint32_t* item_start, uint32_t* item_nq, uint32_t chunk, cudaStream_t s,
                       unsigned long long* live_entries = nullptr);
// K4r: exact ADC distance of every filter candidate (reference order), and
// the per-query count of candidates at or below tau.
bool recheck_supported(uint32_t d, uint32_t m, uint32_t w);
void launch_recheck(const float* xq, uint32_t d, uint32_t m, const float* coarse,
                    const float* books, const uint32_t* probes, uint32_t w, const uint8_t* codes,
                    const uint32_t* cand_cnt, uint32_t cap, const uint32_t* cand_pos,
                    float* cand_dist, const float* tau, size_t nq, uint32_t* cand_le,
                    cudaStream_t s, uint32_t* cand_mm = nullptr, const uint64_t* cand_code = nullptr,
                    const uint32_t* cand_used = nullptr);

// Build the scan work items from the probes.
void launch_items_build(const uint32_t* list_cnt, const uint32_t* list_first,
                        const uint32_t* list_len, uint32_t nlists, const uint32_t* item_off,
                        uint32_t* item_list, uint32_t* item_start, uint32_t* item_nq,
                        uint32_t* item_e0, uint32_t* item_e1, uint32_t* sort_key, uint32_t qt,
                        cudaStream_t s, uint32_t chunk, uint32_t n_items);
// Small-batch probe inversion in shared memory (k_invert.cu): one launch for
// the sorted pairs, per-list counts / first pair, and for two item sets (qt
// queries per item, lists cut into `chunk` entries) the item offsets, the
// items and their longest-first order.
static const size_t kInvertSmallMaxPairs = 4096;
static const uint32_t kInvertSmallMaxItems = 4096;
bool invert_small_supported(size_t np, uint32_t c);
struct SmallItems {
    uint32_t* item_off;  // [c + 1]
    uint32_t *item_list, *item_start, *item_nq, *item_e0, *item_e1, *item_order;
    uint32_t qt, chunk;
    uint32_t bound;  // >= the real item count, <= kInvertSmallMaxItems; 0: offsets only
};
void launch_invert_small(const uint32_t* probes, uint32_t np, uint32_t w, const float* D, uint32_t c,
                         const uint32_t* list_len, uint32_t* pair_sorted, uint32_t* list_cnt,
                         uint32_t* list_first, const SmallItems& a, const SmallItems& b, cudaStream_t s);
void launch_items_per_list(const uint32_t* list_cnt, const uint32_t* list_len, uint32_t nlists,
                           uint32_t* items, uint32_t qt, cudaStream_t s, uint32_t chunk = 1u << 30);
// Per query: N_q = sum of probed list lengths; per pair sample counts.
void launch_query_sizes(const uint32_t* probes, size_t nq, uint32_t w, const uint32_t* list_len,
                        uint32_t stride, int tiered, uint32_t cap, uint64_t* nq_entries,
                        uint8_t* query_sampled, uint64_t* pair_samples, uint64_t* grand_total,
                        cudaStream_t s, uint32_t max_rank = 0xffffffffu);
// Small batches (<= 8192 pairs): sizes and the exclusive scan of the pairs'
// sample counts (sample_off, nq * w + 1 entries) in one single-CTA launch.
bool launch_query_sizes_small(const uint32_t* probes, size_t nq, uint32_t w, const uint32_t* list_len,
                              uint32_t stride, int tiered, uint32_t cap, uint64_t* nq_entries,
                              uint8_t* query_sampled, uint64_t* sample_off, uint64_t* grand_total,
                              cudaStream_t s, uint32_t max_rank);
// tau_q = rank-th smallest sample of query q (sampled queries), +inf otherwise.
void launch_sample_threshold(const float* sample_dist, const uint64_t* sample_off, uint32_t w,
                             size_t nq, const uint8_t* query_sampled, float alpha_k,
                             uint32_t stride, int tiered, uint32_t max_samples, float* tau,
                             cudaStream_t s);
// Exact top-kprime under (dist, id) from each query's candidates.
void launch_select_topk(const float* cand_dist, const uint32_t* cand_pos, const uint32_t* cand_cnt,
                        uint32_t cap, uint32_t max_n, size_t nq, const uint32_t* ids,
                        uint32_t kprime, bool sorted, uint64_t* sl_key, uint32_t* sl_pos,
                        uint32_t* sl_cnt, cudaStream_t s,
                        const uint32_t* cand_mm = nullptr, bool need_ids = true);
// Re-rank the shortlist with the 3-term reconstruction, keep the k best.
void launch_rerank(const uint64_t* sl_key, const uint32_t* sl_pos, const uint32_t* sl_cnt,
                   uint32_t sl_stride, size_t nq, const float* xq, uint32_t d,
                   const uint16_t* block_list, const float* coarse,
                   const uint8_t* codes, const float* books, uint32_t m, const uint8_t* rcodes,
                   const float* rbooks, uint32_t mprime, uint32_t ks, uint32_t k,
                   uint32_t* out_ids, float* out_dists, uint32_t* out_cnt, cudaStream_t s,
                   cudaEvent_t ev_dist_done = nullptr, const uint32_t* ids_for_keys = nullptr);
// Add-path coarse assignment on the tensor cores (k_assign_tc.cu): u8 rows,
// d = 128, nc % 128 == 0; certified equal to launch_argmin's result.
bool assign_tc_supported(uint32_t d, uint32_t nc);
struct AssignTc {
    bool ready = false, usable = false;
    uint32_t nc = 0;
    float cmax = 0.f;
    void* hi = nullptr;
    void* lo = nullptr;
    float* cn = nullptr;
    AssignTc() = default;
    AssignTc(const AssignTc&) = delete;
    AssignTc& operator=(const AssignTc&) = delete;
    ~AssignTc();
    // one-time split of the centroids (false: keep the exact CUDA-core path)
    bool prepare(const float* coarse, uint32_t nc, cudaStream_t s);
    void assign(const uint8_t* y, size_t n, const float* coarse, uint32_t* out, cudaStream_t s);
    // search side: D~ rows of n u8-valued f32 queries (+ per-row min / max keys)
    void dtilde(const float* x, size_t n, float* Dt, uint32_t* kmm, cudaStream_t s);
};
// K5a on CTA pairs (k_rerank.cu): refined distance + id of every shortlist
// entry (rows of `stride`, sl_cnt[q] valid) into rdist / rid.
bool rerank_pair_supported(uint32_t d, uint32_t m, uint32_t ks, uint32_t mprime);
void launch_rerank_pair(const uint64_t* sl_key, const uint32_t* sl_pos, const uint32_t* sl_cnt,
                        uint32_t stride, size_t nq, const float* xq, const uint16_t* block_list,
                        const float* coarse, const uint8_t* codes, const float* books,
                        const uint8_t* rcodes, const float* rbooks, uint32_t mprime, float* rdist,
                        uint32_t* rid, cudaStream_t s, const uint32_t* ids = nullptr);
// Merge per-shard ranked lists into the top-k (K7).  Part p's rows are
// ids/dists + p * ps (nq x width) and counts + p * cs (nq); ps = cs = 0 means
// the stacked layout [parts][nq][width] + [parts][nq].
void launch_merge_topk(const uint32_t* ids, const float* dists, const uint32_t* counts, size_t nq,
                       uint32_t parts, uint32_t width, uint32_t k, uint32_t* out_ids,
                       float* out_dists, uint32_t* out_cnt, cudaStream_t s, size_t ps = 0,
                       size_t cs = 0);
// K1 on the tensor cores with certified exact top-w (k_coarse_tc.cu).
bool coarse_tc_supported(uint32_t d, uint32_t w);
void launch_coarse_norms(const float* c, uint32_t n, uint32_t d, float* out, cudaStream_t s);
// atc (prepared, non-null) and u8-valued queries: D~ on tcgen05 (k_assign_tc.cu)
// with the certification window 2^-13 (|x|^2 + max |c|^2); otherwise mma.sync TF32.
struct AssignTc;
void launch_coarse_tc(const float* x, size_t nq, const float* c, uint32_t nc, const float* cnorm,
                      float cnorm_max, uint32_t w, float* Dt, uint32_t* out_idx, uint32_t* overflow,
                      cudaStream_t s, AssignTc* atc = nullptr);
// Warp-per-query selections (k_wselect.cu); the bool variants return false
// outside their envelope (caller falls back to the CTA kernels).
bool launch_topw_warp(const float* D, size_t nq, uint32_t nc, uint32_t w, uint32_t* out_idx,
                      float* out_dist, cudaStream_t s);
void launch_select_warp(const float* cand_dist, const uint32_t* cand_pos, const uint32_t* cand_cnt,
                        uint32_t cap, size_t nq, const uint32_t* ids, uint32_t kprime,
                        uint64_t* sl_key, uint32_t* sl_pos, uint32_t* sl_cnt, cudaStream_t s,
                        const uint32_t* cand_mm = nullptr, bool need_ids = true);
void launch_threshold_warp(const float* sample_dist, const uint64_t* sample_off, uint32_t w, size_t nq,
                           const uint8_t* query_sampled, float alpha_k, uint32_t stride, int tiered,
                           float* tau, cudaStream_t s);
bool launch_rerank_topk_warp(const float* rdist, const uint32_t* rid, const uint32_t* cnt,
                             uint32_t stride, size_t nq, uint32_t k, uint32_t* out_ids,
                             float* out_dists, uint32_t* out_cnt, cudaStream_t s);
// Split keys into ids / dists ([nq][stride] -> [nq][stride]).
void launch_unpack_keys(const uint64_t* keys, const uint32_t* cnt, size_t nq, uint32_t stride,
                        uint32_t* ids, float* dists, cudaStream_t s);

// Standalone kernel-seam scan (kernels::scan_topk parity): LUT given.
void launch_lut_scan_all(const float* lut, uint32_t m, uint32_t ks, const uint8_t* codes, size_t n,
                         float* out_dist, cudaStream_t s);
void launch_build_lut(const float* xr, size_t nx, uint32_t d, const float* books, uint32_t m,
                      uint32_t ks, float* out, cudaStream_t s);

}  // namespace pqrr_b200
