/*
 * pqrr_dev.h — C ABI of the B200-native IVFADC+R search path
 * (paper_1102_3828_b200/lib/libpqrr_b200.so).
 *
 * This is the drop-in boundary for the reference's C++ API in namespace
 * pqrr (/root/reference/proj/include/pqrr/).  The reference has no C ABI or
 * plugin registry; its seams are (1) the index API of ivf_index.hpp:48-81,
 * (2) the hot-kernel seam pqrr::kernels of kernels.hpp:13-43, substituted at
 * link time, and (3) the k-means / PQ trainers of kmeans.hpp:38 and
 * product_quantizer.hpp:39-40.  Each entry point below names the reference
 * declaration it replaces.  INTEGRATION.md shows the C++ shim (and a ctypes
 * binding) a maintainer adds on the reference side.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Unless a name ends in _device, every
 *    pointer is a HOST pointer; the library copies in and out.
 *  - Matrices are row-major.  Product-quantizer books are m sub-codebooks of
 *    ks centroids of d/m floats, sub-quantizer-major, centroid-major,
 *    component-minor (storage.hpp:19-20).  A coarse codebook is c x d floats.
 *  - Codes are uint8, m per vector.  Ids are uint32 (ivf_index.hpp:18).
 *  - Every function returns PQRR_OK (0) or a negative status; the message of
 *    the last failure on the calling thread is pqrr_dev_last_error().  Error
 *    messages pinned by the reference spec are reproduced verbatim:
 *    "insufficient training data", "dimension not divisible",
 *    "shortlist too small".
 *  - Arithmetic follows the reference contract bit for bit (distance.hpp:7-33,
 *    product_quantizer.hpp:51-57, types.hpp:45-50): outputs are identical to
 *    the reference path on the same inputs and codebooks.
 *  - There is no CPU fallback: without a usable sm_100 device every call
 *    fails with PQRR_ENODEV.
 */
#ifndef PQRR_DEV_H
#define PQRR_DEV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PQRR_OK = 0,
    PQRR_EINVAL = -1,      /* bad argument (reference std::invalid_argument) */
    PQRR_ECUDA = -2,       /* CUDA runtime failure */
    PQRR_ENODEV = -3,      /* no usable GPU */
    PQRR_EUNSUPPORTED = -4,/* shape outside what the device kernels implement */
    PQRR_ESHORTLIST = -5,  /* "shortlist too small" */
    PQRR_EINTERNAL = -6
};

const char* pqrr_dev_last_error(void);
int pqrr_dev_device_count(int* out);
/* Number of kernels this library has launched in this process. */
uint64_t pqrr_dev_launch_count(void);

/* ------------------------------------------------------------------ kernel seam
 * pqrr::kernels (kernels.hpp:13-43).  One call = one batch on `device`.    */

/* kernels::assign_batch (kernels.hpp:23-25): argmin l2_sq, ties -> lowest index. */
int pqrr_dev_assign_batch(int device, const float* points, size_t n, uint32_t dim,
                          const float* centroids, uint32_t k, uint32_t* out_assign,
                          float* out_dist);
/* assign_batch of u8 rows without distances: the add path's assignment
 * (ivf_index.hpp:54-56).  d = 128 and k % 128 == 0 run the certified
 * tensor-core kernel (k_assign_tc.cu: tcgen05 + TMEM + TMA, ambiguous rows
 * recomputed exactly); other shapes the exact CUDA-core argmin.  Either way
 * out_assign equals kernels::assign_batch on the widened rows.              */
int pqrr_dev_assign_u8(int device, const uint8_t* points, size_t n, uint32_t dim,
                       const float* centroids, uint32_t k, uint32_t* out_assign);
/* kernels::encode_batch (kernels.hpp:28-29) with pq_encode_into semantics. */
int pqrr_dev_encode_batch(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                          const float* data, size_t n, uint8_t* out_codes);
/* kernels::decode_batch (kernels.hpp:32-33). */
int pqrr_dev_decode_batch(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                          const uint8_t* codes, size_t n, float* out_data);
/* build_lut (product_quantizer.hpp:48-49) for nx vectors: out is nx * m * ks. */
int pqrr_dev_build_lut(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                       const float* x, size_t nx, float* out_lut);
/* kernels::scan_topk (kernels.hpp:40-41): ids = id_base + position. */
int pqrr_dev_scan_topk(int device, const float* lut, uint32_t m, uint32_t ks, const uint8_t* codes,
                       size_t n, size_t kprime, uint32_t id_base, uint32_t* out_ids,
                       float* out_dists, size_t* out_count);

/* ------------------------------------------------------------------ training
 * kmeans_train (kmeans.hpp:38), pq_train (product_quantizer.hpp:39-40),
 * ivf_train (ivf_index.hpp:50-52), ivf_refine_train (ivf_index.hpp:68-70).
 * Exact assignment on the device, id-order fp64 update (bit-identical to the
 * serial policy of kmeans.hpp:30-38).                                        */
int pqrr_dev_kmeans_train(int device, const float* points, size_t n, uint32_t dim, uint32_t k,
                          uint32_t iterations, uint64_t seed, uint32_t redo, float* out_centroids,
                          double* out_final_mse, double* out_trace /* iterations or NULL */);
int pqrr_dev_pq_train(int device, const float* training, size_t n, uint32_t d, uint32_t m,
                      uint32_t ks, uint32_t iterations, uint64_t seed, uint32_t redo,
                      float* out_books);
int pqrr_dev_ivf_train(int device, const float* training, size_t n, uint32_t d, uint32_t c,
                       uint32_t m, uint32_t ks, uint32_t iterations, uint64_t seed,
                       float* out_coarse, float* out_books);
int pqrr_dev_ivf_refine_train(int device, const float* coarse, uint32_t c, const float* books,
                              uint32_t d, uint32_t m, uint32_t ks, const float* training,
                              size_t n, uint32_t mprime, uint32_t iterations, uint64_t seed,
                              float* out_rbooks);

/* ------------------------------------------------------------------ synthetic data
 * The BASELINE.json SIFT-like generator: set 0 = centres,
 * 1 = train, 2 = base, 3 = query.  Rows [row0, row0 + n) of `set`.           */
int pqrr_dev_synth(int device, uint64_t seed, uint32_t clusters, uint32_t d, uint32_t set,
                   uint64_t row0, size_t n, uint8_t* out /* host, n * d */);

/* ------------------------------------------------------------------ index
 * IvfIndex + RefineQuantizer + RefineCodes (ivf_index.hpp:27-41,
 * refine.hpp:15-28) resident in one device's HBM.                            */
typedef struct pqrr_dev_index pqrr_dev_index;

/* mprime = 0 / rbooks = NULL: no refinement (plain IVFADC). */
int pqrr_dev_index_create(int device, uint32_t d, uint32_t c, const float* coarse, uint32_t m,
                          const float* books, uint32_t mprime, const float* rbooks, uint32_t ks,
                          pqrr_dev_index** out);
int pqrr_dev_index_destroy(pqrr_dev_index* ix);

/* ivf_build (ivf_index.hpp:54-56) + ivf_refine_encode (:72-73), chunked:
 * vectors get ids id_base .. id_base + n - 1; chunks must arrive in
 * id-ascending order (lists stay id-ascending, ivf_index.hpp:15-16).         */
int pqrr_dev_add_u8(pqrr_dev_index* ix, const uint8_t* y, size_t n, uint32_t id_base);
int pqrr_dev_add_f32(pqrr_dev_index* ix, const float* y, size_t n, uint32_t id_base);
/* Same, vectors generated on the device by the synthetic generator: rows
 * [row0, row0 + n) of the base set get ids id_base + (row - row0).          */
int pqrr_dev_add_synthetic(pqrr_dev_index* ix, uint64_t seed, uint32_t clusters, uint64_t row0,
                           size_t n, uint32_t id_base);
/* Builds the list-major layout of everything added so far (implicit on search). */
int pqrr_dev_finalize(pqrr_dev_index* ix);

typedef struct {
    uint64_t n;            /* indexed vectors */
    uint64_t slots;        /* padded list-major entries */
    uint32_t d, c, m, mprime, ks;
    uint32_t max_list_len;
    uint64_t device_bytes; /* bytes held in HBM by the index */
} pqrr_dev_index_info;
int pqrr_dev_index_get_info(pqrr_dev_index* ix, pqrr_dev_index_info* out);

/* Lists in list order without padding: offsets[c + 1], ids[n], codes[n * m],
 * rcodes[n * mprime] (any output may be NULL). */
int pqrr_dev_export_lists(pqrr_dev_index* ix, uint64_t* offsets, uint32_t* ids, uint8_t* codes,
                          uint8_t* rcodes);

/* The lists `lists[0..nl)` only (e.g. the probed lists of a query sample, for
 * an oracle check at 1B without exporting the index): offsets[nl + 1] (always
 * filled), then ids / codes / rcodes of each list id-ascending (NULL = skip). */
int pqrr_dev_export_lists_subset(pqrr_dev_index* ix, const uint32_t* lists, uint32_t nl,
                                 uint64_t* offsets, uint32_t* ids, uint8_t* codes,
                                 uint8_t* rcodes);
/* Trained parameters held by the index (coarse[c*d], books[ks*d],
 * rbooks[ks*d] when mprime > 0; any may be NULL). */
int pqrr_dev_export_codebooks(pqrr_dev_index* ix, float* coarse, float* books, float* rbooks);

/* Inverse of pqrr_dev_export_lists: load an existing inverted file into an
 * EMPTY index (e.g. a host IvfIndex, ivf_index.hpp:27-36, or a PQRR file,
 * storage.hpp:23-25).  Lists in list order, ids ascending within a list;
 * rcodes (list order, mprime bytes per entry) may be NULL when mprime = 0. */
int pqrr_dev_load_lists(pqrr_dev_index* ix, const uint64_t* offsets, const uint32_t* ids,
                        const uint8_t* codes, const uint8_t* rcodes);

/* Fused search: coarse probe of w lists -> LUTs -> ADC scan -> exact top-k'
 * shortlist (ivf_search_batch, ivf_index.hpp:58-64) -> if k > 0, re-rank with
 * the refinement codes to the top-k (ivf_rerank, :79-81).
 * Outputs per query q at row q of width (k > 0 ? k : kprime):
 *   out_ids, out_dists ascending under (dist, id); out_counts[q] entries.
 * k == 0 returns the IVFADC shortlist itself (min(kprime, candidates)).
 * k > min(kprime, candidates) fails with PQRR_ESHORTLIST.                    */
int pqrr_dev_search_u8(pqrr_dev_index* ix, const uint8_t* queries, size_t nq, uint32_t w,
                       size_t kprime, size_t k, uint32_t* out_ids, float* out_dists,
                       uint32_t* out_counts);
int pqrr_dev_search_f32(pqrr_dev_index* ix, const float* queries, size_t nq, uint32_t w,
                        size_t kprime, size_t k, uint32_t* out_ids, float* out_dists,
                        uint32_t* out_counts);
/* Device-resident variant: all pointers are device pointers on the index's
 * device; `stream` is a cudaStream_t (NULL = the legacy default stream). The
 * call is stream-ordered and returns after the results are complete (small
 * batches: one graph launch and one synchronisation; large batches read
 * counts back between stages).                                              */
int pqrr_dev_search_u8_device(pqrr_dev_index* ix, const uint8_t* d_queries, size_t nq,
                              uint32_t w, size_t kprime, size_t k, uint32_t* d_out_ids,
                              float* d_out_dists, uint32_t* d_out_counts, void* stream);
/* Enqueue-only variant for small batches (serving; eval.hpp:49's per-query
 * time is the latency it targets).  The whole search is one CUDA graph,
 * captured on the first call of a (shape, buffers) combination and replayed
 * afterwards: _enqueue returns once the graph is launched, ordered after
 * `stream`'s earlier work, and `stream` waits for the results; no host
 * synchronisation happens inside.  _finish waits for the enqueued search and
 * returns its error code (PQRR_ESHORTLIST as above); in the rare case that a
 * sampled threshold failed its on-device exactness check it redoes the batch
 * on the synchronising path, so the results are the same bits either way.
 * One search may be pending per index.  PQRR_EUNSUPPORTED: the batch is
 * outside the envelope (more than 1024 queries, or bounds too large for the
 * device) — use pqrr_dev_search_u8_device.                                   */
int pqrr_dev_search_u8_enqueue(pqrr_dev_index* ix, const uint8_t* d_queries, size_t nq,
                               uint32_t w, size_t kprime, size_t k, uint32_t* d_out_ids,
                               float* d_out_dists, uint32_t* d_out_counts, void* stream);
int pqrr_dev_search_finish(pqrr_dev_index* ix);
/* enabled = 0: every search of this index takes the synchronising path (per
 * stage times in pqrr_dev_last_search_stats; graph replays report only the
 * total); 1 (default): batches of up to 1024 queries replay captured graphs. */
int pqrr_dev_index_set_graph(pqrr_dev_index* ix, int enabled);

/* ivf_rerank (ivf_index.hpp:79-81) of an explicit shortlist: sl_ids row q
 * holds sl_counts[q] ids (stride sl_stride); outputs k per query. */
int pqrr_dev_rerank_u8(pqrr_dev_index* ix, const uint8_t* queries, size_t nq,
                       const uint32_t* sl_ids, const uint32_t* sl_counts, size_t sl_stride,
                       size_t k, uint32_t* out_ids, float* out_dists);
int pqrr_dev_rerank_f32(pqrr_dev_index* ix, const float* queries, size_t nq,
                        const uint32_t* sl_ids, const uint32_t* sl_counts, size_t sl_stride,
                        size_t k, uint32_t* out_ids, float* out_dists);
/* Exact multi-shard mode: re-rank the entries of a GLOBAL
 * shortlist (the merged top-k' of every shard, rows of sl_stride, d_sl_counts[q]
 * valid) that THIS shard holds; ids held elsewhere are skipped.  Per query the
 * top-min(k, owned) under (dist, id) land in row q of width k and
 * d_out_counts[q].  Merging every shard's rows with pqrr_dev_merge_topk gives
 * the single-index ivf_rerank result (ivf_index.hpp:79-81).  Device pointers,
 * stream-ordered on `stream` (NULL = the legacy default stream).            */
int pqrr_dev_rerank_owned_u8_device(pqrr_dev_index* ix, const uint8_t* d_queries, size_t nq,
                                    const uint32_t* d_sl_ids, const uint32_t* d_sl_counts,
                                    size_t sl_stride, size_t k, uint32_t* d_out_ids,
                                    float* d_out_dists, uint32_t* d_out_counts, void* stream);
/* list_of_id / code_of_id (ivf_index.hpp:33-40) and RefineCodes::code
 * (refine.hpp:27) of n ids: out_list[i] (UINT32_MAX if id i was never
 * added), out_codes[i * m ..], out_rcodes[i * mprime ..] (NULL = skip).
 * The add-path parity check compares these with a CPU re-encode.           */
int pqrr_dev_lookup_ids(pqrr_dev_index* ix, const uint32_t* ids, size_t n, uint32_t* out_list,
                        uint8_t* out_codes, uint8_t* out_rcodes);
/* ivf_reconstruct (ivf_index.hpp:75-77): coarse + decode + refine decode. */
int pqrr_dev_reconstruct(pqrr_dev_index* ix, const uint32_t* ids, size_t n, float* out);

/* Test seam of the two-phase LUT pass (k_bound.cu): certified lower bounds
 * (tensor cores) of sum_j min_c l2_sq(x_q - C_l, B_j[c]) for the pairs
 * (q, l = probes[q w + r]), r >= R1, written to out[q w + r] (other slots are
 * left untouched).  d = 128, m = 8, ks = 256.                               */
int pqrr_dev_pair_bounds(int device, const float* queries, size_t nq, uint32_t d, const float* coarse,
                         uint32_t c, const float* books, uint32_t m, uint32_t ks, const uint32_t* probes,
                         uint32_t w, uint32_t R1, float* out);

/* ------------------------------------------------------------------ ground truth
 * compute_groundtruth / exact_search (eval.hpp:13-19) for u8 vectors, d = 128:
 * per query the min(k, n) nearest base rows, ascending (dist, id) (exact: u8
 * distances are integers < 2^24, computed with integer tensor-core MMA).
 * Rows [k * q, k * q + k) of out_ids / out_dists, out_counts[q] valid.
 * _u8: base rows from host memory (ids 0..n-1); _synthetic: rows
 * [row0, row0 + n) of the synthetic base set generated on the device (the
 * bench's 1B ground truth), ids = row index.  1 <= k <= 16384.              */
int pqrr_dev_exact_knn_u8(int device, const uint8_t* base, size_t n, const uint8_t* queries, size_t nq,
                          uint32_t d, uint32_t k, uint32_t* out_ids, float* out_dists, uint32_t* out_counts);
int pqrr_dev_exact_knn_synthetic(int device, uint64_t seed, uint32_t clusters, uint64_t row0, size_t n,
                                 const uint8_t* queries, size_t nq, uint32_t k, uint32_t* out_ids,
                                 float* out_dists, uint32_t* out_counts);

/* ------------------------------------------------------------------ ADC / ADC+R
 * Exhaustive first stage (adc_index.hpp:13-31) and its re-ranking
 * (refine.hpp:30-53).  An ADC index is an index handle with one all-zero
 * coarse centroid, bit-identical to the ADC definitions:
 *   adc_build        -> pqrr_dev_adc_index_create + pqrr_dev_add_* + pqrr_dev_finalize
 *   adc_search[_batch] -> pqrr_dev_search_*(w = 1, k = 0); with k > 0 the
 *                       search is fused with the ADC+R re-rank (refine.hpp:50-53)
 *   refine_encode    -> create with mprime > 0 (codes of y - decode(encode(y)))
 *   rerank           -> pqrr_dev_rerank_u8/_f32
 * refine_train (refine.hpp:33-36), residual (refine.hpp:30-31) and
 * reconstruct (refine.hpp:42-45) are stand-alone.                                                              */
int pqrr_dev_adc_index_create(int device, uint32_t d, uint32_t m, const float* books,
                              uint32_t mprime, const float* rbooks, uint32_t ks,
                              pqrr_dev_index** out);
int pqrr_dev_refine_train(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                          const float* training, size_t n, uint32_t mprime, uint32_t iterations,
                          uint64_t seed, float* out_rbooks);
int pqrr_dev_residual(int device, const float* books, uint32_t d, uint32_t m, uint32_t ks,
                      const float* y, size_t n, float* out);
int pqrr_dev_reconstruct_codes(int device, const float* books, uint32_t d, uint32_t m,
                               const float* rbooks, uint32_t mprime, uint32_t ks,
                               const uint8_t* codes, const uint8_t* rcodes, size_t n, float* out);

/* ------------------------------------------------------------------ persistence
 * The "PQRR" container (storage.hpp:14-28): magic "PQRR",
 * version byte 1, little-endian.  Host files; index loads create a device
 * index on `device`.  Truncated / oversized / malformed files fail with
 * PQRR_EINVAL "corrupt file".  Layouts: DESIGN.md §10.
 *   save_quantizer / load_quantizer   (also codebooks: m = 1, ks = k)
 *   save_adc_index / load_adc_index   (save_adc_index(ix, rq, codes, path))
 *   save_index / load_index           (save_ivf_index / load_ivf_index)
 *   probe_index_kind                  (probe_index_kind, storage.hpp:59-62)
 * load_quantizer with books = NULL returns the shape only.                  */
enum { PQRR_INDEX_ADC = 0, PQRR_INDEX_IVF = 1 };
int pqrr_dev_save_quantizer(const char* path, uint32_t d, uint32_t m, uint32_t ks,
                            const float* books);
int pqrr_dev_load_quantizer(const char* path, uint32_t* d, uint32_t* m, uint32_t* ks,
                            float* books);
int pqrr_dev_save_index(pqrr_dev_index* ix, const char* path);
int pqrr_dev_load_index(int device, const char* path, pqrr_dev_index** out);
int pqrr_dev_save_adc_index(pqrr_dev_index* ix, const char* path);
int pqrr_dev_load_adc_index(int device, const char* path, pqrr_dev_index** out);
int pqrr_dev_probe_index_kind(const char* path, int* kind);

/* K7 — merge of per-shard ranked lists (multi-GPU id-range sharding, after an
 * all-gather): inputs [parts][nq][width] ids / dists and [parts][nq] counts;
 * output the top-k per query under (dist, id) (types.hpp:47-50).  Host
 * pointers, or device pointers on `device` for the _device variant
 * (stream-ordered on `stream`, a cudaStream_t; NULL = legacy default).     */
int pqrr_dev_merge_topk(int device, const uint32_t* ids, const float* dists,
                        const uint32_t* counts, size_t nq, uint32_t parts, uint32_t width,
                        uint32_t k, uint32_t* out_ids, float* out_dists, uint32_t* out_counts);
int pqrr_dev_merge_topk_device(int device, const uint32_t* ids, const float* dists,
                               const uint32_t* counts, size_t nq, uint32_t parts, uint32_t width,
                               uint32_t k, uint32_t* out_ids, float* out_dists,
                               uint32_t* out_counts, void* stream);
/* K7 on ONE all-gathered buffer: `packed` holds `parts` consecutive blocks of
 * 2 * nq * width + nq 32-bit words, each [ids nq x width | dists nq x width |
 * counts nq] -- the layout a shard's search writes straight into its slice,
 * so a merge needs one all-gather (device pointers, stream-ordered).        */
int pqrr_dev_merge_packed_device(int device, const void* packed, size_t nq, uint32_t parts,
                                 uint32_t width, uint32_t k, uint32_t* d_out_ids,
                                 float* d_out_dists, uint32_t* d_out_counts, void* stream);

/* ------------------------------------------------------------------ multi-GPU group
 * One process driving G id-range shards: shards[r] is an
 * index handle (any device) holding the ids of shard r over all c lists.
 * group_search broadcasts the host queries, searches every shard on its own
 * device, and merges with ONE all-gather per merge of every shard's packed
 * rows (pqrr_dev_merge_packed_device): NCCL (ncclCommInitAll, ncclAllGather in
 * a group call) when the shards sit on distinct devices, device copies when
 * shards share one.  PQRR_GROUP_EXACT (default): global IVFADC top-k', each
 * shard re-ranks the entries it holds -> bit-identical to one index holding
 * every id (ivf_search_batch + ivf_rerank); fails with PQRR_ESHORTLIST exactly
 * when that index would.  PQRR_GROUP_LOCAL: every shard's fused top-k merged
 * (re-ranks up to G k' candidates).  Outputs as pqrr_dev_search_u8.         */
typedef struct pqrr_dev_group pqrr_dev_group;
enum { PQRR_GROUP_EXACT = 0, PQRR_GROUP_LOCAL = 1 };
int pqrr_dev_index_device(pqrr_dev_index* ix, int* device);
int pqrr_dev_group_create(uint32_t G, pqrr_dev_index* const* shards, pqrr_dev_group** out);
int pqrr_dev_group_search_u8(pqrr_dev_group* g, const uint8_t* queries, size_t nq, uint32_t w,
                             size_t kprime, size_t k, int mode, uint32_t* out_ids,
                             float* out_dists, uint32_t* out_counts);
/* shards in the group and whether its all-gathers run on NCCL */
int pqrr_dev_group_size(pqrr_dev_group* g, uint32_t* shards, int* uses_nccl);
int pqrr_dev_group_destroy(pqrr_dev_group* g);

/* Per-stage device times (CUDA events on the index stream) of the last search. */
typedef struct {
    float ms_total, ms_coarse, ms_invert, ms_sample_scan, ms_threshold, ms_scan, ms_select,
        ms_rerank;
    uint64_t nq, scanned_entries, sampled_entries, candidates;
    uint32_t work_items, retries, stride;
    uint32_t kernels;
    float ms_filter;           /* K4f alone (ms_scan = K4f + K4r, or the exact scan) */
    uint64_t exact_candidates; /* candidates with exact ADC <= tau (K4f path) */
    float ms_recheck;          /* K4r alone (exact ADC of the filter's survivors) */
    float ms_rerank_dist;      /* K5 refined distances alone (ms_rerank = K5 + top-k) */
    uint64_t rerank_candidates;/* shortlist entries re-ranked (sum of the k' rows) */
    uint64_t filter_live_entries; /* (live (query, list) pair, entry) combinations K4f tests */
} pqrr_dev_search_stats;
int pqrr_dev_last_search_stats(pqrr_dev_index* ix, pqrr_dev_search_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* PQRR_DEV_H */
