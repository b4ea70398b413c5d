/*
 * pqrr_oracle.h — C ABI of the CPU oracle for the IVFADC+R search path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker or the timed CPU baseline — never as the product.
 *
 * The oracle restates, in plain C++20, the arithmetic contract the reference
 * headers pin down (/root/reference/proj/include/pqrr/ headers) and supplies the
 * bodies the reference declares but never defines.  Every
 * function cites the reference file:line it follows in pqrr_oracle.cpp.
 *
 * Conventions: row-major float32 arrays; codebooks are sub-quantizer-major,
 * centroid-major, component-minor (storage.hpp:19-20); codes are u8, m per
 * vector.  All functions return 0 on success or a negative error code; the
 * message is available from orc_last_error().
 */
#ifndef PQRR_ORACLE_H
#define PQRR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
int orc_set_threads(int t);

/* ---- L0 primitives (distance.hpp, topk.hpp, types.hpp) ---- */
float orc_l2_sq(const float* a, const float* b, size_t d);
double orc_l2_sq_d(const float* a, const float* b, size_t d);
/* k smallest (id, dist) under neighbor_less; returns count written. */
size_t orc_topk(const uint32_t* ids, const float* dists, size_t n, size_t k,
                uint32_t* out_ids, float* out_dists);

/* ---- L1k kernels (kernels.hpp:13-43) ---- */
int orc_assign_batch(const float* points, size_t n, uint32_t dim, const float* centroids,
                     uint32_t k, uint32_t* out_assign, float* out_dist);
/* books: m * ks * (d/m) floats */
int orc_encode_batch(const float* books, uint32_t d, uint32_t m, uint32_t ks, const float* data,
                     size_t n, uint8_t* out_codes);
int orc_decode_batch(const float* books, uint32_t d, uint32_t m, uint32_t ks,
                     const uint8_t* codes, size_t n, float* out_data);
int orc_build_lut(const float* books, uint32_t d, uint32_t m, uint32_t ks, const float* x,
                  float* out_lut /* m*ks */);
float orc_adc_distance(const float* lut, uint32_t m, uint32_t ks, const uint8_t* code);
/* Serial scan + bounded heap (kernels.cpp:55-96 semantics); returns count. */
size_t orc_scan_topk(const float* lut, uint32_t m, uint32_t ks, const uint8_t* codes, size_t n,
                     size_t kprime, uint32_t id_base, uint32_t* out_ids, float* out_dists);

/* ---- training (kmeans.hpp:21-38, product_quantizer.hpp:37-40) ---- */
int orc_kmeans_train(const float* points, size_t n, uint32_t dim, uint32_t k,
                     uint32_t iterations, uint64_t seed, uint32_t redo, float* out_centroids,
                     double* out_final_mse, double* out_trace /* iterations, may be NULL */);
int orc_pq_train(const float* training, size_t n, uint32_t d, uint32_t m, uint32_t ks,
                 uint32_t iterations, uint64_t seed, uint32_t redo, float* out_books);

/* ---- IVF index (ivf_index.hpp:13-83) ---- */
typedef struct orc_ivf orc_ivf;
int orc_ivf_train(const float* training, size_t n, uint32_t d, uint32_t c, uint32_t m,
                  uint32_t ks, uint32_t iterations, uint64_t seed, float* out_coarse,
                  float* out_books);
int orc_ivf_refine_train(const float* coarse, uint32_t c, const float* books, uint32_t d,
                         uint32_t m, uint32_t ks, const float* training, size_t n,
                         uint32_t mprime, uint32_t iterations, uint64_t seed,
                         float* out_rbooks);
orc_ivf* orc_ivf_build(const float* coarse, uint32_t c, const float* books, uint32_t d,
                       uint32_t m, uint32_t ks, const float* base, size_t n);
void orc_ivf_free(orc_ivf* ix);
size_t orc_ivf_list_size(const orc_ivf* ix, uint32_t list);
/* copies list ids (u32) and codes (len*m) */
int orc_ivf_list_get(const orc_ivf* ix, uint32_t list, uint32_t* ids, uint8_t* codes);
int orc_ivf_assignments(const orc_ivf* ix, uint32_t* list_of_id, uint32_t* pos_of_id);
/* Attach refinement codes computed by ivf_refine_encode (id-aligned). */
int orc_ivf_refine_encode(orc_ivf* ix, const float* rbooks, uint32_t mprime,
                          const float* base, size_t n, uint8_t* out_rcodes /* may be NULL */);
/* Per query: counts[q] entries written at out_*[q*kprime]. */
int orc_ivf_search_batch(const orc_ivf* ix, const float* queries, size_t nq, uint32_t v,
                         size_t kprime, uint32_t* out_ids, float* out_dists, uint32_t* counts);
int orc_ivf_reconstruct(const orc_ivf* ix, uint32_t id, float* out /* d */);
/* shortlist: per query counts[q] ids at sl_ids[q*sl_stride]; output top-k per query. */
int orc_ivf_rerank_batch(const orc_ivf* ix, const float* queries, size_t nq,
                         const uint32_t* sl_ids, const uint32_t* sl_counts, size_t sl_stride,
                         size_t k, uint32_t* out_ids, float* out_dists);
/* Coarse probe selection alone (for parity of the first kernel): v ids per query. */
/* ADC / ADC+R (adc_index.hpp:13-31, refine.hpp:30-53), restated directly. */
int orc_adc_encode(const float* books, uint32_t d, uint32_t m, uint32_t ks, const float* base,
                   size_t n, uint8_t* out_codes);
int orc_adc_search_batch(const float* books, uint32_t d, uint32_t m, uint32_t ks,
                         const uint8_t* codes, size_t n, const float* queries, size_t nq,
                         size_t kprime, uint32_t* out_ids, float* out_dists, uint32_t* counts);
int orc_refine_train(const float* books, uint32_t d, uint32_t m, uint32_t ks, const float* training,
                     size_t n, uint32_t mprime, uint32_t iterations, uint64_t seed,
                     float* out_rbooks);
int orc_adc_refine_encode(const float* books, uint32_t d, uint32_t m, const float* rbooks,
                          uint32_t mprime, uint32_t ks, const float* base, size_t n,
                          uint8_t* out_rcodes);
int orc_adc_reconstruct(const float* books, uint32_t d, uint32_t m, const float* rbooks,
                        uint32_t mprime, uint32_t ks, const uint8_t* code, const uint8_t* rcode,
                        float* out);
int orc_adc_rerank_batch(const float* books, uint32_t d, uint32_t m, const float* rbooks,
                         uint32_t mprime, uint32_t ks, const uint8_t* codes, const uint8_t* rcodes,
                         const float* queries, size_t nq, const uint32_t* sl_ids,
                         const uint32_t* sl_counts, size_t sl_stride, size_t k, uint32_t* out_ids,
                         float* out_dists);
int orc_coarse_probe(const float* coarse, uint32_t c, uint32_t d, const float* queries,
                     size_t nq, uint32_t v, uint32_t* out_lists, float* out_dists);

/* ---- eval (eval.hpp:13-33) ---- */
/* nearest id (lowest id among exact ties) and its fp64 distance, per query. */
int orc_exact_nearest(const float* base, size_t n, uint32_t d, const float* queries, size_t nq,
                      uint32_t* out_ids, double* out_dists);
double orc_recall_at_r(const uint32_t* res_ids, const uint32_t* res_counts, size_t stride,
                       size_t nq, const uint32_t* gt_nearest, size_t r);

/* ---- synthetic SIFT-like generator (BASELINE.json configs; rng.hpp:28-56) ---- */
enum { ORC_SET_CENTERS = 0, ORC_SET_TRAIN = 1, ORC_SET_BASE = 2, ORC_SET_QUERY = 3 };
uint64_t orc_splitmix_stream_state(uint64_t seed, uint32_t set, uint64_t row);
uint64_t orc_splitmix_next(uint64_t* state);
void orc_bounded_u32(uint32_t seed, uint32_t bound, size_t n, uint32_t* out);
void orc_uniform01(uint32_t seed, size_t n, float* out);
double orc_ln(double u);
void orc_sincos_2pi(double u, double* s, double* c);
int orc_synth_centers(uint64_t seed, uint32_t clusters, uint32_t d, double* out_centers);
int orc_synth_rows(uint64_t seed, uint32_t set, uint64_t row0, size_t n, uint32_t d,
                   const double* centers, uint32_t clusters, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
