// k_kmeans.cu — device half of deterministic Lloyd k-means (kmeans.hpp:30-38).
// The assignment step reuses the exact argmin tile kernel (k_coarse.cu); the
// update here reproduces the serial id-order fp64 accumulation of the
// reference policy exactly: one thread per (cluster, component) walks the
// cluster's members in ascending id order (a stable sort by cluster), so the
// sequence of double additions is the same as the host loop's.
#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

__global__ void gather_rows_kernel(const float* __restrict__ pts, uint32_t dim,
                                   const uint32_t* __restrict__ rows, uint32_t k,
                                   float* __restrict__ out) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)k * dim) return;
    size_t c = idx / dim, t = idx % dim;
    out[idx] = pts[(size_t)rows[c] * dim + t];
}

__global__ void centroid_update_kernel(const float* __restrict__ pts, uint32_t dim,
                                       const uint32_t* __restrict__ sorted_ids,
                                       const uint32_t* __restrict__ cl_off, uint32_t k,
                                       float* __restrict__ centroids) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)k * dim) return;
    uint32_t c = (uint32_t)(idx / dim), t = (uint32_t)(idx % dim);
    uint32_t lo = cl_off[c], hi = cl_off[c + 1];
    if (lo == hi) return;  // empty cluster: handled by the host split policy
    double s = 0.0;
    for (uint32_t i = lo; i < hi; ++i) s = __dadd_rn(s, (double)pts[(size_t)sorted_ids[i] * dim + t]);
    centroids[idx] = (float)__ddiv_rn(s, (double)(hi - lo));
}

}  // namespace

void launch_gather_rows(const float* pts, uint32_t dim, const uint32_t* rows, uint32_t k,
                        float* out, cudaStream_t s) {
    size_t total = (size_t)k * dim;
    if (!total) return;
    gather_rows_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(pts, dim, rows, k, out);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_centroid_update(const float* pts, uint32_t dim, const uint32_t* sorted_ids,
                            const uint32_t* cl_off, uint32_t k, float* centroids,
                            cudaStream_t s) {
    size_t total = (size_t)k * dim;
    if (!total) return;
    centroid_update_kernel<<<(unsigned)((total + 127) / 128), 128, 0, s>>>(pts, dim, sorted_ids,
                                                                            cl_off, k, centroids);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
