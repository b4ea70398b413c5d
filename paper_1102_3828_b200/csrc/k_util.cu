// k_util.cu — small device utilities: launch accounting, histograms, scans,
// and the stable (list, value) radix sort used by the layout build, probe
// inversion and k-means update (CUB from the CUDA toolkit; data movement only,
// not on the arithmetic path).
#include <atomic>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include "common.cuh"
#include <map>
#include <mutex>
#include <utility>

#include "internal.h"

namespace pqrr_b200 {

static std::atomic<unsigned long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((unsigned long long)n); }
unsigned long long launch_count() { return g_launches.load(); }

int sm_count() {
    int dev = 0;
    PQRR_CUDA(cudaGetDevice(&dev));
    static int cached[64] = {0};
    if (dev < 64 && cached[dev]) return cached[dev];
    int n = 0;
    PQRR_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    if (dev < 64) cached[dev] = n;
    return n;
}

void set_max_smem(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> set;  // (device, kernel) -> limit
    int dev = 0;
    PQRR_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = set[{dev, kernel}];
    if (bytes <= cur) return;
    PQRR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
}

namespace {

__global__ void histogram_kernel(const uint32_t* __restrict__ keys, size_t n, uint32_t nbins,
                                 uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t sh[];
    const bool use_smem = nbins <= 8192;
    if (use_smem)
        for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        uint32_t k = keys[i];
        if (k < nbins) {
            if (use_smem) atomicAdd(&sh[k], 1u);
            else atomicAdd(&hist[k], 1u);
        }
    }
    __syncthreads();
    if (use_smem)
        for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x)
            if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void iota_kernel(uint32_t* out, size_t n) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint32_t)i;
}

}  // namespace

void launch_histogram(const uint32_t* keys, size_t n, uint32_t nbins, uint32_t* hist,
                      cudaStream_t s) {
    PQRR_CUDA(cudaMemsetAsync(hist, 0, nbins * sizeof(uint32_t), s));
    if (n == 0) return;
    size_t smem = nbins <= 8192 ? nbins * sizeof(uint32_t) : 0;
    unsigned grid = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)sm_count() * 4);
    histogram_kernel<<<grid, 256, smem, s>>>(keys, n, nbins, hist);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_iota(uint32_t* out, size_t n, cudaStream_t s) {
    if (n == 0) return;
    iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, n);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

// Small sorts (the work-item inversions of small batches): one CTA, bitonic
// sort of (key << 32 | index) in shared memory — stable like the radix sort,
// one launch instead of CUB's several.
constexpr int kSmallSort = 1024;  // above ~1k the bitonic stages cost more than CUB's passes
__global__ __launch_bounds__(1024) void small_sort_pairs_kernel(const uint32_t* __restrict__ keys_in,
                                                               uint32_t* __restrict__ keys_out,
                                                               const uint32_t* __restrict__ vals_in,
                                                               uint32_t* __restrict__ vals_out, uint32_t n) {
    __shared__ unsigned long long sk[kSmallSort];
    uint32_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x)
        sk[i] = i < n ? (((unsigned long long)keys_in[i] << 32) | i) : ~0ull;
    __syncthreads();
    for (uint32_t size = 2; size <= n2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
                const uint32_t jx = i ^ stride;
                if (jx > i) {
                    const bool up = (i & size) == 0;
                    const unsigned long long a = sk[i], b = sk[jx];
                    if ((a > b) == up) {
                        sk[i] = b;
                        sk[jx] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned long long v = sk[i];
        keys_out[i] = (uint32_t)(v >> 32);
        vals_out[i] = vals_in[(uint32_t)v];
    }
}

void sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                uint32_t* vals_out, size_t n, int bits, cudaStream_t s) {
    if (n == 0) return;
    if (bits < 1) bits = 1;
    if (n <= (size_t)kSmallSort) {
        small_sort_pairs_kernel<<<1, 1024, 0, s>>>(keys_in, keys_out, vals_in, vals_out, (uint32_t)n);
        PQRR_LAUNCH_CHECK();
        count_launch();
        return;
    }
    size_t tmp = 0;
    PQRR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys_in, keys_out, vals_in, vals_out,
                                              (int64_t)n, 0, bits, s));
    void* d_tmp = nullptr;
    PQRR_CUDA(cudaMallocAsync(&d_tmp, tmp, s));
    PQRR_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, keys_in, keys_out, vals_in, vals_out,
                                              (int64_t)n, 0, bits, s));
    PQRR_CUDA(cudaFreeAsync(d_tmp, s));
    count_launch(bits <= 8 ? 2 : 4);
}

void segmented_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                          uint32_t* vals_out, size_t n, uint32_t nseg, const uint64_t* seg_begin,
                          const uint64_t* seg_end, int bits, cudaStream_t s) {
    if (n == 0 || nseg == 0) return;
    size_t tmp = 0;
    PQRR_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp, keys_in, keys_out, vals_in,
                                                       vals_out, (int64_t)n, (int64_t)nseg,
                                                       seg_begin, seg_end, 0, bits, s));
    void* d_tmp = nullptr;
    PQRR_CUDA(cudaMallocAsync(&d_tmp, tmp, s));
    PQRR_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(d_tmp, tmp, keys_in, keys_out, vals_in,
                                                       vals_out, (int64_t)n, (int64_t)nseg,
                                                       seg_begin, seg_end, 0, bits, s));
    PQRR_CUDA(cudaFreeAsync(d_tmp, s));
    count_launch(bits <= 8 ? 1 : 4);
}

void exclusive_scan_u64(const uint64_t* in, uint64_t* out, size_t n, cudaStream_t s) {
    if (n == 0) return;
    size_t tmp = 0;
    PQRR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int64_t)n, s));
    void* d_tmp = nullptr;
    PQRR_CUDA(cudaMallocAsync(&d_tmp, tmp, s));
    PQRR_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, in, out, (int64_t)n, s));
    PQRR_CUDA(cudaFreeAsync(d_tmp, s));
    count_launch(2);
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, cudaStream_t s) {
    if (n == 0) return;
    size_t tmp = 0;
    PQRR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int64_t)n, s));
    void* d_tmp = nullptr;
    PQRR_CUDA(cudaMallocAsync(&d_tmp, tmp, s));
    PQRR_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, in, out, (int64_t)n, s));
    PQRR_CUDA(cudaFreeAsync(d_tmp, s));
    count_launch(2);
}

}  // namespace pqrr_b200
