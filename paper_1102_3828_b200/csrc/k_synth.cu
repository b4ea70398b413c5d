// k_synth.cu — device-side synthetic SIFT-like generator (BASELINE.json configs,
// SURVEY.md §8d).  Bit-identical to the host definition: SplitMix64 streams as
// rng.hpp:30-45, one stream per (seed, set, row), Box-Muller with ln / sin / cos
// spelled out in IEEE double + - * / (all _rn intrinsics, no contraction), so
// every GPU shard generates its own id range with no communication.
#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

__device__ __forceinline__ u64 fmix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ u64 stream_state(u64 seed, uint32_t set, u64 row) {
    return fmix64(fmix64(seed ^ ((u64)(set + 1) * 0xD1B54A32D192ED03ull)) + row);
}
__device__ __forceinline__ u64 sm_next(u64& s) {
    s += 0x9e3779b97f4a7c15ull;
    return fmix64(s);
}
__device__ __forceinline__ double sm_open01(u64& s) {
    return __dmul_rn((double)((sm_next(s) >> 11) + 1), 1.0 / 9007199254740992.0);
}

#define DM(a, b) __dmul_rn((a), (b))
#define DA(a, b) __dadd_rn((a), (b))

__device__ double dev_ln(double u) {
    u64 b = (u64)__double_as_longlong(u);
    int e = (int)((b >> 52) & 0x7ff) - 1023;
    double f = __longlong_as_double((long long)((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
    if (f > 0x1.6a09e667f3bcdp+0) {
        f = DM(f, 0.5);
        e += 1;
    }
    double s = __ddiv_rn(__dsub_rn(f, 1.0), DA(f, 1.0));
    double z = DM(s, s);
    double p = 0x1.8618618618618p-5;
    p = DA(DM(p, z), 0x1.af286bca1af28p-5);
    p = DA(DM(p, z), 0x1.e1e1e1e1e1e1ep-5);
    p = DA(DM(p, z), 0x1.1111111111111p-4);
    p = DA(DM(p, z), 0x1.3b13b13b13b14p-4);
    p = DA(DM(p, z), 0x1.745d1745d1746p-4);
    p = DA(DM(p, z), 0x1.c71c71c71c71cp-4);
    p = DA(DM(p, z), 0x1.2492492492492p-3);
    p = DA(DM(p, z), 0x1.999999999999ap-3);
    p = DA(DM(p, z), 0x1.5555555555555p-2);
    p = DA(DM(p, z), 1.0);
    double lnf = DM(DM(2.0, s), p);
    return DA(DM((double)e, 0x1.62e42fefa39efp-1), lnf);
}

__device__ void dev_sincos_2pi(double u, double& sn, double& cs) {
    double t = DM(u, 4.0);
    double q = floor(t);
    double r = __dsub_rn(t, q);
    double ph = DM(r, 0x1.921fb54442d18p+0);
    double z = DM(ph, ph);
    double ps = -0x1.761b41316381ap-75;
    ps = DA(DM(ps, z), 0x1.71b8ef6dcf572p-66);
    ps = DA(DM(ps, z), -0x1.2f49b46814157p-57);
    ps = DA(DM(ps, z), 0x1.952c77030ad4ap-49);
    ps = DA(DM(ps, z), -0x1.ae7f3e733b81fp-41);
    ps = DA(DM(ps, z), 0x1.6124613a86d09p-33);
    ps = DA(DM(ps, z), -0x1.ae64567f544e4p-26);
    ps = DA(DM(ps, z), 0x1.71de3a556c734p-19);
    ps = DA(DM(ps, z), -0x1.a01a01a01a01ap-13);
    ps = DA(DM(ps, z), 0x1.1111111111111p-7);
    ps = DA(DM(ps, z), -0x1.5555555555555p-3);
    ps = DA(DM(ps, z), 1.0);
    double s = DM(ph, ps);
    double pc = -0x1.0ce396db7f853p-70;
    pc = DA(DM(pc, z), 0x1.e542ba4020225p-62);
    pc = DA(DM(pc, z), -0x1.6827863b97d97p-53);
    pc = DA(DM(pc, z), 0x1.ae7f3e733b81fp-45);
    pc = DA(DM(pc, z), -0x1.93974a8c07c9dp-37);
    pc = DA(DM(pc, z), 0x1.1eed8eff8d898p-29);
    pc = DA(DM(pc, z), -0x1.27e4fb7789f5cp-22);
    pc = DA(DM(pc, z), 0x1.a01a01a01a01ap-16);
    pc = DA(DM(pc, z), -0x1.6c16c16c16c17p-10);
    pc = DA(DM(pc, z), 0x1.5555555555555p-5);
    pc = DA(DM(pc, z), -0x1.0000000000000p-1);
    pc = DA(DM(pc, z), 1.0);
    double c = pc;
    switch ((int)q & 3) {
        case 0: sn = s; cs = c; break;
        case 1: sn = c; cs = -s; break;
        case 2: sn = -s; cs = -c; break;
        default: sn = -c; cs = s; break;
    }
}

__device__ __forceinline__ uint32_t quantize(double v) {
    if (!(v > 0.0)) v = 0.0;
    if (v > 255.0) v = 255.0;
    int iv = __double2int_rn(v);  // round half to even
    return iv < 4 ? 0u : (uint32_t)iv;
}

__global__ void synth_centers_kernel(u64 seed, uint32_t clusters, uint32_t d, double* out) {
    uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= clusters) return;
    u64 s = stream_state(seed, 0, k);
    for (uint32_t t = 0; t < d; ++t) out[(size_t)k * d + t] = DM(-20.0, dev_ln(sm_open01(s)));
}

// One thread per row; bytes packed 4 at a time.
__global__ void synth_rows_kernel(u64 seed, uint32_t set, u64 row0, size_t n, uint32_t d,
                                  const double* __restrict__ centers, uint32_t clusters,
                                  uint8_t* __restrict__ out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    u64 s = stream_state(seed, set, row0 + i);
    u64 comp = __umul64hi(sm_next(s), (u64)clusters);
    const double* mu = centers + comp * d;
    uint8_t* o = out + i * d;
    uint32_t word = 0;
    for (uint32_t t = 0; t < d; t += 2) {
        double u1 = sm_open01(s);
        double u2 = sm_open01(s);
        double r = __dsqrt_rn(DM(-2.0, dev_ln(u1)));
        double sn, cs;
        dev_sincos_2pi(u2, sn, cs);
        uint32_t b0 = quantize(DA(mu[t], DM(10.0, DM(r, cs))));
        word |= b0 << (8 * (t & 3));
        if (t + 1 < d) {
            uint32_t b1 = quantize(DA(mu[t + 1], DM(10.0, DM(r, sn))));
            word |= b1 << (8 * ((t + 1) & 3));
        }
        if (((t + 2) & 3) == 0 || t + 2 >= d) {
            if ((d & 3) == 0) {
                *reinterpret_cast<uint32_t*>(o + (t & ~3u)) = word;
            } else {
                for (uint32_t b = t & ~3u; b < d && b < (t & ~3u) + 4; ++b)
                    o[b] = (uint8_t)(word >> (8 * (b & 3)));
            }
            word = 0;
        }
    }
}

}  // namespace

void launch_synth_centers(uint64_t seed, uint32_t clusters, uint32_t d, double* centers,
                          cudaStream_t s) {
    synth_centers_kernel<<<(clusters + 127) / 128, 128, 0, s>>>(seed, clusters, d, centers);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_synth_rows(uint64_t seed, uint32_t set, uint64_t row0, size_t n, uint32_t d,
                       const double* centers, uint32_t clusters, uint8_t* out, cudaStream_t s) {
    if (n == 0) return;
    synth_rows_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(seed, set, row0, n, d, centers,
                                                                  clusters, out);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace pqrr_b200
