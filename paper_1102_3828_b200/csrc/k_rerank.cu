// k_rerank.cu — K5a: refined distances of every shortlist entry on CTA PAIRS
// (thread-block clusters of 2, distributed shared memory).
//
// ivf_rerank (ivf_index.hpp:79-81) needs, per candidate, the reconstruction
//   yhat[t] = (C_l[t] + B_j[code_j][t - 16 j]) + R_j'[rcode_j'][t - dsr j']
// (ivf_index.hpp:75-77) and l2_sq(x, yhat) in the reference order
// (distance.hpp:16-33): four accumulators s_{t mod 4} summed in ascending t,
// then (s0 + s1) + (s2 + s3).  Per candidate that is 512 B of PQ rows and
// 512 B of refinement rows gathered at random, which must come from on-chip
// memory — but the two code books are 128 KiB each and do not both fit one
// SM's shared memory.
//
// So the two CTAs of a cluster split the DIMENSIONS: CTA r holds, for dims
// 64 r .. 64 r + 63, both books in CODE-MAJOR layout ([code][64 dims], 64 KiB
// each): a lane that owns dims 64 r + 4 g .. + 3 reads its quad of any row at
// bank group g mod 8, so every book gather is conflict-free whatever the
// codes.  Both CTAs walk the same chunks (32 candidates of one query); a warp
// handles 2 candidates per step (half warp each, lane g = one dim quad), the
// squares go to a padded 8-candidate tile, and lanes (candidate, k) add the 16
// terms of s_k of their half in ascending t.  CTA 0's partial sums (16 B per
// candidate) are stored straight into CTA 1's shared memory (distributed shared memory)
// with st.async, which completes CTA 1's mbarrier; CTA 1 continues the same four
// chains over dims 64..127 — the reference's sequential order across the whole
// vector — and forms (s0 + s1) + (s2 + s3).  Per-warp full / empty barriers
// with a 2-slot ring let CTA 0 run a chunk ahead.
#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int RP_WARPS = 16;
constexpr int RP_TLD = 68;  // tile row stride (floats): 4 cc + k + 4 g distinct banks
constexpr int RP_MLD = 40;  // transposed metadata row stride (bytes): 10 j + 2 s banks distinct

__device__ __forceinline__ unsigned s_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cta_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned peer_addr(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// Asynchronous remote store that completes `bytes` of the peer's mbarrier
// transaction count (no fence on the producer side).
__device__ __forceinline__ void st_peer_async(unsigned a, float v, unsigned peer_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(a),
                 "r"(__float_as_uint(v)), "r"(peer_bar) : "memory");
}
__device__ __forceinline__ void expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Remote arrive / local wait with the default (CTA-scope) semantics, as the
// cross-CTA TMA pipelines use them: a cluster-scope acquire would invalidate
// L1 (CCTL.IVALL) and a cluster-scope release fence the GPU on every chunk.
__device__ __forceinline__ void arrive_peer(unsigned a) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void wait_parity(unsigned a, unsigned parity) {
    unsigned done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(a), "r"(parity) : "memory");
}
// Random gathers with no L1 allocation: a candidate's sectors are never
// reused on this SM (the sibling CTA reads the other half), so they would only
// evict the coarse rows and queries L1 does reuse.
__device__ __forceinline__ uint32_t ld_na_u32(const void* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_na_u16(const void* p) {
    unsigned short v;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_na_v2(const void* p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_na_v4(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int DSR>
struct RpSmem {
    static constexpr int HB = (128 / DSR) / 2;  // refinement code bytes per half
    static constexpr size_t books = 2 * 256 * 64 * 4;
    static constexpr size_t tiles = (size_t)RP_WARPS * 8 * RP_TLD * 4;
    static constexpr size_t part = (size_t)RP_WARPS * 2 * 32 * 4 * 4;
    static constexpr size_t mlist = (size_t)RP_WARPS * 32 * 4;
    static constexpr size_t mcode = (size_t)RP_WARPS * 4 * RP_MLD;
    static constexpr size_t mrc = (size_t)RP_WARPS * HB * RP_MLD;
    static constexpr size_t bars = (size_t)RP_WARPS * 2 * 8;
    static constexpr size_t pos = (size_t)RP_WARPS * 33 * 4;
    static constexpr size_t total = books + tiles + part + mlist + mcode + mrc + bars + pos;
};

template <int DSR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(RP_WARPS * 32, 1) rerank_pair_kernel(
    const u64* __restrict__ sl_key, const uint32_t* __restrict__ sl_pos,
    const uint32_t* __restrict__ sl_cnt, uint32_t stride, size_t nq, const float* __restrict__ xq,
    const uint16_t* __restrict__ block_list, const float* __restrict__ coarse,
    const uint8_t* __restrict__ codes, const float* __restrict__ books,
    const uint8_t* __restrict__ rcodes, const float* __restrict__ rbooks, float* __restrict__ rdist,
    uint32_t* __restrict__ rid, const uint32_t* __restrict__ ids, u64 nz) {
    using L = RpSmem<DSR>;
    constexpr int MP = 128 / DSR, HB = L::HB;
    extern __shared__ float4 rp_smem[];
    uint8_t* base = reinterpret_cast<uint8_t*>(rp_smem);
    const float4* bookP = reinterpret_cast<const float4*>(base);            // [256][16] float4
    const float4* bookR = bookP + 256 * 16;                                 // [256][16] float4
    float* tiles = reinterpret_cast<float*>(base + L::books);                // [warps][8][TLD]
    float* part = reinterpret_cast<float*>(base + L::books + L::tiles);      // [warps][2][32][4]
    uint32_t* mlist = reinterpret_cast<uint32_t*>(base + L::books + L::tiles + L::part);
    uint8_t* mcode = reinterpret_cast<uint8_t*>(mlist) + L::mlist;         // [warps][4][MLD]
    uint8_t* mrc = mcode + L::mcode;                                        // [warps][HB][MLD]
    u64* bars = reinterpret_cast<u64*>(mrc + L::mrc);  // [warps][2]: full (rank 1) / empty (rank 0)
    uint32_t* posbuf = reinterpret_cast<uint32_t*>(bars + RP_WARPS * 2);  // [warps][32 positions + count]

    const unsigned r = cta_rank();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // this CTA's half of both code books, code-major
    {
        float4* bp = reinterpret_cast<float4*>(base);
        float4* br = bp + 256 * 16;
        for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) {
            const int c = i >> 4, t = 64 * (int)r + 4 * (i & 15);
            bp[i] = __ldg(reinterpret_cast<const float4*>(books + ((size_t)(t >> 4) * 256 + c) * 16 + (t & 15)));
            br[i] = __ldg(reinterpret_cast<const float4*>(rbooks + ((size_t)(t / DSR) * 256 + c) * DSR + t % DSR));
        }
    }
    if (threadIdx.x < RP_WARPS * 2)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_addr(bars + threadIdx.x)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    cluster_sync();

    float* tile = tiles + warp * 8 * RP_TLD;
    float* wpart = part + warp * 2 * 32 * 4;
    uint32_t* wlist = mlist + warp * 32;
    uint8_t* wcode = mcode + warp * 4 * RP_MLD;
    uint8_t* wrc = mrc + warp * HB * RP_MLD;
    const unsigned bar0 = s_addr(bars + warp * 2);
    // rank 0 writes partials into the peer's shared memory with st.async, each
    // store completing bytes of the peer's "full" barrier (armed by rank 1 with
    // the chunk's byte count); rank 1 releases the slot with one arrive on the
    // peer's "empty" barrier
    const unsigned peer_bar0 = peer_addr(bar0, r ^ 1u);
    const unsigned peer_part = peer_addr(s_addr(wpart), 1u);

    const uint32_t h = lane >> 4, g = lane & 15;  // squares: candidate of the pair, dim quad
    const uint32_t jl = g >> 2;                   // PQ sub-space within the half
    const uint32_t jrl = (4 * g) / DSR;           // refinement sub-space within the half
    const int cc = lane >> 2, kk = lane & 3;      // sums: candidate of the sub-batch, accumulator
    const uint32_t cpq = (stride + 31) / 32;
    const size_t total = nq * (size_t)cpq;
    const size_t tw = (size_t)(gridDim.x >> 1) * RP_WARPS;
    // chunk metadata, software-pipelined (lane = candidate): while chunk i
    // computes, the positions and row counts of chunk i + 2 and the
    // position-dependent gathers (list, code and refinement-code bytes) of
    // chunk i + 1 are in flight, so no warp waits on a dependent DRAM round
    // trip.  Chunk indices advance by the grid stride; chunks past a query's
    // count carry nb = 0 and are skipped by both CTAs alike.
    uint32_t p_id = 0, p_list = 0, p_code = 0;
    uint32_t p_rc[(HB + 3) / 4];
    // the positions and row count of chunk i + 2 travel by cp.async into a
    // per-warp smem slot: a register load here would be the warp's 7th
    // outstanding global load and wait for a free scoreboard (one DRAM round
    // trip per chunk, ncu: 18% of K5a's stall samples at C4)
    uint32_t n_pos = 0, n_cnt = 0;  // chunk i + 1: position of the lane's entry, row count
    uint32_t* wpos = posbuf + warp * 33;
    auto load_pos = [&](size_t c) {  // no dependency: rows are allocated k' wide
        const size_t q = c / cpq;
        const uint32_t i0 = (uint32_t)(c % cpq) * 32;
        cp_async4(wpos + lane, sl_pos + q * stride + i0 + min((uint32_t)lane, stride - 1 - i0));
        if (lane == 0) cp_async4(wpos + 32, sl_cnt + q);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto take_pos = [&]() {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        n_pos = wpos[lane];
        n_cnt = wpos[32];
        __syncwarp();  // read before the next cp.async overwrites the slot
    };
    auto nb_of = [&](size_t c, uint32_t cnt) -> uint32_t {
        const uint32_t i0 = (uint32_t)(c % cpq) * 32;
        return cnt > i0 ? min(32u, cnt - i0) : 0u;
    };
    auto load_meta = [&](size_t c, uint32_t pos, uint32_t nb) {
        const size_t t0 = (c / cpq) * stride + (uint32_t)(c % cpq) * 32;
        if ((uint32_t)lane < nb) {
            // rank 1 writes the ids: from the shortlist keys, or from the id
            // array when the selection left them out of the keys (ids = non-null)
            if (r) p_id = ids ? ld_na_u32(ids + pos) : key_id(sl_key[t0 + lane]);
            p_list = ld_na_u16(block_list + (pos >> 4));
            p_code = ld_na_u32(codes + (size_t)pos * 8 + 4 * r);
            const uint8_t* rs = rcodes + (size_t)pos * MP + r * HB;
            if constexpr (HB == 16) {
                const uint4 v = ld_na_v4(rs);
                p_rc[0] = v.x, p_rc[1] = v.y, p_rc[2] = v.z, p_rc[3] = v.w;
            } else if constexpr (HB == 8) {
                const uint2 v = ld_na_v2(rs);
                p_rc[0] = v.x, p_rc[1] = v.y;
            } else {
                p_rc[0] = ld_na_u32(rs);
            }
        }
    };
    const size_t start = (size_t)(blockIdx.x >> 1) * RP_WARPS + warp;
    uint32_t cur_cnt = 0;
    if (start < total) {
        load_pos(start);
        take_pos();
        cur_cnt = n_cnt;
        load_meta(start, n_pos, nb_of(start, cur_cnt));
        if (start + tw < total) load_pos(start + tw);
    }
    uint32_t it = 0;
    for (size_t ch = start; ch < total; ch += tw) {
        const size_t q = ch / cpq;
        const uint32_t i0 = (uint32_t)(ch % cpq) * 32;
        const uint32_t nb = nb_of(ch, cur_cnt);
        const size_t t0 = q * stride + i0;
        const uint32_t slot = it & 1u, use = it >> 1;
        __syncwarp();  // the previous chunk's metadata reads are done
        if (nb) {
            // lanes past nb repeat the last candidate, so sub-batches run
            // without bounds checks (duplicates are never stored)
            const int src = min(lane, (int)nb - 1);
            wlist[lane] = __shfl_sync(0xffffffffu, p_list, src);
            const uint32_t pc = __shfl_sync(0xffffffffu, p_code, src);
#pragma unroll
            for (int j = 0; j < 4; ++j) wcode[j * RP_MLD + lane] = (uint8_t)(pc >> (8 * j));
#pragma unroll
            for (int v = 0; v < (HB + 3) / 4; ++v) {
                const uint32_t w = __shfl_sync(0xffffffffu, p_rc[v], src);
#pragma unroll
                for (int b = 0; b < 4 && 4 * v + b < HB; ++b) wrc[(4 * v + b) * RP_MLD + lane] = (uint8_t)(w >> (8 * b));
            }
            if (r && (uint32_t)lane < nb) rid[t0 + lane] = p_id;
        }
        if (ch + tw < total) {
            take_pos();
            cur_cnt = n_cnt;
            load_meta(ch + tw, n_pos, nb_of(ch + tw, cur_cnt));
            if (ch + 2 * tw < total) load_pos(ch + 2 * tw);
        }
        if (!nb) continue;
        ++it;
        const float4 x = __ldg(reinterpret_cast<const float4*>(xq + q * 128 + 64 * r) + g);
        const u64 x01 = pk2(x.x, x.y), x23 = pk2(x.z, x.w);
        if (r == 0 && use > 0) wait_parity(bar0 + 8 * slot, (use - 1) & 1u);  // peer done with the slot
        if (r == 1 && lane == 0) expect_tx(bar0 + 8 * slot, 128u * ((nb + 7) / 8));  // partials to come
        __syncwarp();
        uint32_t cur_l = 0xffffffffu;
        float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
        for (uint32_t sb = 0; sb < nb; sb += 8) {
            const uint4 lq0 = reinterpret_cast<const uint4*>(wlist)[sb >> 2];
            const uint4 lq1 = reinterpret_cast<const uint4*>(wlist)[(sb >> 2) + 1];
            const uint32_t la[4] = {h ? lq0.y : lq0.x, h ? lq0.w : lq0.z, h ? lq1.y : lq1.x, h ? lq1.w : lq1.z};
            const u64 cb = *reinterpret_cast<const u64*>(wcode + jl * RP_MLD + sb);
            const u64 rb = *reinterpret_cast<const u64*>(wrc + jrl * RP_MLD + sb);
            float4 bv[4], rv[4];
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                const uint32_t c = 2 * st + h;
                bv[st] = bookP[((uint32_t)(cb >> (8 * c)) & 0xffu) * 16 + g];
                rv[st] = bookR[((uint32_t)(rb >> (8 * c)) & 0xffu) * 16 + g];
            }
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                if (la[st] != cur_l) {  // candidates arrive grouped by list: rare
                    cur_l = la[st];
                    cv = __ldg(reinterpret_cast<const float4*>(coarse + (size_t)cur_l * 128 + 64 * r) + g);
                }
                const u64 y01 = add2(add2(pk2(cv.x, cv.y), pk2(bv[st].x, bv[st].y)), pk2(rv[st].x, rv[st].y));
                const u64 y23 = add2(add2(pk2(cv.z, cv.w), pk2(bv[st].z, bv[st].w)), pk2(rv[st].z, rv[st].w));
                const u64 q01 = sq2(sub2(x01, y01), nz), q23 = sq2(sub2(x23, y23), nz);
                *reinterpret_cast<float4*>(tile + (2 * st + h) * RP_TLD + 4 * g) =
                    make_float4(lo2(q01), hi2(q01), lo2(q23), hi2(q23));
            }
            __syncwarp();
            float t[16];
#pragma unroll
            for (int gg = 0; gg < 16; ++gg) t[gg] = tile[cc * RP_TLD + 4 * gg + kk];
            float sacc = 0.f;  // l2_sq's accumulators start at +0 (distance.hpp:16-33)
            const int pi = (slot * 32 + sb + cc) * 4 + kk;
            if (r) {
                if (sb == 0) wait_parity(bar0 + 8 * slot, use & 1u);  // peer's partials landed
                sacc = wpart[pi];
            }
#pragma unroll
            for (int gg = 0; gg < 16; ++gg) sacc = __fadd_rn(sacc, t[gg]);
            if (r == 0) {
                st_peer_async(peer_part + 4u * pi, sacc, peer_bar0 + 8 * slot);
            } else {
                const float s1 = __shfl_down_sync(0xffffffffu, sacc, 1);
                const float pair = __fadd_rn(sacc, s1);  // kk = 0: s0 + s1, kk = 2: s2 + s3
                const float p23 = __shfl_down_sync(0xffffffffu, pair, 2);
                if (kk == 0 && sb + cc < nb) rdist[t0 + sb + cc] = __fadd_rn(pair, p23);
            }
            __syncwarp();
        }
        // rank 1 hands the slot back once its partials are consumed (rank 0's
        // st.async stores completed the full barrier themselves)
        __syncwarp();
        if (r == 1 && lane == 0) arrive_peer(peer_bar0 + 8 * slot);
    }
    cluster_sync();  // no CTA leaves while its peer may still touch its shared memory
}

void set_smem_attr(const void* f, size_t bytes) {
    set_max_smem((const void*)f, (size_t)((int)bytes));
}

}  // namespace

bool rerank_pair_supported(uint32_t d, uint32_t m, uint32_t ks, uint32_t mprime) {
    return d == 128 && m == 8 && ks == 256 && (mprime == 8 || mprime == 16 || mprime == 32);
}

void launch_rerank_pair(const uint64_t* sl_key, const uint32_t* sl_pos, const uint32_t* sl_cnt,
                        uint32_t stride, size_t nq, const float* xq, const uint16_t* block_list,
                        const float* coarse, const uint8_t* codes, const float* books,
                        const uint8_t* rcodes, const float* rbooks, uint32_t mprime, float* rdist,
                        uint32_t* rid, cudaStream_t s, const uint32_t* ids) {
    auto go = [&](auto kern, size_t smem) {
        static int clusters = 0;  // per instantiation: max co-resident clusters
        set_smem_attr((const void*)kern, smem);
        if (!clusters) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(2 * (unsigned)sm_count());
            cfg.blockDim = dim3(RP_WARPS * 32);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = 2;
            at.val.clusterDim.y = 1;
            at.val.clusterDim.z = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            PQRR_CUDA(cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg));
            if (clusters < 1) throw CudaError("re-ranker: no CTA pair fits an SM pair");
        }
        kern<<<2 * (unsigned)clusters, RP_WARPS * 32, smem, s>>>(
            reinterpret_cast<const u64*>(sl_key), sl_pos, sl_cnt, stride, nq, xq, block_list, coarse,
            codes, books, rcodes, rbooks, rdist, rid, ids, kNegZero2);
        PQRR_LAUNCH_CHECK();
        count_launch();
    };
    if (mprime == 32) go(rerank_pair_kernel<4>, RpSmem<4>::total);
    else if (mprime == 16) go(rerank_pair_kernel<8>, RpSmem<8>::total);
    else go(rerank_pair_kernel<16>, RpSmem<16>::total);
}

}  // namespace pqrr_b200
