// k_filter.cu — K4f + K4r: the main IVFADC scan (ivf_search's hot loop,
// ivf_index.hpp:58-61) as a conservative 4-bit filter followed by an exact
// recheck of the survivors.
//
// The exact scan (k_scan.cu, pass 0) is bound by shared-memory LUT gathers:
// 8 x 4 bytes per (entry, query).  Here a work item is one list and up to 64
// probing queries (four LUT-pass items), and the item's LUT holds 5-bit
// values in bytes, laid out [j][code][64 queries]: a lane's LDS.128 returns 16
// queries' values (8 bytes of gathers per entry-query instead of 32), and a
// 64-byte row keeps the parity-paired list order conflict-free exactly like
// the fp32 [j][code][16] layout.
//
// Conservativeness.  For query q and list l with exact LUT L_j[c] (the same
// values the exact scan sums), m_j = min_c L_j[c] and scale s (k_scan.cu
// quantize_item): v8_j[c] * s <= L_j[c] - m_j.  With Delta = 256 s / mult,
// v5 = min(31, (v8 * mult) >> 8) gives v5 * Delta <= L_j - m_j, so
//     sum_j L_j[c_j] >= sum_j m_j + Delta * sum_j v5_j[c_j].
// The fp32 ADC d = fl(...fl(fl(0 + L_0) + L_1)...) of non-negative terms is
// >= (1 - 8u) sum_j L_j, so d <= tau implies
//     sum_j v5_j <= T = floor((tau (1+e) - sum_m (1-e)) / Delta (1+e)),
// e = 2^-18 covering every rounding.  The filter keeps sum_j v5_j <= T, a
// superset of {d <= tau}; K4r recomputes d exactly for the survivors, so the
// exact shortlist is unchanged.  Delta targets (tau - sum_m) / band_div
// (default 100, FilterArgs): T ~ 100, an average of ~12 per subspace at the
// threshold, well below the clamp at 31.
// Byte sums stay <= 8 * 31 = 248 (no carries); the per-byte unsigned test
// x <= T is SWAR: r = (T | 0x80) - (x & 0x7f) never borrows, and bit 7 of
// (x ^ T) ? T : r is set exactly when x <= T.  Dead slots (no entry of the
// list can reach tau) get an all-31 column and T = 0.
#include <float.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace pqrr_b200 {
namespace {

constexpr int M = 8;
constexpr int KS = 256;
constexpr int FQ = kFQ;      // queries per filter item
constexpr int SUBQ = kQT;    // queries per LUT-pass item
constexpr int NSUB = FQ / SUBQ;
constexpr int FT = 512;
constexpr int FW = FT / 32;
constexpr int LUT8_BYTES = M * KS * FQ;      // 128 KiB
constexpr int Q8_BLOCK = M * KS * SUBQ;      // 32 KiB per LUT-pass item

// Per query slot: multiplier / additive term of the v8 -> v5 conversion and
// the threshold byte T (255 = everything passes).
struct SlotParam {
    uint32_t mult, add, t;
};
__device__ __forceinline__ SlotParam slot_params(float tau, float sc, float summ, float band_div) {
    const float e_up = 1.000003814697265625f, e_dn = 0.999996185302734375f;  // 1 +- 2^-18
    if (!(tau < __int_as_float(0x7f800000))) return {0u, 0u, 255u};  // unsampled: all pass
    const float num = __fsub_rn(__fmul_rn(tau, e_up), __fmul_rn(summ, e_dn));
    if (!(num >= 0.f)) return {0u, 31u, 0u};  // even the closest reconstruction is beyond tau
    if (!(sc > 0.f)) return {0u, 0u, 255u};   // v8 == 0 everywhere and sum_m <= tau
    // mult = floor(256 sc / Delta_target) in [1, 256]
    const float mf = floorf(__fdiv_rn(__fmul_rn(256.f, sc), __fdiv_rn(num, band_div)));
    const uint32_t mult = mf >= 256.f ? 256u : (mf < 1.f ? 1u : (uint32_t)mf);
    // T = floor(num / Delta), Delta = 256 sc / mult
    const float tf = __fmul_rn(__fdiv_rn(__fmul_rn(num, (float)mult), __fmul_rn(256.f, sc)), e_up);
    const float t = floorf(tf);
    return {mult, 0u, t >= 255.f ? 255u : (uint32_t)t};
}

// Four v8 bytes -> v5 bytes: min(31, (b * mult_b >> 8) + add_b).
__device__ __forceinline__ uint32_t v5_of(uint32_t word, const uint32_t* mult, const uint32_t* add) {
    uint32_t out = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const uint32_t v = ((((word >> (8 * b)) & 0xffu) * mult[b]) >> 8) + add[b];
        out |= min(v, 31u) << (8 * b);
    }
    return out;
}

// Bit 7 of each byte set where x <= t (unsigned bytes, see the header).
__device__ __forceinline__ uint32_t le_bytes(uint32_t x, uint32_t t, uint32_t t_hi) {
    const uint32_t r = t_hi - (x & 0x7f7f7f7fu);
    const uint32_t d = x ^ t;
    return ((d & t) | (~d & r)) & 0x80808080u;
}

// Candidates are staged per item in shared memory as (entry << 6 | slot) and
// written out grouped by query slot at the end of the item, so each (query,
// list) run is contiguous in the query's buffer (K4r keeps the run's residual
// in registers).  A full stage falls back to a direct append.
constexpr int STAGE = 16384;  // staged candidates per item (64 KiB)

__device__ __forceinline__ void append_direct(int slot, uint32_t pos, const int* s_q,
                                              const uint32_t* s_r, const FilterArgs& a) {
    const int q = s_q[slot];
    const unsigned o = atomicAdd(a.cand_cnt + q, 1u);
    if (o < a.cap) {
        a.cand_pos[(size_t)q * a.cap + o] = pos;
        a.cand_aux[(size_t)q * a.cap + o] = s_r[slot];
        if (a.cand_code) a.cand_code[(size_t)q * a.cap + o] = __ldg(reinterpret_cast<const u64*>(a.codes) + pos);
    }
    if (a.cand_used) atomicOr(a.cand_used + (size_t)q * 8 + (s_r[slot] >> 5), 1u << (s_r[slot] & 31));
}

// Writes the staged candidates (entry << 6 | slot) of the item to the
// queries' buffers grouped by slot, so each (query, list) run is contiguous
// (K4r keeps the run's residual in registers).  Block-wide; resets the stage.
__device__ __forceinline__ void flush_stage(const FilterArgs& a, const uint32_t* stage, uint32_t* s_nst,
                                            uint32_t* s_scnt, uint32_t* s_sbase, const int* s_q,
                                            const uint32_t* s_r, uint32_t off32) {
    if (threadIdx.x < FQ) s_scnt[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t nst = min(*s_nst, (uint32_t)STAGE);
    for (uint32_t i = threadIdx.x; i < nst; i += FT) atomicAdd(&s_scnt[stage[i] & 63u], 1u);
    __syncthreads();
    if (threadIdx.x < FQ) {
        const uint32_t cnt = s_scnt[threadIdx.x];
        s_sbase[threadIdx.x] = cnt ? atomicAdd(a.cand_cnt + s_q[threadIdx.x], cnt) : 0u;
        s_scnt[threadIdx.x] = 0;
        if (cnt && a.cand_used) {
            const uint32_t r = s_r[threadIdx.x];
            atomicOr(a.cand_used + (size_t)s_q[threadIdx.x] * 8 + (r >> 5), 1u << (r & 31));
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nst; i += FT) {
        const uint32_t v = stage[i];
        const uint32_t sl = v & 63u;
        const uint32_t o = s_sbase[sl] + atomicAdd(&s_scnt[sl], 1u);
        if (o < a.cap) {
            const size_t q = (size_t)s_q[sl];
            const uint32_t pos = off32 + (v >> 6);
            a.cand_pos[q * a.cap + o] = pos;
            a.cand_aux[q * a.cap + o] = s_r[sl];
            if (a.cand_code) a.cand_code[q * a.cap + o] = __ldg(reinterpret_cast<const u64*>(a.codes) + pos);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *s_nst = 0;
    __syncthreads();
}

// The scan of one item's entry range with NQD 16-slot quads per entry
// (NQD = 4: 64 slots, 8 entries per warp step; 2: 32 slots, 16 entries; 1:
// 16 slots, 32 entries).  The 5-bit LUT row always holds 4 16-byte quads;
// quad c carries slot group c % NQD (replicated 4 / NQD times), and lane
// L = 8p + 4h + c reads quad c for entry 2 (p (4 / NQD) + c / NQD) + h of the
// step: the two lanes of a quarter warp that read the same quad position get
// the two entries of a parity pair, so every LDS.128 stays conflict-free
// exactly as in the 64-slot layout.
// NQD = 0 (items with <= 4 or <= 8 live pairs): the LUT row is the pairs'
// bytes as NW = 1 / 2 words, replicated to fill the 64-byte row; a lane reads
// copy (eoff / 2) mod (16 / NW), so the two lanes of a parity pair share a copy
// index and land 16 banks apart -- one LDS.32 per (entry, j) serves the warp
// in one wavefront, one LDS.64 in two (vs 4 for an LDS.128).
template <int NQD, int NW = 1>
__device__ __forceinline__ void filter_scan(const FilterArgs& a, const uint4* __restrict__ lut8v,
                                            const uint8_t* s_t, const int* s_q, const uint32_t* s_r,
                                            uint32_t* s_nst, uint32_t* stage, uint32_t* s_scnt,
                                            uint32_t* s_sbase, const u64* codes, uint32_t len,
                                            uint32_t off32, bool stage_ok) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = lane & 3, h = (lane >> 2) & 1, p = lane >> 3;
    constexpr int NQ = NQD ? NQD : 1;
    const int grp = c % NQ;  // the lane's slot group
    const uint32_t eoff = 2 * (p * (4 / NQ) + c / NQ) + h;
    constexpr uint32_t EPW = 32 / NQ;  // entries per warp step
    const uint32_t* lut32 = reinterpret_cast<const uint32_t*>(lut8v) + NW * ((eoff >> 1) % (16 / NW));
    const uint4 tb = reinterpret_cast<const uint4*>(s_t)[grp];
    const uint4 th = make_uint4(tb.x | 0x80808080u, tb.y | 0x80808080u, tb.z | 0x80808080u,
                                tb.w | 0x80808080u);
    constexpr uint32_t S = FW * EPW;
    const uint32_t wbase = warp * EPW;
    u64 nA, nB, fA, fB;
    {
        const uint32_t e = wbase + eoff;
        nA = e < len ? __ldg(codes + e) : 0ull;
        nB = e + S < len ? __ldg(codes + e + S) : 0ull;
        fA = e + 2 * S < len ? __ldg(codes + e + 2 * S) : 0ull;
        fB = e + 3 * S < len ? __ldg(codes + e + 3 * S) : 0ull;
    }
    // every warp runs the same number of steps (entries past len are masked),
    // so the stage can be flushed at block barriers every FLUSH_EVERY steps
    // once it is half full (a dense item would overflow it otherwise)
    constexpr uint32_t FLUSH_EVERY = 8;
    const uint32_t nsteps = (len + 2 * S - 1) / (2 * S);
    for (uint32_t step = 0; step < nsteps; ++step) {
        const uint32_t wb = wbase + step * 2 * S;
        const uint32_t eA = wb + eoff, eB = eA + S;
        const bool vA = eA < len, vB = eB < len;
        const u64 cA = nA, cB = nB;
        nA = fA;
        nB = fB;
        fA = eA + 4 * S < len ? __ldg(codes + eA + 4 * S) : 0ull;
        fB = eB + 4 * S < len ? __ldg(codes + eB + 4 * S) : 0ull;
        uint32_t a0 = 0u, a1 = 0u, a2 = 0u, a3 = 0u;
        uint32_t b0 = 0u, b1 = 0u, b2 = 0u, b3 = 0u;
        const uint32_t cAl = (uint32_t)cA, cAh = (uint32_t)(cA >> 32);
        const uint32_t cBl = (uint32_t)cB, cBh = (uint32_t)(cB >> 32);
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const uint32_t ca = ((j < 4 ? cAl : cAh) >> (8 * (j & 3))) & 0xffu;
            const uint32_t cb = ((j < 4 ? cBl : cBh) >> (8 * (j & 3))) & 0xffu;
            if (NQD == 0 && NW == 1) {
                a0 += lut32[(j * KS + ca) * 16];
                b0 += lut32[(j * KS + cb) * 16];
            } else if (NQD == 0) {
                const uint2 va = *reinterpret_cast<const uint2*>(lut32 + (j * KS + ca) * 16);
                const uint2 vb = *reinterpret_cast<const uint2*>(lut32 + (j * KS + cb) * 16);
                a0 += va.x; a1 += va.y;
                b0 += vb.x; b1 += vb.y;
            } else {
                const uint4 va = lut8v[(j * KS + ca) * NSUB + c];
                const uint4 vb = lut8v[(j * KS + cb) * NSUB + c];
                a0 += va.x; a1 += va.y; a2 += va.z; a3 += va.w;
                b0 += vb.x; b1 += vb.y; b2 += vb.z; b3 += vb.w;
            }
        }
        // pass bits sit at bit 7 of each byte; gather them into one lane mask
        // (bit 16 s + 4 t + b: step s, word t, byte b -> slot grp * 16 + 4 t
        // + b).  (x >> 7) * 0x00204081 moves bits 0/8/16/24 to bits 21..24
        // without carries.
        auto m4 = [](uint32_t x) { return (((x >> 7) * 0x00204081u) >> 21) & 0xfu; };
        uint32_t mA, mB;
        if (NQD == 0) {
            mA = vA ? m4(le_bytes(a0, tb.x, th.x)) | (NW == 2 ? m4(le_bytes(a1, tb.y, th.y)) << 4 : 0u) : 0u;
            mB = vB ? m4(le_bytes(b0, tb.x, th.x)) | (NW == 2 ? m4(le_bytes(b1, tb.y, th.y)) << 4 : 0u) : 0u;
        } else {
            mA = vA ? (m4(le_bytes(a0, tb.x, th.x)) | (m4(le_bytes(a1, tb.y, th.y)) << 4) |
                       (m4(le_bytes(a2, tb.z, th.z)) << 8) | (m4(le_bytes(a3, tb.w, th.w)) << 12))
                    : 0u;
            mB = vB ? (m4(le_bytes(b0, tb.x, th.x)) | (m4(le_bytes(b1, tb.y, th.y)) << 4) |
                       (m4(le_bytes(b2, tb.z, th.z)) << 8) | (m4(le_bytes(b3, tb.w, th.w)) << 12))
                    : 0u;
        }
        uint32_t mask = mA | (mB << 16);
        while (mask) {
            const int bpos = __ffs(mask) - 1;
            mask &= mask - 1;
            const int sl = grp * 16 + (bpos & 15);
            const uint32_t e = bpos < 16 ? eA : eB;
            const uint32_t k = stage_ok ? atomicAdd(s_nst, 1u) : (uint32_t)STAGE;
            if (k < (uint32_t)STAGE)
                stage[k] = (e << 6) | (uint32_t)sl;
            else
                append_direct(sl, off32 + e, s_q, s_r, a);
        }
        if (step % FLUSH_EVERY == FLUSH_EVERY - 1 && step + 1 < nsteps) {
            __syncthreads();
            if (*s_nst >= (uint32_t)STAGE / 2) flush_stage(a, stage, s_nst, s_scnt, s_sbase, s_q, s_r, off32);
        }
    }
}

__global__ __launch_bounds__(FT, 1) void ivf_filter_kernel(const FilterArgs a) {
    extern __shared__ uint4 smem_f[];
    uint8_t* lut8 = reinterpret_cast<uint8_t*>(smem_f);  // [M][KS][FQ]
    const uint4* lut8v = smem_f;
    __shared__ uint32_t s_item;
    __shared__ int s_q[FQ];
    __shared__ uint32_t s_r[FQ];
    __shared__ __align__(16) uint8_t s_t[FQ];
    __shared__ uint32_t s_mult[FQ], s_add[FQ];
    __shared__ uint64_t s_src[FQ];  // byte offset of the slot's lane column in q8_cache
    __shared__ uint32_t s_nst, s_scnt[FQ], s_sbase[FQ];
    uint32_t* stage = reinterpret_cast<uint32_t*>(lut8 + LUT8_BYTES);

    const uint32_t n_items = *a.num_items;

    for (;;) {
        if (threadIdx.x == 0) {
            const uint32_t c = atomicAdd(a.item_counter, 1u);
            s_item = c < n_items ? a.item_order[c] : 0xffffffffu;
            s_nst = 0;
        }
        __syncthreads();
        const uint32_t it = s_item;
        if (it == 0xffffffffu) break;
        const uint32_t nqi = a.item_nq[it];
        if (nqi == 0) {  // every pair of this item's group is dead (launch_live_pairs)
            __syncthreads();  // all threads read s_item before thread 0 claims the next item
            continue;
        }
        const uint32_t l = a.item_list[it];
        const uint32_t start = a.item_start[it];
        if (threadIdx.x < FQ) {
            const uint32_t t = threadIdx.x;
            int q = -1;
            uint32_t r = 0;
            SlotParam sp{0u, 31u, 0u};  // empty slot: dead
            uint64_t src = 0;
            if (t < nqi) {
                const uint32_t slot = a.live_slot[start + t];
                const uint32_t blk = slot / SUBQ, ln = slot % SUBQ;
                const uint32_t p = a.live_pair[start + t];
                q = (int)(p / a.w);
                r = p % a.w;
                const float* prm = a.q8_param + ((size_t)blk * SUBQ + ln) * 2;
                sp = slot_params(a.tau[q], prm[0], prm[1], a.band_div);
                if (a.pass_all) sp = {0u, 0u, 255u};
                src = (uint64_t)blk * Q8_BLOCK + (uint64_t)ln * (M * KS);
            }
            s_q[t] = q;
            s_r[t] = r;
            s_mult[t] = sp.mult;
            s_add[t] = sp.add;
            s_t[t] = (uint8_t)sp.t;
            s_src[t] = src;
        }
        __syncthreads();
        // NQD = 1 / 2 / 4 quads of 16 slots per entry (filter_scan)
        // 0: narrow (<= 4 / <= 8 pairs: nw replicated words per row); else quads per entry
        const int nqd = nqi <= 8 ? 0 : (nqi <= 16 ? 1 : (nqi <= 32 ? 2 : 4));
        const int nw = nqi <= 4 ? 1 : 2;

        // ---- 5-bit LUT of the item: the live slots' 8-bit lane columns
        // (lane-major LUT-pass blocks, q8_put_rows) are staged 32 at a time in
        // shared memory (2052-byte stride: conflict-free byte reads), then
        // transposed into [j][code][quad] rows; quad position c holds slot
        // group c % nqd
        {
            uint8_t* colbuf = reinterpret_cast<uint8_t*>(stage);  // [32][2052]
            uint32_t* colw = stage;
            constexpr int CST = M * KS + 4;  // bytes per staged column
            const int nsl = nqd ? 16 * nqd : 4 * nw;
            for (int h = 0; 32 * h < nsl; ++h) {
                const int ns = min(32, nsl - 32 * h);
                for (int x = threadIdx.x; x < ns * (M * KS / 16); x += FT) {
                    const int sl = x / (M * KS / 16), ch = x % (M * KS / 16);
                    if ((uint32_t)(32 * h + sl) < nqi) {
                        const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.q8_cache + s_src[32 * h + sl]) + ch);
                        uint32_t* d = colw + sl * (CST / 4) + ch * 4;
                        d[0] = v.x;
                        d[1] = v.y;
                        d[2] = v.z;
                        d[3] = v.w;
                    }
                }
                __syncthreads();
                const int sq = threadIdx.x & 7;
                if (nqd == 0) {
                    // every thread converts whole rows: the pairs' nw words, replicated
                    uint32_t mu[8], ad[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        mu[k] = s_mult[k];
                        ad[k] = s_add[k];
                    }
                    for (int row = threadIdx.x; row < M * KS; row += FT) {
                        const uint8_t* cb = colbuf + row;
                        const uint32_t word = (uint32_t)cb[0] | ((uint32_t)cb[CST] << 8) |
                                              ((uint32_t)cb[2 * CST] << 16) | ((uint32_t)cb[3 * CST] << 24);
                        const uint32_t v5 = v5_of(word, mu, ad);
                        uint32_t v5b = v5;
                        if (nw == 2) {
                            const uint8_t* cc = cb + 4 * CST;
                            const uint32_t w2 = (uint32_t)cc[0] | ((uint32_t)cc[CST] << 8) |
                                                ((uint32_t)cc[2 * CST] << 16) | ((uint32_t)cc[3 * CST] << 24);
                            v5b = v5_of(w2, mu + 4, ad + 4);
                        }
                        const uint4 v4 = make_uint4(v5, v5b, nw == 2 ? v5 : v5b, v5b);
#pragma unroll
                        for (int i = 0; i < 4; ++i)  // rotated: the 8 lanes of a phase hit 8 bank groups
                            reinterpret_cast<uint4*>(lut8 + row * FQ)[(i + (row >> 1)) & 3] = v4;
                    }
                } else if (4 * sq < ns) {
                    const int s0 = 32 * h + 4 * sq;  // first slot of this thread's word
                    uint32_t mu[4], ad[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        mu[k] = s_mult[s0 + k];
                        ad[k] = s_add[s0 + k];
                    }
                    const int quad = s0 / 16, byte0 = s0 % 16;
                    for (int row = threadIdx.x >> 3; row < M * KS; row += FT / 8) {
                        const uint8_t* cb = colbuf + (4 * sq) * CST + row;
                        const uint32_t word = (uint32_t)cb[0] | ((uint32_t)cb[CST] << 8) |
                                              ((uint32_t)cb[2 * CST] << 16) | ((uint32_t)cb[3 * CST] << 24);
                        const uint32_t v5 = v5_of(word, mu, ad);
                        for (int c = quad; c < NSUB; c += nqd)
                            *reinterpret_cast<uint32_t*>(lut8 + row * FQ + c * 16 + byte0) = v5;
                    }
                }
                __syncthreads();
            }
        }

        const uint32_t ie0 = a.item_e0[it];
        const uint64_t off = a.list_off[l] + ie0;  // this item's entry range [e0, e1)
        const uint32_t len = a.item_e1[it] - ie0;
        const uint32_t off32 = (uint32_t)off;
        const bool stage_ok = len < (1u << 26);
        const u64* codes = reinterpret_cast<const u64*>(a.codes) + off;
        if (nqd == 0 && nw == 1)
            filter_scan<0, 1>(a, lut8v, s_t, s_q, s_r, &s_nst, stage, s_scnt, s_sbase, codes, len, off32, stage_ok);
        else if (nqd == 0)
            filter_scan<0, 2>(a, lut8v, s_t, s_q, s_r, &s_nst, stage, s_scnt, s_sbase, codes, len, off32, stage_ok);
        else if (nqd == 1)
            filter_scan<1>(a, lut8v, s_t, s_q, s_r, &s_nst, stage, s_scnt, s_sbase, codes, len, off32, stage_ok);
        else if (nqd == 2)
            filter_scan<2>(a, lut8v, s_t, s_q, s_r, &s_nst, stage, s_scnt, s_sbase, codes, len, off32, stage_ok);
        else
            filter_scan<4>(a, lut8v, s_t, s_q, s_r, &s_nst, stage, s_scnt, s_sbase, codes, len, off32, stage_ok);
        // ---- flush the remaining staged candidates
        __syncthreads();
        flush_stage(a, stage, &s_nst, s_scnt, s_sbase, s_q, s_r, off32);
    }
}

// K4r: one CTA per query.  The query's residuals x - C_l for its w probes are
// staged in shared memory; each candidate's distance is the j-ascending fp32
// sum of l2_sq(residual_j, B_j[c_j]) in the reference order — bit-identical to
// the LUT value the exact scan would have added (build_luts, k_scan.cu).
template <int DSUB>
__global__ __launch_bounds__(256) void recheck_kernel(
    const float* __restrict__ xq, uint32_t d, const float* __restrict__ coarse,
    const float* __restrict__ books, const uint32_t* __restrict__ probes, uint32_t w,
    const u64* __restrict__ codes, const uint32_t* __restrict__ cand_cnt, uint32_t cap,
    const uint32_t* __restrict__ cand_pos, float* __restrict__ cand_dist,
    const float* __restrict__ tau, uint32_t* __restrict__ cand_le, const u64 nz) {
    extern __shared__ float4 smem_r[];
    float* res = reinterpret_cast<float*>(smem_r);  // [w][d]
    __shared__ uint32_t s_le;
    const size_t q = blockIdx.x;
    const uint32_t n = min(cand_cnt[q], cap);
    if (threadIdx.x == 0) s_le = 0;
    if (n == 0) {
        if (threadIdx.x == 0) cand_le[q] = 0;
        return;
    }
    for (uint32_t idx = threadIdx.x; idx < w * d; idx += blockDim.x) {
        const uint32_t r = idx / d, t = idx % d;
        const uint32_t l = probes[q * w + r];
        res[idx] = __fsub_rn(xq[q * d + t], coarse[(size_t)l * d + t]);
    }
    __syncthreads();
    const float tq = tau[q];
    uint32_t le = 0;
    const uint32_t* aux = reinterpret_cast<const uint32_t*>(cand_dist) + q * cap;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t pos = cand_pos[q * cap + i];
        const uint32_t r = aux[i];
        const u64 code = __ldg(codes + pos);
        const float* rr = res + (size_t)r * d;
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const uint32_t c = (uint32_t)(code >> (8 * j)) & 0xffu;
            acc = __fadd_rn(acc, l2sq_packed<DSUB>(rr + j * DSUB, books + ((size_t)j * KS + c) * DSUB, nz));
        }
        cand_dist[q * cap + i] = acc;
        le += acc <= tq ? 1u : 0u;
    }
    atomicAdd(&s_le, le);
    __syncthreads();
    if (threadIdx.x == 0) cand_le[q] = s_le;
}

// K4r, shared-memory variant (d/m <= 16): persistent CTAs hold the whole
// codebook (8 x 256 x DSUB floats) in shared memory and walk the queries.
// Per query the w residuals are staged with chunk swizzle
// phys = c ^ ((c >> 3) & 3) (16-byte chunks), and a warp rechecks 4
// candidates per step with 8 lanes each (lane = subspace j): the 8 lanes of a
// quarter-warp read residual chunk p of 8 different subspaces at 8 distinct
// bank groups, and codebook rows (stored with the same per-subspace swizzle)
// at ~2 wavefronts.  Each lane computes l2_sq(residual_j, B_j[c_j]) in the
// reference order; the 8 values are gathered by shuffles and summed
// j-ascending — the same fp32 operations as the exact scan's LUT + ADC.
// A survivor's 8 code bytes: a random sector never reused on this SM, read
// without allocating in L1.
__device__ __forceinline__ u64 ld_code_na(const u64* p) {
    u64 v;
    asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

template <int DSUB>
__global__ __launch_bounds__(512, 1) void recheck_smem_kernel(
    const float* __restrict__ xq, uint32_t d, const float* __restrict__ coarse,
    const float* __restrict__ books, const uint32_t* __restrict__ probes, uint32_t w,
    const u64* __restrict__ codes, const uint32_t* __restrict__ cand_cnt, uint32_t cap,
    const uint32_t* __restrict__ cand_pos, float* __restrict__ cand_dist,
    const float* __restrict__ tau, size_t nq, uint32_t* __restrict__ cand_le,
    uint32_t* __restrict__ counter, const u64 nz, uint32_t* __restrict__ cand_mm) {
    constexpr int CH = DSUB / 4;  // 16-byte chunks per subspace row
    extern __shared__ float4 smem_k[];
    float4* bk = smem_k;                      // [KS][M][CH]: code-major, chunks rotated
    float4* res = smem_k + M * KS * CH;       // [w][d / 4], swizzled
    __shared__ uint32_t s_q, s_le, s_mn, s_mx;
    // per-warp exchange of the 8 sub-space terms of 4 x 4 candidates:
    // [round u][slot][j], rows of 36 floats (conflict-free writes and reads)
    __shared__ __align__(16) float s_x[16][4 * 36];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane & 7, slot = lane >> 3;
    const uint32_t dch = d / 4;
    // swizzled chunk index within a row of subspace j (CH chunks per subspace)
    auto sw = [](uint32_t c) { return CH >= 4 ? (c ^ ((c >> 3) & 3)) : c; };
    // Code-major book: row `code` holds all M sub-spaces' centroids for that
    // code (the candidate's 8 lanes read 8 different rows), and sub-space j's
    // chunk p sits at chunk (p + j / 2) mod CH of its slot, so at any p the 8
    // lanes of a quarter warp land in 8 distinct 16-byte bank groups whatever
    // the codes: 4 (j & 1) + ((p + j / 2) & 3).
    auto bslot = [](uint32_t code, uint32_t jj, uint32_t p) {
        return code * (M * CH) + jj * CH + ((p + (jj >> 1)) & (CH - 1));
    };
    for (uint32_t i = threadIdx.x; i < (uint32_t)(M * KS * CH); i += blockDim.x) {
        const uint32_t row = i / CH, p = i % CH;  // row = j * KS + code
        bk[bslot(row % KS, row / KS, p)] = reinterpret_cast<const float4*>(books)[i];
    }
    for (;;) {
        __syncthreads();  // previous query done (and books staged)
        if (threadIdx.x == 0) {
            s_q = atomicAdd(counter, 1u);
            s_le = 0;
            s_mn = 0xffffffffu;
            s_mx = 0u;
        }
        __syncthreads();
        const size_t q = s_q;
        if (q >= nq) break;
        const uint32_t n = min(cand_cnt[q], cap);
        if (n == 0) {
            if (threadIdx.x == 0) cand_le[q] = 0;
            continue;
        }
        uint32_t dmn = 0xffffffffu, dmx = 0u;  // the exact distances' range (select_warp)
        for (uint32_t i = threadIdx.x; i < w * dch; i += blockDim.x) {
            const uint32_t r = i / dch, c = i % dch;
            const uint32_t l = probes[q * w + r];
            const float4 x = reinterpret_cast<const float4*>(xq + q * d)[c];
            const float4 y = reinterpret_cast<const float4*>(coarse + (size_t)l * d)[c];
            res[r * dch + sw(c)] = make_float4(__fsub_rn(x.x, y.x), __fsub_rn(x.y, y.y),
                                               __fsub_rn(x.z, y.z), __fsub_rn(x.w, y.w));
        }
        __syncthreads();
        const float tq = tau[q];
        const uint32_t* aux = reinterpret_cast<const uint32_t*>(cand_dist) + q * cap;
        uint32_t le = 0;
        // each warp takes 16 candidates per iteration (4 rounds of 4); the
        // position / probe-rank loads of the next iteration are issued before
        // this one's arithmetic, the codes of all 4 rounds together.  Slots of
        // odd parity read the second 8-byte half of every chunk first, so the
        // two candidates of a half-warp never share a bank; the halves feed the
        // separate (s0,s1) / (s2,s3) accumulators, so the order is unchanged.
        // The residual chunk stays in registers while the probe rank repeats
        // (K4f writes each (query, list) run contiguously).
        constexpr int U = 4;
        constexpr uint32_t STEP = 16 * 4 * U;
        uint32_t npos[U], nr[U];
        auto fetch = [&](uint32_t b) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = min(b + u * 4 + slot, n - 1);
                npos[u] = cand_pos[q * cap + i];
                nr[u] = aux[i];
            }
        };
        // 16-byte loads: a quarter-warp is one candidate's 8 sub-spaces, so the
        // swizzled residual chunks and the code-major book rows (bslot) sit in
        // 8 distinct bank groups
        const ulonglong2* res128 = reinterpret_cast<const ulonglong2*>(res);
        const ulonglong2* bk128 = reinterpret_cast<const ulonglong2*>(bk);
        u64 xa[CH], xb[CH];  // residual chunk halves (t, t+1) / (t+2, t+3)
        uint32_t cur_r = 0xffffffffu;
        // software pipeline: positions run two iterations ahead, codes one
        // (the random 8-byte code gathers are the kernel's long-latency loads)
        u64 ncode[U];
        fetch(warp * 4 * U);
#pragma unroll
        for (int u = 0; u < U; ++u) ncode[u] = ld_code_na(codes + npos[u]);
        uint32_t cpos_r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cpos_r[u] = nr[u];
        if (warp * 4 * U + STEP < n) fetch(warp * 4 * U + STEP);
        for (uint32_t base = warp * 4 * U; base < n; base += STEP) {
            uint32_t rr[U];
            u64 code[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                code[u] = ncode[u];
                rr[u] = cpos_r[u];
            }
            if (base + STEP < n) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    ncode[u] = ld_code_na(codes + npos[u]);
                    cpos_r[u] = nr[u];
                }
                if (base + 2 * STEP < n) fetch(base + 2 * STEP);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = base + u * 4 + slot;
                if (rr[u] != cur_r) {
                    cur_r = rr[u];
#pragma unroll
                    for (int p = 0; p < CH; ++p) {
                        const ulonglong2 v = res128[cur_r * dch + sw(j * CH + p)];
                        xa[p] = v.x;
                        xb[p] = v.y;
                    }
                }
                const uint32_t c = (uint32_t)(code[u] >> (8 * j)) & 0xffu;
                u64 sa = 0, sb = 0;
#pragma unroll
                for (int p = 0; p < CH; ++p) {
                    const ulonglong2 bv = bk128[bslot(c, j, p)];
                    if (p == 0) {  // 0 + x == x for the rounded square x >= +0
                        sa = sq2(sub2(xa[p], bv.x), nz);
                        sb = sq2(sub2(xb[p], bv.y), nz);
                    } else {
                        sa = acc_sq2(sa, xa[p], bv.x, nz);
                        sb = acc_sq2(sb, xb[p], bv.y, nz);
                    }
                }
                const u64 s01 = sa, s23 = sb;
                const float Lj = __fadd_rn(__fadd_rn(lo2(s01), hi2(s01)), __fadd_rn(lo2(s23), hi2(s23)));
                (void)i;
                s_x[warp][u * 36 + slot * 8 + j] = Lj;
            }
            __syncwarp();
            // lane j < 4 of a quarter warp sums round u = j's 8 terms
            // j-ascending (adc_distance, product_quantizer.hpp:53-57)
            if (j < U) {
                const float4 t0 = *reinterpret_cast<const float4*>(&s_x[warp][j * 36 + slot * 8]);
                const float4 t1 = *reinterpret_cast<const float4*>(&s_x[warp][j * 36 + slot * 8 + 4]);
                float acc = __fadd_rn(__fadd_rn(__fadd_rn(t0.x, t0.y), t0.z), t0.w);  // 0 + L0 == L0
                acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, t1.x), t1.y), t1.z), t1.w);
                const uint32_t i = base + j * 4 + slot;
                if (i < n) {
                    cand_dist[q * cap + i] = acc;
                    le += acc <= tq ? 1u : 0u;
                    dmn = min(dmn, __float_as_uint(acc));
                    dmx = max(dmx, __float_as_uint(acc));
                }
            }
            __syncwarp();
        }
        if (le) atomicAdd(&s_le, le);
        if (cand_mm) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                dmn = min(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
                dmx = max(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
            }
            if (lane == 0) {
                atomicMin(&s_mn, dmn);
                atomicMax(&s_mx, dmx);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            cand_le[q] = s_le;
            if (cand_mm) {
                cand_mm[2 * q] = s_mn;
                cand_mm[2 * q + 1] = s_mx;
            }
        }
    }
}

template <int DSUB>
void recheck_t(const float* xq, uint32_t d, const float* coarse, const float* books,
               const uint32_t* probes, uint32_t w, const uint8_t* codes, const uint32_t* cand_cnt,
               uint32_t cap, const uint32_t* cand_pos, float* cand_dist, const float* tau, size_t nq,
               uint32_t* cand_le, cudaStream_t s) {
    const size_t smem = (size_t)w * d * sizeof(float);
    set_max_smem((const void*)recheck_kernel<DSUB>, (size_t)((int)std::max<size_t>(smem, 1)));
    recheck_kernel<DSUB><<<(unsigned)nq, 256, smem, s>>>(
        xq, d, coarse, books, probes, w, reinterpret_cast<const u64*>(codes), cand_cnt, cap, cand_pos,
        cand_dist, tau, cand_le, kNegZero2);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

}  // namespace

// Per list (one CTA): the live pairs of the list from both pair sets (near /
// far probes of the two-phase LUT pass; one set otherwise), compacted from
// all_first[l] on as (q8 slot, pair id).  Ballot per warp + a prefix over the
// CTA's warps per 256-pair chunk.
__global__ __launch_bounds__(256) void live_pairs_kernel(const FilterArgs a, PairSet s0, PairSet s1,
                                                         const uint32_t* __restrict__ all_first,
                                                         uint32_t* __restrict__ live_slot,
                                                         uint32_t* __restrict__ live_pair,
                                                         uint32_t* __restrict__ live_cnt,
                                                         unsigned long long* __restrict__ live_entries) {
    __shared__ uint32_t s_wc[8];
    const uint32_t l = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = all_first[l];
    uint32_t o = 0;
    for (int set = 0; set < 2; ++set) {
        const PairSet& ps = set ? s1 : s0;
        if (!ps.list_cnt) continue;
        const uint32_t n = ps.list_cnt[l], f = ps.list_first[l], b0 = ps.blk_base + ps.sub_item_off[l];
        for (uint32_t i0 = 0; i0 < n; i0 += 256) {
            const uint32_t i = i0 + threadIdx.x;
            bool live = false;
            uint32_t p = 0, slot = 0;
            if (i < n) {
                p = ps.pair_sorted[f + i];
                slot = (b0 + i / SUBQ) * SUBQ + i % SUBQ;
                // (a bound-dead pair's item may have been skipped: its q8_param is then unset)
                live = a.pass_all || ((!ps.pair_bound || pair_live(a.tau[p / a.w], ps.pair_bound[p])) &&
                                      pair_live(a.tau[p / a.w], a.q8_param[(size_t)slot * 2 + 1]));
            }
            const unsigned bal = __ballot_sync(0xffffffffu, live);
            if (lane == 0) s_wc[warp] = __popc(bal);
            __syncthreads();
            uint32_t before = o;
            for (int k = 0; k < warp; ++k) before += s_wc[k];
            if (live) {
                const uint32_t d = base + before + __popc(bal & ((1u << lane) - 1u));
                live_slot[d] = slot;
                live_pair[d] = p;
            }
            for (int k = 0; k < 8; ++k) o += s_wc[k];
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        live_cnt[l] = o;
        // (live pair, entry) lookups K4f executes for this list (measurement)
        if (live_entries && o) atomicAdd(live_entries, (unsigned long long)o * a.list_len[l]);
    }
}

// The K4f items of a list (groups of FQ pairs x entry chunks, items_build
// order) re-pointed at its live pairs; groups past the live count are empty.
__global__ void live_items_kernel(const FilterArgs a, const uint32_t* __restrict__ list_cnt,
                                  const uint32_t* __restrict__ list_first,
                                  const uint32_t* __restrict__ live_cnt, uint32_t nlists,
                                  const uint32_t* __restrict__ item_off, uint32_t* __restrict__ item_start,
                                  uint32_t* __restrict__ item_nq, uint32_t chunk) {
    const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= nlists) return;
    const uint32_t c = list_cnt[l], lc = live_cnt[l], L = a.list_len[l];
    const uint32_t chunks = max(1u, (L + chunk - 1) / chunk);
    uint32_t o = item_off[l];
    for (uint32_t g = 0; g < c; g += FQ)
        for (uint32_t ch = 0; ch < chunks; ++ch, ++o) {
            item_start[o] = list_first[l] + g;
            item_nq[o] = g < lc ? min((uint32_t)FQ, lc - g) : 0u;
        }
}

void launch_ivf_filter(const FilterArgs& a, cudaStream_t s) {
    // + 1 KiB: 32 staged 2052-byte lane columns (the LUT build) exceed the
    // 64 KiB candidate stage
    const int smem = LUT8_BYTES + STAGE * (int)sizeof(uint32_t) + 1024;
    set_max_smem((const void*)ivf_filter_kernel, (size_t)(smem));
    ivf_filter_kernel<<<sm_count(), FT, smem, s>>>(a);
    PQRR_LAUNCH_CHECK();
    count_launch();
}

void launch_live_pairs(const FilterArgs& a, PairSet s0, PairSet s1, const uint32_t* all_first,
                       const uint32_t* all_cnt, uint32_t nlists, uint32_t* live_slot,
                       uint32_t* live_pair, uint32_t* live_cnt, const uint32_t* item_off,
                       uint32_t* item_start, uint32_t* item_nq, uint32_t chunk, cudaStream_t s,
                       unsigned long long* live_entries) {
    live_pairs_kernel<<<nlists, 256, 0, s>>>(a, s0, s1, all_first, live_slot, live_pair, live_cnt,
                                             live_entries);
    PQRR_LAUNCH_CHECK();
    live_items_kernel<<<(nlists + 255) / 256, 256, 0, s>>>(a, all_cnt, all_first, live_cnt, nlists, item_off,
                                                          item_start, item_nq, chunk);
    PQRR_LAUNCH_CHECK();
    count_launch(2);
}

bool recheck_supported(uint32_t d, uint32_t m, uint32_t w) {
    if (m != M) return false;
    const uint32_t ds = d / m;
    if (ds != 4 && ds != 8 && ds != 16 && ds != 32) return false;
    return (size_t)w * d * sizeof(float) <= 200 * 1024;
}

// K4r with per-pair LUTs (d = 128, m = 8, ks = 256).  A query's survivors
// come from few (query, list) pairs (at C4 ~8 of the 64 probes), each with
// hundreds to thousands of survivors, so the CTA builds the exact LUT of every
// pair that has survivors -- L_j[c] = l2_sq(x - C_l restricted to sub-space
// j, B_j[c]), 2048 values in the reference order, 8 KiB in shared memory --
// and each survivor's exact ADC distance is then 8 shared-memory lookups
// summed j-ascending (adc_distance, product_quantizer.hpp:53-57): the same
// fp32 values in the same order as recomputing the 8 terms per survivor.
// Pairs are taken LUT_SLOTS at a time (a query with more such pairs makes one
// pass over its survivors per batch).  The pairs with survivors come from
// K4f's per-query rank mask (cand_used) or, without it, from a pass over the
// survivors' ranks.  Survivors are handled 4 per thread with vector loads and
// two groups' loads in flight before the first store (the kernel is bound by
// load latency, not by its shared-memory lookups).
constexpr int LUT_SLOTS = 16;

__device__ __forceinline__ float subspace_l2(const float* __restrict__ r, const float* __restrict__ b, u64 nz) {
    // l2_sq(r[0..16), b[0..16)) in the reference order (distance.hpp:16-33)
    const ulonglong2* r2 = reinterpret_cast<const ulonglong2*>(r);
    const ulonglong2* b2 = reinterpret_cast<const ulonglong2*>(b);
    u64 sa = 0, sb = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const ulonglong2 rv = r2[p], bv = b2[p];
        if (p == 0) {  // 0 + x == x for the rounded square x >= +0
            sa = sq2(sub2(rv.x, bv.x), nz);
            sb = sq2(sub2(rv.y, bv.y), nz);
        } else {
            sa = acc_sq2(sa, rv.x, bv.x, nz);
            sb = acc_sq2(sb, rv.y, bv.y, nz);
        }
    }
    return __fadd_rn(__fadd_rn(lo2(sa), hi2(sa)), __fadd_rn(lo2(sb), hi2(sb)));
}

// One group of 4 survivors (i0 .. i0+3 of the query's buffer): ranks and codes.
struct SurvGroup {
    uint32_t r[4];
    u64 c[4];
    uint32_t cnt;  // valid survivors in the group (0..4)
};

__device__ __forceinline__ SurvGroup load_group(const uint32_t* aux, const u64* cq, const uint32_t* pq,
                                                const u64* codes, uint32_t i0, uint32_t n) {
    SurvGroup g;
    g.cnt = i0 < n ? min(4u, n - i0) : 0u;
    if (g.cnt == 4) {
        const uint4 a4 = *reinterpret_cast<const uint4*>(aux + i0);
        g.r[0] = a4.x, g.r[1] = a4.y, g.r[2] = a4.z, g.r[3] = a4.w;
        if (cq) {
            const ulonglong2 c01 = *reinterpret_cast<const ulonglong2*>(cq + i0);
            const ulonglong2 c23 = *reinterpret_cast<const ulonglong2*>(cq + i0 + 2);
            g.c[0] = c01.x, g.c[1] = c01.y, g.c[2] = c23.x, g.c[3] = c23.y;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) g.c[u] = __ldg(codes + pq[i0 + u]);
        }
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool v = (uint32_t)u < g.cnt;
            g.r[u] = v ? aux[i0 + u] : 0u;
            g.c[u] = v ? (cq ? cq[i0 + u] : __ldg(codes + pq[i0 + u])) : 0ull;
        }
    }
    return g;
}

__global__ __launch_bounds__(512, 1) void recheck_lut_kernel(
    const float* __restrict__ xq, const float* __restrict__ coarse, const float* __restrict__ books,
    const uint32_t* __restrict__ probes, uint32_t w, const u64* __restrict__ codes,
    const uint32_t* __restrict__ cand_cnt, uint32_t cap, const uint32_t* __restrict__ cand_pos,
    float* cand_dist, const float* __restrict__ tau, size_t nq, uint32_t* __restrict__ cand_le,
    uint32_t* __restrict__ counter, const u64 nz, uint32_t* __restrict__ cand_mm,
    const u64* __restrict__ cand_code, const uint32_t* __restrict__ cand_used, float* __restrict__ scratch) {
    constexpr int D = 128, DS = 16;
    extern __shared__ float4 lut4[];
    float* lut = reinterpret_cast<float*>(lut4);  // [LUT_SLOTS][M * KS]
    __shared__ __align__(16) float res[LUT_SLOTS][D];
    __shared__ uint8_t slot_of[256];
    __shared__ uint32_t used[8], s_rank[256];
    __shared__ uint32_t s_q, s_le, s_mn, s_mx, s_nused;
    const int tid = threadIdx.x;
    for (;;) {
        __syncthreads();  // previous query done
        if (tid == 0) {
            s_q = atomicAdd(counter, 1u);
            s_le = 0;
            s_mn = 0xffffffffu;
            s_mx = 0u;
        }
        __syncthreads();
        const size_t q = s_q;
        if (q >= nq) break;
        const uint32_t n = min(cand_cnt[q], cap);
        if (n == 0) {
            if (tid == 0) {
                cand_le[q] = 0;
                if (cand_mm) cand_mm[2 * q] = 0xffffffffu, cand_mm[2 * q + 1] = 0u;
            }
            continue;
        }
        uint32_t* aux = reinterpret_cast<uint32_t*>(cand_dist) + q * cap;  // probe ranks (K4f)
        float* dq = cand_dist + q * cap;
        const uint32_t* pq = cand_pos + q * cap;
        const u64* cq = cand_code ? cand_code + q * cap : nullptr;
        // the probe ranks that have survivors
        if (tid < 8) used[tid] = cand_used ? cand_used[q * 8 + tid] : 0u;
        __syncthreads();
        if (!cand_used) {
            for (uint32_t i = tid; i < n; i += blockDim.x) {
                const uint32_t r = aux[i];
                if (!((used[r >> 5] >> (r & 31)) & 1u)) atomicOr(&used[r >> 5], 1u << (r & 31));
            }
            __syncthreads();
        }
        if (tid < 256 && ((used[tid >> 5] >> (tid & 31)) & 1u)) {
            uint32_t before = __popc(used[tid >> 5] & ((1u << (tid & 31)) - 1u));
            for (int k = 0; k < (tid >> 5); ++k) before += __popc(used[k]);
            slot_of[tid] = (uint8_t)before;
            s_rank[before] = tid;
        }
        if (tid == 0) {
            uint32_t t = 0;
            for (int k = 0; k < 8; ++k) t += __popc(used[k]);
            s_nused = t;
        }
        __syncthreads();
        const uint32_t nused = s_nused;
        const float tq = tau[q];
        uint32_t le = 0, dmn = 0xffffffffu, dmx = 0u;
        // several batches: the ranks are read again by every batch, so the
        // distances go to the CTA's scratch row and are copied over at the end
        float* out = nused > (uint32_t)LUT_SLOTS ? scratch + (size_t)blockIdx.x * cap : dq;
        for (uint32_t b0 = 0; b0 < nused; b0 += LUT_SLOTS) {
            const uint32_t nb = min((uint32_t)LUT_SLOTS, nused - b0);
            if (b0) __syncthreads();  // the previous batch's lookups are done
            // residuals x - C_l of the batch's pairs, then their exact LUTs
            for (uint32_t i = tid; i < nb * D; i += blockDim.x) {
                const uint32_t sl = i / D, t = i % D;
                const uint32_t l = probes[q * w + s_rank[b0 + sl]];
                res[sl][t] = __fsub_rn(xq[q * D + t], coarse[(size_t)l * D + t]);
            }
            __syncthreads();
            for (uint32_t v = tid; v < nb * M * KS; v += blockDim.x) {
                const uint32_t sl = v / (M * KS), jc = v % (M * KS), j = jc / KS, c = jc % KS;
                lut[v] = subspace_l2(&res[sl][j * DS], books + ((size_t)j * KS + c) * DS, nz);
            }
            __syncthreads();
            // survivors of the batch: 8 lookups each, summed j-ascending
            auto run = [&](const SurvGroup& g, uint32_t i0) {
                float d4[4];
                bool done[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t sl = slot_of[g.r[u]] - b0;  // wraps for earlier batches
                    done[u] = (uint32_t)u < g.cnt && sl < nb;
                    const float* L = lut + min(sl, (uint32_t)LUT_SLOTS - 1) * (M * KS);
                    const u64 code = g.c[u];
                    float acc = L[(uint32_t)(code & 0xffu)];  // 0 + L_0 == L_0
#pragma unroll
                    for (int j = 1; j < M; ++j) acc = __fadd_rn(acc, L[j * KS + (uint32_t)((code >> (8 * j)) & 0xffu)]);
                    d4[u] = acc;
                    if (done[u]) {
                        le += acc <= tq ? 1u : 0u;
                        dmn = min(dmn, __float_as_uint(acc));
                        dmx = max(dmx, __float_as_uint(acc));
                    }
                }
                if (done[0] && done[1] && done[2] && done[3]) {
                    *reinterpret_cast<float4*>(out + i0) = make_float4(d4[0], d4[1], d4[2], d4[3]);
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (done[u]) out[i0 + u] = d4[u];
                }
            };
            const uint32_t step = 4 * blockDim.x;
            for (uint32_t i0 = 4 * tid; i0 < n; i0 += 2 * step) {
                const SurvGroup g0 = load_group(aux, cq, pq, codes, i0, n);
                const SurvGroup g1 = load_group(aux, cq, pq, codes, i0 + step, n);
                run(g0, i0);
                if (g1.cnt) run(g1, i0 + step);
            }
        }
        if (out != dq) {
            __syncthreads();
            for (uint32_t i = tid; i < n; i += blockDim.x) dq[i] = out[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            le += __shfl_xor_sync(0xffffffffu, le, o);
            dmn = min(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
            dmx = max(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
        }
        if ((tid & 31) == 0) {
            if (le) atomicAdd(&s_le, le);
            atomicMin(&s_mn, dmn);
            atomicMax(&s_mx, dmx);
        }
        __syncthreads();
        if (tid == 0) {
            cand_le[q] = s_le;
            if (cand_mm) {
                cand_mm[2 * q] = s_mn;
                cand_mm[2 * q + 1] = s_mx;
            }
        }
    }
}

template <int DSUB>
bool recheck_smem_t(const float* xq, uint32_t d, const float* coarse, const float* books,
                    const uint32_t* probes, uint32_t w, const uint8_t* codes, const uint32_t* cand_cnt,
                    uint32_t cap, const uint32_t* cand_pos, float* cand_dist, const float* tau,
                    size_t nq, uint32_t* cand_le, cudaStream_t s, uint32_t* cand_mm) {
    const size_t smem = (size_t)M * KS * DSUB * sizeof(float) + (size_t)w * d * sizeof(float);
    if (smem > 216 * 1024) return false;  // + ~9.3 KiB static (s_x) <= 227 KiB
    set_max_smem((const void*)recheck_smem_kernel<DSUB>, (size_t)((int)smem));
    uint32_t* counter = nullptr;
    PQRR_CUDA(cudaMallocAsync(&counter, sizeof(uint32_t), s));
    PQRR_CUDA(cudaMemsetAsync(counter, 0, sizeof(uint32_t), s));
    recheck_smem_kernel<DSUB><<<sm_count(), 512, smem, s>>>(
        xq, d, coarse, books, probes, w, reinterpret_cast<const u64*>(codes), cand_cnt, cap, cand_pos,
        cand_dist, tau, nq, cand_le, counter, kNegZero2, cand_mm);
    PQRR_LAUNCH_CHECK();
    PQRR_CUDA(cudaFreeAsync(counter, s));
    count_launch();
    return true;
}

void launch_recheck(const float* xq, uint32_t d, uint32_t m, const float* coarse,
                    const float* books, const uint32_t* probes, uint32_t w, const uint8_t* codes,
                    const uint32_t* cand_cnt, uint32_t cap, const uint32_t* cand_pos,
                    float* cand_dist, const float* tau, size_t nq, uint32_t* cand_le,
                    cudaStream_t s, uint32_t* cand_mm, const uint64_t* cand_code,
                    const uint32_t* cand_used) {
    if (!nq) return;
    // per-pair LUTs (the common shape), else the shared-memory code book, else
    // the generic recheck kernels
    if (d == 128 && m == M && d / m == 16 && w <= 256) {
        const size_t smem = (size_t)LUT_SLOTS * M * KS * sizeof(float);
        set_max_smem((const void*)recheck_lut_kernel, smem);
        uint32_t* counter = nullptr;
        float* scratch = nullptr;
        PQRR_CUDA(cudaMallocAsync(&counter, sizeof(uint32_t), s));
        PQRR_CUDA(cudaMallocAsync(&scratch, (size_t)sm_count() * cap * sizeof(float), s));
        PQRR_CUDA(cudaMemsetAsync(counter, 0, sizeof(uint32_t), s));
        recheck_lut_kernel<<<sm_count(), 512, smem, s>>>(xq, coarse, books, probes, w,
                                                        reinterpret_cast<const u64*>(codes), cand_cnt, cap,
                                                        cand_pos, cand_dist, tau, nq, cand_le, counter,
                                                        kNegZero2, cand_mm,
                                                        reinterpret_cast<const u64*>(cand_code), cand_used, scratch);
        PQRR_LAUNCH_CHECK();
        PQRR_CUDA(cudaFreeAsync(scratch, s));
        PQRR_CUDA(cudaFreeAsync(counter, s));
        count_launch();
        return;
    }
    if (d / m == 16 &&
        recheck_smem_t<16>(xq, d, coarse, books, probes, w, codes, cand_cnt, cap, cand_pos, cand_dist,
                           tau, nq, cand_le, s, cand_mm))
        return;
    if (d / m == 8 &&
        recheck_smem_t<8>(xq, d, coarse, books, probes, w, codes, cand_cnt, cap, cand_pos, cand_dist,
                          tau, nq, cand_le, s, cand_mm))
        return;
    switch (d / m) {
        case 16: return recheck_t<16>(xq, d, coarse, books, probes, w, codes, cand_cnt, cap, cand_pos, cand_dist, tau, nq, cand_le, s);
        case 8: return recheck_t<8>(xq, d, coarse, books, probes, w, codes, cand_cnt, cap, cand_pos, cand_dist, tau, nq, cand_le, s);
        case 4: return recheck_t<4>(xq, d, coarse, books, probes, w, codes, cand_cnt, cap, cand_pos, cand_dist, tau, nq, cand_le, s);
        case 32: return recheck_t<32>(xq, d, coarse, books, probes, w, codes, cand_cnt, cap, cand_pos, cand_dist, tau, nq, cand_le, s);
        default: throw ArgError("recheck supports d/m in {4, 8, 16, 32}");
    }
}

}  // namespace pqrr_b200
