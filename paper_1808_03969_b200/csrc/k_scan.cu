// k_scan.cu -- PQ linear scan (Alg. 1 PQLinearScan) on sm_100a.
//
// One CTA = (a batch of B queries) x (a chunk of the linear code array).  The
// ADC table A of every query of the batch is built once in shared
// memory; each thread then streams one uint8 code per step from HBM (coalesced
// 16-byte loads, prefetched one step ahead) and evaluates Eq. 2 for
// all B queries, so every code byte fetched is reused B times from registers.
//
// Bank-conflict-free lookups ("fast" layout, M in {4,8,16,32}): lane l walks the
// subspaces of its code in the order m = j XOR (l mod M) and reads replica
// g = l / M of the table, whose word for (z, m) sits at column g*M + m of row z.
// For a fixed step j the 32 lanes then hit 32 distinct banks whatever their
// code bytes are.  Two queries share each 256-byte row, so one PRMT builds the
// byte offset (z << 8) | 4*(l ^ j) from the code word and the LDS immediate
// selects the query.  The lane-dependent summation order is undone by a
// canonical (CA2, m ascending) rescore of the kept candidates, so the returned
// distances equal the oracle's bit for bit.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "lut.cuh"
#include "topk.cuh"

namespace rii {


template <int W>
__device__ __forceinline__ void ldg256(const uint8_t *p, uint32_t (&w)[W], int o) {
    asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(w[o]), "=r"(w[o + 1]), "=r"(w[o + 2]), "=r"(w[o + 3]), "=r"(w[o + 4]), "=r"(w[o + 5]),
                   "=r"(w[o + 6]), "=r"(w[o + 7])
                 : "l"(p));
}

// The 32-byte code loads need 32-byte aligned code arrays (M >= 32).
static inline void check_code_align(const void *codes, int M) {
    if (M >= 32 && ((uintptr_t)codes & 31u)) throw Error(1, "code array must be 32-byte aligned");
}

template <int W>
__device__ __forceinline__ void load_code(const uint8_t *p, uint32_t (&w)[W]) {
    // M >= 32: 32-byte loads (sm_100 LDG.256): the warp's 32 codes of one load are
    // 1 KB contiguous, 8 L1 wavefronts per load instead of 8 per 16-byte half (the
    // code loads share the L1 data pipe with the table lookups).  Code arrays are
    // 32-byte aligned (checked by the launchers).
    if constexpr (W == 16) {  // M = 64
        ldg256(p, w, 0);
        ldg256(p + 32, w, 8);
    } else if constexpr (W == 8) {
        ldg256(p, w, 0);
    } else if constexpr (W == 4) {
        const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    } else if constexpr (W == 2) {
        const uint2 a = __ldg(reinterpret_cast<const uint2 *>(p));
        w[0] = a.x; w[1] = a.y;
    } else {
        static_assert(W == 1, "code words per thread");
        w[0] = __ldg(reinterpret_cast<const uint32_t *>(p));
    }
}

// Top lists, fresh buffers, counters, thresholds, scratch[16] and the q16 scales.
// (scratch: 32 ints -- [0] compaction max, [1] overflow flag, [2, 2 + B) fill snapshot, [31] rescale flag)
__host__ __device__ constexpr int smem_aux_bytes(int B, int kk) { return B * (kk + NEWCAP) * 8 + B * 8 + 128 + B * 16; }

// Debug counters of one kernel family (0 linear scans, 1 float list items, 2 integer
// list items): RII_DBG_MASK (bit per family, default all) restricts what is counted.
static unsigned long long *debug_counters_for(int family) {
    unsigned long long *d = debug_counters();
    if (!d) return nullptr;
    const char *e = getenv("RII_DBG_MASK");
    return (!e || ((atoi(e) >> family) & 1)) ? d : nullptr;
}

// Window-end read of a query's shared bound (another CTA's published kk-th distance
// tightens this CTA's filter mid-chunk); counted when it lowers the bound.
__device__ __forceinline__ void gqs_update(float *gqs, int qq, float g, unsigned long long *dbg) {
    if (g < gqs[qq]) {
        gqs[qq] = g;
        if (dbg) atomicAdd(dbg + DBG_GTHR_TIGHTEN, 1ull);
    }
}

// TAB: 0 = fp32 pair tables, 1 = bf16-packed quad tables, 2 = u16 fixed-point quad
// tables (integer SWAR sums, linear mode with a per-query bound).
template <int M, int B, bool LISTS, int NTH, int U, int TAB, int VARIANT = 0>
__global__ void __launch_bounds__(NTH, NTH <= 192 ? 2 : 1) scan_fast_kernel(const ScanArgs a) {
    constexpr int W = M / 4, NP = B / 2, NQ = B / 4;
    constexpr bool PACKED = TAB != 0, U6 = TAB == 3, Q16 = TAB == 2 || U6;  // U6: integer path as Q16
    static_assert(!PACKED || B % 4 == 0, "packed tables hold 4 queries each");
    // VARIANT bit 7 (FIXB): the integer tables sit at dynamic-smem offset 0, whose shared
    // address is the compile-time 0x400 (checked at run time), so the LDS carries it as
    // an immediate and no 64 KB-aligned padding is needed (two CTAs fit on an SM).
    constexpr bool FIXB = (VARIANT & 128) != 0;
    constexpr int LDS_BASE = FIXB ? 0x400 : 0;
    static_assert(!U6 || B == 8 || B == 16, "u6 oct tables hold 8 queries");
    static_assert(!(U6 && LISTS) || FIXB, "list-mode u6 uses the fixed-base layout");
    static_assert(!FIXB || U6, "the fixed-base layout is implemented for the u6 tables");
    // u6 options (VARIANT bit 0: 5-bit entries summed over 8 steps; bit 1: two table
    // copies so that the code-word permutation needs one select stage, M = 32 only)
    // (VARIANT bit 8: 7-bit entries, pairs of steps summed bytewise -- finer steps, so
    // the filter passes fewer false candidates, for more widening work)
    constexpr int U6_GJ = ((VARIANT & 1) && M >= 8) ? 8 : (VARIANT & 256) ? 2 : 4;
    constexpr bool U6_R2 = U6 && (VARIANT & 2) && M == 32;
    constexpr float U6_CAP = U6_GJ == 8 ? 31.0f : U6_GJ == 2 ? 127.0f : 63.0f;
    constexpr int H = lut_halves(M), LQF = lut_q_floats(M);  // M = 64: two 32-subspace halves
    static_assert(H == 1 || TAB == 0 || TAB == 3, "M = 64 runs the fp32-pair and u6 tables");
    constexpr int NO = U6 ? B / 8 : 1;  // u6 oct tables (B = 16: two, fixed-base layout, 384 threads)
    static_assert(NO == 1 || (FIXB && H == 1 && !U6_R2), "16-query u6 tables: fixed-base layout, M <= 32");
    constexpr int LUTB = U6 ? (U6_R2 ? 2 : 1) * H * NO * OCT_BYTES : NQ * QUAD_BYTES;  // integer tables
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t *lut = smem;
    const int kk = a.kk;
    uint8_t *aux = smem + (PACKED ? NQ * QUAD_BYTES : NP * H * LUT_PAIR_BYTES);
    if constexpr (Q16 && FIXB) {
        if ((uint32_t)__cvta_generic_to_shared(smem) != (uint32_t)LDS_BASE) __trap();  // layout assumption
        aux = smem + LUTB;
    } else if constexpr (Q16) {
        // The u16 tables start at a 64 KB-aligned shared address, so that one PRMT
        // yields the complete LDS address (bytes 2-3 = table base >> 16); the top
        // lists and buffers go into the padding below it when they fit, else above.
        const uint32_t pad = (0u - (uint32_t)__cvta_generic_to_shared(smem)) & 0xffffu;
        lut = smem + pad;
        aux = pad >= (uint32_t)smem_aux_bytes(B, kk) ? smem : lut + LUTB;
    }
    uint64_t *top = reinterpret_cast<uint64_t *>(aux);
    uint64_t *fresh = top + B * kk;
    int *cnt = reinterpret_cast<int *>(fresh + B * NEWCAP);
    float *thr = reinterpret_cast<float *>(cnt + B);
    int *scratch = reinterpret_cast<int *>(thr + B);
    float *qsc = reinterpret_cast<float *>(scratch + 32);  // q16: per-query scale [B]
    const uint8_t *__restrict__ codes = a.codes;
    const uint8_t *__restrict__ rcodes = LISTS ? a.rcodes : a.codes;  // codes by candidate id

    // (checked build) the whole layout -- tables, top lists, fresh buffers, counters,
    // thresholds, scratch and the per-query scalars below -- fits the launch's smem
    RII_SMEM_CHECK(smem, qsc + 4 * B);
    RII_SMEM_CHECK(smem, lut + LUTB);
    if (a.dbg && threadIdx.x == 0) *reinterpret_cast<long long *>(scratch + 24) = clock64();  // debug cycles
    // Work item: linear mode = (code chunk ci, query batch qb); list mode = (posting
    // list, up to B of the queries that probe it) -- list-major Alg. 2 L7-L13.
    int64_t c0, c1, qstart = 0;
    int ci = 0, qb = 0, nqi = B;
    if constexpr (LISTS) {
        const int4 it = a.items[blockIdx.x];
        c0 = a.offsets[it.x];
        c1 = a.offsets[it.x + 1];
        qstart = it.y;
        nqi = it.z;
        RII_DCHECK(c0 <= c1 && c1 <= a.n_codes && nqi >= 1 && nqi <= B && qstart >= 0 &&
                   qstart + nqi <= a.nq * a.P);
        // The list is one contiguous range of the list-ordered mirror: one bulk prefetch
        // into L2 at item start (overlaps the table fill) instead of a DRAM miss per step.
        if (threadIdx.x == 0 && c1 > c0) {
            const uintptr_t b0 = (uintptr_t)(codes + (size_t)c0 * M) & ~(uintptr_t)15;
            const uintptr_t b1 = ((uintptr_t)(codes + (size_t)c1 * M) + 15) & ~(uintptr_t)15;
            for (uintptr_t o = b0; o < b1; o += 65536) {
                const uint32_t n = (uint32_t)min((uintptr_t)65536, b1 - o);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(o), "r"(n) : "memory");
            }
        }
    } else {
        ci = blockIdx.x / a.nb;
        qb = blockIdx.x - ci * a.nb;
        c0 = (int64_t)ci * a.chunk;
        c1 = min(a.n_codes, c0 + a.chunk);
        const int64_t rem = a.nq - (int64_t)qb * B;
        nqi = rem < B ? (int)rem : B;
    }
    // List mode: the item's query indices are read from qlist once into shared memory.
    int *qid_s = reinterpret_cast<int *>(qsc + B);
    float *tsc = qsc + 2 * B;  // integer tables: the bound T each query's scale was set from
    // The query's global bound (list mode: the best kk-th distance any finished item
    // of this query saw, inflated by 1e-5 for the lane-rotated rounding; linear: the
    // sampled bound) also filters.  Kept in shared memory: it is read at window ends
    // only, so it holds no registers across the scan loop.
    float *gqs = qsc + 3 * B;
    if constexpr (LISTS) {
        if (threadIdx.x < B) {
            const int qq = (int)threadIdx.x < nqi ? (int)threadIdx.x : nqi - 1;
            qid_s[threadIdx.x] = (int)(a.qlist[qstart + qq] / a.P);
            RII_DCHECK(a.qlist[qstart + qq] < (uint64_t)(a.nq * a.P));
        }
        __syncthreads();
    }
    auto query_of = [&](int qq) -> int64_t {  // global query index of slot qq
        qq = qq < nqi ? qq : nqi - 1;
        if constexpr (LISTS) return qid_s[qq];
        else return (int64_t)qb * B + qq;
    };
    const int D = M * a.ds, tid = threadIdx.x, lane = tid & 31;
    const uint32_t qmask = nqi >= 32 ? 0xffffffffu : (1u << nqi) - 1u;  // the slots holding real queries

    if constexpr (U6 && LISTS) {
        // precomputed per-query u6 tables (u6_tables_kernel) with their scales
        if (tid < B) qsc[tid] = __ldg(a.qscale + query_of(tid));
#pragma unroll
        for (int o = 0; o < NO; ++o) {
            const uint8_t *tq[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) tq[k] = a.qtab8 + query_of(8 * o + k) * LQF;
            load_lut_oct_u8pre<U6_R2, H, NTH>(reinterpret_cast<uint32_t *>(lut + o * OCT_BYTES), tq);
        }
    } else if constexpr (U6) {
        // u6 tables: per-query scale s = 63 * ALPHA / T (T = +inf -> s = 0: everything passes).
        // The bound is read ONCE per query: the CTAs of other chunks lower it with
        // atomicMin at any moment, and threads that quantised with different reads
        // built a table of mixed scales whose filter could drop true candidates (a
        // nondeterministic miss, round 2: ~1 query per run at 1024 queries x 2M codes)
        if (tid < B) {
            const float T = __ldcg(a.gthr + query_of(tid));
            tsc[tid] = T;
            qsc[tid] = __fdiv_rd(U6_CAP * u6_alpha(M), fmaxf(T, 1e-30f));
        }
        __syncthreads();
#pragma unroll
        for (int o = 0; o < NO; ++o) {
            float qs[8];
            const float *tq[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int qq = 8 * o + k;
                qs[k] = qsc[qq];
                tq[k] = a.tables + query_of(qq) * LQF;
            }
            load_lut_oct_u6<U6_R2, H>(reinterpret_cast<uint32_t *>(lut + o * OCT_BYTES), tq, qs, U6_CAP);
        }
    } else if (Q16 && a.qtab16) {
        // precomputed per-query u16 tables (q16_tables_kernel) with their scales
        if (tid < B) qsc[tid] = __ldg(a.qscale + query_of(tid));
#pragma unroll
        for (int p = 0; p < NQ; ++p)
            load_lut_quad_u16(reinterpret_cast<uint32_t *>(lut + p * QUAD_BYTES), a.qtab16 + query_of(4 * p) * LQF,
                              a.qtab16 + query_of(4 * p + 1) * LQF, a.qtab16 + query_of(4 * p + 2) * LQF,
                              a.qtab16 + query_of(4 * p + 3) * LQF);
    } else if constexpr (Q16) {
        // u16 tables: per-query scale s = CAP / T (T = +inf -> s = 0: everything passes);
        // the bound is read once per query (see the u6 branch)
        if (tid < B) {
            const float T = __ldcg(a.gthr + query_of(tid));  // current bound on the kk-th distance
            tsc[tid] = T;
            qsc[tid] = __fdiv_rd((float)q16_cap<M>(), fmaxf(T, 1e-30f));
        }
        __syncthreads();
        float qs[B];
#pragma unroll
        for (int qq = 0; qq < B; ++qq) qs[qq] = qsc[qq];
#pragma unroll
        for (int p = 0; p < NQ; ++p)
            load_lut_quad_q16<M>(reinterpret_cast<uint32_t *>(lut + p * QUAD_BYTES),
                                 a.tables + query_of(4 * p) * LQF, a.tables + query_of(4 * p + 1) * LQF,
                                 a.tables + query_of(4 * p + 2) * LQF,
                                 a.tables + query_of(4 * p + 3) * LQF, qs[4 * p], qs[4 * p + 1],
                                 qs[4 * p + 2], qs[4 * p + 3]);
    } else if constexpr (PACKED) {
#pragma unroll
        for (int p = 0; p < NQ; ++p) {
            uint32_t *dq = reinterpret_cast<uint32_t *>(lut + p * QUAD_BYTES);
            if (a.sdcT)
                load_lut_quad_sdc<M>(dq, a.sdcT, a.qcodes + query_of(4 * p) * M, a.qcodes + query_of(4 * p + 1) * M,
                                     a.qcodes + query_of(4 * p + 2) * M, a.qcodes + query_of(4 * p + 3) * M);
            else
                load_lut_quad(dq, a.tables + query_of(4 * p) * LQF, a.tables + query_of(4 * p + 1) * LQF,
                              a.tables + query_of(4 * p + 2) * LQF,
                              a.tables + query_of(4 * p + 3) * LQF);
        }
    } else {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float *lp = reinterpret_cast<float *>(lut + p * H * LUT_PAIR_BYTES);
            if (a.tables)
                load_lut_pair_h<M>(lp, a.tables + query_of(2 * p) * LQF, a.tables + query_of(2 * p + 1) * LQF);
            else
            {
                if constexpr (H == 1) build_lut_pair<M>(lp, a.q + query_of(2 * p) * D, a.q + query_of(2 * p + 1) * D, a.cb, a.ds);
                else __trap();  // M = 64 always runs with per-query HBM tables
            }
        }
    }
    for (int e = tid; e < B * kk; e += NTH) top[e] = KEY_MAX;
    if (tid < B) {
        cnt[tid] = 0; thr[tid] = __int_as_float(0x7f800000); scratch[2 + tid] = 0;
        // slots past the item's / batch's queries (they repeat its last query's table) get
        // a negative bound: they never pass the filter, push nothing and do not rescale
        gqs[tid] = tid >= nqi ? -1.0f : a.gthr ? __ldcg(a.gthr + query_of(tid)) : __int_as_float(0x7f800000);
    }
    if (tid == 0) scratch[1] = 0;
    __syncthreads();
    // debug cycle accounting: nothing stays live across the scan loop (the timestamp
    // of the loop start is kept in shared memory, scratch[24..25], free for B <= 16)
    if (a.dbg && tid == 0) {
        const long long t = clock64();
        atomicAdd(a.dbg + DBG_CYC_FILL, (unsigned long long)(t - *reinterpret_cast<long long *>(scratch + 24)));
        *reinterpret_cast<long long *>(scratch + 24) = t;
    }

    // u6 tables (one copy, M >= 32): an 8-byte LDS is served per half-warp, so the
    // columns only need to differ within each half: lane l reads column
    // (l mod 16) ^ j at step j (lanes l and l + 16 the same column, in the other
    // wavefront), and the code-word rotation rw < 4 needs two select stages, not three.
    // (the fp32-pair and bf16-packed tables have 8-byte columns too)
    constexpr bool HALFW = ((U6 && !U6_R2) || TAB == 0 || TAB == 1) && M >= 32;
    const uint32_t lr = HALFW ? ((uint32_t)lane & 15u) : (uint32_t)lane;
    const uint32_t r = lr & (M - 1), rw = r >> 2, l8 = lr << 3;
    uint32_t sel[4];
    if constexpr (Q16) make_selectors_q16(r, sel);
    else make_selectors(r, sel);
    // q16 column registers: bytes 0-1 = 8 (l ^ t) for t = 0,1 (colA) and 2,3 (colB),
    // bytes 2-3 = the table's shared address >> 16
    const uint32_t lut_hi = FIXB ? 0u : (uint32_t)__cvta_generic_to_shared(lut) & 0xffff0000u;
    uint32_t colA = lut_hi | ((lr ^ 0u) << 3) | ((lr ^ 1u) << 11);
    uint32_t colB = lut_hi | ((lr ^ 2u) << 3) | ((lr ^ 3u) << 11);
    // two-copy u6 layout: word rotation by bit 2 of the lane only; bit 3 picks the copy
    // (64 KB higher, columns XOR 8), so a half-warp still covers all 32 banks once
    const uint32_t rw2 = ((uint32_t)lane >> 2) & 1u;
    if constexpr (U6_R2) {
        const uint32_t rep = ((uint32_t)lane >> 3) & 1u, r3 = (uint32_t)lane & 3u;
        auto cb = [&](uint32_t t) { return ((rw2 << 5) | (((t ^ r3) & 3u) << 3)) ^ (rep << 6); };
        const uint32_t hi = lut_hi + (rep << 16);
        colA = hi | cb(0) | (cb(1) << 8);
        colB = hi | cb(2) | (cb(3) << 8);
    }
    // The column registers of every word group, computed once with opaque XORs: left
    // to itself the compiler sometimes re-materialises these 16 values inside the
    // loop (16 more ALU ops per code: 127 -> 149 ms on deep10m, build-dependent).
    // (colB = colA ^ 0x1010 in every layout, so only colA's groups are kept: 8 registers)
    uint32_t colv[U6 ? (M / 4 < 8 ? M / 4 : 8) : 1];
    if constexpr (U6) {
#pragma unroll
        for (int aw = 0; aw < (M / 4 < 8 ? M / 4 : 8); ++aw)
            asm volatile("xor.b32 %0, %1, %2;" : "=r"(colv[aw]) : "r"(colA), "r"((uint32_t)(aw * 0x2020)));
    }
    // Filter thresholds: the exact kk-th distance (and list bound); relaxed by
    // PACK_SLACK for the approximate packed sums.
    auto relax = [](float t) { return PACKED ? __fmul_ru(t, PACK_SLACK) : t; };
    float th[B];
    uint32_t thq[Q16 ? B : 1];
    // u6: the thresholds packed per accumulator word, lanes (q, q + 2) as 0x8000 | thq
    uint32_t thp[U6 ? B / 2 : 1];
    auto set_thq = [&]() {
        if constexpr (Q16) {
#pragma unroll
            for (int qq = 0; qq < B; ++qq) thq[qq] = q16_threshold(fminf(thr[qq], gqs[qq]), qsc[qq]);
        }
        if constexpr (U6) {
#pragma unroll
            for (int k = 0; k < B / 2; ++k) {
                const int lo = (k >> 1) * 4 + (k & 1);
                thp[k] = 0x80008000u | min(thq[lo], 0x7fffu) | (min(thq[lo + 2], 0x7fffu) << 16);
            }
        }
    };
#pragma unroll
    for (int qq = 0; qq < B; ++qq) th[qq] = relax(fminf(thr[qq], gqs[qq]));
    set_thq();
    // Integer tables (linear mode): when a query's bound has halved since its scale was
    // set, re-quantise the tables at the new bound (any scale keeps the filter exact;
    // a tight one keeps it selective).  Block-uniform: thread 0 decides from smem.
    auto maybe_rescale = [&]() {
        if constexpr (Q16 && !LISTS) {
            if (tid == 0) {
                int f = 0;
                for (int qq = 0; qq < nqi; ++qq) f |= fminf(thr[qq], gqs[qq]) < 0.5f * tsc[qq];
                if (f) {
                    for (int qq = 0; qq < B; ++qq) {
                        const float T = fminf(thr[qq], gqs[qq]);
                        if (qq >= nqi || !(T < tsc[qq])) continue;
                        tsc[qq] = T;
                        qsc[qq] = U6 ? __fdiv_rd(U6_CAP * u6_alpha(M), fmaxf(T, 1e-30f))
                                     : __fdiv_rd((float)q16_cap<M>(), fmaxf(T, 1e-30f));
                    }
                }
                scratch[31] = f;
                if (f && a.dbg) atomicAdd(a.dbg + DBG_RESCALE, 1ull);
            }
            __syncthreads();
            if (scratch[31]) {
                float qs[B];
#pragma unroll
                for (int qq = 0; qq < B; ++qq) qs[qq] = qsc[qq];
                if constexpr (U6) {
#pragma unroll
                    for (int o = 0; o < NO; ++o) {
                        const float *tq[8];
                        float qo[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            tq[k] = a.tables + query_of(8 * o + k) * LQF;
                            qo[k] = qs[8 * o + k];
                        }
                        load_lut_oct_u6<U6_R2, H>(reinterpret_cast<uint32_t *>(lut + o * OCT_BYTES), tq, qo, U6_CAP);
                    }
                } else {
#pragma unroll
                    for (int p = 0; p < NQ; ++p)
                        load_lut_quad_q16<M>(reinterpret_cast<uint32_t *>(lut + p * QUAD_BYTES),
                                             a.tables + query_of(4 * p) * LQF,
                                             a.tables + query_of(4 * p + 1) * LQF,
                                             a.tables + query_of(4 * p + 2) * LQF,
                                             a.tables + query_of(4 * p + 3) * LQF, qs[4 * p], qs[4 * p + 1],
                                             qs[4 * p + 2], qs[4 * p + 3]);
                }
                __syncthreads();
                set_thq();
            }
        }
    };
    // Packed mode: canonical (CA2) rescore of the fresh entries from the queries'
    // fp32 HBM tables before they are compacted into the exact top lists.
    auto rescore_fresh = [&]() {
        if (a.dbg && tid == 0) {
            int n = 0;
            for (int qq = 0; qq < B; ++qq) n += cnt[qq];
            atomicAdd(a.dbg + DBG_FRESH, (unsigned long long)n);
        }
        if constexpr (PACKED) {
            for (int qq = 0; qq < B; ++qq) {
                const int n = cnt[qq];
                if (a.sdcT) {  // d_S(x, c) = sum_m T_m[x^m][c^m] (CA2)
                    const uint8_t *xq = a.qcodes + query_of(qq) * M;
                    for (int i = tid; i < n; i += NTH) {
                        uint64_t *f = fresh + qq * NEWCAP + i;
                        const uint32_t id = key_id(*f);
                        const uint8_t *cp = rcodes + (size_t)id * M;
                        float d = 0.f;
#pragma unroll
                        for (int m = 0; m < M; ++m)
                            d = __fadd_rn(d, __ldg(a.sdcT + ((size_t)m * KS + xq[m]) * KS + cp[m]));
                        *f = make_key(d, id);
                    }
                    continue;
                }
                const float *tq = a.tables + query_of(qq) * LQF;
                for (int i = tid; i < n; i += NTH) {
                    uint64_t *f = fresh + qq * NEWCAP + i;
                    const uint32_t id = key_id(*f);
                    const uint8_t *cp = rcodes + (size_t)id * M;
                    float d = 0.f;
#pragma unroll
                    for (int m = 0; m < M; ++m) d = __fadd_rn(d, lut_q_entry(tq, m, cp[m]));
                    *f = make_key(d, id);
                }
            }
            __syncthreads();
        }
    };

    // Each thread evaluates U codes per step (positions base + u*NT + tid, coalesced),
    // the next step's codes prefetched into registers.  Block barriers only every
    // WIN steps: a window whose pushes overflow the fresh buffer is rolled back
    // (its pushes dropped, the buffer compacted) and redone one step at a time,
    // which cannot overflow (an empty buffer holds a whole step, NEWCAP >= NT*U).
    // (u16 tables start from the sampled bound, so few pushes: VARIANT bits 2/3 widen the window)
    constexpr int STEP = NTH * U, WIN = (VARIANT & 0x7c) ? (VARIANT & 0x7c) * 2 : 4, SOFT = NEWCAP / 4;
    static_assert(NEWCAP >= STEP, "a single step must fit the fresh buffer");
    int *s_ovf = scratch + 1, *s_cnt0 = scratch + 2;  // flags, fill snapshot at the window start
    uint32_t w[U][W];
    // Codes are read at positions of the linear array (linear mode) or of the
    // list-ordered mirror (list mode: a posting list is the contiguous range
    // [offsets[k], offsets[k+1]) of the mirror, read with the same coalesced loads as a
    // linear chunk).  cid = the candidate's id: the position (linear) or the CSR entry
    // ids[p] (lists), so every tie resolves by (dist, id) (CA4); list-mode rescores
    // read the code by id from the original array (a.rcodes).
    uint32_t cid[U];
    auto key_of = [&](uint32_t id, int64_t) -> uint32_t { return id; };
    // Probe-masked IVF (linear mode, ProbeMask): the CTA's queries whose probed lists
    // contain the code at pos (all ones without a mask).  Read only where some lane of
    // the warp passes the filter, so it costs nothing in the lookup loop.
    auto probe_bits = [&](int64_t pos) -> uint32_t {
        if constexpr (LISTS) return 0xffffffffu;
        else {
            if (a.alist == nullptr || pos >= c1) return 0xffffffffu;
            return __ldg(a.pmask + (int64_t)qb * a.pm_K + __ldg(a.alist + pos));
        }
    };
    auto load_step = [&](int64_t b, uint32_t(&dst)[U][W], uint32_t(&did)[U]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t p = b + u * NTH + tid;
#pragma unroll
            for (int i = 0; i < W; ++i) dst[u][i] = 0;
            did[u] = 0;
            if (p < c1) {
                // the key id: the position (linear) or its CSR entry (lists; an independent
                // coalesced 4-byte load, prefetched with the code one step ahead)
                if constexpr (LISTS) did[u] = __ldg(a.ids + p);
                else did[u] = (uint32_t)p;
                load_code<W>(codes + (size_t)p * M, dst[u]);
            }
        }
    };
    int64_t base = c0;
    load_step(base, w, cid);
    // Adaptive window: without a bound (every threshold +inf) the first window runs one
    // step, and a window that overflowed is redone from one step; the length doubles
    // after every window that fit, up to WIN.  Loose early thresholds therefore cost
    // compactions, not rolled-back windows.
    // (The linear integer-table kernels always start from a sampled bound and keep the
    // fixed scheme -- WIN steps, four single steps after a rollback: their register
    // allocation is at the limit, and the adaptive counter costs them a stack frame.)
    constexpr bool ADAPT = !(Q16 && !LISTS);
    int win = 1;
    if constexpr (ADAPT) {
#pragma unroll
        for (int qq = 0; qq < B; ++qq) win &= qq >= nqi || !(th[qq] < __int_as_float(0x7f800000));
        win = win ? 1 : WIN;
    } else {
        win = 0;  // the `safe` countdown of single-step windows
    }
    while (base < c1) {
        const int64_t wstart = base;
        const int nsteps = ADAPT ? win : (win > 0 ? 1 : WIN);
        bool ovf = false, need = false;
        for (int s = 0; s < nsteps && base < c1; ++s) {
            uint32_t wn[U][W], nid[U];
            // short codes (M <= 16, linear): one thread pulls the codes of step + PFD into L2
            // (a bulk prefetch), so the register prefetch one step ahead waits on L2, not DRAM
            if constexpr (!LISTS && M <= 16 && (VARIANT & 1024)) {
                constexpr int PFD = 6;
                const int64_t pb = base + (int64_t)PFD * STEP;
                if (tid == 0 && pb < c1) {
                    const uintptr_t b0 = (uintptr_t)(codes + (size_t)pb * M) & ~(uintptr_t)15;
                    const uint32_t n = (uint32_t)(min((int64_t)STEP, c1 - pb) * M + 15) & ~15u;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b0), "r"(n) : "memory");
                }
            }
            load_step(base + STEP, wn, nid);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t pos = base + u * NTH + tid;
                if constexpr (Q16) {
                    uint32_t dq[B];
                    if constexpr (U6) {
                        uint32_t acc[4 * NO];
                        adc_u6<M, U6_GJ, U6_R2, LDS_BASE, NO, HALFW ? 4 : 8>(w[u], U6_R2 ? rw2 : rw, sel, colv, a.one,
                                                                             acc);
                        // SWAR compare: lane sums <= M * 63 < 2^15 and thp holds 0x8000 | thq per
                        // lane, so bit 15 / 31 of thp - acc is set exactly when sum <= thq
                        uint32_t t[4 * NO], tor = 0;
#pragma unroll
                        for (int k = 0; k < 4 * NO; ++k) {
                            t[k] = thp[k] - acc[k];
                            tor |= t[k];
                        }
                        const bool anyp = (tor & 0x80008000u) != 0;
                        if (__any_sync(0xffffffffu, anyp && pos < c1)) {
                            // per-lane pass mask (bit qq = query qq; query qq sits in word
                            // (qq / 4) * 2 + qq % 2, bit 15 or 31 by qq & 2), OR-reduced over
                            // the warp: only the queries some lane passes take a ballot
                            uint32_t mk = 0;
#pragma unroll
                            for (int k = 0; k < 4 * NO; ++k)
                                mk |= (t[k] & 0x80008000u) >> (15 - (4 * (k >> 1) + (k & 1)));
                            mk = pos < c1 ? (mk | (mk >> 14)) & qmask : 0u;
                            if (!LISTS && mk && a.alist) mk &= probe_bits(pos);
                            const uint32_t kid = key_of(cid[u], pos);
                            for (uint32_t wm = __reduce_or_sync(0xffffffffu, mk); wm; wm &= wm - 1u) {
                                const int qq = __ffs(wm) - 1;
                                push_candidate_win((mk >> qq) & 1u, (uint64_t)kid, fresh + qq * NEWCAP, cnt + qq,
                                                   lane, SOFT, need, ovf);
                            }
                        }
                        continue;
                    } else {
                        uint32_t acc0[NQ], acc1[NQ];
                        adc_q16<M, NQ>(w[u], rw, sel, colA, colB, acc0, acc1);
#pragma unroll
                        for (int p = 0; p < NQ; ++p) {
                            dq[4 * p] = acc0[p] & 0xffffu;
                            dq[4 * p + 2] = acc0[p] >> 16;
                            dq[4 * p + 1] = acc1[p] & 0xffffu;
                            dq[4 * p + 3] = acc1[p] >> 16;
                        }
                    }
                    uint32_t mk = 0;  // bit qq: query qq passes (the u6 branch's warp-mask loop)
#pragma unroll
                    for (int qq = 0; qq < B; ++qq) mk |= (uint32_t)(dq[qq] <= thq[qq]) << qq;
                    mk = pos < c1 ? mk & qmask : 0u;
                    if (!LISTS && mk && a.alist) mk &= probe_bits(pos);
                    // the key's distance field is replaced by the canonical rescore
                    const uint32_t wmask = __reduce_or_sync(0xffffffffu, mk);
                    const uint32_t kid = wmask ? key_of(cid[u], pos) : 0u;
                    for (uint32_t wm = wmask; wm; wm &= wm - 1u) {
                        const int qq = __ffs(wm) - 1;
                        push_candidate_win((mk >> qq) & 1u, (uint64_t)kid, fresh + qq * NEWCAP, cnt + qq, lane,
                                           SOFT, need, ovf);
                    }
                    continue;
                }
                float d[B];
                if constexpr (PACKED) {
                    float2 ab[NQ], cd[NQ];
                    adc_packed<M, NQ, VARIANT>(lut, w[u], rw, sel, l8, ab, cd);
#pragma unroll
                    for (int p = 0; p < NQ; ++p) {
                        d[4 * p] = ab[p].x;
                        d[4 * p + 1] = ab[p].y;
                        d[4 * p + 2] = cd[p].x;
                        d[4 * p + 3] = cd[p].y;
                    }
                } else {
                    float2 acc2[NP];
                    adc_rotated<M, B, HALFW ? 4 : 8>(lut, w[u], rw, sel, l8, acc2);
#pragma unroll
                    for (int p = 0; p < NP; ++p) {
                        d[2 * p] = acc2[p].x;
                        d[2 * p + 1] = acc2[p].y;
                    }
                }
                // one warp vote per code; per-query ballots only when some lane has a candidate
                bool any = false;
#pragma unroll
                for (int qq = 0; qq < B; ++qq) any |= d[qq] <= th[qq];
                if (__any_sync(0xffffffffu, any && pos < c1)) {
                    const uint32_t kid = key_of(cid[u], pos);
                    const uint32_t pb = probe_bits(pos) & qmask;
#pragma unroll
                    for (int qq = 0; qq < B; ++qq)
                        push_candidate_win(pos < c1 && d[qq] <= th[qq] && ((pb >> qq) & 1u), make_key(d[qq], kid),
                                           fresh + qq * NEWCAP,
                                           cnt + qq, lane, SOFT, need, ovf);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                cid[u] = nid[u];
#pragma unroll
                for (int i = 0; i < W; ++i) w[u][i] = wn[u][i];
            }
            base += STEP;
        }
        if (ovf) *s_ovf = 1;
        if (a.dbg && tid == 0) atomicAdd(a.dbg + DBG_WINDOWS, 1ull);
        if (__syncthreads_or(ovf || need)) {
            const bool rolled = *s_ovf != 0;  // written before the barrier; reset below
            if (a.dbg && tid == 0) atomicAdd(a.dbg + (rolled ? DBG_ROLLBACK : DBG_COMPACT), 1ull);
            if (rolled && tid < B) cnt[tid] = s_cnt0[tid];
            __syncthreads();
            rescore_fresh();
            compact_topk(top, fresh, cnt, thr, B, kk, scratch);
            if (tid == 0) *s_ovf = 0;
            if (tid < B) s_cnt0[tid] = 0;
            if (a.gthr) {
                if (tid < B) gqs_update(gqs, tid, __ldcg(a.gthr + query_of(tid)), a.dbg);
                __syncthreads();
            }
#pragma unroll
            for (int qq = 0; qq < B; ++qq) th[qq] = relax(fminf(thr[qq], gqs[qq]));
            set_thq();
            if (rolled) {
                base = wstart;
                load_step(base, w, cid);
                win = ADAPT ? 1 : 4;
                continue;
            }
        } else {
            if (tid < B) s_cnt0[tid] = cnt[tid];
            if (a.gthr) {
                if (tid < B) gqs_update(gqs, tid, __ldcg(a.gthr + query_of(tid)), a.dbg);
                __syncthreads();
#pragma unroll
                for (int qq = 0; qq < B; ++qq) th[qq] = fminf(th[qq], relax(gqs[qq]));
                set_thq();
            }
            __syncthreads();  // snapshot taken before the next window pushes
        }
        maybe_rescale();
        if constexpr (ADAPT) win = win * 2 < WIN ? win * 2 : WIN;
        else if (win > 0) --win;
    }
    if (a.dbg && tid == 0) {
        const long long t = clock64();
        atomicAdd(a.dbg + DBG_CYC_SCAN, (unsigned long long)(t - *reinterpret_cast<long long *>(scratch + 24)));
        *reinterpret_cast<long long *>(scratch + 24) = t;
    }
    __syncthreads();
    rescore_fresh();
    compact_topk(top, fresh, cnt, thr, B, kk, scratch);
    if (a.gthr) {  // publish this item's kk-th distance as a bound for the query
        if (tid < nqi && thr[tid] < __int_as_float(0x7f800000)) {
            const float bound = __fmul_ru(thr[tid], 1.00001f);
            const int old = atomicMin(reinterpret_cast<int *>(a.gthr + query_of(tid)), __float_as_int(bound));
            if (a.dbg && __float_as_int(bound) < old) atomicAdd(a.dbg + DBG_PUBLISH, 1ull);
        }
    }

    // Canonical rescore (CA2: m ascending, replica 0) of the kept candidates.  List
    // mode defers it to the per-query merge (merge_kernel with a Rescore); packed
    // mode's top lists are exact already.
    const int lkk = ilog2_pow2(kk);
    for (int e = tid; e < ((LISTS || PACKED) ? 0 : B * kk); e += NTH) {
        const uint64_t k = top[e];
        if (k == KEY_MAX) continue;
        const int qq = e >> lkk;
        const uint32_t id = key_id(k);
        const uint8_t *cp = codes + (size_t)id * M;
        const float *lq = reinterpret_cast<const float *>(lut + (qq >> 1) * H * LUT_PAIR_BYTES);
        float d = 0.f;
#pragma unroll
        for (int m = 0; m < M; ++m) d = __fadd_rn(d, lut_pair_entry(lq, qq & 1, m, cp[m]));
        top[e] = make_key(d, id);
    }
    __syncthreads();
    if constexpr (!LISTS && !PACKED) bitonic_sort_rows(top, B, kk, kk);
    for (int e = tid; e < B * kk; e += NTH) {
        const int qq = e >> lkk, i = e & (kk - 1);
        if (qq >= nqi) continue;
        if constexpr (LISTS) {  // [q][probe rank][kk]; an empty list writes its first key only
            if (i == 0 || top[e - i] != KEY_MAX) a.out[a.qlist[qstart + qq] * kk + i] = top[e];
        }
        else {
            RII_DCHECK(((int64_t)qb * B + qq) < a.nq && ci < a.nc);
            a.out[(((int64_t)qb * B + qq) * a.nc + ci) * kk + i] = top[e];
        }
    }
    if (a.dbg && tid == 0) {
        atomicAdd(a.dbg + DBG_CYC_TAIL, (unsigned long long)(clock64() - *reinterpret_cast<long long *>(scratch + 24)));
        atomicAdd(a.dbg + DBG_ITEMS, 1ull);
    }
}

// Generic layout (any M <= 64): table A[q][m][z], canonical m-ascending sums.
template <int B>
__global__ void __launch_bounds__(NT, 1)
    scan_generic_kernel(const uint8_t *__restrict__ codes, int64_t n_codes, const float *__restrict__ q, int64_t nq,
                        const float *__restrict__ cb, int M, int ds, int kk, int nb, int64_t chunk, int nc,
                        uint64_t *__restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    float *lut = reinterpret_cast<float *>(smem);
    uint64_t *top = reinterpret_cast<uint64_t *>(smem + (size_t)B * M * KS * 4);
    uint64_t *fresh = top + B * kk;
    int *cnt = reinterpret_cast<int *>(fresh + B * NEWCAP);
    float *thr = reinterpret_cast<float *>(cnt + B);
    int *scratch = reinterpret_cast<int *>(thr + B);

    const int item = blockIdx.x, ci = item / nb, qb = item - ci * nb;
    const int64_t c0 = (int64_t)ci * chunk, c1 = min(n_codes, c0 + chunk);
    const int D = M * ds, tid = threadIdx.x, lane = tid & 31;

    for (int e = tid; e < B * M * KS; e += NT) {
        const int qq = e / (M * KS), m = (e / KS) % M, z = e % KS;
        const int64_t qi = min((int64_t)qb * B + qq, nq - 1);
        const float *qv = q + qi * D + m * ds, *cv = cb + ((size_t)m * KS + z) * ds;
        float a = 0.f;
        for (int j = 0; j < ds; ++j) a = ca1_step(a, qv[j], cv[j]);
        lut[e] = a;
    }
    for (int e = tid; e < B * kk; e += NT) top[e] = KEY_MAX;
    if (tid < B) { cnt[tid] = 0; thr[tid] = __int_as_float(0x7f800000); }
    __syncthreads();
    float th[B];
#pragma unroll
    for (int qq = 0; qq < B; ++qq) th[qq] = thr[qq];
    bool need = false;
    for (int64_t base = c0; base < c1; base += NT) {
        const int64_t pos = base + tid;
        const bool valid = pos < c1;
        float acc[B];
#pragma unroll
        for (int qq = 0; qq < B; ++qq) acc[qq] = 0.f;
        if (valid) {
            const uint8_t *cp = codes + pos * M;
            for (int m = 0; m < M; ++m) {
                const int z = cp[m];
#pragma unroll
                for (int qq = 0; qq < B; ++qq) acc[qq] = __fadd_rn(acc[qq], lut[(qq * M + m) * KS + z]);
            }
        }
#pragma unroll
        for (int qq = 0; qq < B; ++qq)
            push_candidate(valid && acc[qq] <= th[qq], make_key(acc[qq], (uint32_t)pos), fresh + qq * NEWCAP,
                           cnt + qq, lane, need);
        if (__syncthreads_or(need)) {
            compact_topk(top, fresh, cnt, thr, B, kk, scratch);
#pragma unroll
            for (int qq = 0; qq < B; ++qq) th[qq] = thr[qq];
            need = false;
        }
    }
    compact_topk(top, fresh, cnt, thr, B, kk, scratch);
    for (int e = tid; e < B * kk; e += NT) {
        const int qq = e >> ilog2_pow2(kk), i = e & (kk - 1);
        const int64_t qi = (int64_t)qb * B + qq;
        if (qi < nq) out[(qi * nc + ci) * kk + i] = top[e];
    }
}

// B == 8 means the bf16-packed variant (2 quad tables); otherwise B / 2 fp32 pair tables.
// u16 variant: 64 KB-aligned tables + the aux block below or above them (kernel).
static size_t smem_q16(int kk) { return (size_t)2 * QUAD_BYTES + 2 * (size_t)smem_aux_bytes(8, kk) + 16; }
#ifndef RII_SCAN_M  // common translation unit only
bool q16_supported(int kk) { return smem_q16(kk) <= 227 * 1024; }
#endif  // !RII_SCAN_M
static size_t smem_fast(int B, int kk, int M = 32) {
    const size_t lut = B == 8 ? (size_t)2 * QUAD_BYTES : (size_t)(B / 2) * lut_halves(M) * LUT_PAIR_BYTES;
    return lut + smem_aux_bytes(B, kk);
}
// Integer tables run for scans of at least RII_Q16_MIN (default 2^19) codes.
#ifndef RII_SCAN_M  // common translation unit only
int64_t q16_min_codes() {
    const char *e = getenv("RII_Q16_MIN");
    return e ? atoll(e) : ((int64_t)1 << 19);
}
#endif  // !RII_SCAN_M
// RII_PACKED=0 disables the bf16-packed tables (A/B measurements).
static bool packed_enabled() {
    static bool on = [] {
        const char *e = getenv("RII_PACKED");
        return !(e && e[0] == '0');
    }();
    return on;
}
static size_t smem_generic(int B, int M, int kk) {
    return (size_t)B * M * KS * 4 + (size_t)B * (kk + NEWCAP) * 8 + 64;
}
static constexpr size_t SMEM_CAP = 227 * 1024;
static constexpr int PACKED_MIN_CODES = 16384;  // codes per CTA below which fp32 pair tables win
// Packed-kernel configuration (RII_PACK_CFG, for A/B measurements): 0 = 512 threads,
// shift unpack; 1 = 384 threads, PRMT unpack; 2 = 512 threads, PRMT unpack,
// recomputed column offsets; 3 = 384 threads, shift unpack.
constexpr int PACKED_NTH = 512;  // bf16-packed kernels: 512 threads

#ifndef RII_SCAN_M  // common translation unit only
static int q16_cfg(int M);
static bool fixed_base_ok();
ScanPlan plan_linear(int M, int kk, int64_t nq, int64_t n_codes, int num_sms, bool tables_available, int max_nc,
                     bool int_ok_caller) {
    ScanPlan p{};
    p.fast = (M == 4 || M == 8 || M == 16 || M == 32 || M == 64);
    p.B = 0;
    if (p.fast && M == 64) {
        // two table halves: the u6 oct tables (B = 8, 128 KB) for long scans, else fp32 pairs (B = 2)
        const bool int_ok = int_ok_caller && tables_available && q16_enabled() && q16_supported(kk) &&
                            n_codes >= q16_min_codes();
        if (int_ok) { p.B = 8; p.smem = smem_q16(kk); }
        else if (smem_fast(2, kk, M) <= SMEM_CAP) { p.B = 2; p.smem = smem_fast(2, kk, M); }
    } else if (p.fast && q16_cfg(M) == 9 && int_ok_caller && tables_available && q16_enabled() &&
               n_codes >= q16_min_codes() && fixed_base_ok() &&
               (size_t)2 * OCT_BYTES + smem_aux_bytes(16, kk) + 16 <= SMEM_CAP) {
        p.B = 16;  // u6, two oct tables (RII_Q16_CFG=9)
        p.smem = (size_t)2 * OCT_BYTES + smem_aux_bytes(16, kk) + 16;
    } else if (p.fast) {
        // Packed tables cost a larger per-CTA table build: only for long code ranges.
        const bool pk = packed_enabled() && tables_available && n_codes >= (int64_t)PACKED_MIN_CODES;
        for (int B : {8, 6, 4, 2}) {
            if (B == 8 && !pk) continue;
            if (smem_fast(B, kk) <= SMEM_CAP) { p.B = B; p.smem = smem_fast(B, kk); break; }
        }
    } else {
        for (int B : {4, 2, 1})
            if (smem_generic(B, M, kk) <= SMEM_CAP) { p.B = B; p.smem = smem_generic(B, M, kk); break; }
    }
    if (p.B == 0) throw Error(1, "topk too large for the scan kernel's shared-memory budget");
    p.nb = (int)ceil_div(nq, p.B);
    // Code chunks: minimise waves(nc) / nc (per-CTA work ~ n_codes / nc), >= 8192 codes per
    // chunk, and at most ~40 MB of codes per chunk so that the CTAs of a wave (which all
    // stream the same chunk) hit in the 126 MB L2 even when they drift apart.
    int64_t nc_max = n_codes / 8192;
    if (nc_max > max_nc) nc_max = max_nc;
    if (nc_max < 1) nc_max = 1;
    if (nc_max > 256) nc_max = 256;
    static const int64_t chunk_mb = [] {
        const char *e = getenv("RII_CHUNK_MB");  // A/B: 0 disables the L2 chunk cap
        return (int64_t)(e ? atoi(e) : 40);
    }();
    const int64_t nc_min = chunk_mb > 0 ? std::min<int64_t>(nc_max, ceil_div(n_codes * M, chunk_mb << 20)) : 1;
    // Cost of a chunking: waves x (codes per chunk + a fixed per-CTA cost in code
    // equivalents: table load, final compaction and output, ~25 us ~ 8192 codes).
    static const double fix = [] {
        const char *e = getenv("RII_CTA_FIX");
        return e ? atof(e) : 8192.0;
    }();
    double best = 1e300;
    int bnc = (int)nc_min;
    for (int nc = (int)nc_min; nc <= nc_max; ++nc) {
        const double waves = (double)ceil_div((int64_t)p.nb * nc, num_sms);
        const double t = waves * ((double)n_codes / nc + fix) * (1.0 + 0.002 * nc);
        if (t < best * 0.999) { best = t; bnc = nc; }
    }
    p.nc = bnc;
    p.chunk = ceil_div(n_codes, bnc);
    if (p.chunk < 1) p.chunk = 1;
    // Test knob (multi-window parity tests): a fixed chunk length, so that one CTA
    // scans many barrier windows and chunks end at different times.
    if (const char *e = getenv("RII_CHUNK_CODES")) {
        const int64_t c = atoll(e);
        if (c > 0 && c < n_codes) {
            p.chunk = c;
            p.nc = (int)ceil_div(n_codes, c);
        }
    }
    return p;
}
#endif  // !RII_SCAN_M

// Threads per CTA x codes per thread and step of the lane-rotated kernels
// (RII_SCAN_CFG=0: 256 x 2, 1: 512 x 1; default below).
static int scan_threads() { return 512; }  // fp32 pair kernels

// Linear integer-table kernel (RII_Q16_CFG for A/B; default: u6 oct tables for M = 32,
// where they measured 134.6 ms against 204.1 ms for u16 on deep10m, u16 otherwise
// (sift1m, M = 16: u16 16.0 ms, u6 24.6 ms)).  0 = u16, 384 threads, window 128;
// 1 = u16 window 32; 2 = u16 256 x 2; 3 = u16 512 threads; 4 = u6 384; 5 = u6 512.
static int q16_cfg(int M) {
    const char *e = getenv("RII_Q16_CFG");
    if (M == 64) return 4;  // two halves: u6 oct tables, one copy
    // M = 32: 9 = 16 queries per CTA (two oct tables, fixed-base layout; 117 ms on deep10m),
    // 7 = 8 queries with two table copies (127 ms).  M = 16 and 8 too (round 2: sift1m
    // linear, M = 16, u16 13.0 -> 11.0 ms; the deep10m shape at M = 8 93.8 -> 48.9 ms)
    return e ? atoi(e) : ((M == 32 || M == 16 || M == 8) ? 9 : 0);
}
// M = 64 u6 linear kernel threads (RII_M64_NTH: 384 spills ~200 B of code words and
// took 52.9 ms on sift1m_m64; 256 does not spill: 43.5 ms)
static int m64_nth() {
    const char *e = getenv("RII_M64_NTH");
    return e ? atoi(e) : 256;
}
// Threads of the M = 8, 16-query u6 linear kernel: 512 (118 registers, 16 warps per SM) against 384
// (127 registers, 12 warps) measured deep10m at M = 8 44.2 -> 40.8 ms per 10k queries, 1,024 queries
// 5.22 -> 4.82 ms, a 1e6-id subset 7.50 -> 6.98 ms, 1e8 codes 41.8 -> 40.3 ms per 1,024 queries
// (profiles/r02o_ab_m8nth_*.jsonl).  RII_M8_NTH=384 / 512 forces one (A/B, tests).
// Few query batches over a long scan are the exception (128 queries x 1e7 codes: 1.09 ms at 384
// threads, 1.59 ms at 512; profiles/r02r_ab_m8nth_short.jsonl), so scans of >= 2^22 codes by fewer
// than 512 queries keep 384 threads; shorter scans measured equal or faster at 512 for every batch.
static int m8_nth(int64_t n, int64_t nq) {
    const char *e = getenv("RII_M8_NTH");
    if (e && atoi(e) == 384) return 384;
    if (e && atoi(e) == 512) return 512;
    return (nq >= 512 || n < ((int64_t)1 << 22)) ? 512 : 384;
}
static int q16_nth(int M) { return M == 64 ? m64_nth() : 384; }  // 256 x 2 codes per thread: 150 ms (deep10m)
#ifndef RII_SCAN_M  // common translation unit only
bool q16_is_u6(int M) { const int c = q16_cfg(M); return c == 4 || c == 7 || c == 9; }
#endif  // !RII_SCAN_M
// List-major u6 items (phase B of the two-phase IVF): 0 = u16 items; 3 = u6, 384
// threads, one table copy (deep10m L = 64: 21.4 -> 19.1 ms; 192 threads with two CTAs
// per SM measured 19.2 ms, two table copies 20.7 ms).
#ifndef RII_SCAN_M  // common translation unit only
// The fixed-base layout of the u6 list items assumes the dynamic shared memory of a
// kernel without static shared memory starts at shared address 0x400 (1 KB reserved);
// probed once on the device so that a different base falls back instead of trapping.
static __global__ void smem_base_probe_kernel(uint32_t *out) {
    extern __shared__ uint8_t probe_smem[];
    if (threadIdx.x == 0) *out = (uint32_t)__cvta_generic_to_shared(probe_smem);
}
static bool fixed_base_ok() {
    static const bool ok = [] {
        uint32_t *d = nullptr, h = 0;
        if (cudaMalloc(&d, 4) != cudaSuccess) return false;
        smem_base_probe_kernel<<<1, 32, 1024>>>(d);
        const bool good = cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost) == cudaSuccess && h == 0x400u;
        cudaFree(d);
        return good;
    }();
    return ok;
}
bool smem_fixed_base_ok() { return fixed_base_ok(); }
// 7-bit list-item entries (M = 32; RII_LIST_U7=0 disables): steps twice as fine at the
// same saturation point, pairs of steps summed bytewise (2 * 127 < 256) -- more widening
// work, but the integer items are push-bound, and the finer filter passes fewer false
// candidates (deep10m phase B: 9.6M -> 7.4M pushes; L = 64 13.2 -> 12.6 ms, L = 16 8.7
// -> 8.2, L = 4 5.5 -> 5.1).  The per-query tables are then written with cap 127.
bool list_u7(int M) {
    const char *e = getenv("RII_LIST_U7");
    if (M == 64) return e && atoi(e) == 1;  // A/B (two 32-subspace halves)
    return (M == 32 || M == 16 || M == 8) && !(e && atoi(e) == 0);
}
int list_u6_cfg(int M) {
    if (!fixed_base_ok()) return 0;
    if (M == 64) return 3;  // two halves: only the u6 items fit (128 KB)
    const char *e = getenv("RII_LIST_U6");
    if (M == 32) return e ? atoi(e) : 3;
    // M = 16 and 8: 7-bit oct items too (sift1m L = 64: u16 items 10.2 ms, 7-bit 7.1, 6-bit
    // 7.5; deep10m shape at M = 8, L = 64: u16 11.3 -> 9.1 ms, L = 16 6.1 -> 6.0 ms)
    if (M == 16 || M == 8) return e ? atoi(e) : 3;
    return 0;
}

#endif  // !RII_SCAN_M
// u6 list items: 384 threads (one CTA per SM) or 192 threads with two CTAs per SM, so
// one CTA's table fill, barriers and final compaction overlap the other's scan.
// Measured on deep10m (10k queries): 192 wins at P >= 32 probed lists (L = 64: 15.1
// -> 13.9 ms; with the merged-bound phases 13.9 -> 12.8 ms) and loses below (L = 16:
// 8.8 -> 9.4 ms).  RII_LIST_NTH=192 / 384 forces one (A/B).
// u6 list items with M = 8 load one 8-byte code per thread and step: with 12 warps per
// SM the code stream is latency-bound (configs[4], lists of 31,623 codes: 60 % of the
// stalls on the next step's code load, 14 % warps active), so those items take two
// codes per thread and step: configs[4] IVF L = 64 19.6 -> 13.4 ms per 1,024 queries,
// the deep10m shape at M = 8 8.2 -> 7.5 ms (M = 16, sift1m: 6.7 -> 6.8 ms, not taken).
// RII_LIST_U=1 restores one (A/B).
static bool list_u2() {
    const char *e = getenv("RII_LIST_U");
    return !(e && atoi(e) == 1);
}
// Long linear u6 scans with M = 8: a bulk L2 prefetch of the codes six steps ahead
// (VARIANT bit 10), so the one-step register prefetch of 8-byte codes waits on L2, not
// DRAM: configs[4] linear (1,024 queries x 1e9 codes) 479.5 -> 401.1 ms, the deep10m
// shape at M = 8 49.3 -> 43.5 ms; a 1e6-code subset 1.15 -> 1.23 ms and sift1m (M = 16)
// 11.0 -> 11.5 ms, so only M = 8 scans of >= 2^22 codes take it.  RII_LIN_PF=0 disables.
static bool lin_l2_prefetch(int64_t n) {
    const char *e = getenv("RII_LIN_PF"), *m = getenv("RII_LIN_PF_MIN");  // (MIN: tests)
    return !(e && atoi(e) == 0) && n >= (m ? atoll(m) : ((int64_t)1 << 22));
}
static int list_q16_nth(int M, int64_t P) {
    if (M == 64) return 384;
    const char *e = getenv("RII_LIST_NTH");
    if (e) return atoi(e) == 192 ? 192 : 384;
    return P >= 32 ? 192 : 384;
}
static size_t smem_list_q16(int M, int kk, int B = 8) {
    if (B == 16) return 2 * OCT_BYTES + smem_aux_bytes(16, kk) + 16;
    if (list_u6_cfg(M) < 3) return smem_q16(kk);
    return (size_t)lut_halves(M) * OCT_BYTES + smem_aux_bytes(8, kk) + 16;
}

#ifndef RII_SCAN_M  // common translation unit only
int list_int_B(int M, int kk) {
    return list_u6_cfg(M) == 4 && smem_list_q16(M, kk, 16) <= SMEM_CAP ? 16 : 8;
}
#endif  // !RII_SCAN_M

template <int M, int B, bool LISTS>
static void *fast_kernel_ptr_h1(bool q16, int nth);
template <int M, int B, bool LISTS>
static void *fast_kernel_ptr_b(bool q16, int nth);

template <int M, int B, bool LISTS>
static void *fast_kernel_ptr(bool q16 = false, int nth = 384) {
    if constexpr (lut_halves(M) > 1) {  // M = 64: u6 oct tables (B = 8) or fp32 pairs (B = 2) only
        if constexpr (B == 8) {
            if constexpr (LISTS) {
                if (list_u7(M)) return (void *)scan_fast_kernel<M, 8, true, 384, 1, 3, 256 | 128 | 64>;
                return (void *)scan_fast_kernel<M, 8, true, 384, 1, 3, 128 | 64>;
            } else if (m64_nth() == 256) return (void *)scan_fast_kernel<M, 8, false, 256, 1, 3, 64>;
            else return (void *)scan_fast_kernel<M, 8, false, 384, 1, 3, 64>;
        } else if constexpr (B == 2) {
            return (void *)scan_fast_kernel<M, 2, LISTS, 512, 1, 0>;
        } else {
            return nullptr;
        }
    } else {
        return fast_kernel_ptr_h1<M, B, LISTS>(q16, nth);
    }
}

template <int M, int B, bool LISTS>
static void *fast_kernel_ptr_h1(bool q16, int nth) {
    if constexpr (B == 16) {  // u6, two oct tables, fixed-base layout (list items: M = 32)
        if constexpr (LISTS) {
            if constexpr (M == 32) return (void *)scan_fast_kernel<M, 16, true, 384, 1, 3, 128 | 64>;
            else return nullptr;
        } else {
            return (void *)scan_fast_kernel<M, 16, false, 384, 1, 3, 128 | 64>;
        }
    } else {
        return fast_kernel_ptr_b<M, B, LISTS>(q16, nth);
    }
}

template <int M, int B, bool LISTS>
static void *fast_kernel_ptr_b(bool q16, int nth) {
    // Kernel variants kept for A/B runs (measured on B200, deep10m, 10k queries; the
    // others this round tried are recorded in DESIGN.md and were removed to bound the
    // build time): RII_Q16_CFG 0 = u16 tables (204 ms), 4 = u6 one copy (131 ms),
    // 7 = u6 two copies (125 ms, default for M = 32); RII_LIST_U6 0 = u16 items,
    // 3 = u6 items (default for M = 32); RII_PACKED=0 = fp32 pairs.
    if constexpr (B == 8) {
        if constexpr (LISTS) {
            if (q16) {
                if (list_u6_cfg(M) >= 3 && list_u7(M)) {
                    if constexpr (M <= 8) {  // two codes per thread and step (RII_LIST_U=1: one)
                        if (nth == 192 && list_u2()) return (void *)scan_fast_kernel<M, 8, true, 192, 2, 3, 256 | 128 | 64>;
                    }
                    if (nth == 192) return (void *)scan_fast_kernel<M, 8, true, 192, 1, 3, 256 | 128 | 64>;
                    return (void *)scan_fast_kernel<M, 8, true, 384, 1, 3, 256 | 128 | 64>;
                }
                if (list_u6_cfg(M) >= 3 && nth == 192)
                    return (void *)scan_fast_kernel<M, 8, true, 192, 1, 3, 128 | 64>;
                if (list_u6_cfg(M) >= 3) return (void *)scan_fast_kernel<M, 8, true, 384, 1, 3, 128 | 64>;
                return (void *)scan_fast_kernel<M, 8, true, 384, 1, 2, 64>;  // u16, window 128
            }
        } else {
            if (q16) {
                switch (q16_cfg(M)) {
                    case 4: return (void *)scan_fast_kernel<M, 8, false, 384, 1, 3, 64>;  // u6 oct tables
                    case 7: return (void *)scan_fast_kernel<M, 8, false, 384, 1, 3, 66>;  // two copies
                    default: return (void *)scan_fast_kernel<M, 8, false, 384, 1, 2, 64>;  // u16, window 128
                }
            }
        }
        return (void *)scan_fast_kernel<M, 8, LISTS, 512, 1, 1, 0>;  // bf16-packed quads
    } else {
        return (void *)scan_fast_kernel<M, B, LISTS, 512, 1, 0>;
    }
}

template <int M, int B>
static void launch_fast_t(const ScanPlan &pl, const uint8_t *codes, int64_t n, const float *q, int64_t nq,
                          const float *cb, int ds, int kk, uint64_t *out, cudaStream_t st, const float *tables,
                          float *gthr, bool q16_req, int timer, const ProbeMask &mask) {
    const bool q16 = (B == 8 || B == 16) && q16_req && gthr != nullptr;
    if (mask.alist && mask.B != B) throw Error(1, "probe mask grouped by a different query batch");
    void *kern = fast_kernel_ptr<M, B, false>(q16);
    int nth = q16 ? q16_nth(M) : (B == 8 ? PACKED_NTH : scan_threads());
    if constexpr (M == 8 && B == 16) {
        // M = 8 needs < 128 registers, so 512 threads (16 warps per SM instead of 12) still fit one
        // CTA's register file (m8_nth)
        const bool pf = lin_l2_prefetch(n);
        if (q16 && m8_nth(n, nq) == 512) {
            kern = pf ? (void *)scan_fast_kernel<M, 16, false, 512, 1, 3, 1024 | 128 | 64>
                      : (void *)scan_fast_kernel<M, 16, false, 512, 1, 3, 128 | 64>;
            nth = 512;
        } else if (q16 && pf) {
            kern = (void *)scan_fast_kernel<M, 16, false, 384, 1, 3, 1024 | 128 | 64>;
        }
    }
    // (M = 16 at 512 threads -- 124 registers, no spills -- measured 11.06 -> 16.74 ms on sift1m,
    // 1.62 -> 4.36 ms at 1,024 queries: profiles/r02q_ab_m16nth_sift1m.jsonl; the variant was removed.)
    const size_t smem = q16 && B == 8 ? smem_q16(kk) : pl.smem;
    RII_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    ScanArgs a{};
    a.codes = codes; a.n_codes = n; a.q = q; a.nq = nq; a.cb = cb; a.ds = ds; a.kk = kk;
    a.nb = pl.nb; a.chunk = pl.chunk; a.nc = pl.nc; a.out = out; a.tables = tables;
    a.gthr = gthr;
    a.one = 1;
    a.dbg = debug_counters_for(0);
    a.alist = mask.alist; a.pmask = mask.pm; a.pm_K = mask.K;
    void *args[] = {&a};
    KernelTimer t(timer, st), tp(B >= 8 && timer == TK_LINEAR ? (q16 ? (q16_is_u6(M) ? TK_U6 : TK_Q16) : TK_PACKED) : -1,
                                 st);
    check_code_align(codes, M);
    RII_CUDA(cudaLaunchKernel(kern, dim3(pl.nb * pl.nc), dim3(nth), args, smem, st));
    count_launch();
}

template <int M>
void launch_fast_m(const ScanPlan &pl, const uint8_t *codes, int64_t n, const float *q, int64_t nq,
                          const float *cb, int ds, int kk, uint64_t *out, cudaStream_t st, const float *tables,
                          float *gthr, bool q16, int timer, const ProbeMask &mask) {
    if (pl.B == 16) launch_fast_t<M, 16>(pl, codes, n, q, nq, cb, ds, kk, out, st, tables, gthr, q16, timer, mask);
    else if (pl.B == 8) launch_fast_t<M, 8>(pl, codes, n, q, nq, cb, ds, kk, out, st, tables, gthr, q16, timer, mask);
    else if (pl.B == 6) launch_fast_t<M, 6>(pl, codes, n, q, nq, cb, ds, kk, out, st, tables, gthr, q16, timer, mask);
    else if (pl.B == 4) launch_fast_t<M, 4>(pl, codes, n, q, nq, cb, ds, kk, out, st, tables, gthr, q16, timer, mask);
    else launch_fast_t<M, 2>(pl, codes, n, q, nq, cb, ds, kk, out, st, tables, gthr, q16, timer, mask);
}

template <int B>
static void launch_generic_t(const ScanPlan &pl, const uint8_t *codes, int64_t n, int M, const float *q, int64_t nq,
                             const float *cb, int ds, int kk, uint64_t *out, cudaStream_t st) {
    auto kern = scan_generic_kernel<B>;
    RII_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    KernelTimer t(TK_LINEAR, st);
    kern<<<pl.nb * pl.nc, NT, pl.smem, st>>>(codes, n, q, nq, cb, M, ds, kk, pl.nb, pl.chunk, pl.nc, out);
    RII_LAUNCHED();
}

#ifndef RII_SCAN_M  // common translation unit only
bool list_major_supported(int M) { return M == 4 || M == 8 || M == 16 || M == 32 || M == 64; }
#endif  // !RII_SCAN_M

#ifndef RII_SCAN_M  // common translation unit only
int list_major_B(int kk, double avg_len, int M) {
    if (lut_halves(M) > 1) return smem_fast(2, kk, M) <= SMEM_CAP ? 2 : 0;  // fp32 pairs of two halves
    // bf16-packed B = 8 list items only on request (RII_LIST_PACKED_MIN = shortest average
    // list, A/B): slower than fp32 pairs wherever measured (deep10m rank-0 items 12.4 ->
    // 15.9 ms at 16,384; configs[4], lists of 31,623: 12.8 vs 13.4 ms per 1,024 queries)
    const char *pe = getenv("RII_LIST_PACKED_MIN");
    const double pmin = pe ? atof(pe) : 1e300;
    for (int B : {8, 6, 4, 2}) {
        if (B == 8 && (!packed_enabled() || avg_len < pmin)) continue;
        if (smem_fast(B, kk) <= SMEM_CAP) return B;
    }
    return 0;
}
#endif  // !RII_SCAN_M

template <int M, int B>
static void launch_list_t(const ScanArgs &a, int64_t n_items, cudaStream_t st, bool q16) {
    q16 = q16 && (B == 8 || B == 16);
    const int nth = q16 ? (B == 8 && list_u6_cfg(M) >= 3 ? list_q16_nth(M, a.P) : 384)
                        : (B == 8 ? PACKED_NTH : scan_threads());
    void *kern = fast_kernel_ptr<M, B, true>(q16, nth);
    if (!kern) throw Error(1, "no list-major kernel for this (M, B)");
    const size_t smem = q16 ? smem_list_q16(M, a.kk, B) : smem_fast(B, a.kk, M);
    RII_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    ScanArgs aa = a;
    aa.one = 1;
    aa.dbg = debug_counters_for(q16 ? 2 : 1);
    void *args[] = {&aa};
    KernelTimer t(TK_IVF, st);
    check_code_align(a.codes, M);
    RII_CUDA(cudaLaunchKernel(kern, dim3((unsigned)n_items), dim3(nth), args, smem, st));
    count_launch();
}

template <int M>
void launch_list_m(int B, const ScanArgs &a, int64_t n_items, cudaStream_t st, bool q16) {
    if (B == 16) launch_list_t<M, 16>(a, n_items, st, true);
    else if (B == 8) launch_list_t<M, 8>(a, n_items, st, q16);
    else if (B == 6) launch_list_t<M, 6>(a, n_items, st, false);
    else if (B == 4) launch_list_t<M, 4>(a, n_items, st, false);
    else launch_list_t<M, 2>(a, n_items, st, false);
}

#ifndef RII_SCAN_M  // common translation unit only
// The scan kernels of each M are instantiated in their own translation unit (build.py
// compiles this file once per M with -DRII_SCAN_M): only declared here.
template <int M>
void assign_scan_m(const uint8_t *codes, int64_t n, const uint8_t *centers, int64_t K, const float *T, int32_t *assign,
                   float *dist, cudaStream_t st);
#define RII_EXTERN_M(MM)                                                                                          \
    extern template void launch_fast_m<MM>(const ScanPlan &, const uint8_t *, int64_t, const float *, int64_t,   \
                                           const float *, int, int, uint64_t *, cudaStream_t, const float *,     \
                                           float *, bool, int, const ProbeMask &);                               \
    extern template void launch_list_m<MM>(int, const ScanArgs &, int64_t, cudaStream_t, bool);                  \
    extern template void assign_scan_m<MM>(const uint8_t *, int64_t, const uint8_t *, int64_t, const float *,    \
                                           int32_t *, float *, cudaStream_t);
RII_EXTERN_M(4) RII_EXTERN_M(8) RII_EXTERN_M(16) RII_EXTERN_M(32) RII_EXTERN_M(64)
#undef RII_EXTERN_M
void launch_list_scan(int M, int B, const ScanArgs &a, int64_t n_items, cudaStream_t st, bool q16) {
    if (n_items <= 0) return;
    if (B == 0) throw Error(1, "topk too large for the list-major scan");
    if (q16 && ((B != 8 && B != 16) || !q16_supported(a.kk) || !a.gthr))
        throw Error(1, "integer list scan needs B = 8 or 16, kk <= 256, gthr");
    switch (M) {
        case 4: launch_list_m<4>(B, a, n_items, st, q16); break;
        case 8: launch_list_m<8>(B, a, n_items, st, q16); break;
        case 16: launch_list_m<16>(B, a, n_items, st, q16); break;
        case 64: launch_list_m<64>(B, a, n_items, st, q16); break;
        default: launch_list_m<32>(B, a, n_items, st, q16); break;
    }
}
#endif  // !RII_SCAN_M

#ifndef RII_SCAN_M  // common translation unit only
void launch_linear_scan(const ScanPlan &pl, const uint8_t *codes, int64_t n_codes, int M, const float *q, int64_t nq,
                        const float *cb, int D, int kk, uint64_t *out, cudaStream_t st, const float *tables,
                        float *gthr, bool q16, int timer, const ProbeMask &mask) {
    const int ds = D / M;
    if (pl.fast) {
        switch (M) {
#define RII_LF(MM) launch_fast_m<MM>(pl, codes, n_codes, q, nq, cb, ds, kk, out, st, tables, gthr, q16, timer, mask)
            case 4: RII_LF(4); break;
            case 8: RII_LF(8); break;
            case 16: RII_LF(16); break;
            case 64: RII_LF(64); break;
            default: RII_LF(32); break;
#undef RII_LF
        }
    } else if (mask.alist) {
        throw Error(1, "probe-masked scan: fast-layout plans only");
    } else if (pl.B == 4) {
        launch_generic_t<4>(pl, codes, n_codes, M, q, nq, cb, ds, kk, out, st);
    } else if (pl.B == 2) {
        launch_generic_t<2>(pl, codes, n_codes, M, q, nq, cb, ds, kk, out, st);
    } else {
        launch_generic_t<1>(pl, codes, n_codes, M, q, nq, cb, ds, kk, out, st);
    }
}
#endif  // !RII_SCAN_M

// ---------------------------------------------------- SDC-mode assignment ---
#ifndef RII_SCAN_M  // common translation unit only
bool assign_scan_supported(int M, int64_t K) {
    return (M == 4 || M == 8 || M == 16 || M == 32) && packed_enabled() && K >= 8192 &&
           smem_fast(8, 32) <= SMEM_CAP;
}
#endif  // !RII_SCAN_M

static __global__ void top1_kernel(const uint64_t *__restrict__ keys, int64_t n, int kk, int32_t *__restrict__ assign,
                            float *__restrict__ dist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = keys[i * kk];
    assign[i] = (int32_t)key_id(k);
    if (dist) dist[i] = key_dist(k);
}

template <int M>
void assign_scan_m(const uint8_t *codes, int64_t n, const uint8_t *centers, int64_t K, const float *T,
                          int32_t *assign, float *dist, cudaStream_t st) {
    const int kk = 32, B = 8;
    const size_t smem = smem_fast(B, kk);
    void *kern = fast_kernel_ptr<M, B, false>(false);
    RII_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    const int64_t CH = (int64_t)1 << 23;  // codes per launch: bounds the [chunk][kk] keys
    uint64_t *keys = nullptr;
    RII_CUDA(cudaMallocAsync(&keys, (size_t)std::min(n, CH) * kk * 8, st));
    for (int64_t s0 = 0; s0 < n; s0 += CH) {
        const int64_t cn = std::min(CH, n - s0);
        ScanArgs a{};
        a.codes = centers; a.n_codes = K; a.nq = cn; a.ds = 0; a.kk = kk; a.out = keys;
        a.nb = (int)ceil_div(cn, B); a.chunk = K; a.nc = 1;
        a.sdcT = T; a.qcodes = codes + s0 * M;
        void *args[] = {&a};
        check_code_align(a.codes, M);
        RII_CUDA(cudaLaunchKernel(kern, dim3((unsigned)a.nb), dim3(PACKED_NTH), args, smem, st));
        count_launch();
        top1_kernel<<<(unsigned)ceil_div(cn, 256), 256, 0, st>>>(keys, cn, kk, assign + s0, dist ? dist + s0 : nullptr);
        RII_LAUNCHED();
    }
    RII_CUDA(cudaFreeAsync(keys, st));
}

#ifndef RII_SCAN_M  // common translation unit only
void launch_assign_scan(const uint8_t *codes, int64_t n, const uint8_t *centers, int64_t K, int M, const float *T,
                        int32_t *assign, float *dist, int, cudaStream_t st) {
    if (n <= 0) return;
    switch (M) {
        case 4: assign_scan_m<4>(codes, n, centers, K, T, assign, dist, st); break;
        case 8: assign_scan_m<8>(codes, n, centers, K, T, assign, dist, st); break;
        case 16: assign_scan_m<16>(codes, n, centers, K, T, assign, dist, st); break;
        default: assign_scan_m<32>(codes, n, centers, K, T, assign, dist, st); break;
    }
}
#endif  // !RII_SCAN_M

#ifndef RII_SCAN_M  // common translation unit only: tables, bounds, gather, merge
// ------------------------------------------------------------ LUT tables ---
// One CTA per query, thread z = code word z: the code book rows of subspace m are
// read coalesced (consecutive z), A(m, z) (CA1) goes to a [256][33] smem tile, and
// the rows (column c = A(c mod M, z)) are written out coalesced; M = 64 writes its
// two 32-subspace halves one after the other.
__global__ void __launch_bounds__(256) lut_tables_kernel(const float *__restrict__ q, int64_t nq,
                                                         const float *__restrict__ cb, int M, int ds,
                                                         float *__restrict__ tables) {
    extern __shared__ float qv[];  // [D]
    __shared__ float tile[KS][33];
    const int64_t qi = blockIdx.x;
    const int D = M * ds, z = threadIdx.x, H = lut_halves(M), MH = M < 32 ? M : 32;
    for (int e = threadIdx.x; e < D; e += blockDim.x) qv[e] = q[qi * D + e];
    for (int h = 0; h < H; ++h) {
        __syncthreads();
        for (int mm = 0; mm < MH; ++mm) {
            const int m = 32 * h + mm;
            const float *cv = cb + ((size_t)m * KS + z) * ds;
            float a = 0.f;
            for (int j = 0; j < ds; ++j) a = ca1_step(a, qv[m * ds + j], __ldg(cv + j));
            tile[z][mm] = a;
        }
        __syncthreads();
        float *t = tables + qi * (int64_t)lut_q_floats(M) + h * LUT_Q_FLOATS;
        for (int e = threadIdx.x; e < LUT_Q_FLOATS; e += blockDim.x) t[e] = tile[e >> 5][(e & 31) & (MH - 1)];
    }
}

void launch_lut_tables(const float *q, int64_t nq, const float *cb, int D, int M, float *tables, cudaStream_t st) {
    if (nq <= 0) return;
    lut_tables_kernel<<<(unsigned)nq, 256, (size_t)D * 4, st>>>(q, nq, cb, M, D / M, tables);
    RII_LAUNCHED();
}

// ------------------------------------------------- u16 tables: the bound ---
// RII_Q16=0 disables the u16 fixed-point tables (A/B measurements).
bool q16_enabled() {
    const char *e = getenv("RII_Q16");
    return !(e && e[0] == '0');
}

// out[i] = codes[i * stride] (a strided sample of the scanned codes).
__global__ void strided_gather_kernel(const uint8_t *__restrict__ codes, int M, int64_t stride, int64_t n,
                                      uint8_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t *src = reinterpret_cast<const uint32_t *>(codes + i * stride * M);
    uint32_t *dst = reinterpret_cast<uint32_t *>(out + i * M);
    for (int b = 0; b < M / 4; ++b) dst[b] = __ldg(src + b);
}

void launch_strided_gather(const uint8_t *codes, int M, int64_t stride, int64_t n, uint8_t *out, cudaStream_t st) {
    if (n <= 0) return;
    strided_gather_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(codes, M, stride, n, out);
    RII_LAUNCHED();
}

__global__ void strided_gather_i32_kernel(const int32_t *__restrict__ src, int64_t stride, int64_t n,
                                          int32_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __ldg(src + i * stride);
}

void launch_strided_gather_i32(const int32_t *src, int64_t stride, int64_t n, int32_t *out, cudaStream_t st) {
    if (n <= 0) return;
    strided_gather_i32_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(src, stride, n, out);
    RII_LAUNCHED();
}

// Probe masks of the masked IVF scan (ProbeMask): thread = (query, probe rank).
__global__ void probe_mask_kernel(const int32_t *__restrict__ probes, int64_t nq, int64_t P, int64_t K, int B,
                                  uint32_t *__restrict__ pm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq * P) return;
    const int64_t q = i / P;
    const int32_t k = probes[i];
    if (k < 0 || k >= K) return;
    atomicOr(pm + (q / B) * K + k, 1u << (q % B));
}

void launch_probe_mask(const int32_t *probes, int64_t nq, int64_t P, int64_t K, int B, uint32_t *pm,
                       cudaStream_t st) {
    if (B < 1 || B > 32) throw Error(1, "probe mask: 1 <= B <= 32");
    RII_CUDA(cudaMemsetAsync(pm, 0, (size_t)ceil_div(nq, (int64_t)B) * K * 4, st));
    if (nq * P <= 0) return;
    probe_mask_kernel<<<(unsigned)ceil_div(nq * P, 256), 256, 0, st>>>(probes, nq, P, K, B, pm);
    RII_LAUNCHED();
}

// Group-minimum bound: the sample's ns codes form G = ns / GSZ groups; each group's
// minimum ADC distance is a distance of a distinct sample code, so the kk-th smallest
// of the G group minima is >= the kk-th smallest of the sample, which is >= the final
// kk-th distance (the sample is a subset).  No top-k list is needed: CTA = 6 queries
// (three fp32 pair tables, lane-rotated sums inflated by 1e-5 to bound the canonical
// CA2 value from above), thread = groups, then a bitonic sort of the G minima.
constexpr int GB_NT = 512;
// queries per CTA: three fp32 pair tables (M <= 32) or one pair of two halves (M = 64)
__host__ __device__ constexpr int gb_q(int M) { return M > 32 ? 2 : 6; }

template <int M>
__global__ void __launch_bounds__(GB_NT, 1) group_min_bound_kernel(const uint8_t *__restrict__ samp, int64_t ns,
                                                                   int gsz, const float *__restrict__ tables,
                                                                   int64_t nq, int kk, float *__restrict__ gthr,
                                                                   const int32_t *__restrict__ salist,
                                                                   const uint32_t *__restrict__ pm, int64_t pmK,
                                                                   int pmB) {
    constexpr int GB_Q = gb_q(M), W = M / 4, NP = GB_Q / 2, H = lut_halves(M), LQF = lut_q_floats(M);
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t q0 = (int64_t)blockIdx.x * GB_Q;
    const int G = (int)(ns / gsz);
    auto qidx = [&](int qq) { return min(q0 + qq, nq - 1); };
#pragma unroll
    for (int p = 0; p < NP; ++p)
        load_lut_pair_h<M>(reinterpret_cast<float *>(smem + p * H * LUT_PAIR_BYTES), tables + qidx(2 * p) * LQF,
                           tables + qidx(2 * p + 1) * LQF);
    __syncthreads();
    // half-warp columns (see scan_fast_kernel): lane l reads column (l mod 16) ^ j for M >= 32
    const uint32_t lr = M >= 32 ? ((uint32_t)lane & 15u) : (uint32_t)lane;
    const uint32_t r = lr & (M - 1), rw = r >> 2, l8 = lr << 3;
    uint32_t sel[4];
    make_selectors(r, sel);
    // groups g = tid, tid + NT, ...; per group the min over its gsz codes
    float gmin[2][GB_Q];
    const int ng = (G + GB_NT - 1) / GB_NT;  // <= 2 (G <= 1024)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int qq = 0; qq < GB_Q; ++qq) gmin[h][qq] = __int_as_float(0x7f800000);
    for (int h = 0; h < ng && h < 2; ++h) {
        const int g = tid + h * GB_NT;
        if (g >= G) continue;
        const uint8_t *gp = samp + (int64_t)g * gsz * M;
        uint32_t wn[W];
        load_code<W>(gp, wn);  // the next code is loaded while the current one is summed
        // probe mask (masked IVF): the sample code's list, the mask words of the CTA's
        // first and last query (GB_Q consecutive queries span at most two batches)
        const int64_t b0 = qidx(0) / max(pmB, 1), b1 = qidx(GB_Q - 1) / max(pmB, 1);
        int32_t lst_n = salist ? __ldg(salist + (int64_t)g * gsz) : 0;
        for (int i = 0; i < gsz; ++i) {
            uint32_t w[W];
#pragma unroll
            for (int k = 0; k < W; ++k) w[k] = wn[k];
            const int32_t lst = lst_n;
            if (i + 1 < gsz) {
                load_code<W>(gp + (int64_t)(i + 1) * M, wn);
                if (salist) lst_n = __ldg(salist + (int64_t)g * gsz + i + 1);
            }
            uint32_t m0 = 0xffffffffu, m1 = 0xffffffffu;
            if (salist) {
                m0 = __ldg(pm + b0 * pmK + lst);
                m1 = b1 == b0 ? m0 : __ldg(pm + b1 * pmK + lst);
            }
            float2 acc[NP];
            adc_rotated<M, GB_Q, M >= 32 ? 4 : 8>(smem, w, rw, sel, l8, acc);
            auto probed = [&](int qq) -> bool {
                if (!salist) return true;
                const int64_t qg = qidx(qq);
                return ((qg / pmB == b0 ? m0 : m1) >> (qg % pmB)) & 1u;
            };
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                if (probed(2 * p)) gmin[h][2 * p] = fminf(gmin[h][2 * p], acc[p].x);
                if (probed(2 * p + 1)) gmin[h][2 * p + 1] = fminf(gmin[h][2 * p + 1], acc[p].y);
            }
        }
    }
    __syncthreads();  // tables no longer needed: reuse smem for the sort keys
    uint64_t *keys = reinterpret_cast<uint64_t *>(smem);  // [GB_Q][1024]
    for (int e = tid; e < GB_Q * 1024; e += GB_NT) keys[e] = KEY_MAX;
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int g = tid + h * GB_NT;
        if (g >= G) continue;
#pragma unroll
        for (int qq = 0; qq < GB_Q; ++qq) keys[qq * 1024 + g] = make_key(gmin[h][qq], (uint32_t)g);
    }
    __syncthreads();
    bitonic_sort_rows(keys, GB_Q, 1024, 1024);
    if (tid < GB_Q && q0 + tid < nq) {
        const uint64_t k = keys[tid * 1024 + kk - 1];
        // rotated fp32 order differs from CA2 by < 4e-6 relative: inflate to bound it
        gthr[q0 + tid] = k == KEY_MAX ? __int_as_float(0x7f800000) : __fmul_ru(key_dist(k), 1.00001f);
    }
}

// List-major bound items (IVF, before the integer items): a work item = (posting
// list, <= GB_Q of the queries whose nearest lists it is).  The list's codes are cut
// into G <= 1024 groups of gsz consecutive members; the kk-th smallest group minimum
// of a query is a distance that at least kk members reach (kk distinct groups), so
// it bounds the query's kk-th distance over any superset of the list -- the whole
// probed set.  Lane-rotated fp32 sums, inflated by 1e-5 as in group_min_bound_kernel;
// published with atomicMin (non-negative floats order as ints).  A list shorter
// than kk bounds nothing on its own and is skipped.
template <int M>
__global__ void __launch_bounds__(GB_NT, 1) list_bound_kernel(const uint8_t *__restrict__ codes,
                                                              const int4 *__restrict__ items,
                                                              const int64_t *__restrict__ offsets,
                                                              const uint32_t *__restrict__ ids,
                                                              const uint32_t *__restrict__ qlist, int64_t P,
                                                              const float *__restrict__ tables, int kk,
                                                              float *__restrict__ gthr) {
    constexpr int GB_Q = gb_q(M), W = M / 4, NP = GB_Q / 2, H = lut_halves(M), LQF = lut_q_floats(M);
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int4 it = items[blockIdx.x];
    const int64_t beg = offsets[it.x], len = offsets[it.x + 1] - beg;
    const int nqi = it.z;
    if (len < kk || nqi <= 0) return;  // block-uniform
    auto qidx = [&](int qq) -> int64_t { return (int64_t)(qlist[it.y + (qq < nqi ? qq : nqi - 1)] / P); };
#pragma unroll
    for (int p = 0; p < NP; ++p)
        load_lut_pair_h<M>(reinterpret_cast<float *>(smem + p * H * LUT_PAIR_BYTES), tables + qidx(2 * p) * LQF,
                           tables + qidx(2 * p + 1) * LQF);
    __syncthreads();
    // half-warp columns (see scan_fast_kernel): lane l reads column (l mod 16) ^ j for M >= 32
    const uint32_t lr = M >= 32 ? ((uint32_t)lane & 15u) : (uint32_t)lane;
    const uint32_t r = lr & (M - 1), rw = r >> 2, l8 = lr << 3;
    uint32_t sel[4];
    make_selectors(r, sel);
    const int gsz = (int)((len + 1023) / 1024), G = (int)((len + gsz - 1) / gsz);
    float gmin[2][GB_Q];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int qq = 0; qq < GB_Q; ++qq) gmin[h][qq] = __int_as_float(0x7f800000);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int g = tid + h * GB_NT;
        if (g >= G) continue;
        const int64_t p0 = beg + (int64_t)g * gsz, p1 = min(p0 + gsz, beg + len);
        uint32_t wn[W];
        load_code<W>(codes + (size_t)__ldg(ids + p0) * M, wn);
        for (int64_t p = p0; p < p1; ++p) {
            uint32_t w[W];
#pragma unroll
            for (int k = 0; k < W; ++k) w[k] = wn[k];
            if (p + 1 < p1) load_code<W>(codes + (size_t)__ldg(ids + p + 1) * M, wn);
            float2 acc[NP];
            adc_rotated<M, GB_Q, M >= 32 ? 4 : 8>(smem, w, rw, sel, l8, acc);
#pragma unroll
            for (int q2 = 0; q2 < NP; ++q2) {
                gmin[h][2 * q2] = fminf(gmin[h][2 * q2], acc[q2].x);
                gmin[h][2 * q2 + 1] = fminf(gmin[h][2 * q2 + 1], acc[q2].y);
            }
        }
    }
    __syncthreads();  // tables no longer needed: reuse smem for the sort keys
    uint64_t *keys = reinterpret_cast<uint64_t *>(smem);  // [GB_Q][1024]
    for (int e = tid; e < GB_Q * 1024; e += GB_NT) keys[e] = KEY_MAX;
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int g = tid + h * GB_NT;
        if (g >= G) continue;
#pragma unroll
        for (int qq = 0; qq < GB_Q; ++qq) keys[qq * 1024 + g] = make_key(gmin[h][qq], (uint32_t)g);
    }
    __syncthreads();
    bitonic_sort_rows(keys, GB_Q, 1024, 1024);
    if (tid < nqi) {
        const uint64_t k = keys[tid * 1024 + kk - 1];
        if (k != KEY_MAX)
            atomicMin(reinterpret_cast<int *>(gthr + qidx(tid)), __float_as_int(__fmul_ru(key_dist(k), 1.00001f)));
    }
}

int list_bound_B(int M) { return gb_q(M); }

void launch_list_bound(const uint8_t *codes, int M, const int4 *items, int64_t n_items, const int64_t *offsets,
                       const uint32_t *ids, const uint32_t *qlist, int64_t P, const float *tables, int kk,
                       float *gthr, cudaStream_t st) {
    if (n_items <= 0) return;
    const int GB_Q = gb_q(M);
    const size_t smem = std::max<size_t>((size_t)(GB_Q / 2) * lut_halves(M) * LUT_PAIR_BYTES, (size_t)GB_Q * 1024 * 8);
    check_code_align(codes, M);
    switch (M) {
#define RII_LB(MM)                                                                                                 \
    case MM:                                                                                                       \
        RII_CUDA(cudaFuncSetAttribute(list_bound_kernel<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                                      SMEM_ATTR_MAX));                                                                 \
        list_bound_kernel<MM><<<(unsigned)n_items, GB_NT, smem, st>>>(codes, items, offsets, ids, qlist, P, tables,  \
                                                                      kk, gthr);                                   \
        break;
        RII_LB(4) RII_LB(8) RII_LB(16) RII_LB(32) RII_LB(64)
#undef RII_LB
        default: throw Error(1, "list bound: M outside the fast set");
    }
    RII_LAUNCHED();
}

void launch_group_min_bound(const uint8_t *samp, int64_t ns, int M, const float *tables, int64_t nq, int kk,
                            float *gthr, cudaStream_t st, const ProbeMask &mask) {
    if (nq <= 0) return;
    const int gsz = (int)std::max<int64_t>(1, ceil_div(ns, 1024));  // G = ns / gsz <= 1024 groups
    const int GB_Q = gb_q(M);
    const size_t smem = std::max<size_t>((size_t)(GB_Q / 2) * lut_halves(M) * LUT_PAIR_BYTES, (size_t)GB_Q * 1024 * 8);
    const unsigned grid = (unsigned)ceil_div(nq, GB_Q);
    check_code_align(samp, M);
    switch (M) {
#define RII_GB(MM)                                                                                                 \
    case MM:                                                                                                       \
        RII_CUDA(cudaFuncSetAttribute(group_min_bound_kernel<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                      SMEM_ATTR_MAX));                                                                 \
        group_min_bound_kernel<MM><<<grid, GB_NT, smem, st>>>(samp, ns, gsz, tables, nq, kk, gthr, mask.alist,     \
                                                              mask.pm, mask.K, mask.B);                            \
        break;
        RII_GB(4) RII_GB(8) RII_GB(16) RII_GB(32) RII_GB(64)
#undef RII_GB
        default: throw Error(1, "group-minimum bound: fast M only");
    }
    RII_LAUNCHED();
}

// bound[q] = distance of the kk-th key of keys[q][kk] (+inf when the list is short).
__global__ void kth_bound_kernel(const uint64_t *__restrict__ keys, int64_t nq, int kk, float *__restrict__ bound) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint64_t k = keys[q * kk + kk - 1];
    bound[q] = k == KEY_MAX ? __int_as_float(0x7f800000) : key_dist(k);
}

void launch_kth_bound(const uint64_t *keys, int64_t nq, int kk, float *bound, cudaStream_t st) {
    if (nq <= 0) return;
    kth_bound_kernel<<<(unsigned)ceil_div(nq, 256), 256, 0, st>>>(keys, nq, kk, bound);
    RII_LAUNCHED();
}

// Per-query u16 tables (lut.cuh q16 entries) from the fp32 tables and the current
// bounds: scale[q] = CAP / gthr[q] (rounded down), out[q] = q16(tables[q]).
template <int M>
__global__ void __launch_bounds__(256) q16_tables_kernel(const float *__restrict__ tables, const float *__restrict__ gthr,
                                                         int64_t nq, uint16_t *__restrict__ out, float *__restrict__ scale) {
    const int64_t q = blockIdx.x;
    const float s = __fdiv_rd((float)q16_cap<M>(), fmaxf(__ldcg(gthr + q), 1e-30f));
    if (threadIdx.x == 0) scale[q] = s;
    const float cap = (float)q16_cap<M>();
    const float4 *t4 = reinterpret_cast<const float4 *>(tables + q * LUT_Q_FLOATS);
    uint2 *o = reinterpret_cast<uint2 *>(out + q * LUT_Q_FLOATS);
    for (int e = threadIdx.x; e < LUT_Q_FLOATS / 4; e += blockDim.x) {
        const float4 v = __ldg(t4 + e);
        o[e] = make_uint2(q16_entry(v.x, s, cap) | (q16_entry(v.y, s, cap) << 16),
                          q16_entry(v.z, s, cap) | (q16_entry(v.w, s, cap) << 16));
    }
}

// Per-query u6 tables (lut.cuh u6 entries, bytes [z][32]) at scale 63 * alpha / gthr[q].
template <int M>
__global__ void __launch_bounds__(256) u6_tables_kernel(const float *__restrict__ tables, const float *__restrict__ gthr,
                                                        int64_t nq, uint8_t *__restrict__ out, float *__restrict__ scale,
                                                        float amul, float cap) {
    const int64_t q = blockIdx.x;
    const float s = __fdiv_rd(cap * u6_alpha(M) * amul, fmaxf(__ldcg(gthr + q), 1e-30f));
    if (threadIdx.x == 0) scale[q] = s;
    const float4 *t4 = reinterpret_cast<const float4 *>(tables + q * lut_q_floats(M));
    uint32_t *o = reinterpret_cast<uint32_t *>(out + q * lut_q_floats(M));
    for (int e = threadIdx.x; e < lut_q_floats(M) / 4; e += blockDim.x) {
        const float4 v = __ldg(t4 + e);
        o[e] = u6_entry(v.x, s, cap) | (u6_entry(v.y, s, cap) << 8) | (u6_entry(v.z, s, cap) << 16) |
               (u6_entry(v.w, s, cap) << 24);
    }
}

void launch_u6_tables(const float *tables, const float *gthr, int64_t nq, int M, uint8_t *out, float *scale,
                      cudaStream_t st, bool u7) {
    const float cap = u7 ? 127.f : 63.f;
    if (nq <= 0) return;
    // list items' saturation scale multiplier (RII_U6_LIST_AMUL, A/B): the phase-A bound is tight
    const char *e = getenv("RII_U6_LIST_AMUL");
    const float amul = e ? (float)atof(e) : 1.0f;
    switch (M) {
        case 4: u6_tables_kernel<4><<<(unsigned)nq, 256, 0, st>>>(tables, gthr, nq, out, scale, amul, cap); break;
        case 8: u6_tables_kernel<8><<<(unsigned)nq, 256, 0, st>>>(tables, gthr, nq, out, scale, amul, cap); break;
        case 16: u6_tables_kernel<16><<<(unsigned)nq, 256, 0, st>>>(tables, gthr, nq, out, scale, amul, cap); break;
        case 64: u6_tables_kernel<64><<<(unsigned)nq, 256, 0, st>>>(tables, gthr, nq, out, scale, amul, cap); break;
        default: u6_tables_kernel<32><<<(unsigned)nq, 256, 0, st>>>(tables, gthr, nq, out, scale, amul, cap); break;
    }
    RII_LAUNCHED();
}

void launch_q16_tables(const float *tables, const float *gthr, int64_t nq, int M, uint16_t *out, float *scale,
                       cudaStream_t st) {
    if (nq <= 0) return;
    switch (M) {
        case 4: q16_tables_kernel<4><<<(unsigned)nq, 256, 0, st>>>(tables, gthr, nq, out, scale); break;
        case 8: q16_tables_kernel<8><<<(unsigned)nq, 256, 0, st>>>(tables, gthr, nq, out, scale); break;
        case 16: q16_tables_kernel<16><<<(unsigned)nq, 256, 0, st>>>(tables, gthr, nq, out, scale); break;
        default: q16_tables_kernel<32><<<(unsigned)nq, 256, 0, st>>>(tables, gthr, nq, out, scale); break;
    }
    RII_LAUNCHED();
}

// ---------------------------------------------------------------- gather ---
__global__ void gather_codes_kernel(const uint8_t *__restrict__ codes, int M, const int64_t *__restrict__ pos,
                                    int64_t n, uint8_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t *src = codes + pos[i] * M;
    uint8_t *dst = out + i * M;
    if ((M & 3) == 0) {
        for (int b = 0; b < M; b += 4)
            *reinterpret_cast<uint32_t *>(dst + b) = __ldg(reinterpret_cast<const uint32_t *>(src + b));
    } else {
        for (int b = 0; b < M; ++b) dst[b] = src[b];
    }
}

void launch_gather_codes(const uint8_t *codes, int M, const int64_t *pos, int64_t n, uint8_t *out, cudaStream_t st) {
    if (n <= 0) return;
    gather_codes_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(codes, M, pos, n, out);
    RII_LAUNCHED();
}

__global__ void validate_targets_kernel(const int64_t *__restrict__ ids, int64_t n, int64_t N, int *flag) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t v = ids[i];
    if (v < 0 || v >= N || (i > 0 && v <= ids[i - 1])) atomicOr(flag, 1);
}

void launch_validate_targets(const int64_t *ids, int64_t n, int64_t N, int *flag, cudaStream_t st) {
    if (n <= 0) return;
    validate_targets_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(ids, n, N, flag);
    RII_LAUNCHED();
}

// ----------------------------------------------------------------- merge ---
__global__ void __launch_bounds__(NT) merge_kernel(const uint64_t *__restrict__ keys, int64_t q_stride,
                                                   int64_t p_stride, int parts, int kk, int topk, IdMap map,
                                                   int64_t *__restrict__ out_ids, float *__restrict__ out_dist,
                                                   uint64_t *__restrict__ out_keys, Rescore rs) {
    extern __shared__ __align__(16) uint64_t msm[];
    uint64_t *top = msm, *prt = msm + kk;
    const int64_t q = blockIdx.x;
    const uint64_t *base = keys + q * q_stride;
    uint64_t *first = prt + kk;  // every part's first key, loaded in one round trip
    RII_SMEM_CHECK(msm, first + parts);
    for (int i = threadIdx.x; i < kk; i += blockDim.x) top[i] = KEY_MAX;
    for (int p = threadIdx.x; p < parts; p += blockDim.x) first[p] = __ldg(base + (int64_t)p * p_stride);
    __syncthreads();
    for (int p = 0; p < parts; ++p) {
        // A part whose smallest key (its first: parts are sorted ascending) is not below
        // the current kk-th key cannot change the list: the block skips it without a
        // barrier (top is final since the last barrier).  An empty part may hold only
        // its first key (KEY_MAX; list items write no more).
        const uint64_t *src = base + (int64_t)p * p_stride;
        if (first[p] >= top[kk - 1]) continue;
        for (int i = threadIdx.x; i < kk; i += blockDim.x) prt[i] = src[i];
        __syncthreads();
        for (int i = threadIdx.x; i < kk; i += blockDim.x) {
            const uint64_t v = prt[kk - 1 - i];
            if (v < top[i]) top[i] = v;
        }
        __syncthreads();
        bitonic_merge_rows(top, 1, kk, kk);
    }
    if (rs.tables) {  // canonical (CA2) rescore from the query's HBM table, then re-sort
        const float *tq = rs.tables + q * lut_q_floats(rs.M);
        for (int i = threadIdx.x; i < kk; i += blockDim.x) {
            const uint64_t k = top[i];
            if (k == KEY_MAX) continue;
            const uint32_t id = key_id(k);
            const uint8_t *cp = rs.codes + (size_t)id * rs.M;
            // CA2 in m order; the code bytes and 16 entries at a time are loaded before
            // their adds (a rolled loop serialises two dependent loads per subspace)
            float d = 0.f;
            for (int m0 = 0; m0 < rs.M; m0 += 16) {
                uint32_t cw[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) cw[j] = m0 + 4 * j < rs.M ? __ldg(reinterpret_cast<const uint32_t *>(cp + m0) + j) : 0u;
                float v[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    v[j] = m0 + j < rs.M ? lut_q_entry(tq, m0 + j, (cw[j >> 2] >> (8 * (j & 3))) & 255u) : 0.f;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (m0 + j < rs.M) d = __fadd_rn(d, v[j]);
            }
            top[i] = make_key(d, id);
        }
        __syncthreads();
        bitonic_sort_rows(top, 1, kk, kk);
    }
    if (out_keys) {
        for (int i = threadIdx.x; i < kk; i += blockDim.x) {
            const uint64_t k = top[i];
            out_keys[q * kk + i] = k == KEY_MAX ? KEY_MAX : make_key(key_dist(k), (uint32_t)map_id(map, key_id(k)));
        }
    } else {
        for (int i = threadIdx.x; i < topk; i += blockDim.x) {
            const uint64_t k = top[i];
            out_ids[q * topk + i] = k == KEY_MAX ? -1 : map_id(map, key_id(k));
            out_dist[q * topk + i] = k == KEY_MAX ? __int_as_float(0x7f800000) : key_dist(k);
        }
    }
}

void launch_merge(const uint64_t *keys, int64_t q_stride, int64_t p_stride, int parts, int64_t nq, int kk, int topk,
                  const IdMap &map, int64_t *out_ids, float *out_dist, uint64_t *out_keys, cudaStream_t st,
                  const Rescore &rs) {
    if (nq <= 0) return;
    KernelTimer t(TK_MERGE, st);
    const size_t smem = (size_t)(2 * kk + parts) * 8;
    if (smem > 48 * 1024) RII_CUDA(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    merge_kernel<<<(unsigned)nq, NT, smem, st>>>(keys, q_stride, p_stride, parts, kk, topk, map,
                                                               out_ids, out_dist, out_keys, rs);
    RII_LAUNCHED();
}

#endif  // !RII_SCAN_M

#ifdef RII_SCAN_M  // per-M translation unit: the scan kernels of one M (build.py compiles k_scan.cu once per M)
template void launch_fast_m<RII_SCAN_M>(const ScanPlan &, const uint8_t *, int64_t, const float *, int64_t, const float *,
                                        int, int, uint64_t *, cudaStream_t, const float *, float *, bool, int,
                                        const ProbeMask &);
template void launch_list_m<RII_SCAN_M>(int, const ScanArgs &, int64_t, cudaStream_t, bool);
template void assign_scan_m<RII_SCAN_M>(const uint8_t *, int64_t, const uint8_t *, int64_t, const float *, int32_t *,
                                        float *, cudaStream_t);
#endif

}  // namespace rii
