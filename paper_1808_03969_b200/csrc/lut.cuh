// lut.cuh -- the lane-rotated, bank-conflict-free ADC table of a query pair
// (DESIGN.md §6 "Linear scan").  256 rows (code word z) x 32 columns x 2 queries:
// fp32 word z*64 + 2*c + h holds A_h(c mod M, z) for query h of the pair, so one
// LDS.64 returns the entries of both queries and one packed FADD2 adds them.
// Lane l reads column c = l ^ j at step j: 32 distinct columns -> every 16-lane
// half-warp covers 32 distinct banks whatever the code bytes are.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"

namespace rii {

constexpr int LUT_PAIR_BYTES = 256 * 256;

// Build the table of queries q0, q1 (global memory) from the code book (CA1).
template <int M>
__device__ __forceinline__ void build_lut_pair(float *lutp, const float *q0, const float *q1,
                                               const float *__restrict__ cb, int ds) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int m = lane & (M - 1);
    for (int z = warp; z < KS; z += nwarps) {
        const float *cv = cb + ((size_t)m * KS + z) * ds;
        float a0 = 0.f, a1 = 0.f;
        for (int j = 0; j < ds; ++j) {
            const float c = cv[j];
            a0 = ca1_step(a0, q0[m * ds + j], c);
            a1 = ca1_step(a1, q1[m * ds + j], c);
        }
        reinterpret_cast<float2 *>(lutp)[z * 32 + lane] = make_float2(a0, a1);
    }
}

// Per-query table in HBM (built once per call by lut_tables_kernel): row z holds
// 32 fp32 columns, column c = A(c mod M, z).  32 KB per query for every M <= 32.
// M = 64 (the paper's SIFT1M shape) uses H = 2 such halves, half h holding
// subspaces 32h .. 32h+31: every table (HBM and shared) is H consecutive halves.
constexpr int LUT_Q_FLOATS = KS * 32;
__host__ __device__ constexpr int lut_halves(int M) { return M > 32 ? M / 32 : 1; }
__host__ __device__ constexpr int lut_q_floats(int M) { return LUT_Q_FLOATS * lut_halves(M); }

// Copy the HBM tables of queries qa, qb into the interleaved pair layout:
// coalesced 16-byte loads, 16-byte conflict-free stores.
__device__ __forceinline__ void load_lut_pair(float *lutp, const float *__restrict__ ta,
                                              const float *__restrict__ tb) {
    const float4 *a4 = reinterpret_cast<const float4 *>(ta), *b4 = reinterpret_cast<const float4 *>(tb);
    float4 *d4 = reinterpret_cast<float4 *>(lutp);
    // 8 independent 16-byte loads in flight per thread before the stores (the copy is
    // latency-bound otherwise: one CTA per SM waits on it before scanning)
    constexpr int UNR = 4;
    for (int e0 = threadIdx.x; e0 < LUT_Q_FLOATS / 4; e0 += UNR * blockDim.x) {
        float4 a[UNR], b[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < LUT_Q_FLOATS / 4) { a[u] = __ldg(a4 + e); b[u] = __ldg(b4 + e); }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < LUT_Q_FLOATS / 4) {
                d4[2 * e] = make_float4(a[u].x, b[u].x, a[u].y, b[u].y);
                d4[2 * e + 1] = make_float4(a[u].z, b[u].z, a[u].w, b[u].w);
            }
        }
    }
}

// Pair table of M subspaces (H halves): half h of each query's HBM table -> half h.
template <int M>
__device__ __forceinline__ void load_lut_pair_h(float *lutp, const float *__restrict__ ta,
                                                const float *__restrict__ tb) {
#pragma unroll
    for (int h = 0; h < lut_halves(M); ++h)
        load_lut_pair(lutp + h * (LUT_PAIR_BYTES / 4), ta + h * LUT_Q_FLOATS, tb + h * LUT_Q_FLOATS);
}

// Canonical (replica 0) entry A_h(m, z) of the pair table (halves of 64 KB for M = 64).
__device__ __forceinline__ float lut_pair_entry(const float *lutp, int h, int m, int z) {
    return lutp[(m >> 5) * (LUT_PAIR_BYTES / 4) + z * 64 + 2 * (m & 31) + h];
}

// Entry A(m, z) of a per-query HBM table (lut_tables_kernel layout, H halves).
__device__ __forceinline__ float lut_q_entry(const float *tq, int m, int z) {
    return __ldg(tq + (m >> 5) * LUT_Q_FLOATS + z * 32 + (m & 31));
}

// Packed fp32x2 add (sm_100 FADD2): two IEEE round-to-nearest fp32 adds.
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rc;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rc, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rc;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}

// XOR-permute the code words by the lane's rotation: wp[i] = w[i ^ rw] (rw < 8:
// for M = 64 the rotation stays inside each 32-subspace half).
// (LIM = 4: rw < 4, two select stages -- the half-warp column scheme of adc_u6)
template <int W, int LIM = 8>
__device__ __forceinline__ void permute_words(uint32_t (&w)[W], uint32_t rw) {
#pragma unroll
    for (int b = 1; b < W && b < LIM; b <<= 1) {
        const bool c = (rw & b) != 0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            if (i & b) continue;
            const uint32_t x = w[i], y = w[i | b];
            w[i] = c ? y : x;
            w[i | b] = c ? x : y;
        }
    }
}

// PRMT selectors: byte0 <- b-operand byte 0 (the column offset), byte1 <- code byte
// ((t ^ r) & 3) of the word, bytes 2-3 <- 0.  Result = (z << 8) | col_offset.
__device__ __forceinline__ void make_selectors(uint32_t r, uint32_t (&sel)[4]) {
#pragma unroll
    for (int t = 0; t < 4; ++t) sel[t] = 0x5504u | ((((uint32_t)t ^ r) & 3u) << 4);
}

// Lane-rotated ADC of one code (M bytes in w) against the B tables of the CTA:
// per step j one PRMT builds (z << 8) | 8*(l ^ j); per query pair one LDS.64 +
// one FADD2.
// `wp` = the code words already permuted by permute_words (lane rotation).
template <int M, int B>
__device__ __forceinline__ void adc_rotated_pre(const uint8_t *lut, const uint32_t (&wp)[M / 4],
                                                const uint32_t (&sel)[4], uint32_t l8, float2 (&acc)[B / 2]) {
    constexpr int NP = B / 2, H = lut_halves(M);
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const uint32_t off = __byte_perm(wp[j >> 2], l8 ^ (uint32_t)((j & 31) << 3), sel[j & 3]);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float2 v = *reinterpret_cast<const float2 *>(lut + (p * H + (j >> 5)) * LUT_PAIR_BYTES + off);
            acc[p] = j == 0 ? v : fadd2(acc[p], v);  // 0 + v == v for v >= +0
        }
    }
}


template <int M, int B, int PLIM = 8>
__device__ __forceinline__ void adc_rotated(const uint8_t *lut, const uint32_t (&w)[M / 4], uint32_t rw,
                                            const uint32_t (&sel)[4], uint32_t l8, float2 (&acc)[B / 2]) {
    constexpr int W = M / 4;
    uint32_t wp[W];
#pragma unroll
    for (int i = 0; i < W; ++i) wp[i] = w[i];
    permute_words<W, PLIM>(wp, rw);
    adc_rotated_pre<M, B>(lut, wp, sel, l8, acc);
}

// ---- bf16-packed quad tables (4 queries per 8-byte column) ------------------
// Word 0 of column c in row z = trunc_bf16(A) << 16 | rn_bf16(C), word 1 = the same
// for (B, D).  Read raw as fp32, the high halves give A and B with the low 16
// mantissa bits as noise; shifted left by 16 the low halves give C and D exactly
// as bf16.  Every approximate table value lies within 2^-7 relative of the fp32
// entry, so an approximate ADC sum is within 2^-7 (+ fp32 rounding) of the
// canonical one: the kernels filter with the threshold relaxed by PACK_SLACK and
// rescore every pushed candidate canonically before it can enter a top list.
constexpr int QUAD_BYTES = 256 * 256;
constexpr float PACK_SLACK = 1.008f;  // > (1 + 2^-7) (1 + 1e-5)

__device__ __forceinline__ void load_lut_quad(uint32_t *dst, const float *__restrict__ ta,
                                              const float *__restrict__ tb, const float *__restrict__ tc,
                                              const float *__restrict__ td) {
    const float4 *a4 = reinterpret_cast<const float4 *>(ta), *b4 = reinterpret_cast<const float4 *>(tb);
    const float4 *c4 = reinterpret_cast<const float4 *>(tc), *d4 = reinterpret_cast<const float4 *>(td);
    uint4 *o = reinterpret_cast<uint4 *>(dst);
    auto hi = [](float v) { return __float_as_uint(v) & 0xffff0000u; };
    auto lo = [](float v) { return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v)); };
    constexpr int UNR = 2;  // 8 independent 16-byte loads in flight per thread
    for (int e0 = threadIdx.x; e0 < LUT_Q_FLOATS / 4; e0 += UNR * blockDim.x) {
        float4 A[UNR], B[UNR], C[UNR], D[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < LUT_Q_FLOATS / 4) { A[u] = __ldg(a4 + e); B[u] = __ldg(b4 + e); C[u] = __ldg(c4 + e); D[u] = __ldg(d4 + e); }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e >= LUT_Q_FLOATS / 4) continue;
            o[2 * e] = make_uint4(hi(A[u].x) | lo(C[u].x), hi(B[u].x) | lo(D[u].x), hi(A[u].y) | lo(C[u].y),
                                  hi(B[u].y) | lo(D[u].y));
            o[2 * e + 1] = make_uint4(hi(A[u].z) | lo(C[u].z), hi(B[u].z) | lo(D[u].z), hi(A[u].w) | lo(C[u].w),
                                      hi(B[u].w) | lo(D[u].w));
        }
    }
}

// SDC-mode quad: the table of a PQ code x is T_m[x^m][z] (column c = m = c mod M).
template <int M>
__device__ __forceinline__ void load_lut_quad_sdc(uint32_t *dst, const float *__restrict__ T,
                                                  const uint8_t *__restrict__ xa, const uint8_t *__restrict__ xb,
                                                  const uint8_t *__restrict__ xc, const uint8_t *__restrict__ xd) {
    uint4 *o = reinterpret_cast<uint4 *>(dst);
    auto hi = [](float v) { return __float_as_uint(v) & 0xffff0000u; };
    auto lo = [](float v) { return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v)); };
    auto val = [&](const uint8_t *x, int c, int z) {
        const int m = c & (M - 1);
        return __ldg(T + ((size_t)m * KS + __ldg(x + m)) * KS + z);
    };
    for (int e = threadIdx.x; e < LUT_Q_FLOATS / 4; e += blockDim.x) {
        const int z = e >> 3, c0 = (e & 7) * 4;
        uint32_t w[8];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int c = c0 + t;
            w[2 * t] = hi(val(xa, c, z)) | lo(val(xc, c, z));
            w[2 * t + 1] = hi(val(xb, c, z)) | lo(val(xd, c, z));
        }
        o[2 * e] = make_uint4(w[0], w[1], w[2], w[3]);
        o[2 * e + 1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
}

// Approximate lane-rotated ADC of one pre-loaded code against NQ quad tables:
// per step j one PRMT, per quad one LDS.64, two unpacks and two FADD2 (4 lookups).
// VARIANT bit 0: unpack the low halves with PRMT (ALU pipe) instead of a shift
// (lowered to IMAD on the FMA pipe); bit 1: recompute the column offset l8 ^ 8j per
// step (one LOP) instead of letting the compiler hoist 32 constants into registers.
template <int M, int NQ, int VARIANT>
__device__ __forceinline__ void adc_packed(const uint8_t *lut, const uint32_t (&w)[M / 4], uint32_t rw,
                                           const uint32_t (&sel)[4], uint32_t l8, float2 (&ab)[NQ],
                                           float2 (&cd)[NQ]) {
    constexpr int W = M / 4;
    uint32_t wp[W];
#pragma unroll
    for (int i = 0; i < W; ++i) wp[i] = w[i];
    permute_words<W>(wp, rw);
#pragma unroll
    for (int j = 0; j < M; ++j) {
        uint32_t col;
        if constexpr (VARIANT & 2) asm volatile("xor.b32 %0, %1, %2;" : "=r"(col) : "r"(l8), "r"((uint32_t)(j << 3)));
        else col = l8 ^ (uint32_t)(j << 3);
        const uint32_t off = __byte_perm(wp[j >> 2], col, sel[j & 3]);
#pragma unroll
        for (int p = 0; p < NQ; ++p) {
            const uint2 v = *reinterpret_cast<const uint2 *>(lut + p * QUAD_BYTES + off);
            const float2 x = make_float2(__uint_as_float(v.x), __uint_as_float(v.y));
            float2 y;
            if constexpr (VARIANT & 1)
                y = make_float2(__uint_as_float(__byte_perm(v.x, 0u, 0x1044)), __uint_as_float(__byte_perm(v.y, 0u, 0x1044)));
            else
                y = make_float2(__uint_as_float(v.x << 16), __uint_as_float(v.y << 16));
            ab[p] = j == 0 ? x : fadd2(ab[p], x);
            cd[p] = j == 0 ? y : fadd2(cd[p], y);
        }
    }
}

// ---- u16 fixed-point quad tables (4 queries per 8-byte column, integer SWAR) --
// Entry q(v) = floor(min(v (x)_rd s, CAP)) with a per-query scale s = CAP / T (T an
// upper bound on the query's final kk-th distance, from a sampled exact pass).
// Word 0 of column c in row z = q(A) | q(C) << 16, word 1 = q(B) | q(D) << 16.
// CAP = floor(65535 / M), so a 16-bit lane holding the sum of M entries never
// carries into its neighbour: one IADD3 adds two lookups of two queries.
// Since q(v) <= v*s (real), sum_m q <= s * d_exact (1 + M 2^-24): a code whose
// exact distance is <= thr has quantised sum <= floor(s (x)_ru thr (x)_ru (1 + 2^-16)),
// so the integer filter never drops a candidate that can enter the exact top list
// (every pushed candidate is rescored canonically before compaction).
template <int M>
__host__ __device__ constexpr uint32_t q16_cap() { return 65535u / (uint32_t)M; }

__device__ __forceinline__ uint32_t q16_entry(float v, float s, float cap) {
    return __float2uint_rd(fminf(__fmul_rd(v, s), cap));
}

// Integer threshold of an fp32 distance threshold t (+inf -> pass everything).
__device__ __forceinline__ uint32_t q16_threshold(float t, float s) {
    const float x = __fmul_ru(__fmul_ru(t, s), 1.0000153f);  // (1 + 2^-16), rounded up
    return x >= 4294967040.f ? 0xffffffffu : __float2uint_rd(x);
}

template <int M>
__device__ __forceinline__ void load_lut_quad_q16(uint32_t *dst, const float *__restrict__ ta,
                                                  const float *__restrict__ tb, const float *__restrict__ tc,
                                                  const float *__restrict__ td, float sa, float sb, float sc,
                                                  float sd) {
    const float4 *a4 = reinterpret_cast<const float4 *>(ta), *b4 = reinterpret_cast<const float4 *>(tb);
    const float4 *c4 = reinterpret_cast<const float4 *>(tc), *d4 = reinterpret_cast<const float4 *>(td);
    uint4 *o = reinterpret_cast<uint4 *>(dst);
    const float cap = (float)q16_cap<M>();
    auto pk = [&](float lo, float slo, float hi, float shi) {
        return q16_entry(lo, slo, cap) | (q16_entry(hi, shi, cap) << 16);
    };
    constexpr int UNR = 2;  // 8 independent 16-byte loads in flight per thread
    for (int e0 = threadIdx.x; e0 < LUT_Q_FLOATS / 4; e0 += UNR * blockDim.x) {
        float4 A[UNR], B[UNR], C[UNR], D[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < LUT_Q_FLOATS / 4) { A[u] = __ldg(a4 + e); B[u] = __ldg(b4 + e); C[u] = __ldg(c4 + e); D[u] = __ldg(d4 + e); }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e >= LUT_Q_FLOATS / 4) continue;
            o[2 * e] = make_uint4(pk(A[u].x, sa, C[u].x, sc), pk(B[u].x, sb, D[u].x, sd), pk(A[u].y, sa, C[u].y, sc),
                                  pk(B[u].y, sb, D[u].y, sd));
            o[2 * e + 1] = make_uint4(pk(A[u].z, sa, C[u].z, sc), pk(B[u].z, sb, D[u].z, sd),
                                      pk(A[u].w, sa, C[u].w, sc), pk(B[u].w, sb, D[u].w, sd));
        }
    }
}

// Quad layout from four precomputed per-query u16 tables ([z][32 columns] u16, as
// written by q16_tables_kernel): column word 0 = A | C << 16, word 1 = B | D << 16.
__device__ __forceinline__ void load_lut_quad_u16(uint32_t *dst, const uint16_t *__restrict__ ta,
                                                  const uint16_t *__restrict__ tb, const uint16_t *__restrict__ tc,
                                                  const uint16_t *__restrict__ td) {
    const uint4 *a4 = reinterpret_cast<const uint4 *>(ta), *b4 = reinterpret_cast<const uint4 *>(tb);
    const uint4 *c4 = reinterpret_cast<const uint4 *>(tc), *d4 = reinterpret_cast<const uint4 *>(td);
    uint4 *o = reinterpret_cast<uint4 *>(dst);
    constexpr int N16 = LUT_Q_FLOATS / 8;  // 16-byte chunks (8 columns) per table
    constexpr int UNR = 2;
    for (int e0 = threadIdx.x; e0 < N16; e0 += UNR * blockDim.x) {
        uint4 A[UNR], B[UNR], C[UNR], D[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < N16) { A[u] = __ldg(a4 + e); B[u] = __ldg(b4 + e); C[u] = __ldg(c4 + e); D[u] = __ldg(d4 + e); }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e >= N16) continue;
            // chunk e = columns 8e'..8e'+7 of one row; output 8 columns x 8 bytes = 4 uint4
            const uint32_t a[4] = {A[u].x, A[u].y, A[u].z, A[u].w}, b[4] = {B[u].x, B[u].y, B[u].z, B[u].w};
            const uint32_t c[4] = {C[u].x, C[u].y, C[u].z, C[u].w}, d[4] = {D[u].x, D[u].y, D[u].z, D[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k)  // word k holds columns 2k (low) and 2k+1 (high)
                o[4 * e + k] = make_uint4(__byte_perm(a[k], c[k], 0x5410), __byte_perm(b[k], d[k], 0x5410),
                                          __byte_perm(a[k], c[k], 0x7632), __byte_perm(b[k], d[k], 0x7632));
        }
    }
}

// ---- u6 fixed-point oct tables (8 queries per 8-byte column) ---------------
// Entry q(v) = floor(min(v (x)_rd s, 63)) with s = 63 * alpha / T, alpha = M / 4 (an
// entry saturates at 4x the mean entry of a code at the threshold): an entry may
// saturate (only ever lowering the sum: q(v) <= v s still holds, so the filter
// Sum q <= floor(s thr (1 + 2^-16)) keeps every code with d <= thr -- saturation
// only adds false positives, which the exact rescore removes).  Four lookups of
// one query add in a byte lane (4 * 63 < 256) before the even / odd bytes are
// widened into 16-bit lanes (M * 63 < 65536): one 128-B wavefront carries 128
// lookups.  Column c of row z = bytes [q0 .. q7] (word 0 = queries 0-3).
__host__ __device__ constexpr float u6_alpha(int M) { return M >= 4 ? M / 4.0f : 1.0f; }
constexpr int OCT_BYTES = 256 * 256;  // 256 rows x 32 columns x 8 B: one table for 8 queries

__device__ __forceinline__ uint32_t u6_entry(float v, float s, float cap) {
    return __float2uint_rd(fminf(__fmul_rd(v, s), cap));
}

// Oct table(s) of 8 queries from their fp32 HBM tables (entries capped at `cap`).
// R2 (M = 32): a second copy 64 KB above the first whose column c holds column
// c ^ 8 (a 256-B row covers the 32 banks twice, so column c ^ 8 is the other half
// of c's bank set), so that lanes 8 apart read disjoint banks with the same word
// index.
template <bool R2, int H = 1>
__device__ __forceinline__ void load_lut_oct_u6(uint32_t *dst, const float *const (&t)[8], const float (&s)[8],
                                                float cap) {
    for (int eh = threadIdx.x; eh < H * LUT_Q_FLOATS / 4; eh += blockDim.x) {  // 4 columns of one row
        const int h = eh / (LUT_Q_FLOATS / 4), e = eh - h * (LUT_Q_FLOATS / 4);
        uint2 *o = reinterpret_cast<uint2 *>(dst) + h * (OCT_BYTES / 8);  // half h: 64 KB further
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(reinterpret_cast<const float4 *>(t[k] + h * LUT_Q_FLOATS) + e);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float a = c == 0 ? v[k].x : c == 1 ? v[k].y : c == 2 ? v[k].z : v[k].w;
                const float b = c == 0 ? v[k + 4].x : c == 1 ? v[k + 4].y : c == 2 ? v[k + 4].z : v[k + 4].w;
                lo |= u6_entry(a, s[k], cap) << (8 * k);
                hi |= u6_entry(b, s[k + 4], cap) << (8 * k);
            }
            const int col = 4 * e + c;  // row * 32 + column
            o[col] = make_uint2(lo, hi);
            if constexpr (R2) o[OCT_BYTES / 8 + (col ^ 8)] = make_uint2(lo, hi);
        }
    }
}

// u6 lane-rotated ADC of one code against the oct table: per word index a, the four
// steps' 8-byte loads are summed bytewise, then widened.  acc[0] = queries (0, 2)
// in (low, high) 16-bit lanes, acc[1] = (1, 3), acc[2] = (4, 6), acc[3] = (5, 7).
template <int M, int GJ, bool R2, int BASE = 0, int NO = 1, int PLIM = 8>
__device__ __forceinline__ void adc_u6(const uint32_t (&w)[M / 4], uint32_t rw, const uint32_t (&sel)[4],
                                       const uint32_t (&colv)[M / 4 < 8 ? M / 4 : 8], uint32_t one,
                                       uint32_t (&acc)[4 * NO]);

// Oct layout from 8 precomputed per-query u6 tables ([z][32 columns] bytes, written by
// u6_tables_kernel): column c = [t0[c] .. t7[c]] (an 8 x 8 byte transpose per group of
// 8 columns, 3 PRMT per output word).  R2: the second copy as in load_lut_oct_u6.
template <bool R2, int H = 1, int NTHR = 384>
__device__ __forceinline__ void load_lut_oct_u8pre(uint32_t *dst, const uint8_t *const (&t)[8]) {
    // all loads of a thread are issued before any is used (one L2 round trip, not one
    // per row group): NTHR threads cover the H * 1024 row groups in NIT iterations
    constexpr int NG = H * LUT_Q_FLOATS / 8, NIT = (NG + NTHR - 1) / NTHR;
    uint2 v[NIT][8];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const int eh = (int)threadIdx.x + it * NTHR;
        if (eh < NG) {
            const int h = eh / (LUT_Q_FLOATS / 8), e = eh - h * (LUT_Q_FLOATS / 8);
#pragma unroll
            for (int k = 0; k < 8; ++k) v[it][k] = __ldg(reinterpret_cast<const uint2 *>(t[k] + h * LUT_Q_FLOATS) + e);
        }
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const int eh = (int)threadIdx.x + it * NTHR;
        if (eh >= NG) continue;
        const int h = eh / (LUT_Q_FLOATS / 8), e = eh - h * (LUT_Q_FLOATS / 8);
        uint2 *o = reinterpret_cast<uint2 *>(dst) + h * (OCT_BYTES / 8);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint32_t sc = (uint32_t)(c & 3) | ((uint32_t)(4 + (c & 3)) << 4);  // byte c of a, of b
            auto w_of = [&](int k) { return c < 4 ? v[it][k].x : v[it][k].y; };
            const uint32_t p01 = __byte_perm(w_of(0), w_of(1), sc), p23 = __byte_perm(w_of(2), w_of(3), sc);
            const uint32_t p45 = __byte_perm(w_of(4), w_of(5), sc), p67 = __byte_perm(w_of(6), w_of(7), sc);
            const uint2 col = make_uint2(__byte_perm(p01, p23, 0x5410), __byte_perm(p45, p67, 0x5410));
            const int idx = 8 * e + c;  // row * 32 + column
            o[idx] = col;
            if constexpr (R2) o[OCT_BYTES / 8 + (idx ^ 8)] = col;
        }
    }
}

// a * one + b on the FMA pipe (IMAD): `one` is a runtime 1 the compiler cannot fold,
// which moves the SWAR additions off the integer ALU pipe (the u6 kernel's limiter).
__device__ __forceinline__ uint32_t fma_add(uint32_t a, uint32_t one, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
    return r;
}

// PRMT selectors of the q16 kernel: byte0 <- byte (t & 1) of the column register
// (two column offsets per register), byte1 <- code byte ((t ^ r) & 3) of the
// permuted word, bytes 2-3 <- bytes 2-3 of the column register (table base >> 16).
__device__ __forceinline__ void make_selectors_q16(uint32_t r, uint32_t (&sel)[4]) {
#pragma unroll
    for (int t = 0; t < 4; ++t) sel[t] = 0x7600u | ((((uint32_t)t ^ r) & 3u) << 4) | (4u + ((uint32_t)t & 1u));
}

// 8-byte shared load at address off + IMM (a compile-time offset).
template <int IMM>
__device__ __forceinline__ uint2 lds64_imm(uint32_t off) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+%3];" : "=r"(v.x), "=r"(v.y) : "r"(off), "n"(IMM));
    return v;
}

// 8-byte shared load at address off + p * QUAD_BYTES (p an unrolled constant).
__device__ __forceinline__ uint2 lds64_quad(uint32_t off, int p) {
    uint2 v;
    if (p == 0) asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(off));
    else if (p == 1) asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+65536];" : "=r"(v.x), "=r"(v.y) : "r"(off));
    else if (p == 2) asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+131072];" : "=r"(v.x), "=r"(v.y) : "r"(off));
    else asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+196608];" : "=r"(v.x), "=r"(v.y) : "r"(off));
    return v;
}

// Quantised lane-rotated ADC of one code against NQ u16 quad tables.  colA / colB
// hold the byte offsets 8 (l ^ t) of steps t = 0,1 / 2,3 (bytes 0-1); step
// j = 4a + t reads column (l ^ t) ^ 4a, i.e. the register XOR a * 0x2020.
// acc0[p] = sums of queries (4p, 4p+2) in (low, high) halves; acc1[p] = (4p+1, 4p+3).
template <int M, int NQ>
__device__ __forceinline__ void adc_q16(const uint32_t (&w)[M / 4], uint32_t rw,
                                        const uint32_t (&sel)[4], uint32_t colA, uint32_t colB,
                                        uint32_t (&acc0)[NQ], uint32_t (&acc1)[NQ]) {
    constexpr int W = M / 4;
    uint32_t wp[W];
#pragma unroll
    for (int i = 0; i < W; ++i) wp[i] = w[i];
    permute_words<W>(wp, rw);
    uint2 h[NQ];
#pragma unroll
    for (int aw = 0; aw < W; ++aw) {
        const uint32_t ca = colA ^ (uint32_t)(aw * 0x2020), cb = colB ^ (uint32_t)(aw * 0x2020);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t off = __byte_perm(wp[aw], t < 2 ? ca : cb, sel[t]);
#pragma unroll
            for (int p = 0; p < NQ; ++p) {
                const uint2 v = lds64_quad(off, p);  // off = the complete shared address
                if ((t & 1) == 0) {
                    h[p] = v;
                } else if (aw == 0 && t == 1) {
                    acc0[p] = h[p].x + v.x;
                    acc1[p] = h[p].y + v.y;
                } else {
                    acc0[p] = acc0[p] + h[p].x + v.x;
                    acc1[p] = acc1[p] + h[p].y + v.y;
                }
            }
        }
    }
}

template <int M, int GJ, bool R2, int BASE, int NO, int PLIM>
__device__ __forceinline__ void adc_u6(const uint32_t (&w)[M / 4], uint32_t rw, const uint32_t (&sel)[4],
                                       const uint32_t (&colv)[M / 4 < 8 ? M / 4 : 8], uint32_t one,
                                       uint32_t (&acc)[4 * NO]) {
    // GJ steps (2: 7-bit entries, 4: 6-bit entries, 8: 5-bit entries) are summed bytewise
    // before widening; NO oct tables (8 queries each) 64 KB apart share the offsets of
    // every step
    constexpr int W = M / 4, GW = GJ >= 4 ? GJ / 4 : 1;
    static_assert(W % GW == 0, "word groups");
    uint32_t wp[W];
#pragma unroll
    for (int i = 0; i < W; ++i) wp[i] = w[i];
    if constexpr (R2) {  // rw in {0, 1}: one select stage
        const bool c = rw != 0;
#pragma unroll
        for (int i = 0; i < W; i += 2) {
            const uint32_t x = wp[i], y = wp[i + 1];
            wp[i] = c ? y : x;
            wp[i + 1] = c ? x : y;
        }
    } else {
        permute_words<W, PLIM>(wp, rw);
    }
    auto lds = [&](uint32_t off, int aw, int o) -> uint2 {
        // compile-time immediate: table o (64 KB apart), half aw / 8 (M = 64)
        if constexpr (W <= 8) {
            if constexpr (NO == 1) return lds64_imm<BASE>(off);
            else return o == 0 ? lds64_imm<BASE>(off) : lds64_imm<BASE + 0x10000>(off);
        } else {
            return aw < 8 ? lds64_imm<BASE>(off) : lds64_imm<BASE + 0x10000>(off);
        }
    };
#pragma unroll
    for (int g = 0; g < W / GW; ++g) {
        uint32_t s0[NO], s1[NO];
#pragma unroll
        for (int h = 0; h < GW; ++h) {
            const int aw = g * GW + h;
            const uint32_t ca = colv[aw & 7], cb = ca ^ 0x1010u;  // columns of steps t = 0,1 / 2,3 of group aw
            uint32_t off[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) off[t] = __byte_perm(wp[aw], t < 2 ? ca : cb, sel[t]);
#pragma unroll
            for (int o = 0; o < NO; ++o) {
                uint2 v[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) v[t] = lds(off[t], aw, o);
                if constexpr (GJ == 2) {
                    // 7-bit entries: pairs of steps summed bytewise (2 * 127 < 256), each pair
                    // widened into the 16-bit lanes on its own
                    uint32_t *ac = acc + 4 * o;
#pragma unroll
                    for (int pr = 0; pr < 2; ++pr) {
                        const uint32_t y0 = fma_add(v[2 * pr].x, one, v[2 * pr + 1].x);
                        const uint32_t y1 = fma_add(v[2 * pr].y, one, v[2 * pr + 1].y);
                        const uint32_t e0 = y0 & 0x00ff00ffu, o0 = __byte_perm(y0, 0u, 0x4341);
                        const uint32_t e1 = y1 & 0x00ff00ffu, o1 = __byte_perm(y1, 0u, 0x4341);
                        if (g == 0 && pr == 0) {
                            ac[0] = e0; ac[1] = o0; ac[2] = e1; ac[3] = o1;
                        } else {
                            ac[0] = fma_add(e0, one, ac[0]);
                            ac[1] = fma_add(o0, one, ac[1]);
                            ac[2] = fma_add(e1, one, ac[2]);
                            ac[3] = fma_add(o1, one, ac[3]);
                        }
                    }
                } else {
                    // bytewise (GJ * cap < 256, no carries), as a tree: dependency depth 2
                    const uint32_t x0 = fma_add(fma_add(v[0].x, one, v[1].x), one, fma_add(v[2].x, one, v[3].x));
                    const uint32_t x1 = fma_add(fma_add(v[0].y, one, v[1].y), one, fma_add(v[2].y, one, v[3].y));
                    s0[o] = h == 0 ? x0 : fma_add(x0, one, s0[o]);
                    s1[o] = h == 0 ? x1 : fma_add(x1, one, s1[o]);
                }
            }
        }
        if constexpr (GJ == 2) continue;  // accumulated per pair of steps above
#pragma unroll
        for (int o = 0; o < NO; ++o) {
            const uint32_t e0 = s0[o] & 0x00ff00ffu, o0 = __byte_perm(s0[o], 0u, 0x4341);
            const uint32_t e1 = s1[o] & 0x00ff00ffu, o1 = __byte_perm(s1[o], 0u, 0x4341);
            uint32_t *ac = acc + 4 * o;
            if (g == 0) {
                ac[0] = e0; ac[1] = o0; ac[2] = e1; ac[3] = o1;
            } else {
                ac[0] = fma_add(e0, one, ac[0]);
                ac[1] = fma_add(o0, one, ac[1]);
                ac[2] = fma_add(e1, one, ac[2]);
                ac[3] = fma_add(o1, one, ac[3]);
            }
        }
    }
}

}  // namespace rii
