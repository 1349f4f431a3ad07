// k_ivf.cu -- inverted-index search (Alg. 2 InvertedIndex) on sm_100a.
//
//  coarse_dist   : d0[q][k] = CA2 ADC of q to every centre code cbar_k (L2-L5).
//  select_probes : per query, radix-select the P smallest (d0, k)   (L6, reading R1).
//  ivf_scan      : one CTA per query pair; warps pull (query, list) work items
//                  from a shared counter and stream the list's ids (coalesced)
//                  and codes (16-byte gathers from the linear array),
//                  evaluate ADC with the lane-rotated table of k_scan.cu and keep
//                  the top-kk in shared memory (L7-L16, mode A of reading R2).
#include <algorithm>
#include <cstring>

#include "kernels.cuh"
#include "lut.cuh"
#include "topk.cuh"

namespace rii {

constexpr int CQ = 4;   // queries per CTA in coarse_dist
constexpr int CMC = 32; // subspaces per table chunk in coarse_dist

// d0[q][k] (Alg. 2 L2-L5): CTA = (256 centres, CQ queries); the CA1 table is built
// in chunks of CMC subspaces ([CQ][CMC][256] fp32 in smem), each thread keeps its
// centre's CQ running sums across the chunks, so the sums stay in the canonical m
// order (CA2) for any M (up to 256).
__global__ void __launch_bounds__(NT) coarse_dist_kernel(const uint8_t *__restrict__ centers, int64_t K, int M,
                                                         const float *__restrict__ q, int64_t nq,
                                                         const float *__restrict__ cb, int ds,
                                                         float *__restrict__ d0) {
    extern __shared__ __align__(16) float clut[];  // [CQ][CMC][256]
    const int64_t q0 = (int64_t)blockIdx.y * CQ;
    const int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x;
    const int D = M * ds;
    const uint8_t *cp = centers + min(k, K - 1) * M;
    float acc[CQ];
#pragma unroll
    for (int qq = 0; qq < CQ; ++qq) acc[qq] = 0.f;
    for (int m0 = 0; m0 < M; m0 += CMC) {
        const int mc = min(CMC, M - m0);
        __syncthreads();
        for (int e = threadIdx.x; e < CQ * mc * KS; e += blockDim.x) {
            const int qq = e / (mc * KS), m = (e / KS) % mc, z = e % KS;
            const int64_t qi = min(q0 + qq, nq - 1);
            const float *qv = q + qi * D + (m0 + m) * ds, *cv = cb + ((size_t)(m0 + m) * KS + z) * ds;
            float a = 0.f;
            for (int j = 0; j < ds; ++j) a = ca1_step(a, qv[j], cv[j]);
            clut[(qq * CMC + m) * KS + z] = a;
        }
        __syncthreads();
        if (k < K) {
            for (int m = 0; m < mc; ++m) {
                const int z = cp[m0 + m];
#pragma unroll
                for (int qq = 0; qq < CQ; ++qq) acc[qq] = __fadd_rn(acc[qq], clut[(qq * CMC + m) * KS + z]);
            }
        }
    }
    if (k < K) {
#pragma unroll
        for (int qq = 0; qq < CQ; ++qq)
            if (q0 + qq < nq) d0[(q0 + qq) * K + k] = acc[qq];
    }
}

void launch_coarse_dist(const uint8_t *centers, int64_t K, int M, const float *q, int64_t nq, const float *cb, int D,
                        float *d0, cudaStream_t st) {
    if (nq <= 0 || K <= 0) return;
    const size_t smem = (size_t)CQ * CMC * KS * 4;
    RII_CUDA(cudaFuncSetAttribute(coarse_dist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    dim3 grid((unsigned)ceil_div(K, NT), (unsigned)ceil_div(nq, CQ));
    coarse_dist_kernel<<<grid, NT, smem, st>>>(centers, K, M, q, nq, cb, D / M, d0);
    RII_LAUNCHED();
}

// Block-wide exclusive prefix over a 0/1 flag per thread (NT threads).
__device__ __forceinline__ int block_excl_scan(int flag, int *wsum, int &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < NT / 32; ++w) {
        if (w < warp) off += wsum[w];
        tot += wsum[w];
    }
    __syncthreads();
    total = tot;
    return off + __popc(bal & ((1u << lane) - 1u));
}

// Radix select of the P smallest (d0 bits, k) per query; output in ascending k.
__global__ void __launch_bounds__(NT) select_probes_kernel(const float *__restrict__ d0, int64_t K, int64_t P,
                                                           int32_t *__restrict__ probes) {
    __shared__ int hist[256];
    __shared__ uint32_t s_prefix, s_mask;
    __shared__ int64_t s_rem;
    __shared__ int wsum[NT / 32];
    const int64_t qi = blockIdx.x;
    const uint32_t *u = reinterpret_cast<const uint32_t *>(d0 + qi * K);
    int32_t *outp = probes + qi * P;
    if (P >= K) {  // every list: order does not matter under mode A
        for (int64_t k = threadIdx.x; k < K; k += NT) outp[k] = (int32_t)k;
        return;
    }
    if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_rem = P; }
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        const uint32_t pre = s_prefix, msk = s_mask;
        for (int64_t k = threadIdx.x; k < K; k += NT) {
            const uint32_t v = u[k];
            if ((v & msk) == pre) atomicAdd(&hist[(v >> shift) & 255], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t rem = s_rem, acc = 0;
            int d = 0;
            for (; d < 256; ++d) {
                if (acc + hist[d] >= rem) break;
                acc += hist[d];
            }
            s_rem = rem - acc;
            s_prefix = pre | ((uint32_t)d << shift);
            s_mask = msk | (255u << shift);
        }
        __syncthreads();
    }
    const uint32_t t = s_prefix;
    const int64_t ties = s_rem;  // how many keys equal to t are taken (lowest k first)
    int64_t tie_base = 0, out_base = 0;
    for (int64_t k0 = 0; k0 < K; k0 += NT) {
        const int64_t k = k0 + threadIdx.x;
        const uint32_t v = k < K ? u[k] : 0xffffffffu;
        const int is_tie = (k < K && v == t) ? 1 : 0;
        int ntie;
        const int tie_rank = block_excl_scan(is_tie, wsum, ntie);
        const int take = (k < K && (v < t || (is_tie && tie_base + tie_rank < ties))) ? 1 : 0;
        int ntake;
        const int pos = block_excl_scan(take, wsum, ntake);
        if (take) outp[out_base + pos] = (int32_t)k;
        tie_base += ntie;
        out_base += ntake;
    }
}

// Coarse ranking and probe selection in one kernel (Alg. 2 L2-L6) for the fast-layout M
// (precomputed CA1 tables, lut_tables_kernel, [half][z][32 columns], column c = A(32 h +
// c mod min(M, 32), z)): CTA = one query, thread = centres k.
//  1. Lane-rotated sums: at step j lane l reads column (l + j) mod 32 of its centre's
//     row z, so the 32 lanes of a warp hit 32 distinct banks (no conflicts); a lane's
//     sum runs over the subspaces in a rotated order (not CA2's).
//  2. T = the P-th smallest rotated sum (radix select over the bit patterns, d >= +0).
//  3. Candidates C = {k : d_rot(k) <= T (1 + eps)^2}, eps = 1e-5 >= 2 (M - 1) 2^-24 (the
//     relative gap between any two fp32 summation orders of M non-negative terms,
//     M <= 64): at least P centres have d_rot <= T, hence canonical d0 <= T (1 + eps),
//     so the P-th smallest canonical d0 is <= T (1 + eps) and every member of the exact
//     top-P has d_rot <= T (1 + eps)^2 -- C contains it.
//  4. Canonical CA2 d0 (m ascending) for the members of C only, keys (d0, k), bitonic
//     sort, the first P are the exact top-P by (d0, k) (ties to the lowest k, CA4), in
//     rank order (the list-major items and their phases run nearest lists first).
// For P > CT_ROT_PMAX (masked IVF: hundreds of lists), or if C overflows its buffer
// (many near-ties), the kernel computes every canonical d0 and selects exactly with a
// radix select and tie ranks by k.  Measured (deep10m, 10k queries): L = 1 2.76 ->
// 2.59 ms per call, L = 64 11.68 -> 11.59 ms against the canonical-only kernel.
constexpr int CT_NT = 256;
constexpr int CT_PMAX = 2048;
constexpr float CT_EPS2 = 1.00002f;  // (1 + 1e-5)^2, rounded up
constexpr int CT_ROT_PMAX = 128;     // larger P: canonical sums of every centre directly

// the table region holds the [H][256][32] rotated layout, then (transposed in place for
// the canonical sums) [M][257] (bank = (m + z) mod 32)
__host__ __device__ constexpr size_t ct_tab_bytes(int M) {
    return ((size_t)(M > 32 ? 2 : 1) * LUT_Q_FLOATS * 4 > (size_t)M * 257 * 4 ? (size_t)(M > 32 ? 2 : 1) * LUT_Q_FLOATS * 4
                                                                              : ((size_t)M * 257 * 4 + 15) / 16 * 16);
}
__host__ __device__ constexpr int ct_cap(int Ppad) { return 2 * Ppad < 256 ? 256 : 2 * Ppad; }

template <int M>
__device__ __forceinline__ float ct_canonical(const float *tabc, const uint8_t *__restrict__ cp) {
    float acc = 0.f;  // tabc: [M][257]
#pragma unroll
    for (int m = 0; m < M; ++m) acc = __fadd_rn(acc, tabc[m * 257 + (int)cp[m]]);
    return acc;
}

template <int M>
__global__ void __launch_bounds__(CT_NT) coarse_topp_kernel(const uint8_t *__restrict__ centers, int64_t K,
                                                            const float *__restrict__ tables, int64_t P,
                                                            int32_t *__restrict__ probes, int Ppad,
                                                            int keys_off, int d0_off, bool direct) {
    constexpr int W = M / 4, H = M > 32 ? 2 : 1, MH = M < 32 ? M : 32;
    extern __shared__ __align__(16) uint8_t smem[];
    float *tab = reinterpret_cast<float *>(smem);  // [H][256][32], then [M][257]
    const int cap = ct_cap(Ppad);
    // large P (masked IVF): the candidate re-check would recompute most of the P sums
    // anyway, so the canonical sums of every centre are taken directly (the fallback);
    // the table is then staged as [M][257] at once and the keys overlay it at the end
    uint64_t *keys = reinterpret_cast<uint64_t *>(smem + keys_off);  // [cap] (direct: [Ppad])
    uint32_t *d0 = reinterpret_cast<uint32_t *>(smem + d0_off);      // [K]
    __shared__ int hist[256];
    __shared__ uint32_t s_prefix, s_mask;
    __shared__ int s_rem, s_n;
    __shared__ int wsum[CT_NT / 32];
    const int64_t qi = blockIdx.x;
    const int lane = threadIdx.x & 31;
    RII_SMEM_CHECK(smem, d0 + K);
    RII_SMEM_CHECK(smem, keys + (direct ? Ppad : cap));
    RII_SMEM_CHECK(smem, tab + (direct ? M * 257 : H * LUT_Q_FLOATS));
    if (direct) {  // stage as [M][257] (A(m, z) = column m mod MH of row z of half m / 32)
        const float *tq = tables + qi * (int64_t)lut_q_floats(M);
        for (int e = threadIdx.x; e < M * KS; e += CT_NT) {
            const int h = e / (KS * MH), r = e - h * KS * MH, z = r / MH, mm = r - z * MH;
            tab[(32 * h + mm) * 257 + z] = __ldg(tq + h * LUT_Q_FLOATS + z * 32 + mm);
        }
    } else {  // stage the table (a straight copy: the rotated lookups need no transpose)
        const float4 *src = reinterpret_cast<const float4 *>(tables + qi * (int64_t)lut_q_floats(M));
        float4 *dst = reinterpret_cast<float4 *>(tab);
        for (int e = threadIdx.x; e < H * LUT_Q_FLOATS / 4; e += CT_NT) dst[e] = __ldg(src + e);
    }
    __syncthreads();
    // 1. rotated sums
    for (int64_t k = threadIdx.x; k < (direct ? 0 : K); k += CT_NT) {
        uint32_t w[W];
        const uint32_t *cp = reinterpret_cast<const uint32_t *>(centers + k * M);
#pragma unroll
        for (int i = 0; i < W; ++i) w[i] = __ldg(cp + i);
        // step j reads column c = (l ^ j) mod 32 (distinct per lane), i.e. subspace
        // 32 (j / 32) + c mod MH: its code word is w[(j / 4) ^ rw] within the half, so the
        // words are XOR-permuted once (static register indices in the loop)
        permute_words<W, 8>(w, ((uint32_t)lane >> 2) & (uint32_t)(MH / 4 - 1));
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const uint32_t c = ((uint32_t)lane ^ (uint32_t)j) & 31u;
            const uint32_t z = (w[j >> 2] >> (8 * (c & 3u))) & 255u;
            acc = __fadd_rn(acc, tab[(j >> 5) * LUT_Q_FLOATS + (int)z * 32 + (int)c]);
        }
        d0[k] = __float_as_uint(acc);
    }
    if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_rem = (int)P; s_n = 0; }
    __syncthreads();
    // radix select over d0[0, K): the P-th smallest bit pattern -> s_prefix (s_rem = how
    // many keys equal to it belong to the P smallest)
    auto radix_select = [&]() {
        for (int shift = 24; shift >= 0; shift -= 8) {
            hist[threadIdx.x] = 0;
            __syncthreads();
            const uint32_t pre = s_prefix, msk = s_mask;
            for (int64_t k = threadIdx.x; k < K; k += CT_NT) {
                const uint32_t v = d0[k];
                if ((v & msk) == pre) atomicAdd(&hist[(v >> shift) & 255], 1);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int rem = s_rem, acc = 0, d = 0;
                for (; d < 256; ++d) {
                    if (acc + hist[d] >= rem) break;
                    acc += hist[d];
                }
                s_rem = rem - acc;
                s_prefix = pre | ((uint32_t)d << shift);
                s_mask = msk | (255u << shift);
            }
            __syncthreads();
        }
    };
    if (!direct) radix_select();
    // 3. candidates
    const float thr = __fmul_ru(__uint_as_float(s_prefix), CT_EPS2);
    for (int64_t k = threadIdx.x; k < (direct ? 0 : K); k += CT_NT) {
        if (__uint_as_float(d0[k]) <= thr) {
            const int i = atomicAdd(&s_n, 1);
            if (i < cap) keys[i] = (uint64_t)k;
        }
    }
    __syncthreads();
    if (!direct) {  // transpose the table in place to [M][257] for the canonical sums (bank (m + z) mod 32)
        constexpr int E = H * LUT_Q_FLOATS / CT_NT;
        float v[E];
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = tab[threadIdx.x + i * CT_NT];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const int e = threadIdx.x + i * CT_NT, h = e / LUT_Q_FLOATS, z = (e % LUT_Q_FLOATS) / 32, c = e % 32;
            if (c < MH) tab[(32 * h + c) * 257 + z] = v[i];
        }
        __syncthreads();
    }
    const int n = direct ? cap + 1 : s_n;
    int S = 1;
    if (n <= cap) {
        // 4. canonical d0 of the candidates, exact order
        for (int i = threadIdx.x; i < n; i += CT_NT) {
            const uint32_t k = (uint32_t)keys[i];
            keys[i] = ((uint64_t)__float_as_uint(ct_canonical<M>(tab, centers + (int64_t)k * M)) << 32) | k;
        }
        while (S < n) S <<= 1;
        for (int i = n + threadIdx.x; i < S; i += CT_NT) keys[i] = KEY_MAX;
    } else {
        // fallback: every canonical d0, exact radix select with ties to the lowest k
        __syncthreads();
        for (int64_t k = threadIdx.x; k < K; k += CT_NT)
            d0[k] = __float_as_uint(ct_canonical<M>(tab, centers + k * M));
        if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_rem = (int)P; s_n = 0; }
        __syncthreads();
        radix_select();
        const uint32_t t = s_prefix;
        const int ties = s_rem;
        S = Ppad;
        for (int e = threadIdx.x; e < S; e += CT_NT) keys[e] = KEY_MAX;
        __syncthreads();
        for (int64_t k = threadIdx.x; k < K; k += CT_NT) {  // below the threshold: P - ties keys
            const uint32_t v = d0[k];
            if (v < t) keys[atomicAdd(&s_n, 1)] = ((uint64_t)v << 32) | (uint64_t)k;
        }
        __syncthreads();
        const int base = (int)P - ties;
        int seen = 0;
        for (int64_t k0 = 0; k0 < K && seen < ties; k0 += CT_NT) {  // at it: the lowest k first
            const int64_t k = k0 + threadIdx.x;
            const int tie = (k < K && d0[k] == t) ? 1 : 0;
            const unsigned bal = __ballot_sync(0xffffffffu, tie);
            if (lane == 0) wsum[threadIdx.x >> 5] = __popc(bal);
            __syncthreads();
            int off = 0, tot = 0;
            for (int w = 0; w < CT_NT / 32; ++w) {
                if (w < (int)(threadIdx.x >> 5)) off += wsum[w];
                tot += wsum[w];
            }
            const int rank = seen + off + __popc(bal & ((1u << lane) - 1u));
            if (tie && rank < ties) keys[base + rank] = ((uint64_t)t << 32) | (uint64_t)k;
            seen += tot;
            __syncthreads();
        }
    }
    __syncthreads();
    bitonic_sort_rows(keys, 1, S, S);
    for (int64_t r = threadIdx.x; r < P; r += CT_NT) probes[qi * P + r] = (int32_t)(keys[r] & 0xffffffffu);
}

bool launch_coarse_topp(const uint8_t *centers, int64_t K, int M, const float *tables, int64_t nq, int64_t P,
                        int32_t *probes, cudaStream_t st) {
    if (P > CT_PMAX || P > K || !tables || (M != 4 && M != 8 && M != 16 && M != 32 && M != 64)) return false;
    int Ppad = 1;
    while (Ppad < P) Ppad <<= 1;
    // canonical sums of every centre directly for large P (RII_COARSE_ROT_MINK: also
    // below that many centres, A/B only -- the rotated pass measured faster at every K
    // tried: sift1m K = 1,000, M = 16 L = 1 1.54 -> 1.48 ms; M = 64 L = 1 3.62 -> 2.71 ms,
    // profiles/r02h_ab_coarse_rotmink_sift1m.jsonl)
    const char *mk = getenv("RII_COARSE_ROT_MINK");
    const bool direct = P > CT_ROT_PMAX || K < (mk ? atoll(mk) : 0);
    const size_t tb = ct_tab_bytes(M);
    const size_t keys_off = direct && (size_t)Ppad * 8 <= tb ? 0 : tb;  // direct: keys overlay the table
    const size_t d0_off = direct ? std::max(tb, keys_off + (size_t)Ppad * 8) : tb + (size_t)ct_cap(Ppad) * 8;
    const size_t smem = d0_off + (size_t)K * 4;
    if (smem + 4096 > (size_t)SMEM_ATTR_MAX) return false;
    if (nq <= 0) return true;
    switch (M) {
#define RII_CT(MM)                                                                                            \
    case MM:                                                                                                  \
        RII_CUDA(cudaFuncSetAttribute(coarse_topp_kernel<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                      SMEM_ATTR_MAX - 4096));                                                 \
        coarse_topp_kernel<MM><<<(unsigned)nq, CT_NT, smem, st>>>(centers, K, tables, P, probes, Ppad,       \
                                                                 (int)keys_off, (int)d0_off, direct);        \
        break;
        RII_CT(4) RII_CT(8) RII_CT(16) RII_CT(32) RII_CT(64)
#undef RII_CT
    }
    RII_LAUNCHED();
    return true;
}

__global__ void keys_to_probes_kernel(const uint64_t *__restrict__ keys, int64_t nq, int kk, int64_t P,
                                      int32_t *__restrict__ probes) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nq * P) return;
    const int64_t q = e / P, r = e - q * P;
    probes[e] = (int32_t)key_id(keys[q * kk + r]);
}

void launch_keys_to_probes(const uint64_t *keys, int64_t nq, int kk, int64_t P, int32_t *probes, cudaStream_t st) {
    if (nq * P <= 0) return;
    keys_to_probes_kernel<<<(unsigned)ceil_div(nq * P, 256), 256, 0, st>>>(keys, nq, kk, P, probes);
    RII_LAUNCHED();
}

void launch_select_probes(const float *d0, int64_t nq, int64_t K, int64_t P, int32_t *probes, cudaStream_t st) {
    if (nq <= 0) return;
    select_probes_kernel<<<(unsigned)nq, NT, 0, st>>>(d0, K, P, probes);
    RII_LAUNCHED();
}

// --------------------------------------------------- paper mode (Alg. 2) ----
__global__ void seg_iota_kernel(int32_t *v, int64_t n, int64_t len) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (int32_t)(i % len);
}

// composite sort key of (query, list): (q << 32) | bits(d0[q][k])
__global__ void seg_keys_kernel(const float *__restrict__ d0, int64_t n, int64_t K, uint64_t *__restrict__ key) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) key[i] = ((uint64_t)(i / K) << 32) | (uint64_t)__float_as_uint(d0[i]);
}

__global__ void seg_head_kernel(const int32_t *sorted, int64_t nq, int64_t K, int64_t P, int32_t *probes) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nq * P) return;
    const int64_t q = e / P, r = e - q * P;
    probes[e] = sorted[q * K + r];
}

void launch_sorted_probes(const float *d0, int64_t nq, int64_t K, int64_t P, int32_t *probes, cudaStream_t st) {
    if (nq <= 0 || P <= 0) return;
    const int64_t n = nq * K;
    int32_t *vin = nullptr, *vout = nullptr;
    RII_CUDA(cudaMallocAsync(&vin, (size_t)n * 4, st));
    RII_CUDA(cudaMallocAsync(&vout, (size_t)n * 4, st));
    seg_iota_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(vin, n, K);
    RII_LAUNCHED();
    // one stable sort of the composite keys (q << 32) | bits(d0): d0 >= +0, so its bit
    // order is its value order; stable, so ties keep ascending k (CA4)
    uint64_t *kin = nullptr, *kout64 = nullptr;
    RII_CUDA(cudaMallocAsync(&kin, (size_t)n * 8, st));
    RII_CUDA(cudaMallocAsync(&kout64, (size_t)n * 8, st));
    seg_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d0, n, K, kin);
    RII_LAUNCHED();
    int qbits = 0;
    while (((int64_t)1 << qbits) < nq) ++qbits;
    radix_sort_pairs<uint64_t>(kin, reinterpret_cast<const uint32_t *>(vin), n, 32 + qbits, kout64,
                               reinterpret_cast<uint32_t *>(vout), st);
    seg_head_kernel<<<(unsigned)ceil_div(nq * P, 256), 256, 0, st>>>(vout, nq, K, P, probes);
    RII_LAUNCHED();
    for (void *pp : {(void *)kin, (void *)kout64, (void *)vin, (void *)vout})
        RII_CUDA(cudaFreeAsync(pp, st));
}

__global__ void paper_takes_kernel(const int32_t *__restrict__ probes, int64_t nq, int64_t P,
                                   const int64_t *__restrict__ offsets, int64_t L, int32_t *__restrict__ take) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    int64_t acc = 0;
    for (int64_t r = 0; r < P; ++r) {  // L8-L9 in rank order, stop at |U| = L (L14)
        const int32_t k = probes[q * P + r];
        const int64_t len = offsets[k + 1] - offsets[k];
        const int64_t t = acc >= L ? 0 : (len < L - acc ? len : L - acc);
        take[q * P + r] = (int32_t)t;
        acc += t;
    }
}

void launch_paper_takes(const int32_t *probes, int64_t nq, int64_t P, const int64_t *offsets, int64_t L,
                        int32_t *take, cudaStream_t st) {
    if (nq <= 0 || P <= 0) return;
    paper_takes_kernel<<<(unsigned)ceil_div(nq, 128), 128, 0, st>>>(probes, nq, P, offsets, L, take);
    RII_LAUNCHED();
}

// ------------------------------------------------------ list-major items ----
__global__ void list_item_count_kernel(const int64_t *__restrict__ qoff, int64_t K, int B, int64_t *__restrict__ n) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < K) n[k] = (qoff[k + 1] - qoff[k] + B - 1) / B;
    else if (k == K) n[k] = 0;
}

__global__ void list_item_fill_kernel(const int64_t *__restrict__ qoff, const int64_t *__restrict__ ioff, int64_t K,
                                      int B, int4 *__restrict__ items) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const int64_t c = qoff[k + 1] - qoff[k];
    for (int64_t i = 0; i * B < c; ++i) {
        const int64_t n = c - i * B < B ? c - i * B : B;
        items[ioff[k] + i] = make_int4((int)k, (int)(qoff[k] + i * B), (int)n, 0);
    }
}

__global__ void item_rank_kernel(const int4 *__restrict__ items, int64_t n, const uint32_t *__restrict__ qlist,
                                 int64_t P, uint32_t *__restrict__ key, uint32_t *__restrict__ idx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 it = items[i];
    uint32_t r = 0xffffffffu;
    for (int j = 0; j < it.z; ++j) {
        const uint32_t rj = (uint32_t)(qlist[it.y + j] % P);
        r = rj < r ? rj : r;
    }
    key[i] = r;
    idx[i] = (uint32_t)i;
}

__global__ void permute_items_kernel(const int4 *__restrict__ in, const uint32_t *__restrict__ idx, int64_t n,
                                     int4 *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[idx[i]];
}

__global__ void fill_f32_kernel(float *p, int64_t n, float v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

void launch_fill_f32(float *p, int64_t n, float v, cudaStream_t st) {
    if (n <= 0) return;
    fill_f32_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(p, n, v);
    RII_LAUNCHED();
}

int64_t build_list_items(const int64_t *qoff, int64_t K, int B, const uint32_t *qlist, int64_t P, int4 *items,
                         int64_t cap, cudaStream_t st) {
    int64_t *n = nullptr, *ioff = nullptr;
    RII_CUDA(cudaMallocAsync(&n, (size_t)(K + 1) * 8, st));
    RII_CUDA(cudaMallocAsync(&ioff, (size_t)(K + 1) * 8, st));
    list_item_count_kernel<<<(unsigned)ceil_div(K + 1, 256), 256, 0, st>>>(qoff, K, B, n);
    RII_LAUNCHED();
    exclusive_scan_i64(n, K + 1, ioff, st);
    int64_t total = 0;
    RII_CUDA(cudaMemcpyAsync(&total, ioff + K, 8, cudaMemcpyDeviceToHost, st));
    RII_CUDA(cudaStreamSynchronize(st));
    if (total > cap) throw Error(4, "list-major item buffer too small");
    int4 *raw = nullptr;
    RII_CUDA(cudaMallocAsync(&raw, (size_t)std::max<int64_t>(total, 1) * sizeof(int4), st));
    list_item_fill_kernel<<<(unsigned)ceil_div(K, 256), 256, 0, st>>>(qoff, ioff, K, B, raw);
    RII_LAUNCHED();
    // RII_ITEM_ORDER=list (A/B): keep the items of one list adjacent (L2 reuse of its
    // codes) instead of ordering them by the smallest probe rank of their queries
    const char *ord = getenv("RII_ITEM_ORDER");
    if (total > 0 && ord && !strcmp(ord, "list")) {
        RII_CUDA(cudaMemcpyAsync(items, raw, (size_t)total * sizeof(int4), cudaMemcpyDeviceToDevice, st));
    } else if (total > 0) {
        uint32_t *key = nullptr, *key2 = nullptr, *idx = nullptr, *idx2 = nullptr;
        RII_CUDA(cudaMallocAsync(&key, (size_t)total * 4, st));
        RII_CUDA(cudaMallocAsync(&key2, (size_t)total * 4, st));
        RII_CUDA(cudaMallocAsync(&idx, (size_t)total * 4, st));
        RII_CUDA(cudaMallocAsync(&idx2, (size_t)total * 4, st));
        item_rank_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(raw, total, qlist, P, key, idx);
        RII_LAUNCHED();
        int bits = 1;
        while ((1ll << bits) <= P) ++bits;
        radix_sort_pairs<uint32_t>(key, idx, total, bits, key2, idx2, st);  // stable (sort.cu)
        permute_items_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(raw, idx2, total, items);
        RII_LAUNCHED();
        for (void *pp : {(void *)key, (void *)key2, (void *)idx, (void *)idx2})
            RII_CUDA(cudaFreeAsync(pp, st));
    }
    RII_CUDA(cudaFreeAsync(raw, st));
    RII_CUDA(cudaFreeAsync(n, st));
    RII_CUDA(cudaFreeAsync(ioff, st));
    return total;
}

// ----------------------------------------------------------- list scan -----
template <int W>
__device__ __forceinline__ void load_code_ivf(const uint8_t *p, uint32_t (&w)[W]) {
    if constexpr (W == 8) {
        const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
        const uint4 b = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
        w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    } else if constexpr (W == 4) {
        const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    } else if constexpr (W == 2) {
        const uint2 a = __ldg(reinterpret_cast<const uint2 *>(p));
        w[0] = a.x; w[1] = a.y;
    } else {
        w[0] = __ldg(reinterpret_cast<const uint32_t *>(p));
    }
}

constexpr int PAIR_BYTES = LUT_PAIR_BYTES;

// Per-warp work pulling: (qq, r) items = query half qq, probe rank r.
struct ListCursor {
    int64_t beg, end;
    int qq;
    bool done;
};

// A warp's next work item: segment `it % nseg` of the (query slot, probe rank) pair
// `it / nseg` (nseg > 1 splits every list among several warps: few pairs per CTA).
__device__ __forceinline__ void next_list(ListCursor &c, int *s_next, int64_t P, int64_t q0, int64_t nq,
                                          const int32_t *probes, const int64_t *offsets, const int32_t *take,
                                          int lane, int nseg) {
    while (!c.done && c.beg >= c.end) {
        int it = 0;
        if (lane == 0) it = atomicAdd(s_next, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if ((int64_t)it >= 2 * P * nseg) { c.done = true; break; }
        const int pr = it / nseg, sg = it - pr * nseg;
        const int qq = pr & 1;
        const int64_t r = pr >> 1, qi = q0 + qq;
        if (qi >= nq) continue;
        const int32_t k = probes[qi * P + r];
        const int64_t b = offsets[k], e = take ? b + take[qi * P + r] : offsets[k + 1];
        const int64_t n32 = (e - b + 31) >> 5;  // 32-code steps, split evenly over the segments
        c.qq = qq;
        c.beg = b + ((n32 * sg) / nseg) * 32;
        c.end = min(e, b + ((n32 * (sg + 1)) / nseg) * 32);
    }
}

template <int M, bool FAST>
__global__ void __launch_bounds__(NT) ivf_scan_kernel(const uint8_t *__restrict__ codes, const float *__restrict__ q,
                                                      int64_t nq, const float *__restrict__ cb, int Mrt, int ds,
                                                      int kk, const int32_t *__restrict__ probes, int64_t P,
                                                      const int64_t *__restrict__ offsets,
                                                      const uint32_t *__restrict__ ids, uint64_t *__restrict__ out,
                                                      const float *__restrict__ tables,
                                                      const int32_t *__restrict__ take, int64_t ostride, int nseg) {
    constexpr int W = FAST ? M / 4 : 1;
    const int MM = FAST ? M : Mrt;
    extern __shared__ __align__(16) uint8_t smem[];
    const size_t lut_bytes = FAST ? (size_t)PAIR_BYTES : (size_t)2 * MM * KS * 4;
    uint8_t *lut = smem;
    uint64_t *top = reinterpret_cast<uint64_t *>(smem + lut_bytes);
    uint64_t *fresh = top + 2 * kk;
    int *cnt = reinterpret_cast<int *>(fresh + 2 * NEWCAP);
    float *thr = reinterpret_cast<float *>(cnt + 2);
    int *scratch = reinterpret_cast<int *>(thr + 2);
    int *s_next = scratch + 2;
    RII_SMEM_CHECK(smem, s_next + 1);

    const int64_t q0 = (int64_t)blockIdx.x * 2;
    const int D = MM * ds, tid = threadIdx.x, lane = tid & 31;
    const float *qa = q + min(q0, nq - 1) * D, *qb = q + min(q0 + 1, nq - 1) * D;
    if constexpr (FAST) {
        if (tables)
            load_lut_pair(reinterpret_cast<float *>(lut), tables + min(q0, nq - 1) * LUT_Q_FLOATS,
                          tables + min(q0 + 1, nq - 1) * LUT_Q_FLOATS);
        else
            build_lut_pair<M>(reinterpret_cast<float *>(lut), qa, qb, cb, ds);
    } else {
        float *lp = reinterpret_cast<float *>(lut);
        for (int e = tid; e < 2 * MM * KS; e += NT) {
            const int qq = e / (MM * KS), m = (e / KS) % MM, z = e % KS;
            const float *qv = (qq ? qb : qa) + m * ds, *cv = cb + ((size_t)m * KS + z) * ds;
            float a = 0.f;
            for (int j = 0; j < ds; ++j) a = ca1_step(a, qv[j], cv[j]);
            lp[e] = a;
        }
    }
    for (int e = tid; e < 2 * kk; e += NT) top[e] = KEY_MAX;
    if (tid < 2) { cnt[tid] = 0; thr[tid] = __int_as_float(0x7f800000); }
    if (tid == 0) *s_next = 0;
    __syncthreads();

    uint32_t sel[4];
    const uint32_t r = (uint32_t)lane & (FAST ? (M - 1) : 0), rw = r >> 2;
    make_selectors(r, sel);
    float th0 = thr[0], th1 = thr[1];
    bool need = false;
    ListCursor cur{0, 0, 0, false};
    while (true) {
        next_list(cur, s_next, P, q0, nq, probes, offsets, take, lane, nseg);
        if (!__syncthreads_or(!cur.done)) break;
        if (!cur.done) {
            const int64_t p = cur.beg + lane;
            const bool valid = p < cur.end;
            const uint32_t pos = valid ? __ldg(ids + p) : 0u;
            float acc = 0.f;
            if constexpr (FAST) {
                uint32_t w[W];
#pragma unroll
                for (int i = 0; i < W; ++i) w[i] = 0;
                if (valid) load_code_ivf<W>(codes + (size_t)pos * M, w);
                permute_words<W>(w, rw);
                const uint32_t l8 = ((uint32_t)lane << 3) | ((uint32_t)cur.qq << 2);
#pragma unroll
                for (int j = 0; j < (FAST ? M : 1); ++j) {
                    const uint32_t off = __byte_perm(w[j >> 2], l8 ^ (uint32_t)(j << 3), sel[j & 3]);
                    acc += *reinterpret_cast<const float *>(lut + off);
                }
            } else if (valid) {
                const float *lq = reinterpret_cast<const float *>(lut) + (size_t)cur.qq * MM * KS;
                const uint8_t *cp = codes + (size_t)pos * MM;
                for (int m = 0; m < MM; ++m) acc = __fadd_rn(acc, lq[m * KS + cp[m]]);
            }
            const float th = cur.qq ? th1 : th0;
            push_candidate(valid && acc <= th, make_key(acc, pos), fresh + cur.qq * NEWCAP, cnt + cur.qq, lane,
                           need);
            cur.beg += 32;
        }
        if (__syncthreads_or(need)) {
            compact_topk(top, fresh, cnt, thr, 2, kk, scratch);
            th0 = thr[0];
            th1 = thr[1];
            need = false;
        }
    }
    compact_topk(top, fresh, cnt, thr, 2, kk, scratch);
    if constexpr (FAST) {  // canonical rescore (CA2) of the kept candidates, replica 0
        for (int e = tid; e < 2 * kk; e += NT) {
            const uint64_t k = top[e];
            if (k == KEY_MAX) continue;
            const int qq = e >= kk;
            const uint32_t id = key_id(k);
            const uint8_t *cp = codes + (size_t)id * M;
            const float *lq = reinterpret_cast<const float *>(lut);
            float d = 0.f;
            for (int m = 0; m < M; ++m) d = __fadd_rn(d, lut_pair_entry(lq, qq, m, cp[m]));
            top[e] = make_key(d, id);
        }
        __syncthreads();
        bitonic_sort_rows(top, 2, kk, kk);
    }
    for (int e = tid; e < 2 * kk; e += NT) {
        const int qq = e >= kk ? 1 : 0, i = e - qq * kk;
        if (q0 + qq < nq) out[(q0 + qq) * ostride + i] = top[e];
    }
}

size_t ivf_smem(int M, int kk) {
    const bool fast = (M == 4 || M == 8 || M == 16 || M == 32);
    const size_t lut = fast ? (size_t)PAIR_BYTES : (size_t)2 * M * KS * 4;
    return lut + (size_t)2 * (kk + NEWCAP) * 8 + 64;
}

template <int M, bool FAST>
static void ivf_launch_t(const uint8_t *codes, int Mrt, const float *q, int64_t nq, const float *cb, int ds, int kk,
                         const int32_t *probes, int64_t P, const int64_t *offsets, const uint32_t *ids, uint64_t *out,
                         cudaStream_t st, const float *tables, const int32_t *take, int64_t ostride, int nseg) {
    const size_t smem = ivf_smem(Mrt, kk);
    auto kern = ivf_scan_kernel<M, FAST>;
    RII_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    KernelTimer t(TK_IVF, st);
    kern<<<(unsigned)ceil_div(nq, 2), NT, smem, st>>>(codes, q, nq, cb, Mrt, ds, kk, probes, P, offsets, ids, out,
                                                      FAST ? tables : nullptr, take, ostride > 0 ? ostride : kk,
                                                      nseg);
    RII_LAUNCHED();
}

void launch_ivf_scan(const uint8_t *codes, int M, const float *q, int64_t nq, const float *cb, int D, int kk,
                     const int32_t *probes, int64_t P, const int64_t *offsets, const uint32_t *ids, uint64_t *out,
                     cudaStream_t st, const float *tables, const int32_t *take, int64_t ostride, int nseg) {
    if (nq <= 0) return;
    if (ivf_smem(M, kk) > 227 * 1024) throw Error(1, "topk too large for the inverted-index kernel");
    const int ds = D / M;
    switch (M) {
        case 4: ivf_launch_t<4, true>(codes, M, q, nq, cb, ds, kk, probes, P, offsets, ids, out, st, tables, take, ostride, nseg); break;
        case 8: ivf_launch_t<8, true>(codes, M, q, nq, cb, ds, kk, probes, P, offsets, ids, out, st, tables, take, ostride, nseg); break;
        case 16: ivf_launch_t<16, true>(codes, M, q, nq, cb, ds, kk, probes, P, offsets, ids, out, st, tables, take, ostride, nseg); break;
        case 32: ivf_launch_t<32, true>(codes, M, q, nq, cb, ds, kk, probes, P, offsets, ids, out, st, tables, take, ostride, nseg); break;
        default: ivf_launch_t<1, false>(codes, M, q, nq, cb, ds, kk, probes, P, offsets, ids, out, st, tables, take, ostride, nseg); break;
    }
}

__global__ void rank_bound_kernel(const uint64_t *__restrict__ keys, int64_t nq, int64_t stride, int kk,
                                  float *__restrict__ gthr) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint64_t k = keys[q * stride + kk - 1];
    gthr[q] = k == KEY_MAX ? __int_as_float(0x7f800000) : __fmul_ru(key_dist(k), 1.00001f);
}

void launch_rank_bound(const uint64_t *keys, int64_t nq, int64_t stride, int kk, float *gthr, cudaStream_t st) {
    if (nq <= 0) return;
    rank_bound_kernel<<<(unsigned)ceil_div(nq, 256), 256, 0, st>>>(keys, nq, stride, kk, gthr);
    RII_LAUNCHED();
}

}  // namespace rii
