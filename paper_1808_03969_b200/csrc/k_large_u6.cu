// k_large_u6.cu -- linear ADC scan (Alg. 1) for large M (SURVEY 8(f) F3:
// GIST-like D = 960, M = 240; MET M = 192), on the u6 fixed-point oct tables of the
// M = 32 kernels, one 32-subspace chunk at a time.
//
// For M > 64 the 8 queries' oct tables (M/32 chunks x 64 KB) do not fit shared
// memory, so a CTA (8 queries x a range of codes) walks its codes in tiles of
// NTH x U codes and, for each tile, loops over the subspace chunks: load chunk c's
// oct table (8 precomputed per-query u6 tables of 8 KB, transposed into the
// interleaved layout), add every code's 32 chunk lookups for the 8 queries into
// SWAR accumulators (16-bit lanes; M * 63 < 2^15, so the lanes never carry and the
// threshold test stays one subtraction per pair of queries), next chunk.  After
// the last chunk the per-query sums are complete and filtered exactly as in the
// M <= 64 kernels: q(v) = floor(min(v s, 63)) <= v s, so a code with d <= thr has
// Sum q <= floor(s thr (1 + 2^-16)); every pushed candidate is rescored in the
// canonical CA2 order from the query's fp32 table before it can enter the top
// list, so results equal the oracle's bit for bit.
//
// The scale s = 63 (M / 4) / T needs an upper bound T on the query's final kk-th
// distance: the exact kk-th over a strided sample of the codes (the one-query
// bf16 kernel of k_large.cu over <= 8192 codes), a subset, so it bounds the kk-th
// over all codes.  That bound is loose (~ the 1.6 % quantile), and the integer
// filter's slack is additive in it (M floor errors ~ 6 % of T), so the scan runs in
// two passes: the first 1/16 of the codes at that scale, then -- tables rebuilt at
// the kk-th over the first pass's exact results, a much tighter bound -- the rest.
#include <algorithm>

#include "kernels.cuh"
#include "lut.cuh"
#include "topk.cuh"

namespace rii {

namespace {
constexpr int LU_B = 8;      // queries per CTA (one oct table)
constexpr int LU_U = 8;      // codes per thread per tile
constexpr int LU_CH = 32;    // subspaces per chunk
constexpr int LU_CHB = KS * LU_CH;  // bytes of one query's u6 table chunk: [256][32]
// 7-bit entries (cap 127, pairs of steps summed bytewise): half the filter's floor
// error of 6-bit entries at the same saturation point; lane sums <= M * 127 < 2^15 for
// M <= 256.  The filter's slack is what the rescores pay for (see below).
static_assert(256 * 127 < 32768, "SWAR lanes");
// RII_LARGE_U7=0: 6-bit entries (A/B)
bool large_u7() {
    const char *e = getenv("RII_LARGE_U7");
    return !(e && atoi(e) == 0);
}

struct LargeU6Args {
    const uint8_t *codes;
    int64_t n_codes;  // codes [base, base + n_codes) of the array are scanned
    int64_t base;     // keys are absolute positions in `codes`
    int M, nch, kk;
    int64_t nq;
    int nb, nc;
    int64_t chunk;
    const uint8_t *qtab8;  // [nb][nch] oct tables of 64 KB (u6_tables_large_kernel)
    const float *qscale;   // [nq]
    const float *tables;   // [nq][M][256] fp32 (canonical layout, rescore)
    float *gthr;           // [nq] bound: filter, lowered with each CTA's kk-th
    uint64_t *out;         // [nb * 8][nc_out][kk]: this launch writes slots [ci_off, ci_off + nc)
    int nc_out, ci_off;
    uint32_t one;
};

__host__ __device__ constexpr size_t lu_aux_bytes(int kk) {
    return (size_t)LU_B * (kk + NEWCAP) * 8 + LU_B * 8 + 128 + LU_B * 16;
}
}  // namespace

// u6 oct tables of large M, ready to copy: out[b][c] = the 64 KB oct table of query
// batch b (queries 8b .. 8b+7, the last batch padded with its last query) and
// subspace chunk c: row z, column j, byte k = u6(A(8b + k, 32 c + j, z) s) (0 for
// 32 c + j >= M), s = 63 (M / 4) / gthr[q] rounded down.  One CTA per (padded) query.
__global__ void __launch_bounds__(256) u6_tables_large_kernel(const float *__restrict__ tables,
                                                              const float *__restrict__ gthr, int64_t nq, int M,
                                                              int nch, uint8_t *__restrict__ out,
                                                              float *__restrict__ scale, float amul, float cap) {
    const int64_t qp = blockIdx.x, q = qp < nq ? qp : nq - 1;
    const float s = __fdiv_rd(cap * u6_alpha(M) * amul, fmaxf(__ldcg(gthr + q), 1e-30f));
    if (threadIdx.x == 0 && qp < nq) scale[q] = s;
    const float *tq = tables + q * (int64_t)M * KS;
    uint8_t *o = out + (qp >> 3) * (int64_t)nch * OCT_BYTES + (qp & 7);
    for (int e = threadIdx.x; e < nch * LU_CHB; e += blockDim.x) {
        const int c = e / LU_CHB, r = e - c * LU_CHB, z = r / LU_CH, j = r - z * LU_CH, m = c * LU_CH + j;
        o[(int64_t)c * OCT_BYTES + (int64_t)r * 8] =
            m < M ? (uint8_t)u6_entry(__ldg(tq + (int64_t)m * KS + z), s, cap) : (uint8_t)0;
    }
}

// 1-D bulk copy global -> shared completing on an mbarrier (TMA engine, sm_90+).
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    for (uint32_t o = 0; o < bytes; o += 16384)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared((uint8_t *)dst + o)),
                     "l"((const uint8_t *)src + o), "r"(min(16384u, bytes - o)), "r"(b)
                     : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n LAB_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra LAB_WAIT_%=;\n}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(bar)),
        "r"(parity)
        : "memory");
}

// Exact CA2 rescore of the fresh candidates (from the queries' fp32 tables), fold
// into the top lists, refresh the shared bounds.  Not inlined: the push rounds that
// call it stay unrolled (their accumulators stay in registers).
template <int NTH>
__device__ __noinline__ void lu_compact(uint64_t *top, uint64_t *fresh, int *cnt, float *thr, float *gqs, int *scratch,
                                        const float *tables, const uint8_t *codes, const float *gthr, int qb, int nqi,
                                        int M, int kk) {
    const int tid = threadIdx.x;
    for (int qq = 0; qq < LU_B; ++qq) {
        const int n = cnt[qq];
        const int64_t q = (int64_t)qb * LU_B + (qq < nqi ? qq : nqi - 1);
        const float *tq = tables + q * (int64_t)M * KS;
        for (int i = tid; i < n; i += NTH) {
            uint64_t *f = fresh + qq * NEWCAP + i;
            const uint32_t id = key_id(*f);
            *f = make_key(rescore_ca2_16(tq, codes + (size_t)id * M, M), id);
        }
    }
    __syncthreads();
    compact_topk(top, fresh, cnt, thr, LU_B, kk, scratch);
    if (tid < LU_B) gqs[tid] = fminf(gqs[tid], __ldcg(gthr + (int64_t)qb * LU_B + (tid < nqi ? tid : nqi - 1)));
    __syncthreads();
}

template <int NTH, int LU_GJ>
__global__ void __launch_bounds__(NTH, 1) scan_large_u6_kernel(const LargeU6Args a) {
    constexpr int B = LU_B, U = LU_U, STEP = NTH;
    static_assert(NEWCAP >= STEP, "one round of pushes must fit the fresh buffer");
    extern __shared__ __align__(16) uint8_t smem[];
    if ((uint32_t)__cvta_generic_to_shared(smem) != 0x400u) __trap();  // fixed-base LDS immediates
    // two oct-table buffers (64 KB each, shared addresses 0x400 and 0x10400: LDS
    // immediates), filled by bulk copies one chunk ahead of the lookups
    uint8_t *lut = smem;
    uint8_t *aux = smem + 2 * OCT_BYTES;
    const int kk = a.kk, M = a.M, tid = threadIdx.x, lane = tid & 31;
    uint64_t *top = reinterpret_cast<uint64_t *>(aux);
    uint64_t *fresh = top + B * kk;
    int *cnt = reinterpret_cast<int *>(fresh + B * NEWCAP);
    float *thr = reinterpret_cast<float *>(cnt + B);
    int *scratch = reinterpret_cast<int *>(thr + B);
    float *qsc = reinterpret_cast<float *>(scratch + 32);
    float *gqs = qsc + B;
    uint64_t *bars = reinterpret_cast<uint64_t *>(aux + lu_aux_bytes(kk));  // [2], 8-byte aligned
    RII_SMEM_CHECK(smem, gqs + B);
    RII_SMEM_CHECK(smem, bars + 2);

    // chunk-major grid: the CTAs of a wave (all query batches of one code chunk) stream
    // the same codes (query-batch-major measured worse: 212 -> 277 ms, GIST-like)
    const int ci = blockIdx.x / a.nb, qb = blockIdx.x - ci * a.nb;
    const int64_t c0 = a.base + (int64_t)ci * a.chunk, c1 = a.base + min(a.n_codes, (int64_t)ci * a.chunk + a.chunk);
    const int64_t rem = a.nq - (int64_t)qb * B;
    const int nqi = rem < B ? (int)rem : B;
    RII_DCHECK(nqi >= 1 && c0 <= c1);
    auto query_of = [&](int qq) -> int64_t { return (int64_t)qb * B + (qq < nqi ? qq : nqi - 1); };
    const uint8_t *__restrict__ codes = a.codes;

    const int nch = a.nch;
    const int64_t ntiles = c1 > c0 ? ceil_div(c1 - c0, (int64_t)NTH * U) : 0;
    const int64_t nload = ntiles * nch;  // (tile, chunk) table loads of this CTA
    const uint8_t *tab_b = a.qtab8 + (int64_t)qb * nch * OCT_BYTES;
    if (tid == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (nload > 0) bulk_g2s(lut, tab_b, OCT_BYTES, bars);  // load 0: tile 0, chunk 0
    }
    for (int e = tid; e < B * kk; e += NTH) top[e] = KEY_MAX;
    if (tid < B) {
        cnt[tid] = 0;
        thr[tid] = __int_as_float(0x7f800000);
        qsc[tid] = __ldg(a.qscale + query_of(tid));
        gqs[tid] = __ldcg(a.gthr + query_of(tid));
    }
    __syncthreads();

    // lane geometry of the M = 32 u6 kernels (half-warp columns, one table copy)
    const uint32_t lr = (uint32_t)lane & 15u, rw = lr >> 2;
    uint32_t sel[4];
    make_selectors_q16(lr, sel);
    const uint32_t colA = (lr << 3) | ((lr ^ 1u) << 11);
    uint32_t colv[8];
#pragma unroll
    for (int aw = 0; aw < 8; ++aw) asm volatile("xor.b32 %0, %1, %2;" : "=r"(colv[aw]) : "r"(colA), "r"((uint32_t)(aw * 0x2020)));

    uint32_t thp[4];
    auto set_thp = [&]() {
        uint32_t thq[B];
#pragma unroll
        for (int qq = 0; qq < B; ++qq) thq[qq] = q16_threshold(fminf(thr[qq], gqs[qq]), qsc[qq]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int lo = (k >> 1) * 4 + (k & 1);
            thp[k] = 0x80008000u | min(thq[lo], 0x7fffu) | (min(thq[lo + 2], 0x7fffu) << 16);
        }
    };
    set_thp();

    auto compact = [&]() {
        lu_compact<NTH>(top, fresh, cnt, thr, gqs, scratch, a.tables, codes, a.gthr, qb, nqi, M, kk);
        set_thp();
    };

    const int M16 = M & ~15;  // bytes of a code row loaded with 16-byte loads (M % 16 == 0 on this path)
    int64_t g = 0;              // index of the (tile, chunk) table load being consumed
    for (int64_t tile = c0; tile < c1; tile += (int64_t)STEP * U) {
        uint32_t acc[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[u][k] = 0;
        for (int ch = 0; ch < nch; ++ch, ++g) {
            // buffer (g + 1) & 1 was last read by load g - 1, finished before the barrier
            // that ended that chunk: refill it with load g + 1 while load g is consumed
            if (tid == 0 && g + 1 < nload) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior LDS reads before the async writes
                const int nch1 = (int)((g + 1) % nch);
                bulk_g2s(lut + ((g + 1) & 1) * OCT_BYTES, tab_b + (int64_t)nch1 * OCT_BYTES, OCT_BYTES, bars + ((g + 1) & 1));
            }
            // this chunk's 32 code bytes, one code ahead of its lookups (bytes past the
            // row end of the last chunk are not read; their table columns are zero)
            const int b0 = ch * LU_CH;
            auto load_w = [&](int u, uint32_t (&w)[8]) {
                const int64_t p = tile + u * STEP + tid;
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = 0;
                if (p < c1) {
                    const uint8_t *cp = codes + (size_t)p * M + b0;
                    const uint4 x = __ldg(reinterpret_cast<const uint4 *>(cp));
                    w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
                    if (b0 + 16 < M16) {
                        const uint4 y = __ldg(reinterpret_cast<const uint4 *>(cp + 16));
                        w[4] = y.x; w[5] = y.y; w[6] = y.z; w[7] = y.w;
                    }
                }
            };
            uint32_t w[8], wn[8];
            load_w(0, w);
            mbar_wait(bars + (g & 1), (uint32_t)((g >> 1) & 1));  // table of load g has landed
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (u + 1 < U) load_w(u + 1, wn);
                uint32_t s6[4];
                if (g & 1) adc_u6<32, LU_GJ, false, 0x400 + OCT_BYTES, 1, 4>(w, rw, sel, colv, a.one, s6);
                else adc_u6<32, LU_GJ, false, 0x400, 1, 4>(w, rw, sel, colv, a.one, s6);
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[u][k] = fma_add(s6[k], a.one, acc[u][k]);
                if (u + 1 < U) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) w[i] = wn[i];
                }
            }
            __syncthreads();  // every warp is done with buffer g & 1
        }
        // complete sums: SWAR threshold test (lanes <= M * 63 < 2^15), pushes by round
#pragma unroll
        for (int u = 0; u < U; ++u) {
            // every push of the previous round must have landed before the fill is read
            // (reading it before the barrier let two rounds of pushes overflow the buffer)
            __syncthreads();
            if (__syncthreads_or(tid < B && cnt[tid] > NEWCAP - STEP)) compact();
            const int64_t p = tile + u * STEP + tid;
            uint32_t t[4], tor = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                t[k] = thp[k] - acc[u][k];
                tor |= t[k];
            }
            const bool anyp = (tor & 0x80008000u) != 0 && p < c1;
            if (__any_sync(0xffffffffu, anyp)) {
                uint32_t mk = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) mk |= (t[k] & 0x80008000u) >> (15 - (4 * (k >> 1) + (k & 1)));
                mk = p < c1 ? (mk | (mk >> 14)) & 0xffu : 0u;
                bool need = false;
                for (uint32_t wm = __reduce_or_sync(0xffffffffu, mk); wm; wm &= wm - 1u) {
                    const int qq = __ffs(wm) - 1;
                    push_candidate((mk >> qq) & 1u, (uint64_t)(uint32_t)p, fresh + qq * NEWCAP, cnt + qq, lane, need);
                }
            }
        }
    }
    __syncthreads();
    compact();
    if (tid < nqi && thr[tid] < __int_as_float(0x7f800000))  // publish this CTA's kk-th as a bound
        atomicMin(reinterpret_cast<int *>(a.gthr + query_of(tid)), __float_as_int(thr[tid]));
    for (int e = tid; e < B * kk; e += NTH) {
        const int qq = e / kk, i = e - qq * kk;
        if (qq < nqi) a.out[(((int64_t)qb * B + qq) * a.nc_out + a.ci_off + ci) * kk + i] = top[e];
    }
}

namespace {
constexpr int LU_NTH = 384;
size_t large_u6_smem(int kk) { return (size_t)2 * OCT_BYTES + lu_aux_bytes(kk) + 32; }
}  // namespace

bool large_u6_supported(int M, int kk) {
    return M > 64 && M <= 256 && M % 16 == 0 && kk <= 256 && large_u6_smem(kk) <= 227 * 1024;
}

int large_u6_nch(int M) { return (M + LU_CH - 1) / LU_CH; }

void launch_u6_tables_large(const float *tables, const float *gthr, int64_t nq, int M, uint8_t *out, float *scale,
                            cudaStream_t st) {
    if (nq <= 0) return;
    // RII_LARGE_U6_AMUL (A/B): saturation at 4 / amul times the mean entry of a code at the
    // bound; a larger multiplier means finer steps (less filter slack) and more saturation
    const char *e = getenv("RII_LARGE_U6_AMUL");
    const float amul = e ? (float)atof(e) : 1.0f;
    u6_tables_large_kernel<<<(unsigned)(ceil_div(nq, LU_B) * LU_B), 256, 0, st>>>(tables, gthr, nq, M, large_u6_nch(M),
                                                                                   out, scale, amul,
                                                                                   large_u7() ? 127.f : 63.f);
    RII_LAUNCHED();
}

int large_u6_chunks(int64_t nq, int64_t n_codes, int M, int num_sms) {
    // Code chunks of <= 64 MB (RII_LARGE_U6_CHUNK_MB): CTAs are ordered chunk-major, so
    // the CTAs of a wave (all query batches of one chunk) stream the same codes.
    // GIST-like (1M x 240 B, 10k queries): one 240 MB chunk 276 ms, 64 MB 258 ms,
    // 32 MB 276, 8 MB 359, 4 MB 378 ms -- the exact rescores of the candidates that pass
    // the u6 filter (240 scattered fp32 reads each) are the larger DRAM stream.  At
    // least ~2 waves of CTAs.
    const int64_t nb = ceil_div(nq, LU_B), tile = (int64_t)LU_NTH * LU_U;
    const char *e = getenv("RII_LARGE_U6_CHUNK_MB");
    const int64_t mb = e ? std::max(1, atoi(e)) : 64;
    int64_t nc = std::max<int64_t>(ceil_div(n_codes * M, mb << 20), ceil_div((int64_t)2 * num_sms, nb));
    nc = std::min<int64_t>(nc, std::max<int64_t>(1, n_codes / (2 * tile)));
    return (int)std::max<int64_t>(1, std::min<int64_t>(nc, 256));
}

void launch_large_u6_linear(const uint8_t *codes, int64_t base, int64_t n_codes, int M, const uint8_t *qtab8,
                            const float *qscale, const float *tables, float *gthr, int64_t nq, int kk, int nc,
                            uint64_t *out, int nc_out, int ci_off, cudaStream_t st) {
    if (nq <= 0 || n_codes <= 0) return;
    LargeU6Args a{};
    a.codes = codes; a.base = base; a.n_codes = n_codes; a.M = M; a.nch = large_u6_nch(M); a.kk = kk; a.nq = nq;
    a.nb = (int)ceil_div(nq, LU_B); a.nc = nc; a.chunk = ceil_div(n_codes, nc);
    a.nc_out = nc_out; a.ci_off = ci_off;
    a.qtab8 = qtab8; a.qscale = qscale; a.tables = tables; a.gthr = gthr; a.out = out; a.one = 1;
    const size_t smem = large_u6_smem(kk);
    auto kern = large_u7() ? scan_large_u6_kernel<LU_NTH, 2> : scan_large_u6_kernel<LU_NTH, 4>;
    RII_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    KernelTimer t(TK_LINEAR, st), tu(TK_U6, st);
    kern<<<(unsigned)(a.nb * nc), LU_NTH, smem, st>>>(a);
    RII_LAUNCHED();
}

}  // namespace rii
