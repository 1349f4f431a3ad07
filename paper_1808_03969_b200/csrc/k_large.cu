// k_large.cu -- large-M shapes (GIST-like D = 960, M = 240; MET
// M = 192; the paper's range 8 <= M <= 240, Table 2).
//
// For M > 64 the per-query fp32 table (M KB) no longer fits shared memory next to
// anything else (240 KB at M = 240), and re-streaming subspace chunks of it per
// code tile costs ~M KB of L2 traffic per (query, tile).  So one query per CTA
// keeps its whole table resident as bf16 (M * 512 B <= 128 KB), sums the bf16
// entries in fp32 in the canonical m order, filters with the threshold relaxed by
// LARGE_SLACK (a bf16-rounded entry is within 2^-9 of its fp32 value and all terms
// are >= 0), and rescores every pushed candidate exactly (CA2, from the query's
// fp32 table in HBM) before it can enter the top list -- so results equal the
// oracle's bit for bit.
//
// Modes: 0 = linear scan over [c0, c1) of a code array (Alg. 1, whole or gathered
// subset); 1 = the query's probed posting lists (Alg. 2, mode A, or mode B with
// per-(query, rank) takes); 2 = SDC: the "query" is a PQ code x whose
// table rows are T_m[x^m][.], scanned against the centre codes (assignment a(n)).
#include <cuda_bf16.h>

#include "kernels.cuh"
#include "topk.cuh"

namespace rii {

constexpr float LARGE_SLACK = 1.0025f;  // > (1 + 2^-9)(1 + 256 * 2^-24)^2

struct LargeArgs {
    const uint8_t *codes;  // scanned codes [.][M]
    int M, kk;
    int64_t nq;
    // mode 0: chunks of the code array
    int64_t n_codes, chunk;
    int nc;
    // mode 1: probed lists
    const int32_t *probes;
    int64_t P;
    const int64_t *offsets;
    const uint32_t *ids;
    const int32_t *take;
    // tables: mode 0/1 per-query fp32 [nq][M][256]; mode 2 SDC tables T [M][256][256] + query codes
    const float *tables;
    const float *sdcT;
    const uint8_t *qcodes;
    uint64_t *out;  // mode 0: [nq][nc][kk]; modes 1/2: [nq][kk]
};

template <int MODE>
__global__ void __launch_bounds__(NT, 1) scan_large_kernel(const LargeArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int M = a.M, kk = a.kk, tid = threadIdx.x, lane = tid & 31;
    uint16_t *lut = reinterpret_cast<uint16_t *>(smem);  // [M][256] bf16
    uint64_t *top = reinterpret_cast<uint64_t *>(smem + (((size_t)M * KS * 2 + 15) & ~(size_t)15));
    uint64_t *fresh = top + kk;
    int *cnt = reinterpret_cast<int *>(fresh + NEWCAP);
    float *thr = reinterpret_cast<float *>(cnt + 1);
    int *scratch = reinterpret_cast<int *>(thr + 1);
    RII_SMEM_CHECK(smem, scratch + 8);

    int64_t q, ci = 0;
    if constexpr (MODE == 0) {
        ci = blockIdx.x / a.nq;
        q = blockIdx.x - ci * a.nq;
    } else {
        q = blockIdx.x;
    }
    // exact (fp32, canonical layout [m][z]) table entry of this query
    const uint8_t *xq = MODE == 2 ? a.qcodes + q * M : nullptr;
    auto entry = [&](int m, int z) -> float {
        if constexpr (MODE == 2) return __ldg(a.sdcT + ((size_t)m * KS + xq[m]) * KS + z);
        else return __ldg(a.tables + ((size_t)q * M + m) * KS + z);
    };
    for (int e = tid; e < M * KS; e += NT) {
        const int m = e >> 8, z = e & 255;
        lut[e] = __bfloat16_as_ushort(__float2bfloat16_rn(entry(m, z)));
    }
    for (int e = tid; e < kk; e += NT) top[e] = KEY_MAX;
    if (tid == 0) { cnt[0] = 0; thr[0] = __int_as_float(0x7f800000); }
    __syncthreads();

    float th = __int_as_float(0x7f800000);
    bool need = false;
    const uint8_t *__restrict__ codes = a.codes;
    auto rescore_fresh = [&]() {
        const int n = cnt[0];
        for (int i = tid; i < n; i += NT) {
            const uint32_t id = key_id(fresh[i]);
            const uint8_t *cp = codes + (size_t)id * M;
            float d = 0.f;
            if (MODE != 2 && (M & 15) == 0) {
                d = rescore_ca2_16(a.tables + (size_t)q * M * KS, cp, M);  // loads in flight per 16 subspaces
            } else {
                for (int m = 0; m < M; ++m) d = __fadd_rn(d, entry(m, cp[m]));
            }
            fresh[i] = make_key(d, id);
        }
        __syncthreads();
    };
    auto scan_range = [&](int64_t beg, int64_t end, bool indirect) {
        for (int64_t base = beg; base < end; base += NT) {
            const int64_t p = base + tid;
            const bool valid = p < end;
            uint32_t id = 0;
            float acc = 0.f;
            if (valid) {
                id = indirect ? __ldg(a.ids + p) : (uint32_t)p;
                const uint8_t *cp = codes + (size_t)id * M;
                if ((M & 3) == 0) {
                    for (int m4 = 0; m4 < M; m4 += 4) {
                        const uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(cp + m4));
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            acc = __fadd_rn(acc, __uint_as_float((uint32_t)lut[(m4 + b) * KS + ((w >> (8 * b)) & 255)]
                                                                 << 16));
                    }
                } else {
                    for (int m = 0; m < M; ++m)
                        acc = __fadd_rn(acc, __uint_as_float((uint32_t)lut[m * KS + cp[m]] << 16));
                }
            }
            push_candidate(valid && acc <= th, (uint64_t)id, fresh, cnt, lane, need);
            if (__syncthreads_or(need)) {
                rescore_fresh();
                compact_topk(top, fresh, cnt, thr, 1, kk, scratch);
                th = __fmul_ru(thr[0], LARGE_SLACK);
                need = false;
            }
        }
    };
    if constexpr (MODE == 1) {
        for (int64_t r = 0; r < a.P; ++r) {
            const int32_t k = a.probes[q * a.P + r];
            const int64_t beg = a.offsets[k];
            const int64_t end = a.take ? beg + a.take[q * a.P + r] : a.offsets[k + 1];
            scan_range(beg, end, true);
        }
    } else {
        const int64_t c0 = MODE == 0 ? ci * a.chunk : 0;
        const int64_t c1 = MODE == 0 ? min(a.n_codes, c0 + a.chunk) : a.n_codes;
        scan_range(c0, c1, false);
    }
    __syncthreads();
    rescore_fresh();
    compact_topk(top, fresh, cnt, thr, 1, kk, scratch);
    uint64_t *o = a.out + (MODE == 0 ? (q * a.nc + ci) * kk : q * kk);
    for (int e = tid; e < kk; e += NT) o[e] = top[e];
}

static size_t large_smem(int M, int kk) {
    return (((size_t)M * KS * 2 + 15) & ~(size_t)15) + (size_t)(kk + NEWCAP) * 8 + 64;
}

bool large_supported(int M, int kk) { return large_smem(M, kk) <= 227 * 1024; }

template <int MODE>
static void launch_large(const LargeArgs &a, int64_t grid, cudaStream_t st, int timer) {
    if (grid <= 0) return;
    const size_t smem = large_smem(a.M, a.kk);
    if (smem > 227 * 1024) throw Error(1, "topk too large for the large-M scan");
    RII_CUDA(cudaFuncSetAttribute(scan_large_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    KernelTimer t(timer, st);
    scan_large_kernel<MODE><<<(unsigned)grid, NT, smem, st>>>(a);
    RII_LAUNCHED();
}

// Canonical per-query fp32 tables [nq][M][256] (CA1), one CTA per query.
__global__ void __launch_bounds__(256) lut_large_kernel(const float *__restrict__ q, int64_t nq,
                                                        const float *__restrict__ cb, int M, int ds,
                                                        float *__restrict__ tables) {
    const int64_t qi = blockIdx.x;
    const float *qv = q + qi * (int64_t)M * ds;
    for (int e = threadIdx.x; e < M * KS; e += blockDim.x) {
        const int m = e >> 8, z = e & 255;
        const float *cv = cb + ((size_t)m * KS + z) * ds;
        float acc = 0.f;
        for (int j = 0; j < ds; ++j) acc = ca1_step(acc, qv[m * ds + j], cv[j]);
        tables[qi * (int64_t)M * KS + e] = acc;
    }
}

void launch_lut_large(const float *q, int64_t nq, const float *cb, int D, int M, float *tables, cudaStream_t st) {
    if (nq <= 0) return;
    lut_large_kernel<<<(unsigned)nq, 256, 0, st>>>(q, nq, cb, M, D / M, tables);
    RII_LAUNCHED();
}

int large_linear_chunks(int64_t nq, int64_t n_codes, int num_sms) {
    // enough CTAs for ~4 waves of 1 CTA per SM, chunks of >= 4096 codes
    int64_t nc = ceil_div((int64_t)4 * num_sms, std::max<int64_t>(nq, 1));
    nc = std::min<int64_t>(nc, std::max<int64_t>(1, n_codes / 4096));
    return (int)std::max<int64_t>(1, std::min<int64_t>(nc, 256));
}

void launch_large_linear(const uint8_t *codes, int64_t n_codes, int M, const float *tables, int64_t nq, int kk, int nc,
                         uint64_t *out, cudaStream_t st, int timer) {
    LargeArgs a{};
    a.codes = codes; a.M = M; a.kk = kk; a.nq = nq; a.n_codes = n_codes; a.nc = nc;
    a.chunk = ceil_div(n_codes, nc); a.tables = tables; a.out = out;
    launch_large<0>(a, nq * nc, st, timer);
}

void launch_large_ivf(const uint8_t *codes, int M, const float *tables, int64_t nq, int kk, const int32_t *probes,
                      int64_t P, const int64_t *offsets, const uint32_t *ids, const int32_t *take, uint64_t *out,
                      cudaStream_t st) {
    LargeArgs a{};
    a.codes = codes; a.M = M; a.kk = kk; a.nq = nq; a.probes = probes; a.P = P; a.offsets = offsets;
    a.ids = ids; a.take = take; a.tables = tables; a.out = out;
    launch_large<1>(a, nq, st, TK_IVF);
}

__global__ void large_top1_kernel(const uint64_t *__restrict__ keys, int64_t n, int kk, int32_t *__restrict__ assign,
                                  float *__restrict__ dist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = keys[i * kk];
    assign[i] = (int32_t)key_id(k);
    if (dist) dist[i] = key_dist(k);
}

void launch_large_assign(const uint8_t *codes, int64_t n, const uint8_t *centers, int64_t K, int M, const float *T,
                         int32_t *assign, float *dist, cudaStream_t st) {
    if (n <= 0) return;
    const int kk = 32;
    const int64_t CH = (int64_t)1 << 20;  // codes per launch: bounds the [n][kk] keys
    uint64_t *keys = nullptr;
    RII_CUDA(cudaMallocAsync(&keys, (size_t)std::min(n, CH) * kk * 8, st));
    for (int64_t s0 = 0; s0 < n; s0 += CH) {
        const int64_t cn = std::min(CH, n - s0);
        LargeArgs a{};
        a.codes = centers; a.M = M; a.kk = kk; a.nq = cn; a.n_codes = K; a.sdcT = T; a.qcodes = codes + s0 * M;
        a.out = keys;
        launch_large<2>(a, cn, st, -1);
        large_top1_kernel<<<(unsigned)ceil_div(cn, 256), 256, 0, st>>>(keys, cn, kk, assign + s0,
                                                                      dist ? dist + s0 : nullptr);
        RII_LAUNCHED();
    }
    RII_CUDA(cudaFreeAsync(keys, st));
}

}  // namespace rii
