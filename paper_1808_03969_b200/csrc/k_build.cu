// k_build.cu -- build-side kernels: PQ encode (Eq. 1), SDC tables (d_S), SDC
// assignment a(n), posting-list CSR (Eq. 4), reconfigure sample
// (R10), PQk-means (Alg. 4 L1, reading R9) and code-book k-means (R8).
// All arithmetic follows the canonical orders of DESIGN.md (CA1/CA2, ties to
// the lowest index) so codes, assignments and centres equal the oracle's.
#include <cub/cub.cuh>
#include <cstring>

#include "kernels.cuh"
#include "lut.cuh"

namespace rii {

// ------------------------------------------------------------------ encode --
// Eq. 1: one thread per vector, one grid row per subspace m; the
// code words of subspace m and the CTA's sub-vectors (transposed) sit in smem.
__global__ void __launch_bounds__(256) encode_kernel(const float *__restrict__ x, int64_t n, int D, int M, int ds,
                                                     const float *__restrict__ cb, uint8_t *__restrict__ codes) {
    extern __shared__ float esm[];
    float *cbs = esm;            // [256][ds]
    float *xs = esm + KS * ds;   // [ds][256]
    const int m = blockIdx.y, tid = threadIdx.x;
    const int64_t i0 = (int64_t)blockIdx.x * 256;
    for (int e = tid; e < KS * ds; e += 256) cbs[e] = cb[(size_t)m * KS * ds + e];
    for (int e = tid; e < 256 * ds; e += 256) {
        const int r = e / ds, j = e - r * ds;
        const int64_t i = i0 + r;
        xs[j * 256 + r] = i < n ? x[i * D + m * ds + j] : 0.f;
    }
    __syncthreads();
    float best = __int_as_float(0x7f800000);
    int bz = 0;
    for (int z = 0; z < KS; ++z) {
        float acc = 0.f;
        for (int j = 0; j < ds; ++j) acc = ca1_step(acc, xs[j * 256 + tid], cbs[z * ds + j]);
        if (acc < best) { best = acc; bz = z; }
    }
    const int64_t i = i0 + tid;
    if (i < n) codes[i * M + m] = (uint8_t)bz;
}

void launch_encode(const float *x, int64_t n, int D, int M, const float *cb, uint8_t *codes, cudaStream_t st) {
    if (n <= 0) return;
    const int ds = D / M;
    const size_t smem = (size_t)2 * KS * ds * 4;
    RII_CUDA(cudaFuncSetAttribute(encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    dim3 grid((unsigned)ceil_div(n, 256), (unsigned)M);
    encode_kernel<<<grid, 256, smem, st>>>(x, n, D, M, ds, cb, codes);
    RII_LAUNCHED();
}

// ------------------------------------------------------------- SDC tables --
__global__ void sdc_tables_kernel(const float *__restrict__ cb, int ds, float *__restrict__ T) {
    const int m = blockIdx.x, i = blockIdx.y, j = threadIdx.x;
    const float *a = cb + ((size_t)m * KS + i) * ds, *b = cb + ((size_t)m * KS + j) * ds;
    float acc = 0.f;
    for (int t = 0; t < ds; ++t) acc = ca1_step(acc, a[t], b[t]);
    T[((size_t)m * KS + i) * KS + j] = acc;
}

void launch_sdc_tables(const float *cb, int D, int M, float *T, cudaStream_t st) {
    sdc_tables_kernel<<<dim3(M, KS), KS, 0, st>>>(cb, D / M, T);
    RII_LAUNCHED();
}

// ----------------------------------------------------------------- assign --
// a(n) = argmin_k sum_m T_m[cbar_k^m][xbar_n^m] (CA2 order, strict <, k ascending).
// CTA = 256*R codes (bytes transposed in smem); centres streamed in batches of
// Bc whose "tables" T_m[cbar_k^m][.] are staged in smem.
constexpr int AR = 4;
__global__ void __launch_bounds__(256) assign_kernel(const uint8_t *__restrict__ codes, int64_t n,
                                                     const uint8_t *__restrict__ centers, int64_t K, int M,
                                                     const float *__restrict__ T, int Bc,
                                                     int32_t *__restrict__ assign, float *__restrict__ dist) {
    extern __shared__ __align__(16) uint8_t asmem[];
    float *alut = reinterpret_cast<float *>(asmem);                         // [Bc][M][256]
    uint8_t *cs = asmem + (size_t)Bc * M * KS * 4;                          // [M][256*AR]
    const int tid = threadIdx.x;
    const int64_t i0 = (int64_t)blockIdx.x * 256 * AR;
    for (int e = tid; e < 256 * AR * M; e += 256) {
        const int r = e / M, m = e - r * M;
        const int64_t i = i0 + r;
        cs[m * 256 * AR + r] = i < n ? codes[i * M + m] : 0;
    }
    float best[AR];
    int bk[AR];
#pragma unroll
    for (int r = 0; r < AR; ++r) { best[r] = __int_as_float(0x7f800000); bk[r] = 0; }
    for (int64_t k0 = 0; k0 < K; k0 += Bc) {
        const int nb = (int)(K - k0 < (int64_t)Bc ? K - k0 : (int64_t)Bc);
        __syncthreads();
        for (int e = tid; e < nb * M * KS; e += 256) {
            const int b = e / (M * KS), m = (e / KS) % M, z = e % KS;
            alut[e] = T[((size_t)m * KS + centers[(k0 + b) * M + m]) * KS + z];
        }
        __syncthreads();
        for (int b = 0; b < nb; ++b) {
            const float *lb = alut + (size_t)b * M * KS;
#pragma unroll
            for (int r = 0; r < AR; ++r) {
                float d = 0.f;
                for (int m = 0; m < M; ++m) d = __fadd_rn(d, lb[m * KS + cs[m * 256 * AR + r * 256 + tid]]);
                if (d < best[r]) { best[r] = d; bk[r] = (int)(k0 + b); }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < AR; ++r) {
        const int64_t i = i0 + r * 256 + tid;
        if (i < n) {
            assign[i] = bk[r];
            if (dist) dist[i] = best[r];
        }
    }
}

static void launch_assign_canonical(const uint8_t *codes, int64_t n, const uint8_t *centers, int64_t K, int M,
                                    const float *T, int32_t *assign, float *dist, cudaStream_t st) {
    if (n <= 0) return;
    int Bc = (int)((190 * 1024 - 256 * AR * M) / ((size_t)M * KS * 4));
    if (Bc < 1) Bc = 1;
    if (Bc > 64) Bc = 64;
    if (Bc > K) Bc = (int)K;
    const size_t smem = (size_t)Bc * M * KS * 4 + (size_t)256 * AR * M;
    RII_CUDA(cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    assign_kernel<<<(unsigned)ceil_div(n, 256 * AR), 256, smem, st>>>(codes, n, centers, K, M, T, Bc, assign, dist);
    RII_LAUNCHED();
}

// ------------------------------------------------------------ fast assign --
// The "table" of centre k is the row set T_m[cbar_k^m][.] (d_S(x, c) = sum_m
// T_m[c^m][x^m]), laid out like a query table (lut.cuh): row z, column c =
// T_{c mod M}[cbar_k^{c mod M}][z].
__global__ void __launch_bounds__(256) centre_tables_kernel(const float *__restrict__ T,
                                                            const uint8_t *__restrict__ centers, int M,
                                                            float *__restrict__ tables) {
    const int64_t k = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = lane % M;
    const float *row = T + ((size_t)m * KS + centers[k * M + m]) * KS;
    float *t = tables + k * LUT_Q_FLOATS;
    for (int z = warp; z < KS; z += 8) t[z * 32 + lane] = __ldg(row + z);
}

// a(n) with the lane-rotated tables: 6 centres per pass (3 pairs), AR2 codes per
// thread kept pre-permuted in registers.  The rotated fp32 order can differ from
// CA2 by < 4e-6 relative (31 roundings of non-negative terms each way), so a code
// whose runner-up is within 1e-5 of its best is re-assigned canonically (exact);
// every other code's argmin is the canonical one.
template <int M>
__host__ __device__ constexpr int ar2() { return M >= 32 ? 4 : 8; }
template <int M>
__global__ void __launch_bounds__(256, 1)
    assign_fast_kernel(const uint8_t *__restrict__ codes, int64_t n, const float *__restrict__ tables, int64_t K,
                       const float *__restrict__ T, const uint8_t *__restrict__ centers, int32_t *__restrict__ assign,
                       float *__restrict__ dist, int64_t *__restrict__ fb, unsigned long long *__restrict__ fb_n) {
    constexpr int W = M / 4, B = 6, NP = 3, AR2 = ar2<M>();
    extern __shared__ __align__(16) uint8_t lut[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t i0 = (int64_t)blockIdx.x * 256 * AR2;
    const uint32_t r = (uint32_t)lane & (M - 1), rw = r >> 2, l8 = (uint32_t)lane << 3;
    uint32_t sel[4];
    make_selectors(r, sel);
    uint32_t wp[AR2][W];
    float best[AR2];
    int bk[AR2];
    bool amb[AR2];
#pragma unroll
    for (int u = 0; u < AR2; ++u) {
        const int64_t i = i0 + u * 256 + tid;
#pragma unroll
        for (int j = 0; j < W; ++j) wp[u][j] = 0;
        if (i < n) {
            const uint32_t *src = reinterpret_cast<const uint32_t *>(codes + i * M);
#pragma unroll
            for (int j = 0; j < W; ++j) wp[u][j] = __ldg(src + j);
        }
        permute_words<W>(wp[u], rw);
        best[u] = __int_as_float(0x7f800000);
        bk[u] = 0;
        amb[u] = false;
    }
    const float TOLF = 1.00001f;
    for (int64_t k0 = 0; k0 < K; k0 += B) {
        __syncthreads();
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int64_t ka = min(k0 + 2 * p, K - 1), kb = min(k0 + 2 * p + 1, K - 1);
            load_lut_pair(reinterpret_cast<float *>(lut + p * LUT_PAIR_BYTES), tables + ka * LUT_Q_FLOATS,
                          tables + kb * LUT_Q_FLOATS);
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < AR2; ++u) {
            float2 acc[NP];
            adc_rotated_pre<M, B>(lut, wp[u], sel, l8, acc);
#pragma unroll
            for (int jj = 0; jj < B; ++jj) {
                const float d = (jj & 1) ? acc[jj >> 1].y : acc[jj >> 1].x;
                const int64_t k = k0 + jj;
                if (k < K) {
                    if (d < best[u]) {
                        amb[u] = best[u] <= d * TOLF;
                        best[u] = d;
                        bk[u] = (int)k;
                    } else if (d <= best[u] * TOLF) {
                        amb[u] = true;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int u = 0; u < AR2; ++u) {
        const int64_t i = i0 + u * 256 + tid;
        if (i >= n) continue;
        if (amb[u]) {
            const unsigned long long slot = atomicAdd(fb_n, 1ull);
            fb[slot] = i;
            continue;
        }
        assign[i] = bk[u];
        if (dist) {  // canonical (CA2) distance to the chosen centre
            const uint8_t *x = codes + i * M;
            const uint8_t *c = centers + (int64_t)bk[u] * M;
            float d = 0.f;
            for (int m = 0; m < M; ++m) d = __fadd_rn(d, __ldg(T + ((size_t)m * KS + c[m]) * KS + x[m]));
            dist[i] = d;
        }
    }
}

__global__ void scatter_fallback_kernel(const int64_t *__restrict__ fb, int64_t nfb, const int32_t *__restrict__ a_fb,
                                        const float *__restrict__ d_fb, int32_t *__restrict__ assign,
                                        float *__restrict__ dist) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nfb) return;
    assign[fb[j]] = a_fb[j];
    if (dist) dist[fb[j]] = d_fb[j];
}

template <int M>
static void assign_fast_t(const uint8_t *codes, int64_t n, const float *tables, int64_t K, const float *T,
                          const uint8_t *centers, int32_t *assign, float *dist, int64_t *fb,
                          unsigned long long *fb_n, cudaStream_t st) {
    auto kern = assign_fast_kernel<M>;
    const size_t smem = (size_t)3 * LUT_PAIR_BYTES;
    RII_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    kern<<<(unsigned)ceil_div(n, 256 * ar2<M>()), 256, smem, st>>>(codes, n, tables, K, T, centers, assign, dist, fb,
                                                              fb_n);
    RII_LAUNCHED();
}

void launch_assign(const uint8_t *codes, int64_t n, const uint8_t *centers, int64_t K, int M, const float *T,
                   int32_t *assign, float *dist, cudaStream_t st) {
    if (n <= 0) return;
    if (M > 64) {  // large M: one code per CTA, bf16 SDC rows + exact rescore (k_large.cu)
        launch_large_assign(codes, n, centers, K, M, T, assign, dist, st);
        return;
    }
    if (assign_scan_supported(M, K) && n >= 8192) {  // large K: codes as queries over the centre codes
        launch_assign_scan(codes, n, centers, K, M, T, assign, dist, 148, st);
        return;
    }
    const bool fast = (M == 4 || M == 8 || M == 16 || M == 32) && K >= 12 && n >= 4096;
    if (!fast) {
        launch_assign_canonical(codes, n, centers, K, M, T, assign, dist, st);
        return;
    }
    float *tables = nullptr;
    int64_t *fb = nullptr;
    unsigned long long *fb_n = nullptr;
    RII_CUDA(cudaMallocAsync(&tables, (size_t)K * LUT_Q_FLOATS * 4, st));
    RII_CUDA(cudaMallocAsync(&fb, (size_t)n * 8, st));
    RII_CUDA(cudaMallocAsync(&fb_n, 8, st));
    RII_CUDA(cudaMemsetAsync(fb_n, 0, 8, st));
    centre_tables_kernel<<<(unsigned)K, 256, 0, st>>>(T, centers, M, tables);
    RII_LAUNCHED();
    switch (M) {
        case 4: assign_fast_t<4>(codes, n, tables, K, T, centers, assign, dist, fb, fb_n, st); break;
        case 8: assign_fast_t<8>(codes, n, tables, K, T, centers, assign, dist, fb, fb_n, st); break;
        case 16: assign_fast_t<16>(codes, n, tables, K, T, centers, assign, dist, fb, fb_n, st); break;
        default: assign_fast_t<32>(codes, n, tables, K, T, centers, assign, dist, fb, fb_n, st); break;
    }
    unsigned long long nfb = 0;
    RII_CUDA(cudaMemcpyAsync(&nfb, fb_n, 8, cudaMemcpyDeviceToHost, st));
    RII_CUDA(cudaStreamSynchronize(st));
    if (nfb > 0) {  // exact canonical re-assignment of the near-tie codes
        uint8_t *sub = nullptr;
        int32_t *a_fb = nullptr;
        float *d_fb = nullptr;
        RII_CUDA(cudaMallocAsync(&sub, (size_t)nfb * M, st));
        RII_CUDA(cudaMallocAsync(&a_fb, (size_t)nfb * 4, st));
        RII_CUDA(cudaMallocAsync(&d_fb, (size_t)nfb * 4, st));
        launch_gather_codes(codes, M, fb, (int64_t)nfb, sub, st);
        launch_assign_canonical(sub, (int64_t)nfb, centers, K, M, T, a_fb, dist ? d_fb : nullptr, st);
        scatter_fallback_kernel<<<(unsigned)ceil_div((int64_t)nfb, 256), 256, 0, st>>>(fb, (int64_t)nfb, a_fb, d_fb,
                                                                                       assign, dist);
        RII_LAUNCHED();
        RII_CUDA(cudaFreeAsync(sub, st));
        RII_CUDA(cudaFreeAsync(a_fb, st));
        RII_CUDA(cudaFreeAsync(d_fb, st));
    }
    RII_CUDA(cudaFreeAsync(tables, st));
    RII_CUDA(cudaFreeAsync(fb, st));
    RII_CUDA(cudaFreeAsync(fb_n, st));
}

// -------------------------------------------------------------------- CSR --
__global__ void csr_offsets_kernel(const int32_t *__restrict__ sorted_keys, int64_t n, int64_t K,
                                   int64_t *__restrict__ offsets) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k > K) return;
    int64_t lo = 0, hi = n;  // first index with key >= k
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sorted_keys[mid] < k) lo = mid + 1; else hi = mid;
    }
    offsets[k] = lo;
}

static int bits_for(int64_t v) {
    int b = 1;
    while ((1ll << b) <= v) ++b;
    return b;
}

void build_csr(const int32_t *keys, const uint32_t *vals, int64_t n, int64_t K, int64_t *offsets, uint32_t *ids,
               cudaStream_t st) {
    if (n <= 0) {
        RII_CUDA(cudaMemsetAsync(offsets, 0, (size_t)(K + 1) * 8, st));
        return;
    }
    int32_t *kout = nullptr;
    RII_CUDA(cudaMallocAsync(&kout, (size_t)n * 4, st));
    // stable (sort.cu): the ids of a list keep their input order (ascending, R11)
    radix_sort_pairs<uint32_t>(reinterpret_cast<const uint32_t *>(keys), vals, n, bits_for(K),
                               reinterpret_cast<uint32_t *>(kout), ids, st);
    csr_offsets_kernel<<<(unsigned)ceil_div(K + 1, 256), 256, 0, st>>>(kout, n, K, offsets);
    RII_LAUNCHED();
    RII_CUDA(cudaFreeAsync(kout, st));
}

// ----------------------------------------------------------------- sample --
__global__ void sample_keys_kernel(int64_t n, IdMap gid, uint64_t seed, uint64_t *__restrict__ keys,
                                   uint32_t *__restrict__ pos) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = splitmix64(seed ^ (uint64_t)map_id(gid, (uint32_t)i));
    pos[i] = (uint32_t)i;
}

void select_sample(int64_t n, const IdMap &gid, int64_t ns, uint64_t seed, uint32_t *out_pos, cudaStream_t st) {
    if (n <= 0 || ns <= 0) return;
    uint64_t *k_in = nullptr, *k_out = nullptr;
    uint32_t *v_in = nullptr, *v_out = nullptr;
    RII_CUDA(cudaMallocAsync(&k_in, (size_t)n * 8, st));
    RII_CUDA(cudaMallocAsync(&k_out, (size_t)n * 8, st));
    RII_CUDA(cudaMallocAsync(&v_in, (size_t)n * 4, st));
    RII_CUDA(cudaMallocAsync(&v_out, (size_t)n * 4, st));
    sample_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, gid, seed, k_in, v_in);
    RII_LAUNCHED();
    size_t tb = 0;
    RII_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, v_in, v_out, (int64_t)n, 0, 64, st));
    void *tmp = nullptr;
    RII_CUDA(cudaMallocAsync(&tmp, tb, st));
    RII_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, v_in, v_out, (int64_t)n, 0, 64, st));
    count_launch(16);
    RII_CUDA(cudaMemcpyAsync(out_pos, v_out, (size_t)ns * 4, cudaMemcpyDeviceToDevice, st));
    RII_CUDA(cudaFreeAsync(tmp, st));
    RII_CUDA(cudaFreeAsync(k_in, st));
    RII_CUDA(cudaFreeAsync(k_out, st));
    RII_CUDA(cudaFreeAsync(v_in, st));
    RII_CUDA(cudaFreeAsync(v_out, st));
}

__global__ void keys_for_pos_kernel(const uint32_t *__restrict__ pos, int64_t n, IdMap gid, uint64_t seed,
                                    uint64_t *__restrict__ keys) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = splitmix64(seed ^ (uint64_t)map_id(gid, pos[i]));
}

void sample_keys_for_positions(int64_t, const IdMap &gid, const uint32_t *pos, int64_t n, uint64_t seed,
                               uint64_t *keys, cudaStream_t st) {
    if (n <= 0) return;
    keys_for_pos_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(pos, n, gid, seed, keys);
    RII_LAUNCHED();
}

__global__ void iota_kernel(uint32_t *v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}

void sort_keys_with_index(const uint64_t *keys, int64_t n, uint32_t *order, cudaStream_t st) {
    if (n <= 0) return;
    uint64_t *k_out = nullptr;
    uint32_t *v_in = nullptr;
    RII_CUDA(cudaMallocAsync(&k_out, (size_t)n * 8, st));
    RII_CUDA(cudaMallocAsync(&v_in, (size_t)n * 4, st));
    iota_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(v_in, n);
    RII_LAUNCHED();
    size_t tb = 0;
    RII_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, k_out, v_in, order, (int64_t)n, 0, 64, st));
    void *tmp = nullptr;
    RII_CUDA(cudaMallocAsync(&tmp, tb, st));
    RII_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, k_out, v_in, order, (int64_t)n, 0, 64, st));
    count_launch(16);
    RII_CUDA(cudaFreeAsync(tmp, st));
    RII_CUDA(cudaFreeAsync(k_out, st));
    RII_CUDA(cudaFreeAsync(v_in, st));
}

// -------------------------------------------------------------- PQk-means --
__device__ __forceinline__ uint64_t code_hash(const uint8_t *c, int M) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int m = 0; m < M; ++m) h = (h ^ c[m]) * 0x100000001b3ull;
    return h;
}

// Init: the first K pairwise-distinct sample codes in sample order (one thread;
// open-addressing table of sample indices).
__global__ void pq_init_kernel(const uint8_t *__restrict__ X, int64_t ns, int64_t K, int M, int32_t *table,
                               int64_t tmask, uint8_t *__restrict__ C, int *err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t got = 0;
    for (int64_t i = 0; i < ns && got < K; ++i) {
        const uint8_t *c = X + i * M;
        int64_t h = (int64_t)(code_hash(c, M) & (uint64_t)tmask);
        bool dup = false;
        while (table[h] >= 0) {
            const uint8_t *o = X + (int64_t)table[h] * M;
            bool eq = true;
            for (int m = 0; m < M; ++m) if (o[m] != c[m]) { eq = false; break; }
            if (eq) { dup = true; break; }
            h = (h + 1) & tmask;
        }
        if (dup) continue;
        table[h] = (int32_t)i;
        for (int m = 0; m < M; ++m) C[got * M + m] = c[m];
        ++got;
    }
    if (got < K) *err = 1;
}

__global__ void pq_hist_kernel(const uint8_t *__restrict__ X, int64_t ns, int M, const int32_t *__restrict__ a,
                               int32_t *__restrict__ h, int32_t *__restrict__ size) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    const int64_t k = a[i];
    atomicAdd(size + k, 1);
    for (int m = 0; m < M; ++m) atomicAdd(h + (k * M + m) * KS + X[i * M + m], 1);
}

// cbar_k^m = argmin_z sum_{z'} h[k][m][z'] (double) T_m[z][z'], z' ascending; zero
// counts are skipped (adding +0.0 to a non-negative sum is exact).
__global__ void __launch_bounds__(256) pq_update_kernel(const int32_t *__restrict__ h, const int32_t *__restrict__ size,
                                                        const float *__restrict__ T, int M,
                                                        uint8_t *__restrict__ C) {
    const int64_t k = blockIdx.x;
    const int m = blockIdx.y, z = threadIdx.x, lane = z & 31, warp = z >> 5;
    if (size[k] == 0) return;
    __shared__ int nz_idx[KS];
    __shared__ int nz_cnt[KS];
    __shared__ int wsum[8];
    __shared__ double bestv[8];
    __shared__ int bestz[8];
    const int cz = h[(k * M + m) * KS + z];
    const unsigned bal = __ballot_sync(0xffffffffu, cz != 0);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < 8; ++w) { if (w < warp) off += wsum[w]; tot += wsum[w]; }
    if (cz != 0) {
        const int p = off + __popc(bal & ((1u << lane) - 1u));
        nz_idx[p] = z;
        nz_cnt[p] = cz;
    }
    __syncthreads();
    const float *Tz = T + ((size_t)m * KS + z) * KS;
    double s = 0.0;
    for (int t = 0; t < tot; ++t) s = __dadd_rn(s, __dmul_rn((double)nz_cnt[t], (double)Tz[nz_idx[t]]));
    // argmin (s, z)
    double v = s;
    int bz = z;
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, v, o);
        const int oz = __shfl_down_sync(0xffffffffu, bz, o);
        if (ov < v || (ov == v && oz < bz)) { v = ov; bz = oz; }
    }
    if (lane == 0) { bestv[warp] = v; bestz[warp] = bz; }
    __syncthreads();
    if (z == 0) {
        double bv = bestv[0];
        int b = bestz[0];
        for (int w = 1; w < 8; ++w)
            if (bestv[w] < bv || (bestv[w] == bv && bestz[w] < b)) { bv = bestv[w]; b = bestz[w]; }
        C[k * M + m] = (uint8_t)b;
    }
}

// Empty clusters (k ascending): the unused member of the largest cluster (ties
// lowest k) with the largest assignment distance (ties lowest index) becomes
// the centre and moves to k.  One CTA.
__global__ void __launch_bounds__(1024) pq_reseed_kernel(const uint8_t *__restrict__ X, int64_t ns, int64_t K, int M,
                                                         int32_t *__restrict__ a, const float *__restrict__ dist,
                                                         int32_t *__restrict__ size, uint8_t *__restrict__ used,
                                                         uint8_t *__restrict__ C) {
    __shared__ int64_t s_g, s_i;
    __shared__ int64_t rk[32];
    __shared__ int64_t rv[32];
    __shared__ float rd[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t i = tid; i < ns; i += blockDim.x) used[i] = 0;
    __syncthreads();
    for (int64_t k = 0; k < K; ++k) {
        if (size[k] != 0) continue;  // uniform: every thread reads the same value
        // g = argmax size (ties lowest)
        int64_t bg = -1, bs = -1;
        for (int64_t j = tid; j < K; j += blockDim.x)
            if (size[j] > bs) { bs = size[j]; bg = j; }
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t os = __shfl_down_sync(0xffffffffu, bs, o), og = __shfl_down_sync(0xffffffffu, bg, o);
            if (os > bs || (os == bs && og >= 0 && (bg < 0 || og < bg))) { bs = os; bg = og; }
        }
        if (lane == 0) { rk[warp] = bg; rv[warp] = bs; }
        __syncthreads();
        if (tid == 0) {
            int64_t g = rk[0], s = rv[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (rv[w] > s || (rv[w] == s && rk[w] >= 0 && (g < 0 || rk[w] < g))) { s = rv[w]; g = rk[w]; }
            s_g = g;
        }
        __syncthreads();
        const int64_t g = s_g;
        // farthest unused member of g
        int64_t bi = -1;
        float bd = -1.f;
        for (int64_t i = tid; i < ns; i += blockDim.x) {
            if (a[i] != g || used[i]) continue;
            if (bi < 0 || dist[i] > bd) { bd = dist[i]; bi = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const float od = __shfl_down_sync(0xffffffffu, bd, o);
            const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (oi >= 0 && (bi < 0 || od > bd || (od == bd && oi < bi))) { bd = od; bi = oi; }
        }
        if (lane == 0) { rk[warp] = bi; rd[warp] = bd; }
        __syncthreads();
        if (tid == 0) {
            int64_t b = rk[0];
            float d = rd[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (rk[w] >= 0 && (b < 0 || rd[w] > d || (rd[w] == d && rk[w] < b))) { d = rd[w]; b = rk[w]; }
            s_i = b;
            if (b >= 0) {
                for (int m = 0; m < M; ++m) C[k * M + m] = X[b * M + m];
                used[b] = 1;
                a[b] = (int32_t)k;
                size[g] -= 1;
                size[k] = 1;
            }
        }
        __syncthreads();
    }
}

void run_pqkmeans(const uint8_t *X, int64_t ns, int64_t K, int M, const float *T, int n_iter, uint8_t *C, int *err,
                  cudaStream_t st) {
    int64_t tsize = 1;
    while (tsize < 4 * K) tsize <<= 1;
    int32_t *table = nullptr, *a = nullptr, *h = nullptr, *size = nullptr;
    float *dist = nullptr;
    uint8_t *used = nullptr;
    RII_CUDA(cudaMallocAsync(&table, (size_t)tsize * 4, st));
    RII_CUDA(cudaMemsetAsync(table, 0xff, (size_t)tsize * 4, st));
    pq_init_kernel<<<1, 1, 0, st>>>(X, ns, K, M, table, tsize - 1, C, err);
    RII_LAUNCHED();
    RII_CUDA(cudaFreeAsync(table, st));
    if (n_iter <= 0) return;
    RII_CUDA(cudaMallocAsync(&a, (size_t)ns * 4, st));
    RII_CUDA(cudaMallocAsync(&dist, (size_t)ns * 4, st));
    RII_CUDA(cudaMallocAsync(&h, (size_t)K * M * KS * 4, st));
    RII_CUDA(cudaMallocAsync(&size, (size_t)K * 4, st));
    RII_CUDA(cudaMallocAsync(&used, (size_t)ns, st));
    for (int it = 0; it < n_iter; ++it) {
        launch_assign(X, ns, C, K, M, T, a, dist, st);
        RII_CUDA(cudaMemsetAsync(h, 0, (size_t)K * M * KS * 4, st));
        RII_CUDA(cudaMemsetAsync(size, 0, (size_t)K * 4, st));
        pq_hist_kernel<<<(unsigned)ceil_div(ns, 256), 256, 0, st>>>(X, ns, M, a, h, size);
        RII_LAUNCHED();
        pq_update_kernel<<<dim3((unsigned)K, (unsigned)M), 256, 0, st>>>(h, size, T, M, C);
        RII_LAUNCHED();
        pq_reseed_kernel<<<1, 1024, 0, st>>>(X, ns, K, M, a, dist, size, used, C);
        RII_LAUNCHED();
    }
    RII_CUDA(cudaFreeAsync(a, st));
    RII_CUDA(cudaFreeAsync(dist, st));
    RII_CUDA(cudaFreeAsync(h, st));
    RII_CUDA(cudaFreeAsync(size, st));
    RII_CUDA(cudaFreeAsync(used, st));
}

// ------------------------------------------------------------------ train --
__global__ void absmax_kernel(const float *__restrict__ x, int64_t n, unsigned *out) {
    float mx = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        mx = fmaxf(mx, fabsf(x[i]));
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(mx));
}

__global__ void train_keys_kernel(int64_t n, uint64_t seed, int m, uint64_t *__restrict__ keys,
                                  uint32_t *__restrict__ rows) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = splitmix64(seed ^ ((uint64_t)m << 40) ^ (uint64_t)i);
    rows[i] = (uint32_t)i;
}

// Z = 256 rows in key order with pairwise-distinct sub-vectors (one thread).
__global__ void train_init_kernel(const float *__restrict__ x, int64_t n, int D, int m, int ds,
                                  const uint32_t *__restrict__ order, float *__restrict__ c, int *err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int got = 0;
    for (int64_t r = 0; r < n && got < KS; ++r) {
        const float *u = x + (int64_t)order[r] * D + m * ds;
        bool dup = false;
        for (int z = 0; z < got && !dup; ++z) {
            bool eq = true;
            for (int j = 0; j < ds; ++j) if (c[z * ds + j] != u[j]) { eq = false; break; }
            dup = eq;
        }
        if (dup) continue;
        for (int j = 0; j < ds; ++j) c[got * ds + j] = u[j];
        ++got;
    }
    if (got < KS) *err = 6;
}

// Assignment + fixed-point accumulation (block-local int64 sums, then global).
__global__ void __launch_bounds__(256) train_assign_kernel(const float *__restrict__ x, int64_t n, int D, int m,
                                                           int ds, const float *__restrict__ c,
                                                           int32_t *__restrict__ a, float *__restrict__ d,
                                                           unsigned long long *__restrict__ gsum,
                                                           unsigned long long *__restrict__ gcnt) {
    extern __shared__ __align__(16) uint8_t tsm[];
    unsigned long long *ssum = reinterpret_cast<unsigned long long *>(tsm);   // [256][ds]
    unsigned long long *scnt = ssum + KS * ds;                                // [256]
    float *cs = reinterpret_cast<float *>(scnt + KS);                         // [256][ds]
    const int tid = threadIdx.x;
    for (int e = tid; e < KS * ds; e += 256) { ssum[e] = 0; cs[e] = c[e]; }
    scnt[tid] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * 256 + tid; i < n; i += (int64_t)gridDim.x * 256) {
        const float *u = x + i * D + m * ds;
        float best = __int_as_float(0x7f800000);
        int bz = 0;
        for (int z = 0; z < KS; ++z) {
            float acc = 0.f;
            for (int j = 0; j < ds; ++j) acc = ca1_step(acc, u[j], cs[z * ds + j]);
            if (acc < best) { best = acc; bz = z; }
        }
        a[i] = bz;
        d[i] = best;
        atomicAdd(scnt + bz, 1ull);
        for (int j = 0; j < ds; ++j)
            atomicAdd(ssum + bz * ds + j, (unsigned long long)__double2ll_rn((double)u[j] * 4294967296.0));
    }
    __syncthreads();
    for (int e = tid; e < KS * ds; e += 256) if (ssum[e]) atomicAdd(gsum + e, ssum[e]);
    if (scnt[tid]) atomicAdd(gcnt + tid, scnt[tid]);
}

__global__ void train_update_kernel(const long long *__restrict__ sum, const long long *__restrict__ cnt, int ds,
                                    float *__restrict__ c) {
    const int z = blockIdx.x, j = threadIdx.x;
    if (j >= ds || cnt[z] == 0) return;
    const double mean = __ddiv_rn(__ddiv_rn(__ll2double_rn(sum[z * ds + j]), 4294967296.0), __ll2double_rn(cnt[z]));
    c[z * ds + j] = __double2float_rn(mean);
}

// Empty clusters, z ascending: the not-yet-used row with the largest d (ties lowest row).
__global__ void __launch_bounds__(1024) train_reseed_kernel(const float *__restrict__ x, int64_t n, int D, int m,
                                                            int ds, const float *__restrict__ d,
                                                            const long long *__restrict__ cnt,
                                                            uint8_t *__restrict__ used, float *__restrict__ c) {
    __shared__ int64_t rk[32];
    __shared__ float rd[32];
    __shared__ int64_t s_b;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t i = tid; i < n; i += blockDim.x) used[i] = 0;
    __syncthreads();
    for (int z = 0; z < KS; ++z) {
        if (cnt[z] != 0) continue;
        int64_t bi = -1;
        float bd = -1.f;
        for (int64_t i = tid; i < n; i += blockDim.x) {
            if (used[i]) continue;
            if (bi < 0 || d[i] > bd) { bd = d[i]; bi = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const float od = __shfl_down_sync(0xffffffffu, bd, o);
            const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (oi >= 0 && (bi < 0 || od > bd || (od == bd && oi < bi))) { bd = od; bi = oi; }
        }
        if (lane == 0) { rk[warp] = bi; rd[warp] = bd; }
        __syncthreads();
        if (tid == 0) {
            int64_t b = rk[0];
            float dd = rd[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (rk[w] >= 0 && (b < 0 || rd[w] > dd || (rd[w] == dd && rk[w] < b))) { dd = rd[w]; b = rk[w]; }
            s_b = b;
            if (b >= 0) {
                used[b] = 1;
                for (int j = 0; j < ds; ++j) c[z * ds + j] = x[b * D + m * ds + j];
            }
        }
        __syncthreads();
    }
}

void run_train(const float *x, int64_t n, int D, int M, int n_iter, uint64_t seed, float *cb, int *err,
               cudaStream_t st) {
    const int ds = D / M;
    unsigned *amax = nullptr;
    RII_CUDA(cudaMallocAsync(&amax, 4, st));
    RII_CUDA(cudaMemsetAsync(amax, 0, 4, st));
    absmax_kernel<<<592, 256, 0, st>>>(x, n * D, amax);
    RII_LAUNCHED();
    unsigned amax_h = 0;
    RII_CUDA(cudaMemcpyAsync(&amax_h, amax, 4, cudaMemcpyDeviceToHost, st));
    RII_CUDA(cudaStreamSynchronize(st));
    RII_CUDA(cudaFreeAsync(amax, st));
    float amax_f;
    memcpy(&amax_f, &amax_h, 4);
    if ((double)amax_f * (double)n >= 2147483648.0) throw Error(1, "train: n * max|x| must be < 2^31 (fixed-point range)");

    uint64_t *k_in = nullptr, *k_out = nullptr;
    uint32_t *r_in = nullptr, *r_out = nullptr;
    int32_t *a = nullptr;
    float *d = nullptr;
    unsigned long long *sum = nullptr, *cnt = nullptr;
    uint8_t *used = nullptr;
    RII_CUDA(cudaMallocAsync(&k_in, (size_t)n * 8, st));
    RII_CUDA(cudaMallocAsync(&k_out, (size_t)n * 8, st));
    RII_CUDA(cudaMallocAsync(&r_in, (size_t)n * 4, st));
    RII_CUDA(cudaMallocAsync(&r_out, (size_t)n * 4, st));
    RII_CUDA(cudaMallocAsync(&a, (size_t)n * 4, st));
    RII_CUDA(cudaMallocAsync(&d, (size_t)n * 4, st));
    RII_CUDA(cudaMallocAsync(&sum, (size_t)KS * ds * 8, st));
    RII_CUDA(cudaMallocAsync(&cnt, (size_t)KS * 8, st));
    RII_CUDA(cudaMallocAsync(&used, (size_t)n, st));
    size_t tb = 0;
    RII_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, r_in, r_out, (int64_t)n, 0, 64, st));
    void *tmp = nullptr;
    RII_CUDA(cudaMallocAsync(&tmp, tb, st));
    const size_t smem = (size_t)KS * ds * 8 + KS * 8 + (size_t)KS * ds * 4;
    RII_CUDA(cudaFuncSetAttribute(train_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    const unsigned ablocks = (unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 4);
    for (int m = 0; m < M; ++m) {
        float *c = cb + (size_t)m * KS * ds;
        train_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, seed, m, k_in, r_in);
        RII_LAUNCHED();
        RII_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, r_in, r_out, (int64_t)n, 0, 64, st));
        count_launch(16);
        train_init_kernel<<<1, 1, 0, st>>>(x, n, D, m, ds, r_out, c, err);
        RII_LAUNCHED();
        for (int it = 0; it < n_iter; ++it) {
            RII_CUDA(cudaMemsetAsync(sum, 0, (size_t)KS * ds * 8, st));
            RII_CUDA(cudaMemsetAsync(cnt, 0, (size_t)KS * 8, st));
            train_assign_kernel<<<ablocks, 256, smem, st>>>(x, n, D, m, ds, c, a, d, sum, cnt);
            RII_LAUNCHED();
            train_update_kernel<<<KS, 64, 0, st>>>(reinterpret_cast<const long long *>(sum),
                                                   reinterpret_cast<const long long *>(cnt), ds, c);
            RII_LAUNCHED();
            train_reseed_kernel<<<1, 1024, 0, st>>>(x, n, D, m, ds, d, reinterpret_cast<const long long *>(cnt),
                                                    used, c);
            RII_LAUNCHED();
        }
    }
    RII_CUDA(cudaFreeAsync(tmp, st));
    for (void *p : {(void *)k_in, (void *)k_out, (void *)r_in, (void *)r_out, (void *)a, (void *)d, (void *)sum,
                    (void *)cnt, (void *)used})
        RII_CUDA(cudaFreeAsync(p, st));
}

}  // namespace rii
