// sort.cu -- the library's own stable sorts and scans (no CUB on the query path).
//
// Where they serve the method: grouping (query, probe rank) pairs by posting list
// and restricting the posting lists to a target set S (Alg. 2 L7-L13 executed
// list-major; R7: result-identical alternatives to the paper's binary-search
// membership test), ordering list-major work items by probe rank, the CSR of the
// posting lists after add / reconfigure (ids ascending inside a list, R11), and the
// (d0, k) ranking of the paper-exact mode (Alg. 2 L6, ties to the lowest k, CA4).
//
// Radix sort: LSD, 8-bit digits, stable.  One pass = three kernels:
//   upsweep   -- CTA b counts the digits of its 1024-element tile: hist[d * G + b]
//   scan      -- exclusive scan of hist (digit-major), so hist[d * G + b] becomes the
//                first output slot of digit d in tile b
//   downsweep -- CTA b ranks its elements stably: inside a warp by __match_any_sync
//                (peers with the same digit, lower lanes first), across the CTA's 32
//                warps by a per-digit exclusive scan of the warp counts; element i of
//                tile b with digit d goes to hist[d * G + b] + (earlier warps' d) +
//                (lower lanes' d).
// Each pass is a stable counting sort on one digit, so the passes compose into a
// stable sort on the low `bits` bits of the key (values travel with their keys).
#include <algorithm>

#include "kernels.cuh"

namespace rii {

namespace {

constexpr int SORT_NT = 1024;   // threads per CTA = elements per tile
constexpr int SCAN_NT = 1024;
// elements per thread of a scan tile (a tile of 32 KB in shared memory)
template <class T>
__host__ __device__ constexpr int scan_ipt() { return sizeof(T) == 8 ? 4 : 8; }

// ------------------------------------------------------------------ scan ---
// Block-wide exclusive scan of one value per thread; returns the block total in *total.
template <class T>
__device__ __forceinline__ T block_exclusive_scan(T v, T *warp_sums, T *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        T w = lane < nw ? warp_sums[lane] : T(0);
        T wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < nw) warp_sums[lane] = wi - w;  // exclusive prefix of each warp
        if (lane == nw - 1) *total = wi;
    }
    __syncthreads();
    return inc - v + warp_sums[warp];
}

// partial[b] = sum of tile b
template <class T>
__global__ void __launch_bounds__(SCAN_NT) scan_reduce_kernel(const T *__restrict__ in, int64_t n,
                                                              T *__restrict__ partial) {
    constexpr int SCAN_IPT = scan_ipt<T>(), SCAN_TILE = SCAN_NT * SCAN_IPT;
    __shared__ T ws[32];
    __shared__ T tot;
    const int64_t t0 = (int64_t)blockIdx.x * SCAN_TILE;
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {
        const int64_t e = t0 + (int64_t)i * SCAN_NT + threadIdx.x;
        if (e < n) s += in[e];
    }
    block_exclusive_scan<T>(s, ws, &tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// out[e] = base[b] + exclusive prefix of e inside tile b (in and out may alias)
template <class T>
__global__ void __launch_bounds__(SCAN_NT) scan_apply_kernel(const T *in, int64_t n, const T *__restrict__ base,
                                                             T *out) {
    constexpr int SCAN_IPT = scan_ipt<T>(), SCAN_TILE = SCAN_NT * SCAN_IPT;
    __shared__ T tile[SCAN_TILE];
    __shared__ T ws[32];
    __shared__ T tot;
    const int64_t t0 = (int64_t)blockIdx.x * SCAN_TILE;
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {  // coalesced load into shared memory
        const int64_t e = t0 + (int64_t)i * SCAN_NT + threadIdx.x;
        tile[i * SCAN_NT + threadIdx.x] = e < n ? in[e] : T(0);
    }
    __syncthreads();
    T v[SCAN_IPT], s = 0;  // thread t owns the contiguous elements [t * IPT, (t + 1) * IPT)
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {
        v[i] = tile[threadIdx.x * SCAN_IPT + i];
        s += v[i];
    }
    T run = block_exclusive_scan<T>(s, ws, &tot) + (base ? base[blockIdx.x] : T(0));
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {
        tile[threadIdx.x * SCAN_IPT + i] = run;
        run += v[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {
        const int64_t e = t0 + (int64_t)i * SCAN_NT + threadIdx.x;
        if (e < n) out[e] = tile[i * SCAN_NT + threadIdx.x];
    }
}

template <class T>
void exclusive_scan_t(const T *in, int64_t n, T *out, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t G = ceil_div(n, (int64_t)SCAN_NT * scan_ipt<T>());
    if (G == 1) {
        scan_apply_kernel<T><<<1, SCAN_NT, 0, st>>>(in, n, nullptr, out);
        RII_LAUNCHED();
        return;
    }
    T *partial = nullptr;
    RII_CUDA(cudaMallocAsync(&partial, (size_t)G * sizeof(T), st));
    scan_reduce_kernel<T><<<(unsigned)G, SCAN_NT, 0, st>>>(in, n, partial);
    RII_LAUNCHED();
    exclusive_scan_t<T>(partial, G, partial, st);  // tile bases (recursive: G <= n / 4096)
    scan_apply_kernel<T><<<(unsigned)G, SCAN_NT, 0, st>>>(in, n, partial, out);
    RII_LAUNCHED();
    RII_CUDA(cudaFreeAsync(partial, st));
}

// ------------------------------------------------------------ radix sort ---
template <class K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
    return (uint32_t)(k >> shift) & 0xffu;
}

template <class K>
__global__ void __launch_bounds__(SORT_NT) radix_upsweep_kernel(const K *__restrict__ keys, int64_t n, int shift,
                                                                int64_t G, uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[256];
    if (threadIdx.x < 256) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t e = (int64_t)blockIdx.x * SORT_NT + threadIdx.x;
    if (e < n) atomicAdd(&h[digit_of(keys[e], shift)], 1u);
    __syncthreads();
    if (threadIdx.x < 256) hist[(int64_t)threadIdx.x * G + blockIdx.x] = h[threadIdx.x];
}

template <class K>
__global__ void __launch_bounds__(SORT_NT) radix_downsweep_kernel(const K *__restrict__ keys,
                                                                  const uint32_t *__restrict__ vals, int64_t n,
                                                                  int shift, int64_t G,
                                                                  const uint32_t *__restrict__ hist,
                                                                  K *__restrict__ keys_out,
                                                                  uint32_t *__restrict__ vals_out) {
    __shared__ uint32_t wcnt[32][257];  // [warp][digit] counts, then exclusive prefixes over warps
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 32 * 257; i += SORT_NT) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t e = (int64_t)blockIdx.x * SORT_NT + threadIdx.x;
    const bool valid = e < n;
    K k = 0;
    uint32_t v = 0;
    if (valid) {
        k = keys[e];
        v = vals[e];
    }
    const uint32_t d = valid ? digit_of(k, shift) : 256u;  // 256: past the end
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    if (rank == 0) wcnt[warp][d] = __popc(peers);  // the lowest lane of each digit group
    __syncthreads();
    if (threadIdx.x < 256) {  // per digit: exclusive scan over the 32 warps
        uint32_t run = 0;
        for (int w = 0; w < 32; ++w) {
            const uint32_t c = wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
    if (valid) {
        const uint32_t dst = hist[(int64_t)d * G + blockIdx.x] + wcnt[warp][d] + rank;
        keys_out[dst] = k;
        vals_out[dst] = v;
    }
}

}  // namespace

// Stable sort of (keys, vals) by the low `bits` bits of the key.  keys/vals are
// sorted into keys_out / vals_out (which must not alias the inputs); n < 2^32.
template <class K>
void radix_sort_pairs(const K *keys, const uint32_t *vals, int64_t n, int bits, K *keys_out, uint32_t *vals_out,
                      cudaStream_t st) {
    if (n <= 0) return;
    if (n >= ((int64_t)1 << 32)) throw Error(1, "radix sort: n >= 2^32");
    const int passes = std::max(1, (bits + 7) / 8);
    const int64_t G = ceil_div(n, (int64_t)SORT_NT);
    uint32_t *hist = nullptr;
    K *kb = nullptr;
    uint32_t *vb = nullptr;
    RII_CUDA(cudaMallocAsync(&hist, (size_t)256 * G * 4, st));
    if (passes > 1) {
        RII_CUDA(cudaMallocAsync(&kb, (size_t)n * sizeof(K), st));
        RII_CUDA(cudaMallocAsync(&vb, (size_t)n * 4, st));
    }
    // ping-pong so that the last pass writes keys_out / vals_out
    const K *ki = keys;
    const uint32_t *vi = vals;
    for (int p = 0; p < passes; ++p) {
        K *ko = ((passes - 1 - p) & 1) ? kb : keys_out;
        uint32_t *vo = ((passes - 1 - p) & 1) ? vb : vals_out;
        radix_upsweep_kernel<K><<<(unsigned)G, SORT_NT, 0, st>>>(ki, n, 8 * p, G, hist);
        RII_LAUNCHED();
        exclusive_scan_t<uint32_t>(hist, 256 * G, hist, st);
        radix_downsweep_kernel<K><<<(unsigned)G, SORT_NT, 0, st>>>(ki, vi, n, 8 * p, G, hist, ko, vo);
        RII_LAUNCHED();
        ki = ko;
        vi = vo;
    }
    RII_CUDA(cudaFreeAsync(hist, st));
    if (kb) RII_CUDA(cudaFreeAsync(kb, st));
    if (vb) RII_CUDA(cudaFreeAsync(vb, st));
}

template void radix_sort_pairs<uint32_t>(const uint32_t *, const uint32_t *, int64_t, int, uint32_t *, uint32_t *,
                                         cudaStream_t);
template void radix_sort_pairs<uint64_t>(const uint64_t *, const uint32_t *, int64_t, int, uint64_t *, uint32_t *,
                                         cudaStream_t);

void exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, cudaStream_t st) {
    exclusive_scan_t<int64_t>(in, n, out, st);
}

}  // namespace rii
