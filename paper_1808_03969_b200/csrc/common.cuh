// common.cuh -- shared device helpers of the B200 Rii library (sm_100a only).
// Canonical arithmetic CA1/CA2 and the (dist, id) key order follow DESIGN.md
// "Readings" (CA1: P:292-294; CA2: Eq. 2; CA4: ties to the lowest id).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include <atomic>
#include <string>

#include "error.hpp"

namespace rii {

constexpr int KS = 256;                      // code words per subspace
constexpr uint64_t KEY_MAX = ~0ull;          // empty candidate slot
constexpr int NT = 256;                      // threads per CTA of the scan kernels
// The dynamic shared memory attribute of every kernel is set to the device limit, not
// to one launch's size: concurrent callers (rii.h "Concurrency") launching the same
// kernel with different sizes would otherwise race (one thread's smaller setting
// undercuts the other's launch: cudaLaunchKernel "invalid argument").
constexpr int SMEM_ATTR_MAX = 227 * 1024;

// ---------------------------------------------------------------- errors ---
#define RII_CUDA(call)                                                                            \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            throw ::rii::Error(e_ == cudaErrorMemoryAllocation ? 3 : 4,                           \
                               std::string(#call) + ": " + cudaGetErrorString(e_));               \
    } while (0)

extern std::atomic<uint64_t> g_launches;
inline void count_launch(int n = 1) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

// Checked build (RII_BOUNDS_CHECK, `python -m paper_1808_03969_b200.build --checked` ->
// librii_b200_checked.so, loaded when RII_LIB=checked): the stand-in for compute-sanitizer,
// which this GPU pool does not allow.  Device-side RII_DCHECKs (index and shared-memory
// layout bounds at the risky accesses: work items, gathers by id, append buffers, output
// rows) print the failed condition and trap; every launch is followed by a device
// synchronisation so that a fault is reported by the launch that caused it.
#ifdef RII_BOUNDS_CHECK
#define RII_LAUNCHED()                                                                            \
    do {                                                                                          \
        ::rii::count_launch();                                                                    \
        RII_CUDA(cudaGetLastError());                                                             \
        RII_CUDA(cudaDeviceSynchronize());                                                        \
    } while (0)
#define RII_DCHECK(c)                                                                             \
    do {                                                                                          \
        if (!(c)) {                                                                               \
            printf("RII_DCHECK failed %s:%d: %s (block %d, thread %d)\n", __FILE__, __LINE__, #c, \
                   (int)blockIdx.x, (int)threadIdx.x);                                            \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define RII_LAUNCHED()                                                                            \
    do {                                                                                          \
        ::rii::count_launch();                                                                    \
        RII_CUDA(cudaGetLastError());                                                             \
    } while (0)
#define RII_DCHECK(c) do { } while (0)
#endif
// The dynamic shared memory a launch was given (bytes).
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}
// [base, end) lies inside the launch's dynamic shared memory
#define RII_SMEM_CHECK(base, end) \
    RII_DCHECK((const uint8_t *)(end) >= (const uint8_t *)(base) && \
               (size_t)((const uint8_t *)(end) - (const uint8_t *)(base)) <= (size_t)::rii::dyn_smem_bytes())

// Optional device event counters of the scan kernels (rii_debug_counters): window
// ends, compactions, rollbacks, shared-bound tightenings read at a window end,
// integer-table re-quantisations, bound publications that lowered the bound,
// candidates pushed into the fresh buffers (summed at each compaction), and the
// SM clock cycles thread 0 spent per CTA in table fill / scan loop / final
// compaction + output (summed over CTAs), and the number of CTAs.
enum DebugCounter { DBG_WINDOWS = 0, DBG_COMPACT = 1, DBG_ROLLBACK = 2, DBG_GTHR_TIGHTEN = 3, DBG_RESCALE = 4,
                    DBG_PUBLISH = 5, DBG_FRESH = 6, DBG_CYC_FILL = 7, DBG_CYC_SCAN = 8,
                    DBG_CYC_TAIL = 9, DBG_ITEMS = 10, DBG_COUNT = 16 };
unsigned long long *debug_counters();  // device array [DBG_COUNT] or nullptr (counting off)

// Optional per-kernel event timing (rii_kernel_timing).
enum TimedKernel { TK_LINEAR = 0, TK_IVF = 1, TK_MERGE = 2, TK_PACKED = 3, TK_BOUND = 4, TK_Q16 = 5, TK_U6 = 6, TK_COUNT = 7 };
struct KernelTimer {
    cudaStream_t st;
    int which;
    cudaEvent_t a = nullptr, b = nullptr;
    KernelTimer(int w, cudaStream_t s);   // records the start event if timing is on
    ~KernelTimer();                       // records the stop event
};

// -------------------------------------------------------- arithmetic ------
// CA1: t = u - c; acc = acc + t*t; fp32 round-to-nearest, no contraction.
__device__ __forceinline__ float ca1_step(float acc, float u, float c) {
    float t = __fsub_rn(u, c);
    return __fadd_rn(acc, __fmul_rn(t, t));
}

// CA2 sum d = ((0 + A[0][c0]) + A[1][c1]) + ... of a code of M bytes (M % 16 == 0,
// 16-byte aligned) against a canonical [M][256] fp32 table in global memory.  The
// loads of 16 subspaces are issued before their in-order adds: a rolled loop would
// serialise two dependent memory round trips per subspace (code byte, then entry).
__device__ __forceinline__ float rescore_ca2_16(const float *__restrict__ tq, const uint8_t *__restrict__ cp, int M) {
    float d = 0.f;
    for (int m0 = 0; m0 < M; m0 += 16) {
        const uint4 c = __ldg(reinterpret_cast<const uint4 *>(cp + m0));
        const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __ldg(tq + (int64_t)(m0 + j) * 256 + ((cw[j >> 2] >> (8 * (j & 3))) & 255u));
#pragma unroll
        for (int j = 0; j < 16; ++j) d = __fadd_rn(d, v[j]);
    }
    return d;
}

// (dist, id) packed so that unsigned order == (dist asc, id asc) for dist >= +0.
__device__ __forceinline__ uint64_t make_key(float d, uint32_t id) {
    return ((uint64_t)__float_as_uint(d) << 32) | (uint64_t)id;
}
__device__ __forceinline__ float key_dist(uint64_t k) { return __uint_as_float((uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t key_id(uint64_t k) { return (uint32_t)(k & 0xffffffffu); }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// splitmix64 finaliser (counter-based hash for every seeded choice, R8 / R10).
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

inline int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// Width of the per-query candidate lists kept by every kernel: a power of two
// with at least 16 slots of slack above topk.
inline int partial_width(int topk) { return next_pow2(topk + 16 < 32 ? 32 : topk + 16); }

// Mapping of the 32-bit candidate index stored in a key to a global id.
struct IdMap {
    int kind = 0;                 // 0 identity, 1 table (int64 global ids), 2 ranges
    const int64_t *table = nullptr;
    const int64_t *seg_local = nullptr;  // ranges: local offset of each segment (ascending)
    const int64_t *seg_global = nullptr; // ranges: global id of the segment's first code
    int nseg = 0;
};

__device__ __forceinline__ int64_t map_id(const IdMap &m, uint32_t i) {
    if (m.kind == 0) return (int64_t)i;
    if (m.kind == 1) return m.table[i];
    int lo = 0, hi = m.nseg - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (m.seg_local[mid] <= (int64_t)i) lo = mid; else hi = mid - 1;
    }
    return m.seg_global[lo] + ((int64_t)i - m.seg_local[lo]);
}

}  // namespace rii
