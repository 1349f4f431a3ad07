// topk.cuh -- exact (dist, id) top-kk selection in shared memory (Alg. 1 L6-L7
// "PartialSort / Take", re-designed for a CTA of NT threads).
//
// Per query the CTA keeps `top[kk]` (ascending keys, kk a power of two) and a
// `fresh[NEWCAP]` append buffer.  Lanes push candidates whose distance is <=
// the current kk-th best (warp-aggregated atomics).  When a step may overflow
// `fresh`, the CTA bitonic-sorts the fresh keys, folds them into `top` with a
// bitonic half-cleaner (min(top[i], fresh[kk-1-i]) keeps the kk smallest of the
// union as a bitonic sequence) and bitonic-merges `top` back to ascending order.
#pragma once
#include "common.cuh"

namespace rii {

constexpr int NEWCAP = 512;                 // fresh slots per query
constexpr int PUSH_TRIGGER = NEWCAP - NT;   // compaction once a step could overflow

// Warp-aggregated push of one candidate per lane into fresh_q; sets `need` when
// the buffer passed the trigger.  The whole warp must call it (converged).
__device__ __forceinline__ void push_candidate(bool pred, uint64_t key, uint64_t *fresh_q, int *cnt_q, int lane,
                                               bool &need) {
    unsigned bal = __ballot_sync(0xffffffffu, pred);
    if (bal) {
        int n = __popc(bal);
        int leader = __ffs(bal) - 1;
        int base = 0;
        if (lane == leader) {
            base = atomicAdd(cnt_q, n);
            if (base + n > PUSH_TRIGGER) need = true;
        }
        base = __shfl_sync(0xffffffffu, base, leader);
        if (pred) fresh_q[base + __popc(bal & ((1u << lane) - 1u))] = key;
    }
}

// Windowed variant: never writes past NEWCAP; a push that does not fit sets
// `ovf` (the caller rolls the window back and redoes it) and a fill above
// `soft` sets `need` (compaction at the window end).
__device__ __forceinline__ void push_candidate_win(bool pred, uint64_t key, uint64_t *fresh_q, int *cnt_q, int lane,
                                                   int soft, bool &need, bool &ovf) {
    unsigned bal = __ballot_sync(0xffffffffu, pred);
    if (bal) {
        int n = __popc(bal);
        int leader = __ffs(bal) - 1;
        int base = 0;
        if (lane == leader) {
            base = atomicAdd(cnt_q, n);
            if (base + n > soft) need = true;
        }
        base = __shfl_sync(0xffffffffu, base, leader);
        const int slot = base + __popc(bal & ((1u << lane) - 1u));
        if (pred) {
            if (slot < NEWCAP) fresh_q[slot] = key;
            else ovf = true;
        }
    }
}

__device__ __forceinline__ void cas_asc(uint64_t *a, int i, int p) {
    uint64_t x = a[i], y = a[p];
    if (x > y) { a[i] = y; a[p] = x; }
}

__device__ __forceinline__ int ilog2_pow2(int v) { return __ffs(v) - 1; }  // v a power of two

// Bitonic sort of `nq` independent arrays a[q*stride .. + S), S a power of two.
__device__ inline void bitonic_sort_rows(uint64_t *a, int nq, int stride, int S) {
    const int half = S >> 1, lh = ilog2_pow2(half > 0 ? half : 1);
    for (int k = 2; k <= S; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int e = threadIdx.x; e < nq * half; e += blockDim.x) {
                int q = e >> lh, t = e & (half - 1);
                int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                int p = i | j;
                uint64_t *r = a + (size_t)q * stride;
                uint64_t x = r[i], y = r[p];
                bool up = (i & k) == 0;
                if ((x > y) == up) { r[i] = y; r[p] = x; }
            }
            __syncthreads();
        }
    }
}

// Sort a bitonic sequence a[q*stride .. + S) ascending (merge network).
__device__ inline void bitonic_merge_rows(uint64_t *a, int nq, int stride, int S) {
    const int half = S >> 1, lh = ilog2_pow2(half > 0 ? half : 1);
    for (int len = half; len > 0; len >>= 1) {
        for (int e = threadIdx.x; e < nq * half; e += blockDim.x) {
            int q = e >> lh, t = e & (half - 1);
            int i = ((t & ~(len - 1)) << 1) | (t & (len - 1));
            cas_asc(a + (size_t)q * stride, i, i | len);
        }
        __syncthreads();
    }
}

// Fold the fresh candidates of `nq` queries into their top lists.
// top: [nq][kk] ascending; fresh: [nq][NEWCAP]; cnt[nq]; thr[nq] updated.
__device__ inline void compact_topk(uint64_t *top, uint64_t *fresh, int *cnt, float *thr, int nq, int kk,
                                    int *scratch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        int mx = 0;
        for (int q = 0; q < nq; ++q) mx = cnt[q] > mx ? cnt[q] : mx;
        scratch[0] = mx;
    }
    __syncthreads();
    const int mx = scratch[0];
    if (mx > 0) {
        int S = 2;
        while (S < mx) S <<= 1;
        const int ls = ilog2_pow2(S);
        for (int e = threadIdx.x; e < nq * S; e += blockDim.x) {
            int q = e >> ls, i = e & (S - 1);
            if (i >= cnt[q]) fresh[(size_t)q * NEWCAP + i] = KEY_MAX;
        }
        __syncthreads();
        bitonic_sort_rows(fresh, nq, NEWCAP, S);
        const int lk = ilog2_pow2(kk);
        for (int e = threadIdx.x; e < nq * kk; e += blockDim.x) {
            int q = e >> lk, i = e & (kk - 1);
            int x = kk - 1 - i;
            uint64_t v = x < S ? fresh[(size_t)q * NEWCAP + x] : KEY_MAX;
            uint64_t *t = top + (size_t)q * kk + i;
            if (v < *t) *t = v;
        }
        __syncthreads();
        bitonic_merge_rows(top, nq, kk, kk);
    }
    if (threadIdx.x < nq) {
        uint64_t last = top[(size_t)threadIdx.x * kk + kk - 1];
        thr[threadIdx.x] = last == KEY_MAX ? __int_as_float(0x7f800000) : key_dist(last);
        cnt[threadIdx.x] = 0;
    }
    __syncthreads();
}

}  // namespace rii
