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
        const int slot = base + __popc(bal & ((1u << lane) - 1u));
        if (pred) {
            RII_DCHECK(slot < NEWCAP);  // the trigger leaves room for one more step of pushes
            fresh_q[slot] = key;
        }
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

// ---- warp-level compaction (few fresh candidates: no block barriers) -------
// Element i of a warp-distributed array of 32*E keys sits in lane i / E, slot i % E.
template <int E>
__device__ __forceinline__ void warp_cas_stage(uint64_t (&v)[E], int lane, int k, int j) {
    if (j < E) {  // partner in the same lane
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int p = e ^ j;
            if (p <= e) continue;
            const bool up = ((lane * E + e) & k) == 0;
            const uint64_t x = v[e], y = v[p];
            if ((x > y) == up) { v[e] = y; v[p] = x; }
        }
    } else {
        const int lj = j / E;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint64_t y = __shfl_xor_sync(0xffffffffu, v[e], lj);
            const bool up = ((lane * E + e) & k) == 0;
            v[e] = (lower == up) ? (v[e] < y ? v[e] : y) : (v[e] > y ? v[e] : y);
        }
    }
}

template <int E>
__device__ __forceinline__ void warp_bitonic_sort(uint64_t (&v)[E], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) warp_cas_stage<E>(v, lane, k, j);
}

// Ascending sort of a bitonic warp-distributed sequence (merge network only).
template <int E>
__device__ __forceinline__ void warp_bitonic_merge(uint64_t (&v)[E], int lane) {
#pragma unroll
    for (int j = 16 * E; j > 0; j >>= 1) warp_cas_stage<E>(v, lane, 32 * E, j);
}

// One warp folds fresh_q[0..n) (n <= 32 * EF) into top_q[kk] (kk = 32 * E,
// ascending): sort the fresh keys (EF per lane), then top[i] = min(top[i],
// fresh[kk-1-i]) keeps the kk smallest of the union as a bitonic sequence, which
// the merge sorts.
template <int E, int EF>
__device__ __forceinline__ float warp_compact_query(uint64_t *top_q, uint64_t *fresh_q, int n, int lane) {
    uint64_t f[EF];
#pragma unroll
    for (int e = 0; e < EF; ++e) f[e] = lane * EF + e < n ? fresh_q[lane * EF + e] : KEY_MAX;
    warp_bitonic_sort<EF>(f, lane);
#pragma unroll
    for (int e = 0; e < EF; ++e) fresh_q[lane * EF + e] = f[e];
    __syncwarp();
    uint64_t v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e, x = 32 * E - 1 - i;
        const uint64_t t = top_q[i], c = x < 32 * EF ? fresh_q[x] : KEY_MAX;
        v[e] = c < t ? c : t;
    }
    warp_bitonic_merge<E>(v, lane);
#pragma unroll
    for (int e = 0; e < E; ++e) top_q[lane * E + e] = v[e];
    const uint64_t last = __shfl_sync(0xffffffffu, v[E - 1], 31);
    return last == KEY_MAX ? __int_as_float(0x7f800000) : key_dist(last);
}

template <int E>
__device__ __forceinline__ void warp_compact_all(uint64_t *top, uint64_t *fresh, int *cnt, float *thr, int nq) {
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int q = threadIdx.x >> 5; q < nq; q += nw) {
        const int n = cnt[q];
        if (n > 0) {
            uint64_t *tq = top + (size_t)q * (32 * E), *fq = fresh + (size_t)q * NEWCAP;
            float t;
            if (n <= 64) t = warp_compact_query<E, 2>(tq, fq, n, lane);
            else t = warp_compact_query<E, 8>(tq, fq, n, lane);
            if (lane == 0) thr[q] = t;
        }
        __syncwarp();
    }
}

// Fold the fresh candidates of `nq` queries into their top lists.
// top: [nq][kk] ascending; fresh: [nq][NEWCAP]; cnt[nq]; thr[nq] updated.
__device__ inline void compact_topk(uint64_t *top, uint64_t *fresh, int *cnt, float *thr, int nq, int kk,
                                    int *scratch) {
    __syncthreads();
    if (threadIdx.x < 32) {
        int m = 0;
        for (int q = threadIdx.x; q < nq; q += 32) m = max(m, cnt[q]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) scratch[0] = m;
    }
    __syncthreads();
    const int mx = scratch[0];
    if (mx > 0 && mx <= 256 && kk >= 32 && kk <= 256) {  // warp per query
        switch (kk) {
            case 32: warp_compact_all<1>(top, fresh, cnt, thr, nq); break;
            case 64: warp_compact_all<2>(top, fresh, cnt, thr, nq); break;
            case 128: warp_compact_all<4>(top, fresh, cnt, thr, nq); break;
            default: warp_compact_all<8>(top, fresh, cnt, thr, nq); break;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < nq; q += blockDim.x) cnt[q] = 0;
        __syncthreads();
        return;
    }
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
