// capi.cu -- the C ABI of include/rii.h: argument checks, the index state held in
// HBM (Sec. 4.1), and the orchestration of the kernels of
// k_scan.cu / k_ivf.cu / k_build.cu for train, add, reconfigure and query.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/rii.h"
#include "comm.hpp"
#include "kernels.cuh"
#include "opq.hpp"
#include "lut.cuh"

namespace rii {
std::atomic<uint64_t> g_launches{0};

// rii_debug_counters: device event counters of the scan kernels (common.cuh)
std::atomic<unsigned long long *> g_dbg{nullptr};
unsigned long long *debug_counters() { return g_dbg.load(std::memory_order_relaxed); }

namespace timing {
std::mutex g_tmu;
bool g_timing = false;
struct TimedPair { int which; cudaEvent_t a, b; };
std::vector<TimedPair> g_pairs;
double g_total_ms[TK_COUNT] = {};
int64_t g_count[TK_COUNT] = {};

void drain_pairs() {  // caller holds g_tmu
    for (auto &p : g_pairs) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            g_total_ms[p.which] += ms;
            g_count[p.which] += 1;
        }
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    g_pairs.clear();
}
}  // namespace timing
using namespace timing;

KernelTimer::KernelTimer(int w, cudaStream_t s) : st(s), which(w) {
    std::lock_guard<std::mutex> lk(g_tmu);
    if (!g_timing || w < 0) return;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) { a = b = nullptr; return; }
    cudaEventRecord(a, st);
}

KernelTimer::~KernelTimer() {
    if (!a) return;
    cudaEventRecord(b, st);
    std::lock_guard<std::mutex> lk(g_tmu);
    g_pairs.push_back({which, a, b});
}

// Grow-only device buffer (scratch and index arrays).
struct Buf {
    void *p = nullptr;
    size_t cap = 0;
    Buf() = default;
    Buf(const Buf &) = delete;
    Buf &operator=(const Buf &) = delete;
    ~Buf() { if (p) cudaFree(p); }
    template <class T>
    T *get(size_t count) {
        const size_t b = std::max<size_t>(count * sizeof(T), 16);
        if (b > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            RII_CUDA(cudaMalloc(&p, b));
            cap = b;
        }
        return reinterpret_cast<T *>(p);
    }
    template <class T>
    T *as() const { return reinterpret_cast<T *>(p); }
    // keep the first `keep` bytes when growing
    template <class T>
    T *grow(size_t count, size_t keep, cudaStream_t st) {
        const size_t b = std::max<size_t>(count * sizeof(T), 16);
        if (b <= cap) return reinterpret_cast<T *>(p);
        size_t nb = std::max(b, cap + cap / 2);
        void *np = nullptr;
        RII_CUDA(cudaMalloc(&np, nb));
        if (keep) RII_CUDA(cudaMemcpyAsync(np, p, keep, cudaMemcpyDeviceToDevice, st));
        RII_CUDA(cudaStreamSynchronize(st));
        if (p) cudaFree(p);
        p = np;
        cap = nb;
        return reinterpret_cast<T *>(p);
    }
};

// Stream-ordered scratch owned by one call (rii.h "Concurrency"): cudaMallocAsync
// on the call's stream from the device pool that rii_create keeps warm, released
// with cudaFreeAsync when the call's scratch goes out of scope, so concurrent
// readers on different streams never share (or free) each other's buffers.
struct SBuf {
    const cudaStream_t *st;
    void *p = nullptr;
    size_t cap = 0;
    explicit SBuf(const cudaStream_t *s) : st(s) {}
    SBuf(const SBuf &) = delete;
    SBuf &operator=(const SBuf &) = delete;
    ~SBuf() { if (p) cudaFreeAsync(p, *st); }
    template <class T>
    T *get(size_t count) {
        const size_t b = std::max<size_t>(count * sizeof(T), 16);
        if (b > cap) {
            if (p) cudaFreeAsync(p, *st);
            p = nullptr;
            cap = 0;
            RII_CUDA(cudaMallocAsync(&p, b, *st));
            cap = b;
        }
        return reinterpret_cast<T *>(p);
    }
    template <class T>
    T *as() const { return reinterpret_cast<T *>(p); }
};

// Every scratch buffer of one rii_query / rii_query_partial call.
struct QueryScratch {
    cudaStream_t st;
    SBuf s_q{&st}, s_S{&st}, s_pos{&st}, s_sub{&st}, s_part{&st}, s_keys{&st}, s_gather{&st}, s_d0{&st},
        s_probe{&st}, s_roff{&st}, s_rids{&st}, s_rkey{&st}, s_rval{&st}, s_out_ids{&st}, s_out_dist{&st},
        s_flag{&st}, s_lq{&st}, s_qoff{&st}, s_ql{&st}, s_qoff2{&st}, s_ql2{&st}, s_items{&st}, s_gthr{&st},
        s_tables{&st}, s_cpart{&st}, s_ckeys{&st}, s_take{&st}, s_samp{&st}, s_spart{&st}, s_bound{&st},
        s_skey{&st}, s_tab16{&st}, s_qscale{&st}, s_qrot{&st}, s_route{&st}, s_rmirror{&st}, s_alist{&st}, s_pr0{&st},
        s_pmask{&st}, s_salist{&st};
    explicit QueryScratch(cudaStream_t s) : st(s) {}
};

struct Seg {
    int64_t local_off, global_first, count;
};

}  // namespace rii

using namespace rii;

struct rii_index {
    int D = 0, M = 0, ds = 0, device = 0, rank = 0, world = 1, num_sms = 148;
    Comm *comm = nullptr;  // NCCL or host transport (world > 1); nullptr = single GPU / detached shard
    bool trained = false, T_valid = false;
    Buf cb, T;
    int64_t N = 0, n_local = 0;
    Buf codes, assign;
    std::vector<Seg> segs;
    Buf seg_local, seg_global, seg_count;
    int64_t K = 0;
    Buf centers, offsets, ids;
    Buf mirror;  // codes in posting-list order: mirror[p] = codes[ids[p]] (list-major IVF scans)
    int64_t theta = -1;
    int ivf_mode = 0;        // RII_IVF_LISTS / RII_IVF_PAPER
    bool theta_fit = false;  // rii_calibrate_theta result in use (theta(L) = fit_a * L + fit_b)
    bool has_rot = false;    // OPQ rotation (rii_set_rotation / rii_train_opq): R and R^T, D x D fp32
    Buf rot, rotT;
    std::vector<float> rot_host;
    double fit_a = 0.0, fit_b = 0.0;
    // writer-side scratch (train / add / reconfigure; single writer).  Queries use a
    // per-call QueryScratch instead.
    Buf s_x, s_flag, s_xrot, s_rval;
};

namespace {
thread_local std::string t_err;

rii_status fail(int st, const std::string &msg) {
    t_err = msg;
    return (rii_status)st;
}

template <class F>
rii_status guarded(F &&f) {
    try {
        t_err.clear();
        f();
        return RII_OK;
    } catch (const rii::Error &e) {
        return fail(e.status, e.what());
    } catch (const std::bad_alloc &) {
        return fail(RII_ERR_OOM, "host allocation failed");
    } catch (const std::exception &e) {
        return fail(RII_ERR_CUDA, e.what());
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        RII_CUDA(cudaGetDevice(&prev));
        if (prev != dev) RII_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

void arg_check(bool ok, const char *msg) {
    if (!ok) throw Error(RII_ERR_ARG, msg);
}
void state_check(bool ok, const char *msg) {
    if (!ok) throw Error(RII_ERR_STATE, msg);
}

IdMap local_map(const rii_index *x) {
    IdMap m;
    if (x->world == 1) return m;  // local position == global id
    m.kind = 2;
    m.seg_local = x->seg_local.as<int64_t>();
    m.seg_global = x->seg_global.as<int64_t>();
    m.nseg = (int)x->segs.size();
    return m;
}

void upload_segs(rii_index *x, cudaStream_t st) {
    std::vector<int64_t> lo, gl, ct;
    for (auto &s : x->segs) { lo.push_back(s.local_off); gl.push_back(s.global_first); ct.push_back(s.count); }
    int64_t *dl = x->seg_local.get<int64_t>(lo.size() + 1), *dg = x->seg_global.get<int64_t>(gl.size() + 1);
    int64_t *dc = x->seg_count.get<int64_t>(ct.size() + 1);
    if (!lo.empty()) {
        RII_CUDA(cudaMemcpyAsync(dl, lo.data(), lo.size() * 8, cudaMemcpyHostToDevice, st));
        RII_CUDA(cudaMemcpyAsync(dg, gl.data(), gl.size() * 8, cudaMemcpyHostToDevice, st));
        RII_CUDA(cudaMemcpyAsync(dc, ct.data(), ct.size() * 8, cudaMemcpyHostToDevice, st));
    }
    RII_CUDA(cudaStreamSynchronize(st));
}

void ensure_T(rii_index *x, cudaStream_t st) {
    if (x->T_valid) return;
    float *T = x->T.get<float>((size_t)x->M * KS * KS);
    launch_sdc_tables(x->cb.as<float>(), x->D, x->M, T, st);
    x->T_valid = true;
}

__global__ void iota_u32_kernel(uint32_t *v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}

// List-major phase split: pair (q, r) goes to bucket ph * K + probes[q][r], ph = the
// phase whose rank range [rb[ph], rb[ph + 1]) holds r (phase 0: float tables; later
// phases: integer tables re-quantised at the bounds the earlier phases published).
struct PhaseBounds { int64_t rb[8]; int n; };
__global__ void split_keys_kernel(const int32_t *probes, int64_t npairs, int64_t P, PhaseBounds pb, int64_t K,
                                  int32_t *keys) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npairs) return;
    const int64_t r = i % P;
    int ph = 0;
    while (ph + 1 < pb.n && r >= pb.rb[ph + 1]) ++ph;
    keys[i] = probes[i] + ph * (int32_t)K;
}

// gthr[q] = min(gthr[q], the kk-th distance of keys[q][kk] inflated by 1e-5 (it may
// be a lane-rotated fp32 sum, within 4e-6 relative of the canonical CA2 value)):
// the kk-th smallest over a subset of a query's candidates bounds its final kk-th.
__global__ void merged_bound_kernel(const uint64_t *keys, int64_t nq, int kk, float *gthr) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint64_t k = keys[q * kk + kk - 1];
    if (k == KEY_MAX) return;
    const float b = __fmul_ru(key_dist(k), 1.00001f);
    if (b < gthr[q]) gthr[q] = b;
}

__global__ void gather_i32_kernel(const int32_t *src, const int64_t *pos, int64_t n, int32_t *dst, uint32_t *val) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { dst[i] = src[pos[i]]; val[i] = (uint32_t)pos[i]; }
}

__global__ void assign_from_csr_kernel(const int64_t *off, int64_t K, const uint32_t *ids, int32_t *a) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    for (int64_t p = off[k]; p < off[k + 1]; ++p) a[ids[p]] = (int32_t)k;
}

__global__ void widen_ids_kernel(const uint32_t *src, int64_t n, IdMap map, int64_t *dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = map_id(map, src[i]);
}

__global__ void gather_u32pos_codes_kernel(const uint8_t *codes, int M, const uint32_t *pos, int64_t n, uint8_t *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if ((M & 3) == 0) {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(codes + (int64_t)pos[i] * M);
        uint32_t *dst = reinterpret_cast<uint32_t *>(out + i * M);
        for (int m = 0; m < M / 4; ++m) dst[m] = __ldg(src + m);
    } else {
        for (int m = 0; m < M; ++m) out[i * M + m] = codes[(int64_t)pos[i] * M + m];
    }
}

// out[p] = codes[ids[p]] for the n positions of a CSR: the codes in posting-list order
// (list-major IVF reads a list as one contiguous range).
void build_mirror(const uint8_t *codes, int M, const uint32_t *ids, int64_t n, uint8_t *out, cudaStream_t st) {
    if (n <= 0) return;
    gather_u32pos_codes_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(codes, M, ids, n, out);
    RII_LAUNCHED();
}

void rebuild_csr(rii_index *x, cudaStream_t st) {
    uint32_t *vals = x->s_rval.get<uint32_t>(x->n_local + 1);
    if (x->n_local > 0) {
        iota_u32_kernel<<<(unsigned)ceil_div(x->n_local, 256), 256, 0, st>>>(vals, x->n_local);
        RII_LAUNCHED();
    }
    int64_t *off = x->offsets.get<int64_t>(x->K + 1);
    uint32_t *ids = x->ids.get<uint32_t>(x->n_local + 1);
    build_csr(x->assign.as<int32_t>(), vals, x->n_local, x->K, off, ids, st);
    build_mirror(x->codes.as<uint8_t>(), x->M, ids, x->n_local,
                 x->mirror.get<uint8_t>((size_t)std::max<int64_t>(x->n_local, 1) * x->M + 64), st);
}

// Rows [lo, hi) of this rank in a batch of n rows split into `world` chunks.
void rank_rows(int64_t n, int rank, int world, int64_t &lo, int64_t &hi) {
    const int64_t per = ceil_div(n, world);
    lo = std::min<int64_t>(n, per * rank);
    hi = std::min<int64_t>(n, lo + per);
}

// Subset routing (SURVEY 8(e) "S is routed by binary search over the range table"):
// S is sorted and each segment of this rank is a contiguous id range, so the ids of
// S a segment owns form one contiguous range [b_j, e_j) of S.  One block finds those
// ranges (two binary searches per segment) and their output offsets; then every
// element of S finds its segment's range by a binary search over the b_j and, if
// owned, writes its global id and local position.  Only the owned count goes to the
// host (one 8-byte read), not S itself.
__device__ __forceinline__ int64_t lower_bound_i64(const int64_t *a, int64_t n, int64_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void route_ranges_kernel(const int64_t *__restrict__ S, int64_t nS, const int64_t *__restrict__ seg_global,
                                    const int64_t *__restrict__ seg_count, int nseg, int64_t *__restrict__ rb,
                                    int64_t *__restrict__ re, int64_t *__restrict__ roff, int64_t *__restrict__ total) {
    for (int j = threadIdx.x; j < nseg; j += blockDim.x) {
        rb[j] = lower_bound_i64(S, nS, seg_global[j]);
        re[j] = lower_bound_i64(S, nS, seg_global[j] + seg_count[j]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // segments are few (one per add batch): a serial prefix sum
        int64_t acc = 0;
        for (int j = 0; j < nseg; ++j) {
            roff[j] = acc;
            acc += re[j] - rb[j];
        }
        *total = acc;
    }
}

__global__ void route_scatter_kernel(const int64_t *__restrict__ S, int64_t nS, const int64_t *__restrict__ seg_local,
                                     const int64_t *__restrict__ seg_global, int nseg, const int64_t *__restrict__ rb,
                                     const int64_t *__restrict__ re, const int64_t *__restrict__ roff,
                                     int64_t *__restrict__ S_loc, int64_t *__restrict__ pos) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nS) return;
    // last segment j with rb[j] <= i (rb is non-decreasing: segments ascend in id)
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (rb[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    if (i < rb[lo] || i >= re[lo]) return;  // owned by another rank
    const int64_t o = roff[lo] + (i - rb[lo]), s = S[i];
    S_loc[o] = s;
    pos[o] = s - seg_global[lo] + seg_local[lo];
}

// Target ids of this rank: global ids (device) and local positions (device).
// world == 1: positions == ids (no copy).  Returns the local count.
int64_t route_targets(const rii_index *x, QueryScratch &sc, const int64_t *S, int64_t nS, cudaStream_t st,
                      const int64_t **S_loc, const int64_t **pos_loc) {
    if (x->world == 1) {
        *S_loc = S;
        *pos_loc = S;
        return nS;
    }
    const int nseg = (int)x->segs.size();
    if (nseg == 0 || nS == 0) {
        *S_loc = *pos_loc = sc.s_S.get<int64_t>(1);
        return 0;
    }
    int64_t *r = sc.s_route.get<int64_t>((size_t)3 * nseg + 1);  // rb, re, roff, total
    route_ranges_kernel<<<1, 256, 0, st>>>(S, nS, x->seg_global.as<int64_t>(), x->seg_count.as<int64_t>(), nseg, r,
                                          r + nseg, r + 2 * nseg, r + 3 * nseg);
    RII_LAUNCHED();
    int64_t *dS = sc.s_S.get<int64_t>(nS + 1), *dP = sc.s_pos.get<int64_t>(nS + 1);
    route_scatter_kernel<<<(unsigned)ceil_div(nS, 256), 256, 0, st>>>(S, nS, x->seg_local.as<int64_t>(),
                                                                     x->seg_global.as<int64_t>(), nseg, r, r + nseg,
                                                                     r + 2 * nseg, dS, dP);
    RII_LAUNCHED();
    int64_t n_loc = 0;
    RII_CUDA(cudaMemcpyAsync(&n_loc, r + 3 * nseg, 8, cudaMemcpyDeviceToHost, st));
    RII_CUDA(cudaStreamSynchronize(st));
    *S_loc = dS;
    *pos_loc = dP;
    return n_loc;
}

struct QueryArgs {
    const float *q;          // device
    int64_t nq;
    int topk, kk;
    const int64_t *S;        // device global ids or nullptr
    int64_t nS;
    int L;
    int path;                // how the call executes: LINEAR / IVF / EXEC_MASKED (decide_exec)
    bool collective;         // rii_query with world > 1 and a communicator: every rank runs this call
};

// Execution of an IVF call in mode A (reading R2: every S-member of the P probed lists
// is a candidate, ranked by (d, id)).  Its candidate set is (union of the P probed
// lists) ∩ S, so:
//  - P == K probes every list: the candidates are S itself and the result is the
//    linear scan's (Alg. 1) -- run it (path_used still reports IVF);
//  - many probed lists (P * RII_MASKED_RATIO >= K, default 8): a probe-masked linear
//    scan of S (EXEC_MASKED, ProbeMask) -- each code of S is evaluated only for the
//    queries that probe its list, at the linear scan's rate, instead of list-major
//    items over short restricted lists;
//  - otherwise the posting-list traversal.
// Every quantity is global (N, K, |S|, L), so all ranks decide alike.
constexpr int EXEC_MASKED = 3;
int64_t ivf_num_probes(const rii_index *x, bool has_S, int64_t nS, int L) {
    return has_S ? std::min<int64_t>(x->K, ceil_div((int64_t)L * x->N, std::max<int64_t>(nS, 1)))
                 : std::min<int64_t>(L, x->K);  // P:492-502, R1
}
static int masked_ratio() {
    const char *e = getenv("RII_MASKED_RATIO");  // 0 disables both shortcuts (A/B, tests)
    return e ? atoi(e) : 8;
}
// warps sharing one list in the query-major rank-0 phase (8 warps per 2-query CTA)
static int r0q_nseg() {
    const char *e = getenv("RII_R0_NSEG");
    return e ? std::max(1, atoi(e)) : 4;
}
int decide_exec(const rii_index *x, int used, bool has_S, int64_t nS, int L) {
    if (used != RII_PATH_IVF || x->ivf_mode == RII_IVF_PAPER) return used;
    // RII_IVF_MODE (tests / tuning): "list" / "query" force a traversal, "masked" the
    // masked scan whenever P < K
    const char *mode = getenv("RII_IVF_MODE");
    const bool force_trav = mode && (!strcmp(mode, "list") || !strcmp(mode, "query"));
    const bool force_mask = mode && !strcmp(mode, "masked");
    const int r = masked_ratio();
    if (force_trav || (r <= 0 && !force_mask)) return used;
    const int64_t P = ivf_num_probes(x, has_S, nS, L);
    if (P >= x->K) return RII_PATH_LINEAR;
    const bool fast = list_major_supported(x->M);  // the fast-layout scan kernels carry the mask
    if (fast && (force_mask || P * r >= x->K)) return EXEC_MASKED;
    return used;
}

// OPQ: the rotated copy R x of n device rows in `buf`, or x itself
// when the index has no rotation.
template <class B>
const float *rotate_input(const rii_index *x, B &buf, const float *dx, int64_t n, cudaStream_t st) {
    if (!x->has_rot || n <= 0) return dx;
    float *o = buf.template get<float>((size_t)n * x->D);
    launch_rotate(x->rotT.as<float>(), dx, n, x->D, o, st);
    return o;
}

int resolve_path(const rii_index *x, int64_t nS_global, bool has_S, int L, rii_path path) {
    if (x->K == 0) {
        state_check(path != RII_PATH_IVF, "inverted-index path requested but the index has no coarse centres (K == 0)");
        return RII_PATH_LINEAR;
    }
    if (path != RII_PATH_AUTO) return path;
    const int64_t ns = has_S ? nS_global : x->N;
    int64_t th = x->theta >= 0 ? x->theta
                 : x->ivf_mode == RII_IVF_PAPER ? (int64_t)L + x->K          // L candidates + K coarse
                                                : ceil_div((int64_t)L * x->N, x->K) + x->K;  // R3
    if (x->theta < 0 && x->theta_fit) th = (int64_t)std::max(0.0, std::ceil(x->fit_a * L + x->fit_b));
    return ns < th ? RII_PATH_LINEAR : RII_PATH_IVF;  // Alg. 3 L1
}

// RII_TRACE=1: synchronise and print the host-side duration of each query phase.
struct PhaseTrace {
    bool on;
    cudaStream_t st;
    std::chrono::steady_clock::time_point t;
    explicit PhaseTrace(cudaStream_t s) : on(getenv("RII_TRACE") != nullptr), st(s), t(std::chrono::steady_clock::now()) {}
    void mark(const char *what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[rii] %-24s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

// Per-call preparation of the target set S on this rank (R7): the local slice of
// S, its gathered codes (linear path) or the posting lists restricted to it (IVF).
struct Targets {
    const int64_t *S_loc = nullptr, *pos = nullptr;
    int64_t n_loc = 0;
    const uint8_t *sub_codes = nullptr;     // linear path
    const int64_t *roff = nullptr;          // IVF path
    const uint32_t *rids = nullptr;
    const uint8_t *rmirror = nullptr;       // codes of the restricted lists in list order
    const int32_t *alist = nullptr;         // masked IVF: list of each gathered code
};

Targets prepare_targets(const rii_index *x, QueryScratch &sc, const QueryArgs &a, cudaStream_t st) {
    Targets t;
    if (!a.S) {
        if (a.path == EXEC_MASKED) t.alist = x->assign.as<int32_t>();
        return t;
    }
    t.n_loc = route_targets(x, sc, a.S, a.nS, st, &t.S_loc, &t.pos);
    if (a.path == RII_PATH_LINEAR || a.path == EXEC_MASKED) {
        uint8_t *sub = sc.s_sub.get<uint8_t>((size_t)std::max<int64_t>(t.n_loc, 1) * x->M + 64);
        launch_gather_codes(x->codes.as<uint8_t>(), x->M, t.pos, t.n_loc, sub, st);
        t.sub_codes = sub;
        if (a.path == EXEC_MASKED) {
            int32_t *al = sc.s_alist.get<int32_t>(t.n_loc + 1);
            uint32_t *scratch = sc.s_rval.get<uint32_t>(t.n_loc + 1);
            if (t.n_loc > 0) {
                gather_i32_kernel<<<(unsigned)ceil_div(t.n_loc, 256), 256, 0, st>>>(x->assign.as<int32_t>(), t.pos,
                                                                                   t.n_loc, al, scratch);
                RII_LAUNCHED();
            }
            t.alist = al;
        }
    } else {
        int32_t *rk = sc.s_rkey.get<int32_t>(t.n_loc + 1);
        uint32_t *rv = sc.s_rval.get<uint32_t>(t.n_loc + 1);
        if (t.n_loc > 0) {
            gather_i32_kernel<<<(unsigned)ceil_div(t.n_loc, 256), 256, 0, st>>>(x->assign.as<int32_t>(), t.pos,
                                                                               t.n_loc, rk, rv);
            RII_LAUNCHED();
        }
        int64_t *roff = sc.s_roff.get<int64_t>(x->K + 1);
        uint32_t *rids = sc.s_rids.get<uint32_t>(t.n_loc + 1);
        build_csr(rk, rv, t.n_loc, x->K, roff, rids, st);
        t.roff = roff;
        t.rids = rids;
        uint8_t *rm = sc.s_rmirror.get<uint8_t>((size_t)std::max<int64_t>(t.n_loc, 1) * x->M + 64);
        build_mirror(x->codes.as<uint8_t>(), x->M, rids, t.n_loc, rm, st);
        t.rmirror = rm;
    }
    return t;
}

// u16 tables: scans of at least RII_Q16_MIN (default 2^19) codes; the bound comes
// from min(Q16_SAMPLE, n / 4) strided codes.
// Non-fast M at or above this use the large-M kernels (k_large.cu); below, the fp32
// generic kernels (RII_LARGE_MIN_M for A/B; M > 64 always needs the large kernels).
// The paper's SIFT1M shape (M = 64, Table 2): generic 856 ms, large 496 ms per 10k
// queries over 1M codes; IVF L = 5: 22.4 -> 13.7 ms.
static int large_min_m() {
    const char *e = getenv("RII_LARGE_MIN_M");
    return std::min(65, e ? atoi(e) : 33);
}
static double list_q16_min_len() {  // RII_LIST_Q16_MIN: average list length for two-phase u16
    const char *e = getenv("RII_LIST_Q16_MIN");
    return e ? atof(e) : 1024.0;
}
static int64_t large_u6_min_codes() {  // RII_LARGE_U6_MIN: shortest large-M scan on the u6 chunk kernel
    const char *e = getenv("RII_LARGE_U6_MIN");
    return e ? atoll(e) : 65536;
}
static int64_t q16_sample() {
    const char *e = getenv("RII_Q16_SAMPLE");
    return e ? atoll(e) : ((int64_t)1 << 15);
}
static int ns_chunks() {
    const char *e = getenv("RII_Q16_SAMPLE_NC");
    return e ? atoi(e) : 1;
}


// Coarse ranking (Alg. 2 L2-L5) and probe selection (L6): the P nearest lists of every
// query by (d0, k), [nq][P] int32.
const int32_t *coarse_probes(const rii_index *x, QueryScratch &sc, const QueryArgs &a, const float *tables, int64_t P,
                             cudaStream_t st) {
    const float *cb = x->cb.as<float>();
    const bool fast = list_major_supported(x->M);
    int32_t *probes = sc.s_probe.get<int32_t>((size_t)a.nq * std::max<int64_t>(P, 1));
    const int kkc = partial_width((int)std::min<int64_t>(P, 1024));
    const char *cte = getenv("RII_COARSE_TOPP");  // 0: the scan-based coarse ranking (A/B)
    if (P >= x->K) {
        launch_select_probes(nullptr, a.nq, x->K, P, probes, st);  // every list
    } else if (fast && !(cte && cte[0] == '0') && (x->K <= 8192 || P > 1008 || (cte && cte[0] == '1')) &&
               launch_coarse_topp(x->centers.as<uint8_t>(), x->K, x->M, tables, a.nq, P, probes, st)) {
        // one CTA per query: canonical d0 of every centre, radix-selected top-P (k_ivf.cu).
        // Measured against the scan-based ranking below: deep10m (K = 3,162) 0.7 vs 0.7 ms
        // at L <= 16, 0.7 vs 1.2 ms at L = 64, 1.2 vs 4.5 ms at P = 640; configs[4]
        // (K = 31,623, 1,024 queries: one CTA per SM for the 126 KB of d0) 0.57 vs 0.29 ms,
        // so large K keeps the scan unless P > 1008 (RII_COARSE_TOPP=1 forces it)
    } else if (fast && P <= 1008) {
        // coarse ranking (L2-L5) with the lane-rotated scan over the K centre codes,
        // canonical rescore, top-P by (d0, k) (L6)
        ScanPlan pc = plan_linear(x->M, kkc, a.nq, x->K, x->num_sms, tables != nullptr, 1 << 30, false);
        uint64_t *cp = sc.s_cpart.get<uint64_t>((size_t)pc.nb * pc.B * pc.nc * kkc);
        // RII_COARSE_BOUND=1 (A/B, off): seed the filter with the kkc-th smallest of the
        // group minima over all K centre codes (>= kkc groups: a valid bound on the
        // kkc-th d0).  Fewer pushes, but the bound pass costs more than it saves
        // (deep10m L = 64 13.22 -> 13.37 ms, L = 1 2.79 -> 3.05 ms).
        float *cg = nullptr;
        const char *cbe = getenv("RII_COARSE_BOUND");
        const int64_t cgs = ceil_div(x->K, 1024);
        if (tables && pc.fast && kkc <= 512 && x->K / cgs >= kkc && cbe && cbe[0] == '1') {
            cg = sc.s_bound.get<float>(a.nq);
            launch_group_min_bound(x->centers.as<uint8_t>(), x->K, x->M, tables, a.nq, kkc, cg, st);
        }
        launch_linear_scan(pc, x->centers.as<uint8_t>(), x->K, x->M, a.q, a.nq, cb, x->D, kkc, cp, st, tables, cg);
        uint64_t *ck = sc.s_ckeys.get<uint64_t>((size_t)a.nq * kkc);
        launch_merge(cp, (int64_t)pc.nc * kkc, kkc, pc.nc, a.nq, kkc, (int)P, IdMap(), nullptr, nullptr, ck, st);
        launch_keys_to_probes(ck, a.nq, kkc, P, probes, st);
    } else {
        float *d0 = sc.s_d0.get<float>((size_t)a.nq * x->K);
        launch_coarse_dist(x->centers.as<uint8_t>(), x->K, x->M, a.q, a.nq, cb, x->D, d0, st);
        launch_select_probes(d0, a.nq, x->K, P, probes, st);
    }
    return probes;
}

// One batch of queries (a.q, a.nq) against this rank's shard.  Writes either the
// final result (world == 1, out_keys == nullptr) or this rank's top-kk keys with
// global ids (out_keys, device [nq][kk]).
void search_batch(const rii_index *x, QueryScratch &sc, const QueryArgs &a, const Targets &t, cudaStream_t st,
                  int64_t *out_ids, float *out_dist, uint64_t *out_keys) {
    const int kk = a.kk;
    const float *cb = x->cb.as<float>();
    const uint8_t *codes = x->codes.as<uint8_t>();
    const bool fast = list_major_supported(x->M);
    IdMap map = local_map(x);
    PhaseTrace tr(st);
    // per-query rotated ADC tables, built once per batch (a1)
    const float *tables = nullptr;
    const bool large = !fast && x->M >= large_min_m();  // k_large.cu: one query per CTA, bf16 resident table
    if (fast) {
        float *tb = sc.s_tables.get<float>((size_t)a.nq * lut_q_floats(x->M));
        launch_lut_tables(a.q, a.nq, cb, x->D, x->M, tb, st);
        tables = tb;
    } else if (large) {
        float *tb = sc.s_tables.get<float>((size_t)a.nq * x->M * KS);
        launch_lut_large(a.q, a.nq, cb, x->D, x->M, tb, st);
        tables = tb;
    }
    tr.mark("tables");
    const uint64_t *parts = nullptr;
    int64_t q_stride = kk, p_stride = kk;
    int nparts = 1;
    Rescore rs;  // set when the partials hold lane-rotated (not yet canonical) distances
    if (a.path == RII_PATH_LINEAR || a.path == EXEC_MASKED) {  // Alg. 1 (masked: Alg. 2 mode A, decide_exec)
        const uint8_t *scan_codes = a.S ? t.sub_codes : codes;
        const int64_t n_codes = a.S ? t.n_loc : x->n_local;
        // masked IVF: every query's P probed lists (Alg. 2 L2-L6), as the traversal ranks them
        const bool masked = a.path == EXEC_MASKED;
        int64_t P_m = 0;
        const int32_t *probes_m = nullptr;
        if (masked) {
            P_m = ivf_num_probes(x, a.S != nullptr, a.nS, a.L);
            probes_m = coarse_probes(x, sc, a, tables, P_m, st);
            tr.mark("coarse+probes");
        }
        if (a.S) {
            map = IdMap();
            map.kind = 1;
            map.table = t.S_loc;
        }
        // Whole-database scans on several ranks share the bound pass of the integer
        // tables: rank r bounds the queries of its slice from its own shard's sample (a
        // subset of the database, so the bound holds globally) and the slices are
        // all-gathered.  Whether the ranks enter that all-gather is decided from global
        // quantities only (N, world, M, kk, nq), so every rank -- also one whose shard
        // is empty or short -- joins the same collectives; each rank then decides
        // locally whether its own scan runs the integer tables.
        float *gthr_shared = nullptr;
        if (!a.S && a.collective && fast && !large && !masked) {
            const int64_t n_dec = ceil_div(x->N, x->world);
            const ScanPlan pd = plan_linear(x->M, kk, a.nq, std::max<int64_t>(n_dec, 1), x->num_sms, tables != nullptr);
            const bool q16_glob = (pd.B == 8 || pd.B == 16) && pd.fast && q16_enabled() && q16_supported(kk) &&
                                  n_dec >= q16_min_codes() && std::min<int64_t>(q16_sample(), n_dec / 4) >= 4 * kk;
            if (q16_glob) {
                KernelTimer tb(TK_BOUND, st);
                const int64_t qs = ceil_div(a.nq, (int64_t)x->world), q_lo = std::min<int64_t>(a.nq, x->rank * qs);
                const int64_t nloc = std::min<int64_t>(a.nq, q_lo + qs) - q_lo;
                float *slice = sc.s_bound.get<float>((size_t)qs + 1);
                float *all = sc.s_spart.get<float>((size_t)qs * x->world + 1);
                launch_fill_f32(slice, qs, INFINITY, st);  // no bound: filter from +inf
                const int64_t ns = std::min<int64_t>(q16_sample(), x->n_local / 4);
                if (nloc > 0 && ns >= 4096 && kk <= 512) {
                    uint8_t *samp = sc.s_samp.get<uint8_t>((size_t)ns * x->M);
                    launch_strided_gather(codes, x->M, x->n_local / ns, ns, samp, st);
                    launch_group_min_bound(samp, ns, x->M, tables + q_lo * lut_q_floats(x->M), nloc, kk, slice, st);
                }
                x->comm->allgather(slice, all, (size_t)qs * 4, st);
                gthr_shared = all;
                tr.mark("shared q16 bound");
            }
        }
        if (n_codes == 0) {
            uint64_t *pp = sc.s_part.get<uint64_t>((size_t)a.nq * kk);
            RII_CUDA(cudaMemsetAsync(pp, 0xff, (size_t)a.nq * kk * 8, st));
            parts = pp;
        } else if (large && large_u6_supported(x->M, kk) && q16_enabled() && smem_fixed_base_ok() &&
                   n_codes >= large_u6_min_codes() && std::min<int64_t>(8192, n_codes / 8) >= 4 * kk) {
            // chunked u6 oct tables (k_large_u6.cu), scaled by the exact kk-th distance
            // over a strided sample of the codes (a subset: it bounds the final kk-th)
            KernelTimer tb(TK_BOUND, st);
            const int64_t ns = std::min<int64_t>(8192, n_codes / 8);
            uint8_t *samp = sc.s_samp.get<uint8_t>((size_t)ns * x->M + 64);
            launch_strided_gather(scan_codes, x->M, n_codes / ns, ns, samp, st);
            const int ncs = large_linear_chunks(a.nq, ns, x->num_sms);
            uint64_t *sp = sc.s_spart.get<uint64_t>((size_t)a.nq * ncs * kk);
            launch_large_linear(samp, ns, x->M, tables, a.nq, kk, ncs, sp, st, -1);
            uint64_t *sk = sc.s_ckeys.get<uint64_t>((size_t)a.nq * kk);
            launch_merge(sp, (int64_t)ncs * kk, kk, ncs, a.nq, kk, kk, IdMap(), nullptr, nullptr, sk, st);
            float *gthr = sc.s_gthr.get<float>(a.nq);
            launch_kth_bound(sk, a.nq, kk, gthr, st);
            uint8_t *qt = sc.s_tab16.get<uint8_t>((size_t)ceil_div(a.nq, 8) * 8 * large_u6_nch(x->M) * KS * 32);
            float *qsc = sc.s_qscale.get<float>(a.nq);
            launch_u6_tables_large(tables, gthr, a.nq, x->M, qt, qsc, st);
            tr.mark("large u6 bound + tables");
            // pass 1: the first 1/16 of the codes at the sample bound's scale; pass 2: the
            // rest, with tables rebuilt at the kk-th over pass 1's exact top lists
            const int64_t n1 = std::max<int64_t>(ceil_div(n_codes, 16), std::min<int64_t>(n_codes, 16 * kk));
            const int64_t n2 = n_codes - n1;
            const int nc1 = large_u6_chunks(a.nq, n1, x->M, x->num_sms),
                      nc2 = n2 > 0 ? large_u6_chunks(a.nq, n2, x->M, x->num_sms) : 0;
            const int nct = nc1 + nc2;
            uint64_t *pp = sc.s_part.get<uint64_t>((size_t)ceil_div(a.nq, 8) * 8 * nct * kk);
            launch_large_u6_linear(scan_codes, 0, n1, x->M, qt, qsc, tables, gthr, a.nq, kk, nc1, pp, nct, 0, st);
            tr.mark("large u6 pass 1");
            if (n2 > 0) {
                launch_merge(pp, (int64_t)nct * kk, kk, nc1, a.nq, kk, kk, IdMap(), nullptr, nullptr, sk, st);
                // min with the sample bound: pass 1 may have kept fewer than kk candidates
                // of a query (its filter already had the sample bound), then its kk-th is +inf
                merged_bound_kernel<<<(unsigned)ceil_div(a.nq, 256), 256, 0, st>>>(sk, a.nq, kk, gthr);
                RII_LAUNCHED();
                launch_u6_tables_large(tables, gthr, a.nq, x->M, qt, qsc, st);
                launch_large_u6_linear(scan_codes, n1, n2, x->M, qt, qsc, tables, gthr, a.nq, kk, nc2, pp, nct, nc1,
                                       st);
            }
            parts = pp;
            q_stride = (int64_t)nct * kk;
            p_stride = kk;
            nparts = nct;
        } else if (large) {
            const int nc = large_linear_chunks(a.nq, n_codes, x->num_sms);
            uint64_t *pp = sc.s_part.get<uint64_t>((size_t)a.nq * nc * kk);
            launch_large_linear(scan_codes, n_codes, x->M, tables, a.nq, kk, nc, pp, st);
            parts = pp;
            q_stride = (int64_t)nc * kk;
            p_stride = kk;
            nparts = nc;
        } else {
            ScanPlan pl = plan_linear(x->M, kk, a.nq, n_codes, x->num_sms, tables != nullptr);
            ProbeMask mask;
            auto make_mask = [&](int B) {  // grouped by the plan's query batch
                if (!masked) return;
                uint32_t *pm = sc.s_pmask.get<uint32_t>((size_t)ceil_div(a.nq, (int64_t)B) * x->K);
                launch_probe_mask(probes_m, a.nq, P_m, x->K, B, pm, st);
                mask.alist = t.alist;
                mask.pm = pm;
                mask.K = x->K;
                mask.B = B;
            };
            make_mask(pl.B);
            // u16 / u6 fixed-point tables for long scans: an upper bound on each query's
            // final kk-th distance (the group minima of a strided sample of the codes --
            // a subset) scales the tables and seeds the filter; every CTA filters with,
            // and publishes its kk-th distance into, gthr.
            float *gthr = gthr_shared;
            bool q16;
            if (gthr_shared) {
                q16 = (pl.B == 8 || pl.B == 16) && pl.fast && q16_enabled() && q16_supported(kk);
            } else {
                gthr = sc.s_gthr.get<float>(a.nq);
                const int64_t ns = std::min<int64_t>(q16_sample(), n_codes / 4);
                q16 = (pl.B == 8 || pl.B == 16) && pl.fast && q16_enabled() && q16_supported(kk) &&
                      n_codes >= q16_min_codes() && ns >= 4 * kk;
                if (q16) {
                    KernelTimer tb(TK_BOUND, st);
                    const int64_t stride = n_codes / ns;
                    uint8_t *samp = sc.s_samp.get<uint8_t>((size_t)ns * x->M);
                    launch_strided_gather(scan_codes, x->M, stride, ns, samp, st);
                    ProbeMask smask = mask;  // masked: the sample's lists
                    if (masked) {
                        int32_t *sal = sc.s_salist.get<int32_t>(ns);
                        launch_strided_gather_i32(t.alist, stride, ns, sal, st);
                        smask.alist = sal;
                    }
                    if (ns >= 4096 && kk <= 512 && (masked || !getenv("RII_BOUND_TOPK"))) {
                        // kk-th smallest of 1024 group minima (no top-k lists; k_scan.cu)
                        launch_group_min_bound(samp, ns, x->M, tables, a.nq, kk, gthr, st, smask);
                    } else if (masked) {
                        launch_fill_f32(gthr, a.nq, INFINITY, st);  // no sampled bound: filter from +inf
                    } else {
                        // exact kk-th over the sample: one chunk per query batch
                        ScanPlan ps = plan_linear(x->M, kk, a.nq, ns, x->num_sms, true, ns_chunks(), false);
                        uint64_t *sp = sc.s_spart.get<uint64_t>((size_t)ps.nb * ps.B * ps.nc * kk);
                        launch_linear_scan(ps, samp, ns, x->M, a.q, a.nq, cb, x->D, kk, sp, st, tables, nullptr, false,
                                           -1);
                        uint64_t *sk = sc.s_ckeys.get<uint64_t>((size_t)a.nq * kk);
                        launch_merge(sp, (int64_t)ps.nc * kk, kk, ps.nc, a.nq, kk, kk, IdMap(), nullptr, nullptr, sk,
                                     st);
                        launch_kth_bound(sk, a.nq, kk, gthr, st);
                    }
                    tr.mark("q16 bound");
                }
            }
            if (!q16 && pl.B == 8 && lut_halves(x->M) > 1) {  // M = 64 has no float B = 8 kernel
                pl = plan_linear(x->M, kk, a.nq, n_codes, x->num_sms, tables != nullptr, 1 << 30, false);
                make_mask(pl.B);
            }
            if (!pl.fast) gthr = nullptr;
            else if (!q16 && !gthr_shared) launch_fill_f32(gthr, a.nq, INFINITY, st);
            uint64_t *pp = sc.s_part.get<uint64_t>((size_t)pl.nb * pl.B * pl.nc * kk);
            launch_linear_scan(pl, scan_codes, n_codes, x->M, a.q, a.nq, cb, x->D, kk, pp, st, tables, gthr, q16,
                               TK_LINEAR, mask);
            parts = pp;
            q_stride = (int64_t)pl.nc * kk;
            p_stride = kk;
            nparts = pl.nc;
        }
    } else if (x->ivf_mode == RII_IVF_PAPER) {  // Alg. 2 exactly as printed (mode B)
        const int64_t ns = a.S ? std::max<int64_t>(a.nS, 1) : x->N;
        const int64_t P = std::min<int64_t>(x->K, ceil_div(x->K * (int64_t)a.L, ns));  // ceil(KL/|S|)
        int32_t *probes = sc.s_probe.get<int32_t>((size_t)a.nq * std::max<int64_t>(P, 1));
        float *d0 = sc.s_d0.get<float>((size_t)a.nq * x->K);
        launch_coarse_dist(x->centers.as<uint8_t>(), x->K, x->M, a.q, a.nq, cb, x->D, d0, st);  // L2-L5
        launch_sorted_probes(d0, a.nq, x->K, P, probes, st);                                     // L6
        const int64_t *off = a.S ? t.roff : x->offsets.as<int64_t>();
        const uint32_t *ids = a.S ? t.rids : x->ids.as<uint32_t>();
        int32_t *take = sc.s_take.get<int32_t>((size_t)a.nq * std::max<int64_t>(P, 1));
        launch_paper_takes(probes, a.nq, P, off, a.L, take, st);                                  // L14 cut
        uint64_t *pp = sc.s_part.get<uint64_t>((size_t)a.nq * kk);
        if (large) launch_large_ivf(codes, x->M, tables, a.nq, kk, probes, P, off, ids, take, pp, st);
        else launch_ivf_scan(codes, x->M, a.q, a.nq, cb, x->D, kk, probes, P, off, ids, pp, st, tables, take);
        parts = pp;
    } else {  // Alg. 2, mode A (reading R2)
        const int64_t P = ivf_num_probes(x, a.S != nullptr, a.nS, a.L);
        const int32_t *probes = coarse_probes(x, sc, a, tables, P, st);
        tr.mark("coarse+probes");
        const int64_t *off = a.S ? t.roff : x->offsets.as<int64_t>();
        const uint32_t *ids = a.S ? t.rids : x->ids.as<uint32_t>();
        // List-major (B queries share one list's codes) when lists are long and the
        // [nq][P][kk] partials stay small; otherwise query-major (one table per query).
        const int64_t n_cand = a.S ? std::max<int64_t>(t.n_loc, 1) : x->n_local;
        const double avg_len = (double)n_cand / (double)x->K;
        const int Bl = fast ? list_major_B(kk, avg_len, x->M) : 0;
        // (items store the start of their query run in qlist as an int32: nq * P < 2^31)
        const bool pairs_fit = (double)a.nq * P < 2147483647.0;
        bool list_major = Bl > 0 && avg_len >= 768.0 && (double)a.nq * P * kk * 8 <= 4e9 && pairs_fit;
        if (const char *mode = getenv("RII_IVF_MODE")) {  // test / tuning override: "list" or "query"
            if (!strcmp(mode, "list")) list_major = Bl > 0 && pairs_fit;
            if (!strcmp(mode, "query")) list_major = false;
        }
        if (list_major) {
            const int64_t npairs = a.nq * P;
            uint32_t *vals = sc.s_lq.get<uint32_t>(npairs);
            iota_u32_kernel<<<(unsigned)ceil_div(npairs, 256), 256, 0, st>>>(vals, npairs);
            RII_LAUNCHED();
            // Two phases (u16 tables): the pairs of the r0 nearest lists of every query run
            // first with fp32 / bf16 tables and publish each query's kk-th distance as its
            // bound; the remaining pairs run with u16 tables scaled by those bounds.
            const int64_t r0 = std::max<int64_t>(1, std::min<int64_t>(P, ceil_div(4 * kk, (int64_t)std::max(avg_len, 1.0))));
            // integer phases when the lists are long, or half as long but probed many times
            // (sift1m, lists of 1000 codes: L = 64 12.0 -> 7.1 ms on 7-bit items; L = 16
            // 5.0 -> 5.4 ms, so not there)
            const double qmin = list_q16_min_len();
            const bool q16l = q16_enabled() && q16_supported(kk) && P > r0 &&
                              (avg_len >= qmin || (avg_len >= qmin / 2 && P >= 32)) &&
                              (lut_halves(x->M) == 1 || list_u6_cfg(x->M) == 3);  // M = 64 needs the u6 items
            // Integer phases over growing rank ranges (RII_LIST_PHASES = the first rank of
            // each integer phase, e.g. "1,4,16"; default: one integer phase from r0).  Before
            // each integer phase the partial top-kk lists of every rank already scanned are
            // merged and each query's kk-th distance over them -- a bound on its final kk-th
            // (a subset of its candidates) -- re-scales its u6 tables and seeds the filter.
            PhaseBounds pb{};
            pb.rb[0] = 0;
            pb.n = 1;
            if (q16l) {
                // default: a merged-bound phase boundary at 4 r0 when at least 16 lists are
                // probed (deep10m L = 64: 15.1 -> 13.9 ms, L = 16: 8.8 -> 8.3 ms; no effect
                // at smaller L or on sift1m's u16 items)
                std::vector<int64_t> starts{r0};
                if (P >= 16 && 4 * r0 < P) starts.push_back(4 * r0);
                if (const char *e = getenv("RII_LIST_PHASES")) {
                    starts.clear();
                    for (const char *c = e; *c;) {
                        char *end = nullptr;
                        const long v = strtol(c, &end, 10);
                        if (end == c) break;
                        starts.push_back(v);
                        c = *end ? end + 1 : end;
                    }
                }
                for (int64_t r : starts)
                    if (r > pb.rb[pb.n - 1] && r < P && pb.n < 6) pb.rb[pb.n++] = r;
                pb.rb[pb.n] = P;
            }
            const int64_t nb = pb.n * x->K;
            const int32_t *keys = probes;
            if (q16l) {
                int32_t *k2 = sc.s_skey.get<int32_t>(npairs);
                split_keys_kernel<<<(unsigned)ceil_div(npairs, 256), 256, 0, st>>>(probes, npairs, P, pb, x->K, k2);
                RII_LAUNCHED();
                keys = k2;
            }
            int64_t *qoff = sc.s_qoff.get<int64_t>(nb + 1);
            uint32_t *qlist = sc.s_ql.get<uint32_t>(npairs);
            build_csr(keys, vals, npairs, nb, qoff, qlist, st);  // (query, rank) pairs grouped by list
            // RII_LIST_BOUND=1 (A/B knob): the ranks < r0 only publish a group-minimum
            // bound per query (list_bound_kernel) and the integer items cover every rank
            // (deep10m L = 64: 16.3 ms against 16.1 ms for the exact phase-A items).
            const char *lbe = getenv("RII_LIST_BOUND");
            const bool lbound = q16l && pb.n == 2 && lbe && atoi(lbe) != 0;
            const int B0 = lbound ? list_bound_B(x->M) : Bl;
            const int64_t cap = npairs / std::min(B0, 8) + npairs / 8 + 2 * nb + 2;
            int4 *items = sc.s_items.get<int4>(cap);
            tr.mark("pairs csr");
            int64_t n_ph_items[4] = {0, 0, 0, 0};
            // RII_R0_QMAJOR=1 (A/B knob, off): rank 0 alone (r0 = 1) on the query-major
            // traversal -- each query's nearest list scanned with its own table, the list
            // split over RII_R0_NSEG warps, partials written in place, their kk-th distance
            // published as the bound -- instead of list items holding the ~nq / K queries
            // whose nearest list it is.  Measured slower (deep10m L = 64: 11.54 ms with
            // list items, 12.40 / 12.55 / 12.64 ms with 4 / 8 / 16 warps per list, 15.79
            // with one; profiles/r02k_ab_rank0_qmajor_deep10m.jsonl); parity-tested.
            const char *r0e = getenv("RII_R0_QMAJOR");
            const bool r0q = q16l && !lbound && r0 == 1 && pb.n >= 2 && x->M <= 32 && tables != nullptr &&
                             r0e && atoi(r0e) != 0;
            if (!r0q) n_ph_items[0] = build_list_items(qoff, x->K, B0, qlist, P, items, cap, st);
            int64_t n_items = n_ph_items[0];
            const int Bi = list_int_B(x->M, kk);  // queries per integer item
            const int64_t *qoff_i = qoff + x->K;
            const uint32_t *qlist_i = qlist;
            if (lbound) {  // integer items over all ranks: the unsplit (query, rank) CSR
                int64_t *qoff2 = sc.s_qoff2.get<int64_t>(x->K + 1);
                uint32_t *ql2 = sc.s_ql2.get<uint32_t>(npairs);
                build_csr(probes, vals, npairs, x->K, qoff2, ql2, st);
                qoff_i = qoff2;
                qlist_i = ql2;
            }
            for (int ph = 1; ph < pb.n; ++ph) {
                n_ph_items[ph] = build_list_items(lbound ? qoff_i : qoff + ph * x->K, x->K, Bi, qlist_i, P,
                                                  items + n_items, cap - n_items, st);
                n_items += n_ph_items[ph];
            }
            tr.mark("items");
            uint64_t *pp = sc.s_part.get<uint64_t>((size_t)npairs * kk);
            float *gthr = sc.s_gthr.get<float>(a.nq);
            launch_fill_f32(gthr, a.nq, INFINITY, st);
            tr.mark("alloc partials");
            // items stream their list as a contiguous range of the list-ordered mirror;
            // keys carry ids (the CSR entry of the position), so ties resolve by id (CA4)
            const uint8_t *lcodes = a.S ? t.rmirror : x->mirror.as<uint8_t>();
            ScanArgs sa{};
            sa.codes = lcodes; sa.n_codes = a.S ? t.n_loc : x->n_local;  // mirror rows
            sa.rcodes = codes; sa.q = a.q; sa.nq = a.nq; sa.cb = cb; sa.ds = x->ds; sa.kk = kk;
            sa.out = pp;
            sa.items = items; sa.qlist = qlist; sa.P = P; sa.offsets = off; sa.ids = ids; sa.gthr = gthr;
            sa.tables = tables;
            if (lbound)
                launch_list_bound(codes, x->M, items, n_ph_items[0], off, ids, qlist, P, tables, kk, gthr, st);
            else if (r0q) {
                int32_t *pr0 = sc.s_pr0.get<int32_t>(a.nq);
                launch_strided_gather_i32(probes, P, a.nq, pr0, st);  // every query's nearest list
                launch_ivf_scan(codes, x->M, a.q, a.nq, cb, x->D, kk, pr0, 1, off, ids, pp, st, tables, nullptr,
                                P * kk, r0q_nseg());
                launch_rank_bound(pp, a.nq, P * kk, kk, gthr, st);
            } else
                launch_list_scan(x->M, Bl, sa, n_ph_items[0], st);
            int64_t done = n_ph_items[0];
            if (lbound) sa.qlist = qlist_i;
            for (int ph = 1; ph < pb.n; ++ph) {
                if (n_ph_items[ph] == 0) continue;
                tr.mark("list scan phase");
                if (pb.rb[ph] > 1 && !lbound) {  // merged bound over the ranks [0, rb[ph]) scanned so far
                    uint64_t *mk = sc.s_ckeys.get<uint64_t>((size_t)a.nq * kk);
                    launch_merge(pp, P * kk, kk, (int)pb.rb[ph], a.nq, kk, kk, IdMap(), nullptr, nullptr, mk, st);
                    merged_bound_kernel<<<(unsigned)ceil_div(a.nq, 256), 256, 0, st>>>(mk, a.nq, kk, gthr);
                    RII_LAUNCHED();
                }
                float *qsc = sc.s_qscale.get<float>(a.nq);
                if (list_u6_cfg(x->M) >= 3) {  // u6 oct items
                    uint8_t *t8 = sc.s_tab16.get<uint8_t>((size_t)a.nq * lut_q_floats(x->M));
                    launch_u6_tables(tables, gthr, a.nq, x->M, t8, qsc, st, list_u7(x->M));
                    sa.qtab8 = t8;
                } else {
                    uint16_t *t16 = sc.s_tab16.get<uint16_t>((size_t)a.nq * LUT_Q_FLOATS);
                    launch_q16_tables(tables, gthr, a.nq, x->M, t16, qsc, st);
                    sa.qtab16 = t16;
                }
                sa.qscale = qsc;
                sa.items = items + done;
                launch_list_scan(x->M, Bi, sa, n_ph_items[ph], st, true);
                done += n_ph_items[ph];
            }
            tr.mark("list scan");
            parts = pp;
            if (Bl != 8 && !lbound) {  // fp32-pair items keep lane-rotated keys: rescore in the merge
                rs.codes = codes;
                rs.tables = tables;
                rs.M = x->M;
            }
            q_stride = P * kk;
            p_stride = kk;
            nparts = (int)P;
        } else {
            uint64_t *pp = sc.s_part.get<uint64_t>((size_t)a.nq * kk);
            if (large) launch_large_ivf(codes, x->M, tables, a.nq, kk, probes, P, off, ids, nullptr, pp, st);
            else launch_ivf_scan(codes, x->M, a.q, a.nq, cb, x->D, kk, probes, P, off, ids, pp, st, tables);
            parts = pp;
        }
    }
    tr.mark("scan");
    launch_merge(parts, q_stride, p_stride, nparts, a.nq, kk, a.topk, map, out_ids, out_dist, out_keys, st, rs);
    tr.mark("merge");
}

// Query batches of at most QBATCH queries bound the per-call scratch (tables:
// 32 KB per query; partials).
constexpr int64_t QBATCH = 16384;

void search_local(const rii_index *x, QueryScratch &sc, const QueryArgs &a, cudaStream_t st, int64_t *out_ids,
                  float *out_dist, uint64_t *out_keys) {
    const Targets t = prepare_targets(x, sc, a, st);
    // IVF: smaller batches keep the batch's per-query tables (32 KB each) L2-resident
    // while the list-major items re-read them once per probed list.
    int64_t qb = QBATCH;
    if (a.path == RII_PATH_IVF) {
        const char *e = getenv("RII_IVF_QBATCH");
        qb = e ? std::max<int64_t>(atoll(e), 1) : QBATCH;
    }
    for (int64_t q0 = 0; q0 < a.nq; q0 += qb) {
        QueryArgs b = a;
        b.q = a.q + q0 * x->D;
        b.nq = std::min<int64_t>(qb, a.nq - q0);
        search_batch(x, sc, b, t, st, out_ids ? out_ids + q0 * a.topk : nullptr, out_dist ? out_dist + q0 * a.topk : nullptr,
                     out_keys ? out_keys + q0 * a.kk : nullptr);
    }
}

void check_targets(const rii_index *x, QueryScratch &sc, const int64_t *S, int64_t nS, cudaStream_t st) {
    if (!S || nS == 0) return;
    int *flag = sc.s_flag.get<int>(1);
    RII_CUDA(cudaMemsetAsync(flag, 0, 4, st));
    launch_validate_targets(S, nS, x->N, flag, st);
    int h = 0;
    RII_CUDA(cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, st));
    RII_CUDA(cudaStreamSynchronize(st));
    arg_check(h == 0, "target_ids must be strictly ascending and inside [0, N)");
}

void common_query_checks(const rii_index *x, int64_t nq, int topk, const int64_t *S, int64_t nS, int L,
                         rii_path path) {
    arg_check(x != nullptr, "index is NULL");
    state_check(x->trained, "index has no code book (call rii_train or rii_set_codebook)");
    arg_check(nq >= 0, "nq must be >= 0");
    arg_check(topk >= 1 && topk <= 1024, "topk must be in [1, 1024]");
    arg_check(!S || nS >= 0, "n_target must be >= 0");
    arg_check(!S || nS <= x->N, "n_target larger than N");
    arg_check(L >= 1, "L must be >= 1");
    arg_check(path == RII_PATH_AUTO || path == RII_PATH_LINEAR || path == RII_PATH_IVF, "unknown path");
}

}  // namespace

extern "C" {

const char *rii_last_error(const rii_index *) { return t_err.c_str(); }

uint64_t rii_launch_count(void) { return g_launches.load(); }

void rii_kernel_timing(int32_t enable) {
    std::lock_guard<std::mutex> lk(g_tmu);
    drain_pairs();
    for (int i = 0; i < TK_COUNT; ++i) { g_total_ms[i] = 0; g_count[i] = 0; }
    g_timing = enable != 0;
}

rii_status rii_kernel_timing_read(int32_t which, double *total_ms, int64_t *launches) {
    return guarded([&] {
        arg_check(which >= 0 && which < TK_COUNT, "which must be in [0, 7)");
        std::lock_guard<std::mutex> lk(g_tmu);
        drain_pairs();
        if (total_ms) *total_ms = g_total_ms[which];
        if (launches) *launches = g_count[which];
    });
}

rii_status rii_debug_counters(int32_t enable) {
    return guarded([&] {
        unsigned long long *d = g_dbg.load();
        if (enable) {
            if (!d) {
                RII_CUDA(cudaMalloc(&d, DBG_COUNT * sizeof(unsigned long long)));
                g_dbg.store(d);
            }
            RII_CUDA(cudaMemset(d, 0, DBG_COUNT * sizeof(unsigned long long)));
            RII_CUDA(cudaDeviceSynchronize());
        } else if (d) {
            g_dbg.store(nullptr);
            RII_CUDA(cudaDeviceSynchronize());
            cudaFree(d);
        }
    });
}

rii_status rii_debug_counters_read(int64_t *out, int32_t n) {
    return guarded([&] {
        arg_check(out != nullptr && n >= 0, "bad arguments");
        unsigned long long h[DBG_COUNT] = {};
        if (unsigned long long *d = g_dbg.load()) {
            RII_CUDA(cudaDeviceSynchronize());
            RII_CUDA(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
        }
        for (int i = 0; i < n; ++i) out[i] = i < DBG_COUNT ? (int64_t)h[i] : 0;
    });
}

int32_t rii_partial_width(int32_t topk) { return partial_width(topk); }

rii_status rii_shard_range(int64_t n, int32_t rank, int32_t world, int64_t *lo, int64_t *hi) {
    return guarded([&] {
        arg_check(lo && hi, "NULL argument");
        arg_check(n >= 0 && world >= 1 && rank >= 0 && rank < world, "need n >= 0 and 0 <= rank < world");
        rank_rows(n, rank, world, *lo, *hi);
    });
}

rii_status rii_nccl_unique_id(void *out) {
    return guarded([&] {
        arg_check(out != nullptr, "out is NULL");
        nccl_unique_id(out);
    });
}

static rii_status create_impl(int32_t D, int32_t M, int32_t Ks, int32_t device, int32_t rank, int32_t world,
                              const void *nccl_id, const rii_transport *tr, rii_index **out) {
    if (out) *out = nullptr;
    return guarded([&] {
        arg_check(out != nullptr, "out is NULL");
        arg_check(M >= 1 && M <= 256, "M must be in [1, 256]");
        arg_check(D >= M && D % M == 0, "D must be a positive multiple of M");
        arg_check(D / M <= 64, "D / M must be <= 64");
        arg_check(Ks == 256, "Ks must be 256 (one byte per subspace, P:287)");
        arg_check(world >= 1 && rank >= 0 && rank < world, "need 0 <= rank < world");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw Error(RII_ERR_CUDA, "no CUDA device");
        arg_check(device >= 0 && device < ndev, "device ordinal out of range");
        DeviceGuard g(device);
        auto *x = new rii_index();
        x->D = D;
        x->M = M;
        x->ds = D / M;
        x->device = device;
        x->rank = rank;
        x->world = world;
        RII_CUDA(cudaDeviceGetAttribute(&x->num_sms, cudaDevAttrMultiProcessorCount, device));
        // keep memory freed by cudaFreeAsync cached in the pool (no re-mapping per call:
        // every query allocates its scratch from it)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        try {
            x->cb.get<float>((size_t)M * KS * x->ds);
            if (world > 1 && tr) x->comm = host_comm_create(*tr, rank, world);
            else if (world > 1 && nccl_id) x->comm = nccl_comm_create(nccl_id, rank, world);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

rii_status rii_create(int32_t D, int32_t M, int32_t Ks, int32_t device, int32_t rank, int32_t world,
                      const void *nccl_id, rii_index **out) {
    return create_impl(D, M, Ks, device, rank, world, nccl_id, nullptr, out);
}

rii_status rii_create_with_transport(int32_t D, int32_t M, int32_t Ks, int32_t device, int32_t rank, int32_t world,
                                     const rii_transport *transport, rii_index **out) {
    if (out) *out = nullptr;
    if (!transport || !transport->allgather || world < 2)
        return fail(RII_ERR_ARG, "rii_create_with_transport needs world > 1 and a transport with allgather");
    return create_impl(D, M, Ks, device, rank, world, nullptr, transport, out);
}

void rii_destroy(rii_index *x) {
    if (!x) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(x->device);
    delete x->comm;
    delete x;
    if (prev >= 0) cudaSetDevice(prev);
}

rii_status rii_train(rii_index *x, const float *xs, int64_t n, int32_t n_iter, uint64_t seed, rii_mem where,
                     void *stream) {
    return guarded([&] {
        arg_check(x && xs, "NULL argument");
        arg_check(n_iter >= 0, "n_iter must be >= 0");
        state_check(x->N == 0, "the code book can only be (re)trained while the index is empty");
        if (n < KS) throw Error(RII_ERR_TRAIN, "training needs n >= 256 rows");
        DeviceGuard g(x->device);
        cudaStream_t st = (cudaStream_t)stream;
        const float *dx = xs;
        if (where == RII_MEM_HOST) {
            float *b = x->s_x.get<float>((size_t)n * x->D);
            RII_CUDA(cudaMemcpyAsync(b, xs, (size_t)n * x->D * 4, cudaMemcpyHostToDevice, st));
            dx = b;
        }
        dx = rotate_input(x, x->s_xrot, dx, n, st);  // OPQ: train on R x
        int *err = x->s_flag.get<int>(1);
        RII_CUDA(cudaMemsetAsync(err, 0, 4, st));
        Buf tmp;
        float *cb = tmp.get<float>((size_t)x->M * KS * x->ds);
        run_train(dx, n, x->D, x->M, n_iter, seed, cb, err, st);
        int h = 0;
        RII_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, st));
        RII_CUDA(cudaStreamSynchronize(st));
        if (h) throw Error(RII_ERR_TRAIN, "fewer than 256 distinct sub-vectors in some subspace");
        RII_CUDA(cudaMemcpyAsync(x->cb.as<float>(), cb, (size_t)x->M * KS * x->ds * 4, cudaMemcpyDeviceToDevice, st));
        RII_CUDA(cudaStreamSynchronize(st));
        x->trained = true;
        x->T_valid = false;
    });
}

rii_status rii_set_rotation(rii_index *x, const float *R) {
    return guarded([&] {
        arg_check(x != nullptr, "index is NULL");
        state_check(x->N == 0, "the rotation can only be set while the index is empty");
        DeviceGuard g(x->device);
        if (!R) {
            x->has_rot = false;
        } else {
            const size_t DD = (size_t)x->D * x->D;
            x->rot_host.assign(R, R + DD);
            std::vector<float> Rt(DD);
            for (int i = 0; i < x->D; ++i)
                for (int j = 0; j < x->D; ++j) Rt[(size_t)j * x->D + i] = R[(size_t)i * x->D + j];
            RII_CUDA(cudaMemcpy(x->rot.get<float>(DD), R, DD * 4, cudaMemcpyHostToDevice));
            RII_CUDA(cudaMemcpy(x->rotT.get<float>(DD), Rt.data(), DD * 4, cudaMemcpyHostToDevice));
            x->has_rot = true;
        }
        x->trained = false;  // the code book lives in the rotated space: train or set it afterwards
        x->T_valid = false;
    });
}

rii_status rii_get_rotation(const rii_index *x, float *R, int32_t *has_rotation) {
    return guarded([&] {
        arg_check(x != nullptr, "index is NULL");
        if (has_rotation) *has_rotation = x->has_rot ? 1 : 0;
        if (R) {
            for (int i = 0; i < x->D; ++i)
                for (int j = 0; j < x->D; ++j)
                    R[(size_t)i * x->D + j] = x->has_rot ? x->rot_host[(size_t)i * x->D + j] : (i == j ? 1.f : 0.f);
        }
    });
}

rii_status rii_rotate(const rii_index *x, const float *in, int64_t n, float *out, void *stream) {
    return guarded([&] {
        arg_check(x && (n == 0 || (in && out)) && n >= 0, "bad arguments");
        DeviceGuard g(x->device);
        cudaStream_t st = (cudaStream_t)stream;
        if (n == 0) return;
        if (x->has_rot) launch_rotate(x->rotT.as<float>(), in, n, x->D, out, st);
        else RII_CUDA(cudaMemcpyAsync(out, in, (size_t)n * x->D * 4, cudaMemcpyDeviceToDevice, st));
        RII_CUDA(cudaStreamSynchronize(st));
    });
}

rii_status rii_train_opq(rii_index *x, const float *xs, int64_t n, int32_t n_opq_iter, int32_t n_iter,
                         uint64_t seed, rii_mem where, void *stream) {
    return guarded([&] {
        arg_check(x && xs, "NULL argument");
        arg_check(n_opq_iter >= 0 && n_iter >= 0, "iteration counts must be >= 0");
        state_check(x->N == 0, "the rotation can only be trained while the index is empty");
        if (n < KS) throw Error(RII_ERR_TRAIN, "training needs n >= 256 rows");
        DeviceGuard g(x->device);
        cudaStream_t st = (cudaStream_t)stream;
        const int D = x->D;
        const size_t DD = (size_t)D * D;
        Buf xb, yb, xr, cbb, cod, Cb;
        const float *dx = xs;
        if (where == RII_MEM_HOST) {
            float *b = xb.get<float>((size_t)n * D);
            RII_CUDA(cudaMemcpyAsync(b, xs, (size_t)n * D * 4, cudaMemcpyHostToDevice, st));
            dx = b;
        }
        std::vector<float> R(DD, 0.f);
        for (int i = 0; i < D; ++i) R[(size_t)i * D + i] = 1.f;  // R_0 = I
        std::vector<double> Ch(DD);
        int *err = x->s_flag.get<int>(1);
        float *cb = cbb.get<float>((size_t)x->M * KS * x->ds);
        uint8_t *codes = cod.get<uint8_t>((size_t)n * x->M);
        float *y = yb.get<float>((size_t)n * D);
        double *Cd = Cb.get<double>(DD);
        for (int it = 0; it < n_opq_iter; ++it) {
            // (1) PQ on the rotated data, (2) orthogonal Procrustes R = argmin sum ||y - R x||^2
            RII_CUDA(cudaStreamSynchronize(st));
            const rii_status s1 = rii_set_rotation(x, R.data());
            if (s1 != RII_OK) throw Error(s1, t_err);
            const float *rx = rotate_input(x, xr, dx, n, st);
            RII_CUDA(cudaMemsetAsync(err, 0, 4, st));
            run_train(rx, n, D, x->M, std::max(1, n_iter / 2), seed + (uint64_t)it, cb, err, st);
            launch_encode(rx, n, D, x->M, cb, codes, st);
            launch_decode(codes, n, x->M, D, cb, y, st);
            launch_cross(y, dx, n, D, Cd, st);
            RII_CUDA(cudaMemcpyAsync(Ch.data(), Cd, DD * 8, cudaMemcpyDeviceToHost, st));
            RII_CUDA(cudaStreamSynchronize(st));
            procrustes_rotation(Ch.data(), D, R.data());
        }
        RII_CUDA(cudaStreamSynchronize(st));
        const rii_status s2 = rii_set_rotation(x, R.data());
        if (s2 != RII_OK) throw Error(s2, t_err);
        const rii_status s3 = rii_train(x, dx, n, n_iter, seed, RII_MEM_DEVICE, stream);  // final code book on R x
        if (s3 != RII_OK) throw Error(s3, t_err);
    });
}

rii_status rii_set_codebook(rii_index *x, const float *cb) {
    return guarded([&] {
        arg_check(x && cb, "NULL argument");
        state_check(x->N == 0, "the code book can only be set while the index is empty");
        DeviceGuard g(x->device);
        RII_CUDA(cudaMemcpy(x->cb.as<float>(), cb, (size_t)x->M * KS * x->ds * 4, cudaMemcpyHostToDevice));
        x->trained = true;
        x->T_valid = false;
    });
}

rii_status rii_get_codebook(const rii_index *x, float *out) {
    return guarded([&] {
        arg_check(x && out, "NULL argument");
        state_check(x->trained, "no code book");
        DeviceGuard g(x->device);
        RII_CUDA(cudaMemcpy(out, x->cb.as<float>(), (size_t)x->M * KS * x->ds * 4, cudaMemcpyDeviceToHost));
    });
}

rii_status rii_add(rii_index *x, const float *xs, int64_t n, rii_mem where, void *stream, int64_t *first_id) {
    return guarded([&] {
        arg_check(x != nullptr, "index is NULL");
        arg_check(n >= 0 && (n == 0 || xs), "bad x / n");
        state_check(x->trained, "index has no code book");
        arg_check(x->N + n < (1ll << 32), "at most 2^32 ids");
        DeviceGuard g(x->device);
        cudaStream_t st = (cudaStream_t)stream;
        const int64_t first = x->N;
        if (first_id) *first_id = first;
        int64_t lo, hi;
        rank_rows(n, x->rank, x->world, lo, hi);
        const int64_t cnt = hi - lo;
        if (cnt > 0) {
            uint8_t *codes = x->codes.grow<uint8_t>((size_t)(x->n_local + cnt) * x->M, (size_t)x->n_local * x->M, st);
            const int64_t chunk = (int64_t)1 << 22;  // bound the staging buffer for host input
            for (int64_t s = lo; s < hi; s += chunk) {
                const int64_t e = std::min(hi, s + chunk);
                const float *dx = xs + s * x->D;
                if (where == RII_MEM_HOST) {
                    float *b = x->s_x.get<float>((size_t)(e - s) * x->D);
                    RII_CUDA(cudaMemcpyAsync(b, dx, (size_t)(e - s) * x->D * 4, cudaMemcpyHostToDevice, st));
                    dx = b;
                }
                dx = rotate_input(x, x->s_xrot, dx, e - s, st);  // OPQ: encode R x
                launch_encode(dx, e - s, x->D, x->M, x->cb.as<float>(), codes + (x->n_local + (s - lo)) * x->M, st);
            }
            if (x->K > 0) {
                ensure_T(x, st);
                int32_t *as = x->assign.grow<int32_t>((size_t)(x->n_local + cnt), (size_t)x->n_local * 4, st);
                launch_assign(codes + x->n_local * x->M, cnt, x->centers.as<uint8_t>(), x->K, x->M, x->T.as<float>(),
                              as + x->n_local, nullptr, st);
            }
            x->segs.push_back({x->n_local, first + lo, cnt});
            x->n_local += cnt;
            upload_segs(x, st);
            if (x->K > 0) rebuild_csr(x, st);  // PushBack(W_a(n), n): lists stay ascending
        }
        x->N += n;
        RII_CUDA(cudaStreamSynchronize(st));
    });
}

rii_status rii_reconfigure(rii_index *x, int32_t nlist, int32_t n_iter, uint64_t seed, void *stream) {
    return guarded([&] {
        arg_check(x != nullptr, "index is NULL");
        state_check(x->trained, "index has no code book");
        arg_check(nlist >= 1 && nlist <= x->N, "nlist must be in [1, N]");
        arg_check(n_iter >= 0, "n_iter must be >= 0");
        DeviceGuard g(x->device);
        cudaStream_t st = (cudaStream_t)stream;
        ensure_T(x, st);
        const int M = x->M;
        const int64_t ns = std::min<int64_t>(x->N, (int64_t)100 * nlist);
        Buf pos_b, X_b;
        uint8_t *X = X_b.get<uint8_t>((size_t)ns * M);
        if (x->world == 1) {
            uint32_t *pos = pos_b.get<uint32_t>(ns);
            select_sample(x->n_local, IdMap(), ns, seed, pos, st);
            gather_u32pos_codes_kernel<<<(unsigned)ceil_div(ns, 256), 256, 0, st>>>(x->codes.as<uint8_t>(), M, pos, ns,
                                                                                   X);
            RII_LAUNCHED();
        } else {
            state_check(x->comm != nullptr, "multi-rank reconfigure needs a communicator (NCCL id or transport)");
            // each rank contributes its ns smallest keys; the global ns smallest are
            // selected identically on every rank after an all-gather.
            const int64_t nl = std::min<int64_t>(x->n_local, ns);
            Buf lk, lc, gk, gc, sk, sv, iv;
            uint32_t *pos = pos_b.get<uint32_t>(std::max<int64_t>(nl, 1));
            uint64_t *keys = lk.get<uint64_t>(ns);
            uint8_t *lcodes = lc.get<uint8_t>((size_t)ns * M);
            RII_CUDA(cudaMemsetAsync(keys, 0xff, (size_t)ns * 8, st));
            RII_CUDA(cudaMemsetAsync(lcodes, 0, (size_t)ns * M, st));
            if (nl > 0) {
                select_sample(x->n_local, local_map(x), nl, seed, pos, st);
                gather_u32pos_codes_kernel<<<(unsigned)ceil_div(nl, 256), 256, 0, st>>>(x->codes.as<uint8_t>(), M,
                                                                                        pos, nl, lcodes);
                RII_LAUNCHED();
                sample_keys_for_positions(x->n_local, local_map(x), pos, nl, seed, keys, st);
            }
            uint64_t *gkeys = gk.get<uint64_t>((size_t)ns * x->world);
            uint8_t *gcodes = gc.get<uint8_t>((size_t)ns * x->world * M);
            x->comm->allgather(keys, gkeys, (size_t)ns * 8, st);
            x->comm->allgather(lcodes, gcodes, (size_t)ns * M, st);
            const int64_t tot = ns * x->world;
            uint32_t *order = sv.get<uint32_t>(tot);
            sort_keys_with_index(gkeys, tot, order, st);
            gather_u32pos_codes_kernel<<<(unsigned)ceil_div(ns, 256), 256, 0, st>>>(gcodes, M, order, ns, X);
            RII_LAUNCHED();
        }
        Buf newc;
        uint8_t *C = newc.get<uint8_t>((size_t)nlist * M);
        int *err = x->s_flag.get<int>(1);
        RII_CUDA(cudaMemsetAsync(err, 0, 4, st));
        run_pqkmeans(X, ns, nlist, M, x->T.as<float>(), n_iter, C, err, st);
        int h = 0;
        RII_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, st));
        RII_CUDA(cudaStreamSynchronize(st));
        arg_check(h == 0, "fewer than nlist distinct codes in the reconfigure sample");
        uint8_t *cent = x->centers.get<uint8_t>((size_t)nlist * M);
        RII_CUDA(cudaMemcpyAsync(cent, C, (size_t)nlist * M, cudaMemcpyDeviceToDevice, st));
        x->K = nlist;
        x->theta_fit = false;
        int32_t *as = x->assign.get<int32_t>(x->n_local + 1);
        launch_assign(x->codes.as<uint8_t>(), x->n_local, cent, x->K, M, x->T.as<float>(), as, nullptr, st);
        rebuild_csr(x, st);
        x->theta = -1;
        RII_CUDA(cudaStreamSynchronize(st));
    });
}

static rii_status query_impl(const rii_index *x, const float *q, int64_t nq, int32_t topk, const int64_t *S,
                             int64_t nS, int32_t L, rii_path path, rii_mem where, void *stream, int64_t *out_ids,
                             float *out_dist, int32_t *path_used, uint64_t *out_keys) {
    return guarded([&] {
        common_query_checks(x, nq, topk, S, nS, L, path);
        DeviceGuard g(x->device);
        cudaStream_t st = (cudaStream_t)stream;
        const int used = resolve_path(x, nS, S != nullptr, L, path);
        state_check(!(used == RII_PATH_IVF && x->ivf_mode == RII_IVF_PAPER && x->world > 1),
                    "RII_IVF_PAPER (global early stop) is single-GPU only");
        if (path_used) *path_used = used;
        if (nq == 0) return;
        arg_check(q && (out_keys || (out_ids && out_dist)), "NULL argument");
        state_check(out_keys || x->world == 1 || x->comm != nullptr,
                    "detached shard (world > 1, no communicator): use rii_query_partial + rii_merge_partials");
        QueryScratch sc(st);  // this call's own scratch (concurrent readers)
        const bool host = where == RII_MEM_HOST && !out_keys;
        const float *dq = q;
        const int64_t *dS = S;
        if (host) {
            float *b = sc.s_q.get<float>((size_t)nq * x->D);
            RII_CUDA(cudaMemcpyAsync(b, q, (size_t)nq * x->D * 4, cudaMemcpyHostToDevice, st));
            dq = b;
            if (S && nS > 0) {
                int64_t *sb = sc.s_gather.get<int64_t>(nS);
                RII_CUDA(cudaMemcpyAsync(sb, S, (size_t)nS * 8, cudaMemcpyHostToDevice, st));
                dS = sb;
            }
        }
        check_targets(x, sc, dS, S ? nS : 0, st);
        dq = rotate_input(x, sc.s_qrot, dq, nq, st);  // OPQ: "an input vector is first rotated"
        const bool collective = !out_keys && x->world > 1 && x->comm != nullptr;
        const int exec = decide_exec(x, used, S != nullptr, S ? nS : 0, L);
        QueryArgs a{dq, nq, topk, partial_width(topk), S ? dS : nullptr, S ? nS : 0, L, exec, collective};
        int64_t *oid = out_ids;
        float *od = out_dist;
        if (host) {
            oid = sc.s_out_ids.get<int64_t>((size_t)nq * topk);
            od = sc.s_out_dist.get<float>((size_t)nq * topk);
        }
        if (out_keys) {
            search_local(x, sc, a, st, nullptr, nullptr, out_keys);
        } else if (x->world == 1) {
            search_local(x, sc, a, st, oid, od, nullptr);
        } else {
            // the one exchange step: all-gather of every rank's top-kk
            // keys (global ids), then the same merge on every rank
            const int kk = a.kk;
            uint64_t *lk = sc.s_keys.get<uint64_t>((size_t)nq * kk * (x->world + 1));
            uint64_t *gk = lk + (size_t)nq * kk;
            search_local(x, sc, a, st, nullptr, nullptr, lk);
            x->comm->allgather(lk, gk, (size_t)nq * kk * 8, st);
            launch_merge(gk, kk, (int64_t)nq * kk, x->world, nq, kk, topk, IdMap(), oid, od, nullptr, st);
        }
        if (host) {
            RII_CUDA(cudaMemcpyAsync(out_ids, oid, (size_t)nq * topk * 8, cudaMemcpyDeviceToHost, st));
            RII_CUDA(cudaMemcpyAsync(out_dist, od, (size_t)nq * topk * 4, cudaMemcpyDeviceToHost, st));
        }
        RII_CUDA(cudaStreamSynchronize(st));
    });
}

rii_status rii_query(const rii_index *x, const float *q, int64_t nq, int32_t topk, const int64_t *target_ids,
                     int64_t n_target, int32_t L, rii_path path, rii_mem where, void *stream, int64_t *out_ids,
                     float *out_dist, int32_t *path_used) {
    return query_impl(x, q, nq, topk, target_ids, n_target, L, path, where, stream, out_ids, out_dist, path_used,
                      nullptr);
}

rii_status rii_query_partial(const rii_index *x, const float *q, int64_t nq, int32_t topk, const int64_t *target_ids,
                             int64_t n_target, int32_t L, rii_path path, void *stream, uint64_t *out_keys,
                             int32_t *path_used) {
    return query_impl(x, q, nq, topk, target_ids, n_target, L, path, RII_MEM_DEVICE, stream, nullptr, nullptr,
                      path_used, out_keys);
}

rii_status rii_merge_partials(const uint64_t *keys, int32_t parts, int64_t nq, int32_t topk, void *stream,
                              int64_t *out_ids, float *out_dist) {
    return guarded([&] {
        arg_check(keys && out_ids && out_dist, "NULL argument");
        arg_check(parts >= 1 && nq >= 0 && topk >= 1 && topk <= 1024, "bad parts / nq / topk");
        const int kk = partial_width(topk);
        cudaStream_t st = (cudaStream_t)stream;
        launch_merge(keys, kk, (int64_t)nq * kk, parts, nq, kk, topk, IdMap(), out_ids, out_dist, nullptr, st);
        RII_CUDA(cudaStreamSynchronize(st));
    });
}

rii_status rii_get_codes(const rii_index *x, int64_t first, int64_t n, uint8_t *out) {
    return guarded([&] {
        arg_check(x && (n == 0 || out), "NULL argument");
        arg_check(first >= 0 && n >= 0 && first + n <= x->N, "range outside [0, N)");
        DeviceGuard g(x->device);
        int64_t done = 0;
        for (auto &s : x->segs) {  // copy the parts of [first, first+n) stored here
            const int64_t a = std::max(first, s.global_first), b = std::min(first + n, s.global_first + s.count);
            if (a >= b) continue;
            RII_CUDA(cudaMemcpy(out + (a - first) * x->M, x->codes.as<uint8_t>() + (a - s.global_first + s.local_off) * x->M,
                                (size_t)(b - a) * x->M, cudaMemcpyDeviceToHost));
            done += b - a;
        }
        arg_check(done == n, "part of the requested range is stored on another rank");
    });
}

rii_status rii_get_centers(const rii_index *x, uint8_t *out) {
    return guarded([&] {
        arg_check(x && out, "NULL argument");
        DeviceGuard g(x->device);
        if (x->K) RII_CUDA(cudaMemcpy(out, x->centers.as<uint8_t>(), (size_t)x->K * x->M, cudaMemcpyDeviceToHost));
    });
}

rii_status rii_get_postings(const rii_index *x, int64_t *offsets, int64_t *ids) {
    return guarded([&] {
        arg_check(x && offsets && ids, "NULL argument");
        state_check(x->K > 0, "no posting lists (K == 0)");
        DeviceGuard g(x->device);
        RII_CUDA(cudaMemcpy(offsets, x->offsets.as<int64_t>(), (size_t)(x->K + 1) * 8, cudaMemcpyDeviceToHost));
        if (x->n_local) {
            Buf w;
            int64_t *d = w.get<int64_t>(x->n_local);
            widen_ids_kernel<<<(unsigned)ceil_div(x->n_local, 256), 256>>>(x->ids.as<uint32_t>(), x->n_local,
                                                                           local_map(x), d);
            RII_LAUNCHED();
            RII_CUDA(cudaMemcpy(ids, d, (size_t)x->n_local * 8, cudaMemcpyDeviceToHost));
        }
    });
}

}  // extern "C"

namespace {
struct FileW {
    FILE *f;
    void put(const void *p, size_t n) {
        if (n && fwrite(p, 1, n, f) != n) throw Error(RII_ERR_ARG, "write failed");
    }
    template <class T>
    void val(T v) { put(&v, sizeof(T)); }
};
struct FileR {
    FILE *f;
    void get(void *p, size_t n, const char *what) {
        if (n && fread(p, 1, n, f) != n) throw Error(RII_ERR_ARG, std::string("truncated index file: ") + what);
    }
    template <class T>
    T val(const char *what) { T v; get(&v, sizeof(T), what); return v; }
};
template <class T>
void dev_to_file(FileW &w, const T *d, size_t n) {
    std::vector<T> h(n);
    if (n) RII_CUDA(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
    w.put(h.data(), n * sizeof(T));
}
template <class T>
void file_to_dev(FileR &r, T *d, size_t n, const char *what) {
    std::vector<T> h(n);
    r.get(h.data(), n * sizeof(T), what);
    if (n) RII_CUDA(cudaMemcpy(d, h.data(), n * sizeof(T), cudaMemcpyHostToDevice));
}
}  // namespace

extern "C" {

rii_status rii_save(const rii_index *x, const char *path) {
    return guarded([&] {
        arg_check(x && path, "NULL argument");
        state_check(x->trained, "nothing to save: no code book");
        DeviceGuard g(x->device);
        FILE *f = fopen(path, "wb");
        arg_check(f != nullptr, "cannot open file for writing");
        FileW w{f};
        try {
            if (x->world == 1) {
                // SPEC's RII1 layout, bit for bit
                w.put("RII1", 4);
                const bool analytic = x->theta < 0 && !x->theta_fit;
                for (uint32_t v : {1u, (uint32_t)x->D, (uint32_t)x->M, (uint32_t)KS, (uint32_t)x->N, (uint32_t)x->K})
                    w.val(v);
                w.val<uint64_t>(x->theta >= 0 ? (uint64_t)x->theta : 0);
                w.val<uint32_t>(1);  // default_L
                w.val<uint32_t>((x->has_rot ? 1u : 0u) | (analytic ? 2u : 0u));
                dev_to_file(w, x->cb.as<float>(), (size_t)x->M * KS * x->ds);
                if (x->has_rot) w.put(x->rot_host.data(), x->rot_host.size() * 4);
                dev_to_file(w, x->codes.as<uint8_t>(), (size_t)x->n_local * x->M);
                if (x->K > 0) {
                    dev_to_file(w, x->centers.as<uint8_t>(), (size_t)x->K * x->M);
                    std::vector<int64_t> off((size_t)x->K + 1);
                    std::vector<uint32_t> ids((size_t)x->n_local);
                    RII_CUDA(cudaMemcpy(off.data(), x->offsets.as<int64_t>(), off.size() * 8, cudaMemcpyDeviceToHost));
                    if (x->n_local)
                        RII_CUDA(cudaMemcpy(ids.data(), x->ids.as<uint32_t>(), ids.size() * 4, cudaMemcpyDeviceToHost));
                    for (int64_t k = 0; k < x->K; ++k) {
                        w.val<uint32_t>((uint32_t)(off[k + 1] - off[k]));
                        w.put(ids.data() + off[k], (size_t)(off[k + 1] - off[k]) * 4);
                    }
                }
                if (x->ivf_mode != 0 || x->theta_fit) {  // state SPEC has no field for
                    w.put("RIIX", 4);
                    w.val<uint32_t>((uint32_t)x->ivf_mode);
                    w.val<uint32_t>(x->theta_fit ? 1u : 0u);
                    w.val(x->fit_a);
                    w.val(x->fit_b);
                }
            } else {
                w.put("RIIS", 4);  // a shard of a world > 1 job: this library's own layout
                w.val<uint32_t>(1);
                for (uint32_t v : {(uint32_t)x->D, (uint32_t)x->M, (uint32_t)KS, (uint32_t)x->world, (uint32_t)x->rank,
                                   (uint32_t)x->ivf_mode, (uint32_t)((x->theta_fit ? 1 : 0) | (x->has_rot ? 2 : 0)),
                                   (uint32_t)x->segs.size()})
                    w.val(v);
                for (int64_t v : {x->N, x->n_local, x->K, x->theta}) w.val(v);
                w.val(x->fit_a);
                w.val(x->fit_b);
                if (x->has_rot) w.put(x->rot_host.data(), x->rot_host.size() * 4);
                dev_to_file(w, x->cb.as<float>(), (size_t)x->M * KS * x->ds);
                for (auto &sg : x->segs) { w.val(sg.local_off); w.val(sg.global_first); w.val(sg.count); }
                dev_to_file(w, x->codes.as<uint8_t>(), (size_t)x->n_local * x->M);
                if (x->K > 0) {
                    dev_to_file(w, x->centers.as<uint8_t>(), (size_t)x->K * x->M);
                    dev_to_file(w, x->offsets.as<int64_t>(), (size_t)x->K + 1);
                    dev_to_file(w, x->ids.as<uint32_t>(), (size_t)x->n_local);
                }
            }
        } catch (...) {
            fclose(f);
            throw;
        }
        arg_check(fclose(f) == 0, "close failed");
    });
}

namespace {
// Posting lists read from a file must be a partition of [0, n_local) into lists
// with ascending ids (Eq. 4, R11) before anything indexes device memory with them.
void check_postings(const std::vector<int64_t> &off, const std::vector<uint32_t> &ids, int64_t K, int64_t n_local) {
    arg_check(off.size() == (size_t)K + 1 && off[0] == 0 && off[K] == n_local, "posting offsets do not span the codes");
    std::vector<uint8_t> seen((size_t)n_local, 0);
    for (int64_t k = 0; k < K; ++k) {
        arg_check(off[k + 1] >= off[k], "posting offsets are not monotone");
        for (int64_t p = off[k]; p < off[k + 1]; ++p) {
            arg_check((int64_t)ids[p] < n_local, "posting id out of range");
            arg_check(p == off[k] || ids[p] > ids[p - 1], "posting list not strictly ascending");
            arg_check(!seen[ids[p]], "posting id listed twice");
            seen[ids[p]] = 1;
        }
    }
}

void upload_postings(rii_index *x, const std::vector<int64_t> &off, const std::vector<uint32_t> &ids) {
    const int64_t K = x->K, n = x->n_local;
    RII_CUDA(cudaMemcpy(x->offsets.get<int64_t>((size_t)K + 1), off.data(), off.size() * 8, cudaMemcpyHostToDevice));
    uint32_t *dids = x->ids.get<uint32_t>((size_t)std::max<int64_t>(n, 1));
    if (n) RII_CUDA(cudaMemcpy(dids, ids.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
    // a(n) is implied by W (Eq. 4): rebuilt on the device, not stored
    int32_t *as = x->assign.get<int32_t>((size_t)std::max<int64_t>(n, 1));
    if (K > 0 && n > 0) {
        assign_from_csr_kernel<<<(unsigned)ceil_div(K, 64), 64>>>(x->offsets.as<int64_t>(), K, dids, as);
        RII_LAUNCHED();
    }
    build_mirror(x->codes.as<uint8_t>(), x->M, dids, n, x->mirror.get<uint8_t>((size_t)std::max<int64_t>(n, 1) * x->M + 64),
                 nullptr);
    RII_CUDA(cudaDeviceSynchronize());
}
}  // namespace

rii_status rii_load(const char *path, int32_t device, const void *nccl_id, rii_index **out) {
    if (out) *out = nullptr;
    return guarded([&] {
        arg_check(path && out, "NULL argument");
        FILE *f = fopen(path, "rb");
        arg_check(f != nullptr, "cannot open index file");
        FileR r{f};
        rii_index *x = nullptr;
        try {
            char magic[4];
            r.get(magic, 4, "magic");
            const bool spec = memcmp(magic, "RII1", 4) == 0, shard = memcmp(magic, "RIIS", 4) == 0;
            arg_check(spec || shard, "not an index file (magic is neither RII1 nor RIIS)");
            arg_check(r.val<uint32_t>("version") == 1, "unsupported index file version");
            if (spec) {  // SPEC's RII1 (single-GPU index)
                const uint32_t D = r.val<uint32_t>("header"), M = r.val<uint32_t>("header"), Z = r.val<uint32_t>("header");
                const uint32_t N = r.val<uint32_t>("header"), K = r.val<uint32_t>("header");
                const uint64_t theta = r.val<uint64_t>("header");
                r.val<uint32_t>("header");  // default_L (unused: L is a query argument)
                const uint32_t flags = r.val<uint32_t>("header");
                arg_check(Z == KS && M >= 1 && M <= 256 && D >= M && D % M == 0 && D / M <= 64, "bad shape in header");
                arg_check((flags & ~3u) == 0 && K <= N && K < (1u << 31), "bad header");
                arg_check(theta <= (uint64_t)INT64_MAX, "theta out of range");
                const rii_status st = create_impl((int32_t)D, (int32_t)M, (int32_t)Z, device, 0, 1, nullptr, nullptr, &x);
                if (st != RII_OK) throw Error(st, t_err);
                DeviceGuard g(device);
                file_to_dev(r, x->cb.as<float>(), (size_t)M * KS * (D / M), "code book");
                if (flags & 1u) {  // OPQ rotation
                    std::vector<float> R((size_t)D * D);
                    r.get(R.data(), R.size() * 4, "rotation");
                    const rii_status sr = rii_set_rotation(x, R.data());
                    if (sr != RII_OK) throw Error(sr, t_err);
                }
                x->trained = true;
                x->N = x->n_local = N;
                file_to_dev(r, x->codes.get<uint8_t>((size_t)std::max<uint32_t>(N, 1) * M + 64), (size_t)N * M, "codes");
                if (N) x->segs.push_back({0, 0, (int64_t)N});
                x->K = K;
                if (K > 0) {
                    file_to_dev(r, x->centers.get<uint8_t>((size_t)K * M), (size_t)K * M, "centres");
                    std::vector<int64_t> off((size_t)K + 1, 0);
                    std::vector<uint32_t> ids((size_t)N);
                    for (uint32_t k = 0; k < K; ++k) {
                        const uint32_t len = r.val<uint32_t>("posting length");
                        arg_check((uint64_t)off[k] + len <= N, "posting lists longer than N");
                        off[k + 1] = off[k] + len;
                        r.get(ids.data() + off[k], (size_t)len * 4, "posting ids");
                    }
                    check_postings(off, ids, K, N);
                    upload_postings(x, off, ids);
                }
                x->theta = (flags & 2u) ? -1 : (int64_t)theta;
                char ext[4];
                const size_t got = fread(ext, 1, 4, f);
                if (got == 4) {
                    arg_check(memcmp(ext, "RIIX", 4) == 0, "trailing bytes after the index");
                    const uint32_t mode = r.val<uint32_t>("extension"), fit = r.val<uint32_t>("extension");
                    arg_check(mode <= 1 && fit <= 1, "bad extension block");
                    x->ivf_mode = (int)mode;
                    x->theta_fit = fit != 0;
                    x->fit_a = r.val<double>("extension");
                    x->fit_b = r.val<double>("extension");
                } else {
                    arg_check(got == 0, "trailing bytes after the index");
                }
            } else {  // RIIS: one shard of a world > 1 job
                const uint32_t D = r.val<uint32_t>("header"), M = r.val<uint32_t>("header"), Ks = r.val<uint32_t>("header");
                const uint32_t world = r.val<uint32_t>("header"), rank = r.val<uint32_t>("header");
                const uint32_t mode = r.val<uint32_t>("header"), flags = r.val<uint32_t>("header");
                const uint32_t nseg = r.val<uint32_t>("header");
                const int64_t N = r.val<int64_t>("header"), n_local = r.val<int64_t>("header");
                const int64_t K = r.val<int64_t>("header"), theta = r.val<int64_t>("header");
                const double fa = r.val<double>("header"), fb = r.val<double>("header");
                arg_check(Ks == KS && M >= 1 && M <= 256 && D >= M && D % M == 0 && D / M <= 64, "bad shape in header");
                arg_check(world >= 1 && world <= 4096 && rank < world && (flags & ~3u) == 0 && mode <= 1, "bad header");
                arg_check(N >= 0 && N < (1ll << 32) && n_local >= 0 && n_local <= N && K >= 0 && K <= N &&
                              K < (1ll << 31) && theta >= -1,
                          "bad header");
                arg_check(nseg <= (uint64_t)n_local, "more segments than codes");
                const rii_status st = create_impl((int32_t)D, (int32_t)M, (int32_t)Ks, device, (int32_t)rank,
                                                  (int32_t)world, nccl_id, nullptr, &x);
                if (st != RII_OK) throw Error(st, t_err);
                DeviceGuard g(device);
                if (flags & 2u) {  // OPQ rotation
                    std::vector<float> R((size_t)D * D);
                    r.get(R.data(), R.size() * 4, "rotation");
                    const rii_status sr = rii_set_rotation(x, R.data());
                    if (sr != RII_OK) throw Error(sr, t_err);
                }
                file_to_dev(r, x->cb.as<float>(), (size_t)M * KS * (D / M), "code book");
                x->trained = true;
                int64_t tiled = 0, prev_end = 0;
                for (uint32_t i = 0; i < nseg; ++i) {  // segments tile [0, n_local), ascending global ranges
                    Seg sg;
                    sg.local_off = r.val<int64_t>("segments");
                    sg.global_first = r.val<int64_t>("segments");
                    sg.count = r.val<int64_t>("segments");
                    arg_check(sg.local_off == tiled && sg.count > 0 && sg.global_first >= prev_end &&
                                  sg.global_first + sg.count <= N,
                              "segments do not tile the shard");
                    tiled += sg.count;
                    prev_end = sg.global_first + sg.count;
                    x->segs.push_back(sg);
                }
                arg_check(tiled == n_local, "segments do not tile the shard");
                x->N = N;
                x->n_local = n_local;
                file_to_dev(r, x->codes.get<uint8_t>((size_t)std::max<int64_t>(n_local, 1) * M + 64),
                            (size_t)n_local * M, "codes");
                x->K = K;
                if (K > 0) {
                    file_to_dev(r, x->centers.get<uint8_t>((size_t)K * M), (size_t)K * M, "centres");
                    std::vector<int64_t> off((size_t)K + 1);
                    std::vector<uint32_t> ids((size_t)n_local);
                    r.get(off.data(), off.size() * 8, "posting offsets");
                    r.get(ids.data(), ids.size() * 4, "posting ids");
                    check_postings(off, ids, K, n_local);
                    upload_postings(x, off, ids);
                }
                char extra;
                arg_check(fread(&extra, 1, 1, f) == 0, "trailing bytes after the index");
                x->theta = theta;
                x->ivf_mode = (int)mode;
                x->theta_fit = (flags & 1) != 0;
                x->fit_a = fa;
                x->fit_b = fb;
            }
            upload_segs(x, nullptr);
        } catch (...) {
            fclose(f);
            rii_destroy(x);
            throw;
        }
        fclose(f);
        *out = x;
    });
}

rii_status rii_set_centers(rii_index *x, const uint8_t *centers, int32_t K, void *stream) {
    return guarded([&] {
        arg_check(x && centers, "NULL argument");
        arg_check(K >= 1, "K must be >= 1");
        state_check(x->trained, "index has no code book");
        DeviceGuard g(x->device);
        cudaStream_t st = (cudaStream_t)stream;
        ensure_T(x, st);
        uint8_t *cent = x->centers.get<uint8_t>((size_t)K * x->M);
        RII_CUDA(cudaMemcpyAsync(cent, centers, (size_t)K * x->M, cudaMemcpyHostToDevice, st));
        x->K = K;
        int32_t *as = x->assign.get<int32_t>(x->n_local + 1);
        launch_assign(x->codes.as<uint8_t>(), x->n_local, cent, x->K, x->M, x->T.as<float>(), as, nullptr, st);
        rebuild_csr(x, st);
        x->theta = -1;
        x->theta_fit = false;
        RII_CUDA(cudaStreamSynchronize(st));
    });
}

rii_status rii_set_ivf_mode(rii_index *x, int32_t mode) {
    return guarded([&] {
        arg_check(x != nullptr, "index is NULL");
        arg_check(mode == RII_IVF_LISTS || mode == RII_IVF_PAPER, "mode must be RII_IVF_LISTS or RII_IVF_PAPER");
        x->ivf_mode = mode;
        x->theta_fit = false;
    });
}

rii_status rii_set_theta(rii_index *x, int64_t theta) {
    return guarded([&] {
        arg_check(x != nullptr, "index is NULL");
        x->theta = theta < 0 ? -1 : theta;
        x->theta_fit = false;
    });
}

__global__ void strided_ids_kernel(int64_t *out, int64_t s, int64_t N) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < s) out[i] = (int64_t)(((__int128)i * N) / s);
}

rii_status rii_calibrate_theta(rii_index *x, const float *q, int64_t nq, int32_t topk, const int32_t *L_grid,
                               int32_t n_L, rii_mem where, void *stream, double *a_out, double *b_out,
                               double *crossovers) {
    return guarded([&] {
        arg_check(x && q && L_grid && n_L >= 1 && nq >= 1, "bad arguments");
        state_check(x->trained && x->K > 0, "calibration needs coarse centres (K > 0)");
        arg_check(topk >= 1 && topk <= 1024, "topk must be in [1, 1024]");
        DeviceGuard g(x->device);
        cudaStream_t st = (cudaStream_t)stream;
        const float *dq = q;
        Buf qb, Sb, oi, od, kb;
        if (where == RII_MEM_HOST) {
            float *b = qb.get<float>((size_t)nq * x->D);
            RII_CUDA(cudaMemcpyAsync(b, q, (size_t)nq * x->D * 4, cudaMemcpyHostToDevice, st));
            dq = b;
        }
        std::vector<int64_t> sizes;
        for (int64_t s = 128; s <= x->N; s *= 4) sizes.push_back(s);
        if (sizes.empty() || sizes.back() != x->N) sizes.push_back(x->N);
        int64_t *S = Sb.get<int64_t>(x->N);
        int64_t *ids = oi.get<int64_t>((size_t)nq * topk);
        float *dist = od.get<float>((size_t)nq * topk);
        cudaEvent_t e0, e1;
        RII_CUDA(cudaEventCreate(&e0));
        RII_CUDA(cudaEventCreate(&e1));
        auto time_query = [&](int64_t s, int L, int path) -> int64_t {  // ns, max over ranks
            for (int rep = 0; rep < 2; ++rep) {
                if (rep == 1) RII_CUDA(cudaEventRecord(e0, st));
                const rii_status r = query_impl(x, dq, nq, topk, S, s, L, (rii_path)path, RII_MEM_DEVICE, st, ids,
                                                dist, nullptr, nullptr);
                if (r != RII_OK) throw Error(r, t_err);
                if (rep == 1) RII_CUDA(cudaEventRecord(e1, st));
            }
            RII_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            RII_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            int64_t ns = (int64_t)(ms * 1e6), mx = ns;
            if (x->world > 1 && x->comm) {
                int64_t *d = kb.get<int64_t>(2);
                RII_CUDA(cudaMemcpyAsync(d, &ns, 8, cudaMemcpyHostToDevice, st));
                x->comm->allreduce_max_i64(d, d + 1, 1, st);
                RII_CUDA(cudaMemcpyAsync(&mx, d + 1, 8, cudaMemcpyDeviceToHost, st));
                RII_CUDA(cudaStreamSynchronize(st));
            }
            return mx;
        };
        std::vector<double> Ls, cross;
        for (int li = 0; li < n_L; ++li) {
            const int L = L_grid[li];
            arg_check(L >= 1, "L_grid values must be >= 1");
            double prev_s = 0.0, prev_r = 0.0, c = -1.0;
            for (size_t si = 0; si < sizes.size(); ++si) {
                const int64_t s = sizes[si];
                if (decide_exec(x, RII_PATH_IVF, true, s, L) == RII_PATH_LINEAR) {
                    // P = K: the inverted index executes as the linear scan (same candidates,
                    // same time), so the crossover lies above s
                    prev_s = (double)s;
                    prev_r = 0.0;
                    continue;
                }
                strided_ids_kernel<<<(unsigned)ceil_div(s, 256), 256, 0, st>>>(S, s, x->N);
                RII_LAUNCHED();
                const double tl = (double)time_query(s, L, RII_PATH_LINEAR);
                const double ti = (double)time_query(s, L, RII_PATH_IVF);
                const double r = std::log(tl / std::max(ti, 1.0));  // > 0: the inverted index is faster
                if (r > 0) {
                    if (si == 0) c = 0.0;
                    else {  // log-linear interpolation of the sign change of log(t_lin / t_ivf)
                        const double f = prev_r / (prev_r - r);
                        c = std::exp(std::log(prev_s) + f * (std::log((double)s) - std::log(prev_s)));
                    }
                    break;
                }
                prev_s = (double)s;
                prev_r = r;
            }
            if (c < 0) c = (double)x->N;
            Ls.push_back((double)L);
            cross.push_back(c);
            if (crossovers) crossovers[li] = c;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        double a = 0.0, b = cross[0];
        if (n_L > 1) {  // least squares theta = a L + b
            double mL = 0, mC = 0;
            for (int i = 0; i < n_L; ++i) { mL += Ls[i]; mC += cross[i]; }
            mL /= n_L;
            mC /= n_L;
            double sxy = 0, sxx = 0;
            for (int i = 0; i < n_L; ++i) { sxy += (Ls[i] - mL) * (cross[i] - mC); sxx += (Ls[i] - mL) * (Ls[i] - mL); }
            a = sxx > 0 ? sxy / sxx : 0.0;
            b = mC - a * mL;
        }
        x->fit_a = a;
        x->fit_b = b;
        x->theta_fit = true;
        x->theta = -1;
        if (a_out) *a_out = a;
        if (b_out) *b_out = b;
    });
}

rii_status rii_get_info(const rii_index *x, int64_t *N, int32_t *K, int64_t *theta, int64_t *n_local,
                        int64_t *bytes) {
    return guarded([&] {
        arg_check(x != nullptr, "index is NULL");
        if (N) *N = x->N;
        if (K) *K = (int32_t)x->K;
        if (theta) *theta = x->theta;
        if (n_local) *n_local = x->n_local;
        if (bytes) *bytes = x->n_local * x->M + x->K * x->M + (x->K ? 4 * x->n_local : 0);
    });
}

}  // extern "C"
