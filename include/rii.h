/*
 * rii.h -- C ABI of the B200-native Rii hot path (Reconfigurable Inverted Index,
 * Matsui, Hinami, Satoh, ACM MM 2018, arXiv 1808.03969).
 *
 * Citation keys: "P:n" = PAPER.md line n (section / equation / algorithm named),
 * "S:n" = SPEC.md line n, "R#" = a reading of the paper listed in DESIGN.md.
 *
 * General conventions (every entry point):
 *  - Every call returns rii_status; RII_OK == 0.  On failure nothing the call was
 *    asked to produce is valid, and rii_last_error() returns a message for the
 *    calling thread.  The index stays usable after RII_ERR_ARG / RII_ERR_STATE.
 *  - Ids are 0-based and dense (the paper's 1..N is 0..N-1, R4), int64 at the
 *    boundary.  A vector added as the n-th row overall has id n.
 *  - Distances are squared L2 ADC values in fp32 (Eq. 3; R17), computed
 *    in the canonical order of DESIGN.md (CA1 / CA2), so they equal the oracle's.
 *  - Code books have Ks = 256 code words per subspace ("we set Z to 256");
 *    codes are M bytes per vector.
 *  - `where` says where the caller's arrays of that call live: RII_MEM_HOST
 *    (pageable or pinned host memory; copied in/out inside the call, the call
 *    returns after results are on the host) or RII_MEM_DEVICE (device pointers
 *    on the index's device; results are complete when the call returns).
 *  - `stream` is a cudaStream_t (NULL = the legacy default stream); all device
 *    work of a call is ordered on it.  Caller arrays are borrowed for the call.
 *  - Ownership: the index owns every device buffer it allocates (code book,
 *    codes, centres, posting lists, scratch) and frees them in rii_destroy.
 *  - Concurrency: one writer (train / add / reconfigure / set_*) or many readers
 *    (query / query_partial / get_*) at a time per index.  Readers may run
 *    concurrently from several host threads on several streams: every query
 *    allocates its scratch per call (cudaMallocAsync on its own stream from the
 *    device's memory pool, freed before it returns), so no two calls share a
 *    buffer.  A writer must not overlap any other call on the same index.
 *  - Multi-GPU (world > 1): one process per GPU, every rank calls every function
 *    collectively with identical arguments (full x, q, S).  The database is
 *    sharded by id range; each rank scans its shard and the per-rank top-k lists
 *    are merged after an NCCL all-gather, so every rank receives the full result.
 *  - The library never falls back to the CPU: without a usable CUDA device every
 *    call that needs one returns RII_ERR_CUDA.
 */
#ifndef RII_H_
#define RII_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rii_index rii_index; /* opaque */

typedef enum {
    RII_OK = 0,
    RII_ERR_ARG = 1,   /* invalid argument (shape, range, unsorted target ids, ...) */
    RII_ERR_STATE = 2, /* call not valid in the current state (e.g. untrained)    */
    RII_ERR_OOM = 3,   /* device or host allocation failed                         */
    RII_ERR_CUDA = 4,  /* CUDA runtime error, or no usable device                  */
    RII_ERR_NCCL = 5,  /* NCCL error (world > 1)                                   */
    RII_ERR_TRAIN = 6  /* code-book training impossible (n < Ks, < Ks distinct rows) */
} rii_status;

typedef enum { RII_PATH_AUTO = 0, RII_PATH_LINEAR = 1, RII_PATH_IVF = 2 } rii_path;
typedef enum { RII_MEM_HOST = 0, RII_MEM_DEVICE = 1 } rii_mem;

/* Size of the opaque NCCL unique id accepted by rii_create. */
#define RII_NCCL_ID_BYTES 128

/* Message of the last failed call on the calling thread ("" if none); never NULL.
 * The message is thread-local, so idx only documents which index the caller means
 * (SURVEY 8(b) signature); it may be NULL (e.g. after a failed rii_create). */
const char *rii_last_error(const rii_index *idx);

/* Number of CUDA kernels this library has launched in this process (all
 * indexes).  Used by bench.py to report "gpu_launches". */
uint64_t rii_launch_count(void);

/* Optional CUDA-event timing of the dominant kernels, recorded on the stream each
 * kernel is launched on (used by bench.py for the roofline's "achieved").
 * rii_kernel_timing(1) clears the totals and starts recording; (0) stops.
 * which: 0 = linear ADC scan kernel, 1 = inverted-index list-scan kernel,
 * 2 = top-k merge kernel, 3 = the linear-scan launches that used the
 * bf16-packed tables (a subset of 0), 4 = the u16-table bound pass (strided code
 * sample: gather + exact scan + merge + kk-th distance; one record per call),
 * 5 = the linear-scan launches that used the u16 fixed-point tables, 6 = those that
 * used the u6 fixed-point tables (each a subset of 0).  total_ms / launches cover
 * every launch since the last clear (read synchronises with the recorded events).
 * which outside [0, 7) -> RII_ERR_ARG. */
void rii_kernel_timing(int32_t enable);
rii_status rii_kernel_timing_read(int32_t which, double *total_ms, int64_t *launches);

/* Diagnostic event counters of the scan kernels (device atomics at barrier-window
 * ends, process-wide, for tests; counting costs nothing when off).
 * rii_debug_counters(1) allocates and clears them (on the current device) and
 * starts counting; (0) stops and frees.  rii_debug_counters_read copies n values
 * (synchronises the device): [0] window ends, [1] compactions (a CTA's own kk-th
 * distance tightened), [2] overflowing windows rolled back, [3] window-end reads
 * of the shared per-query bound that lowered it (another CTA's published kk-th,
 * i.e. mid-chunk tightening), [4] integer-table re-quantisations at a tighter
 * bound, [5] bound publications (atomicMin) that lowered the shared bound, [6]
 * candidates pushed past the filter (counted at compactions), [7..9] SM cycles of
 * thread 0 per CTA in table fill / scan loop / final compaction + output (summed),
 * [10] CTAs counted. */
rii_status rii_debug_counters(int32_t enable);
rii_status rii_debug_counters_read(int64_t *out, int32_t n);

/* The rows [*lo, *hi) of an n-row rii_add batch that rank `rank` of `world` stores
 * (contiguous chunks of ceil(n / world) rows; host-only, no device needed). */
rii_status rii_shard_range(int64_t n, int32_t rank, int32_t world, int64_t *lo, int64_t *hi);

/* Rank 0 calls this to obtain the NCCL unique id that every rank then passes to
 * rii_create (distributed by the caller, e.g. through torch.distributed).
 * out: RII_NCCL_ID_BYTES host bytes.  RII_ERR_NCCL if NCCL cannot be loaded. */
rii_status rii_nccl_unique_id(void *out);

/* Create an empty index (Sec. 4.1) of D-dim vectors with M subspaces.
 *  D % M == 0, 1 <= M <= 256, Ks == 256, D/M <= 64 (else RII_ERR_ARG).  M > 64
 *  (GIST-like shapes) runs the one-query-per-CTA large-M kernels.
 *  device: CUDA ordinal this index lives on.  rank/world: this process's place
 *  in a one-process-per-GPU job (world == 1: single GPU).  nccl_id: the 128-byte
 *  id from rii_nccl_unique_id (all ranks identical) or NULL; with world > 1 and
 *  nccl_id == NULL the index is a *detached shard*: rii_query returns
 *  RII_ERR_STATE and the caller combines shards with rii_query_partial +
 *  rii_merge_partials (used for single-GPU logical-shard tests).
 *  *out receives the index (NULL on failure). */
rii_status rii_create(int32_t D, int32_t M, int32_t Ks, int32_t device, int32_t rank, int32_t world,
                      const void *nccl_id, rii_index **out);

/* Host transport for a multi-process job without NCCL (e.g. torch.distributed
 * with the gloo backend): allgather(ctx, send, recv, bytes) must place every
 * rank's `bytes` host bytes (at its `send`) at recv + rank * bytes, recv holding
 * world * bytes, and return 0 (non-zero -> RII_ERR_NCCL).  It is called from
 * inside the library's calls, collectively (every rank, same bytes, same order),
 * after the library synchronised its stream, so no kernel ever waits on another
 * rank.  ctx is passed through; the struct is copied, ctx and the function must
 * outlive the index. */
typedef struct rii_transport {
    void *ctx;
    int32_t (*allgather)(void *ctx, const void *send, void *recv, uint64_t bytes);
} rii_transport;

/* rii_create for a world > 1 job whose exchange step (top-k merge, shared scan
 * bound, reconfigure sample) runs over `transport` instead of NCCL.  Same shard
 * layout, calls and results as with NCCL.  transport == NULL or world == 1 ->
 * RII_ERR_ARG. */
rii_status rii_create_with_transport(int32_t D, int32_t M, int32_t Ks, int32_t device, int32_t rank, int32_t world,
                                     const rii_transport *transport, rii_index **out);

/* Frees every device buffer and the NCCL communicator.  NULL is a no-op. */
void rii_destroy(rii_index *idx);

/* Code-book training (R8; the paper: "preliminarily trained"): per
 * subspace, n_iter Lloyd iterations, seeded distinct-row init, fixed-point
 * mean update (DESIGN.md O-TRAIN).  x: n x D fp32 row-major.  Requires n >= 256
 * and >= 256 distinct sub-vectors per subspace (else RII_ERR_TRAIN) and
 * n * max|x| < 2^31 (else RII_ERR_ARG).  Replaces any code book; only allowed
 * while the index is empty (N == 0), else RII_ERR_STATE.  Every rank trains
 * identically (no communication). */
rii_status rii_train(rii_index *idx, const float *x, int64_t n, int32_t n_iter, uint64_t seed, rii_mem where,
                     void *stream);

/* OPQ variant (Rii-OPQ, Sec. "Advanced Encoding"; Table 2 P:1002,
 * P:1008): "In the search phase, an input vector is first rotated with the
 * matrix.  The remaining process is exactly the same as PQ".
 * rii_set_rotation: R = D x D fp32 row-major host array (copied; NULL removes the
 * rotation).  From then on every vector given to rii_train, rii_add, rii_query,
 * rii_query_partial and rii_calibrate_theta is replaced by y = R x computed in the
 * canonical order y_i = ((0 + R_i0 x_0) + R_i1 x_1) + ... (fp32, no FMA; DESIGN.md
 * CR).  R is not checked for orthogonality.  Only while the index is empty
 * (N == 0, else RII_ERR_STATE); clears the code book (train or set it again).
 * rii_get_rotation: copies R into R (D x D; identity when none) and sets
 * *has_rotation (either pointer may be NULL).
 * rii_rotate: out = R in for n device rows (a copy when no rotation); synchronises.
 * rii_train_opq: non-parametric OPQ (the rotation is "preliminarily trained to
 * minimize the error"): R_0 = I; n_opq_iter times: train a code book on
 * R x (max(1, n_iter / 2) Lloyd iterations, seed + it), reconstruct y = decode(
 * encode(R x)), R <- U V^T for the SVD C = sum y x^T = U S V^T (orthogonal
 * Procrustes; the D x D SVD runs on the host, C on the device); then sets R and
 * trains the final code book on R x with n_iter iterations and `seed` (rii_train).
 * Same requirements and errors as rii_train. */
rii_status rii_set_rotation(rii_index *idx, const float *R);
rii_status rii_get_rotation(const rii_index *idx, float *R, int32_t *has_rotation);
rii_status rii_rotate(const rii_index *idx, const float *in, int64_t n, float *out, void *stream);
rii_status rii_train_opq(rii_index *idx, const float *x, int64_t n, int32_t n_opq_iter, int32_t n_iter, uint64_t seed,
                         rii_mem where, void *stream);

/* Data addition (Sec. 4.3 "Data addition"): encodes x (n x D fp32,
 * Eq. 1) and appends the codes to the linear array (PushBack(Xbar, y));
 * if the index has coarse centres (K > 0) each new id is appended to the posting
 * list of its SDC-nearest centre (PushBack(W_a(n), n); lists stay ascending).
 * Ids first_id .. first_id+n-1 (first_id may be NULL).  Requires a code book
 * (RII_ERR_STATE).  With world > 1 the batch is split into `world` contiguous
 * chunks and rank r stores chunk r. */
rii_status rii_add(rii_index *idx, const float *x, int64_t n, rii_mem where, void *stream, int64_t *first_id);

/* Reconfigure (Alg. 4): PQk-means (reading R9) over the sample of
 * min(N, 100*nlist) ids with the smallest splitmix64(seed ^ id) keys (R10), init
 * = the first nlist distinct sample codes, n_iter iterations; then every code is
 * assigned to its SDC-nearest centre (ties to the lowest k) and the posting lists
 * are rebuilt with ascending ids.  1 <= nlist <= N (RII_ERR_ARG), fewer than nlist
 * distinct sample codes -> RII_ERR_ARG.  Deterministic for (nlist, n_iter, seed)
 * (P:682).  Resets theta to the default (R3). */
rii_status rii_reconfigure(rii_index *idx, int32_t nlist, int32_t n_iter, uint64_t seed, void *stream);

/* Query (Alg. 3), nq queries q (nq x D fp32) sharing one target set:
 *  target_ids: strictly ascending ids in [0, N) (the paper's sorted S, P:366-374;
 *     R6), n_target of them; NULL = the whole database (S = {0..N-1}).
 *     Violations -> RII_ERR_ARG (checked on the device before any result).
 *  topk: R, 1 <= topk <= 1024.
 *  L: the number of nearest coarse lists to probe (reading R1); the inverted
 *     index traverses P = min(L, K) lists for S = ALL and
 *     P = min(K, ceil(L * N / |S|)) lists otherwise, evaluating every
 *     member of S in them (R2 mode A).  L >= 1.
 *  path: RII_PATH_AUTO applies Alg. 3 with the index's theta (|S| < theta ->
 *     PQ linear scan (Alg. 1), else inverted index (Alg. 2)); LINEAR / IVF force
 *     a path.  K == 0 forces LINEAR; IVF with K == 0 -> RII_ERR_STATE.
 *  out_ids / out_dist: nq x topk, each row sorted by (dist asc, id asc); rows
 *     with fewer than topk candidates are padded with id -1 and dist +inf (R18).
 *  path_used (may be NULL): the path taken (Alg. 3's choice).  An inverted-index
 *     query in mode A may execute as a linear scan of S -- every list probed
 *     (P = K), or a scan masked to each query's probed lists when P is a large
 *     fraction of K -- whose candidate set, and so result, is Alg. 2's exactly. */
rii_status rii_query(const rii_index *idx, const float *q, int64_t nq, int32_t topk, const int64_t *target_ids,
                     int64_t n_target, int32_t L, rii_path path, rii_mem where, void *stream, int64_t *out_ids,
                     float *out_dist, int32_t *path_used);

/* Split-phase query for detached shards (world > 1 with nccl_id == NULL) and for
 * custom transports: the same arguments as rii_query, but instead of the final
 * result it writes this rank's top candidates as packed uint64 keys
 * ((fp32 dist bits) << 32 | global id), nq x kk, each row ascending, unused
 * slots = UINT64_MAX.  kk = rii_partial_width(topk).  Arrays in device memory.
 * The path is decided from the global |S| exactly as in rii_query. */
int32_t rii_partial_width(int32_t topk);
rii_status rii_query_partial(const rii_index *idx, const float *q, int64_t nq, int32_t topk,
                             const int64_t *target_ids, int64_t n_target, int32_t L, rii_path path, void *stream,
                             uint64_t *out_keys, int32_t *path_used);

/* Merge `parts` partial key arrays laid out [parts][nq][kk] (device memory) into
 * the final nq x topk result (device memory).  The global top-k is contained in
 * the union of the per-shard top-k, so the result equals the single-index one. */
rii_status rii_merge_partials(const uint64_t *keys, int32_t parts, int64_t nq, int32_t topk, void *stream,
                              int64_t *out_ids, float *out_dist);

/* State hand-off (host memory): code book M x 256 x (D/M) fp32; codes of global
 * ids [first, first+n) (must be stored on this rank, else RII_ERR_ARG); centres
 * K x M; posting lists of this rank as CSR offsets[K+1] + global ids[N_local]
 * ascending within each list; assignment a(id) for this rank's ids [N_local]. */
rii_status rii_get_codebook(const rii_index *idx, float *out);
rii_status rii_set_codebook(rii_index *idx, const float *cb); /* only while N == 0 */
rii_status rii_get_codes(const rii_index *idx, int64_t first, int64_t n, uint8_t *out);
rii_status rii_get_centers(const rii_index *idx, uint8_t *out);
rii_status rii_get_postings(const rii_index *idx, int64_t *offsets, int64_t *ids);

/* Install K coarse centres (K x M PQ codes, host memory) instead of running
 * rii_reconfigure -- e.g. to restore a saved index: every stored code is assigned
 * to its SDC-nearest centre (ties to the lowest k) and the posting
 * lists are rebuilt (Alg. 4 L2-L4).  1 <= K < 2^31; resets theta to the default. */
rii_status rii_set_centers(rii_index *idx, const uint8_t *centers, int32_t K, void *stream);

/* Threshold calibration (Alg. 3 / P:589-598: "we simply run the search with several
 * parameter combinations when the data structure is constructed ... fit a 1D line
 * in the parameter space"; the supplement with the details is missing, reading R3).
 * For every L in L_grid (n_L >= 1 values) and target-set sizes |S| = 2^7, 2^9, ...
 * <= N (evenly spaced sorted ids), times rii_query on the GPU with path LINEAR and
 * path IVF (CUDA events, one warm-up each; max over ranks), locates the crossover
 * |S|*(L) by log-linear interpolation (N if the linear scan always wins, 0 if the
 * inverted index always wins) and fits theta(L) = a*L + b by least squares.
 * AUTO then uses max(0, a*L + b) at each call's L until rii_set_theta or
 * rii_reconfigure.  q: nq x D queries (`where`).  Needs K > 0 (RII_ERR_STATE).
 * a_out / b_out / crossovers (n_L values) may be NULL.  The value is
 * machine-dependent by construction (parity unpinned). */
rii_status rii_calibrate_theta(rii_index *idx, const float *q, int64_t nq, int32_t topk, const int32_t *L_grid,
                               int32_t n_L, rii_mem where, void *stream, double *a_out, double *b_out,
                               double *crossovers);

/* Persistence (the paper pickles the index; SPEC's persistence
 * module).  All little-endian.
 *  Single-GPU index (world == 1): SPEC's "RII1" layout bit for bit -- magic
 *    "RII1", u32 version (1), u32 D, M, Z (256), N, K, u64 theta, u32 default_L
 *    (always 1 here), u32 flags (bit 0: OPQ rotation present, bit 1: theta is the
 *    analytic default of reading R3, stored value 0); the code book (M*Z*(D/M)
 *    f32); the rotation (D*D f32) if bit 0; the codes (N*M u8); the centres (K*M
 *    u8); the postings (for k < K: u32 length, then that many u32 ids, ascending).
 *    Payload (N+K)M + 4N(+4K) bytes.  State SPEC has no field for follows
 *    in an optional trailing block: "RIIX", u32 ivf_mode, u32 fitted-theta flag,
 *    f64 fit_a, f64 fit_b (written only when ivf_mode != 0 or theta was fitted).
 *  Shard of a world > 1 job: magic "RIIS" (not SPEC's layout), u32 version (1),
 *    u32 D, M, Ks, world, rank, ivf_mode, flags (bit 0: fitted theta, bit 1: OPQ),
 *    n_segments; i64 N, n_local, K, theta; f64 fit_a, fit_b; rotation (if bit 1);
 *    code book; n_segments x (i64 local offset, i64 global first id, i64 count);
 *    codes (n_local*M u8); centres; CSR offsets (K+1) i64; ids n_local u32 (local
 *    positions).  Each rank saves its own shard; rii_load restores it on the same
 *    rank/world (nccl_id as in rii_create).
 * rii_load validates everything before upload (header ranges, segments tiling
 * [0, n_local), posting lists a partition with ascending in-range ids, no trailing
 * bytes beyond the optional block): format errors -> RII_ERR_ARG. */
rii_status rii_save(const rii_index *idx, const char *path);
rii_status rii_load(const char *path, int32_t device, const void *nccl_id, rii_index **out);

/* Meaning of L in the inverted index (reading R2).
 *  RII_IVF_LISTS (default, mode A): L = the number of nearest coarse lists; every
 *    member of S in them is evaluated (BASELINE.json's "posting lists of the L
 *    nearest coarse centres").
 *  RII_IVF_PAPER (mode B, Alg. 2 exactly as printed): L = the number of
 *    candidates; the ceil(K*L/|S|) (<= K) nearest lists by (d0, k) are traversed
 *    in that order, ids ascending in each list, non-members of S skipped, and the
 *    traversal stops once L candidates were evaluated.  AUTO's default threshold
 *    becomes theta(L) = L + K.  Single-GPU only (world > 1 -> RII_ERR_STATE at query). */
typedef enum { RII_IVF_LISTS = 0, RII_IVF_PAPER = 1 } rii_ivf_mode;
rii_status rii_set_ivf_mode(rii_index *idx, int32_t mode);

/* theta of Alg. 3 (reading R3).  theta < 0 restores the default
 * theta(L) = ceil(L*N/K) + K evaluated at each call's L. */
rii_status rii_set_theta(rii_index *idx, int64_t theta);

/* N = total ids (all ranks), K = coarse centres, theta = the set value or -1,
 * n_local = ids stored on this rank, bytes = device bytes of codes + centres +
 * posting ids on this rank ((N+K) M + 4N for world == 1).  Any may be NULL. */
rii_status rii_get_info(const rii_index *idx, int64_t *N, int32_t *K, int64_t *theta, int64_t *n_local,
                        int64_t *bytes);

#ifdef __cplusplus
}
#endif
#endif /* RII_H_ */
