// kernels.cuh -- host-side launchers of the sm_100a kernels (internal interface).
#pragma once
#include "common.cuh"

namespace rii {

// ---- search (k_scan.cu) ------------------------------------------------------
// Linear ADC scan (Alg. 1) of n_codes codes (M bytes each) for nq queries.
// Writes out[nq_pad][nc][kk] sorted keys with canonical (CA2) distances and
// key ids = position in `codes`.  Returns nc (number of code chunks).
struct ScanPlan {
    int B;        // queries per CTA
    int nb;       // query batches
    int nc;       // code chunks
    int64_t chunk;
    bool fast;    // lane-rotated conflict-free LUT layout
    size_t smem;
};
// int_ok: the caller will run the integer-table path (sampled bound in gthr) when the
// plan picks B = 8 for M = 64 (its only B = 8 kernel).
ScanPlan plan_linear(int M, int kk, int64_t nq, int64_t n_codes, int num_sms, bool tables_available = false,
                     int max_nc = 1 << 30, bool int_ok = true);

// Probe-masked linear scan (IVF mode A with many probed lists, DESIGN.md §6 "Masked
// IVF"): a code at scan position p belongs to posting list alist[p]; query q of the
// plan's batch b = q / B (B = the scan plan's queries per CTA) evaluates it only if
// bit q % B of pm[b * K + alist[p]] is set, i.e. list alist[p] is among its P probed
// lists.  The candidate set is then exactly Alg. 2's (probed lists) ∩ S.
struct ProbeMask {
    const int32_t *alist = nullptr;  // [n_codes] list of each scanned code; nullptr = no mask
    const uint32_t *pm = nullptr;    // [ceil(nq / B)][K]
    int64_t K = 0;
    int B = 0;                       // query grouping of pm (the scan plan's B)
};

// Arguments of the lane-rotated scan kernel (linear mode, or list-major inverted
// index mode where a work item is (posting list, up to B queries probing it)).
struct ScanArgs {
    const float *tables;  // [nq][256][32] per-query tables (lut.cuh); when set, copied instead of built
    const uint8_t *codes;
    int64_t n_codes;
    const float *q;
    int64_t nq;
    const float *cb;
    int ds, kk;
    int nb;            // linear: query batches
    int64_t chunk;     // linear: codes per chunk
    int nc;            // linear: chunks
    uint64_t *out;     // linear: [nq][nc][kk]; lists: [nq][P][kk]
    const int4 *items; // lists: {list, first entry in qlist, #queries, 0}
    const uint32_t *qlist;  // lists: q * P + probe rank, grouped by list
    int64_t P;
    const int64_t *offsets;  // lists: CSR of the posting lists; `codes` is then the list-ordered
                             // mirror (code of CSR position p at p * M)
    const uint32_t *ids;     // lists: CSR ids (key ids of pushed candidates)
    const uint8_t *rcodes;   // lists: the codes indexed by id (rescores)
    float *gthr;             // per-query upper bound on the global kk-th distance (optional in linear mode)
    // SDC mode (assignment): the "queries" are PQ codes qcodes[nq][M] whose
    // tables are rows of the SDC tables T (T_m[x^m][.]); the scanned codes are centres.
    const float *sdcT;
    const uint8_t *qcodes;
    // u16 list mode: precomputed per-query u16 tables [nq][256][32] and their scales
    const uint16_t *qtab16;
    const uint8_t *qtab8;  // u6 list mode: precomputed per-query u6 tables [nq][256][32]
    const float *qscale;
    uint32_t one;  // = 1 (runtime: keeps the u6 SWAR adds on the FMA pipe, lut.cuh fma_add)
    unsigned long long *dbg;  // debug event counters (rii_debug_counters), nullptr when off
    // linear mode, probe-masked IVF (ProbeMask; alist == nullptr: no mask)
    const int32_t *alist;
    const uint32_t *pmask;
    int64_t pm_K;
};

// List-major inverted-index scan: B queries per CTA share one posting list's codes.
bool list_major_supported(int M);
int list_major_B(int kk, double avg_len, int M);
// q16: u16 fixed-point tables (B == 8, kk <= 256), scaled per item by the queries'
// gthr bounds (items whose queries have no bound yet should run without q16).
void launch_list_scan(int M, int B, const ScanArgs &a, int64_t n_items, cudaStream_t st, bool q16 = false);
// Work items of the list-major scan: for every list k, ceil(#queries probing k / B)
// items {k, first entry of qlist, count, 0}.  qoff = CSR of qlist by list.
// Returns the number of items (synchronises the stream).
// Items are ordered by the smallest probe rank of their queries, so every query's
// nearest lists run first and tighten its global threshold early.
int64_t build_list_items(const int64_t *qoff, int64_t K, int B, const uint32_t *qlist, int64_t P, int4 *items,
                         int64_t cap, cudaStream_t st);
void launch_fill_f32(float *p, int64_t n, float v, cudaStream_t st);
// gthr (fast kernels): per-query upper bound on the global kk-th distance, read by
// every CTA as a filter and lowered (atomicMin) with each CTA's final kk-th distance,
// so chunks scanned later start from the bound of the earlier ones.  q16 (B == 8
// plans only, gthr required): u16 fixed-point tables scaled by the bound at CTA start.
void launch_linear_scan(const ScanPlan &pl, const uint8_t *codes, int64_t n_codes, int M, const float *q, int64_t nq,
                        const float *cb, int D, int kk, uint64_t *out, cudaStream_t st,
                        const float *tables = nullptr, float *gthr = nullptr, bool q16 = false,
                        int timer = TK_LINEAR, const ProbeMask &mask = ProbeMask());
// pm[(q / B) * K + probes[q * P + r]] |= 1 << (q % B) for every (q, r < P); pm zeroed first.
void launch_probe_mask(const int32_t *probes, int64_t nq, int64_t P, int64_t K, int B, uint32_t *pm,
                       cudaStream_t st);
// out[i] = src[i * stride] (int32; the list ids of a strided code sample)
void launch_strided_gather_i32(const int32_t *src, int64_t stride, int64_t n, int32_t *out, cudaStream_t st);
// u16 tables (RII_Q16 != 0), the strided code sample and the kk-th-distance bound.
bool q16_enabled();
int64_t q16_min_codes();  // RII_Q16_MIN (default 2^19): shortest scan that uses integer tables
bool q16_supported(int kk);  // shared-memory budget of the u16 kernels (kk <= 256)
// out[q] = u16 entries of tables[q] with scale[q] = CAP / gthr[q] (u16 list scan).
void launch_q16_tables(const float *tables, const float *gthr, int64_t nq, int M, uint16_t *out, float *scale,
                       cudaStream_t st);
// u6 list items (M = 32, RII_LIST_U6): config (0 = u16 items) and the per-query u6 tables.
int list_u6_cfg(int M);
// queries per integer list-major item: 16 (RII_LIST_U6=4, two u6 oct tables) or 8
int list_int_B(int M, int kk);
// IVF bound items (list_bound_kernel): queries per item, and the launcher that
// publishes every item's kk-th smallest group minimum into gthr (atomicMin).
int list_bound_B(int M);
void launch_list_bound(const uint8_t *codes, int M, const int4 *items, int64_t n_items, const int64_t *offsets,
                       const uint32_t *ids, const uint32_t *qlist, int64_t P, const float *tables, int kk,
                       float *gthr, cudaStream_t st);
bool q16_is_u6(int M);  // the linear integer-table kernel of this M uses u6 tables
void launch_u6_tables(const float *tables, const float *gthr, int64_t nq, int M, uint8_t *out, float *scale,
                      cudaStream_t st, bool u7 = false);
bool list_u7(int M);  // list items on 7-bit entries (RII_LIST_U7)
void launch_strided_gather(const uint8_t *codes, int M, int64_t stride, int64_t n, uint8_t *out, cudaStream_t st);
void launch_kth_bound(const uint64_t *keys, int64_t nq, int kk, float *bound, cudaStream_t st);
// gthr[q] = an upper bound on the kk-th distance over the ns sample codes (the kk-th
// smallest of 1024 group minima, inflated by 1e-5); ns / 1024 codes per group.
// With a mask (alist = the sample's list ids), only the codes of each query's probed
// lists enter its group minima (a group without one has minimum +inf).
void launch_group_min_bound(const uint8_t *samp, int64_t ns, int M, const float *tables, int64_t nq, int kk,
                            float *gthr, cudaStream_t st, const ProbeMask &mask = ProbeMask());

// Per-query rotated tables [nq][256][32] (M in {4,8,16,32}), CA1 values.
void launch_lut_tables(const float *q, int64_t nq, const float *cb, int D, int M, float *tables, cudaStream_t st);

// out[i] = codes[pos[i]] for i < n (subset gather, Alg. 1 "pick up target PQ-codes").
void launch_gather_codes(const uint8_t *codes, int M, const int64_t *pos, int64_t n, uint8_t *out, cudaStream_t st);

// Checks that ids are strictly ascending and inside [0, N); sets *flag != 0 otherwise.
void launch_validate_targets(const int64_t *ids, int64_t n, int64_t N, int *flag, cudaStream_t st);

// Merge `parts` ascending kk-key lists per query into the final result.
// keys addressed as base[q * q_stride + p * p_stride + i].  Either writes
// (out_ids, out_dist) [nq][topk] or, if out_keys != nullptr, [nq][kk] keys with
// ids mapped to global ids.
// Optional canonical rescore inside the merge: key ids are positions in `codes`,
// tables are the per-query HBM tables (lut.cuh layout).
struct Rescore {
    const uint8_t *codes = nullptr;
    const float *tables = nullptr;
    int M = 0;
};
void launch_merge(const uint64_t *keys, int64_t q_stride, int64_t p_stride, int parts, int64_t nq, int kk, int topk,
                  const IdMap &map, int64_t *out_ids, float *out_dist, uint64_t *out_keys, cudaStream_t st,
                  const Rescore &rs = Rescore());

// a[i] = argmin_k d_S(codes[i], centers[k]) with the packed scan kernel in SDC mode
// (exact: top-1 of an exactly rescored top-32).  For large K (the per-centre tables
// of launch_assign would not stay in L2).
bool assign_scan_supported(int M, int64_t K);
void launch_assign_scan(const uint8_t *codes, int64_t n, const uint8_t *centers, int64_t K, int M, const float *T,
                        int32_t *assign, float *dist, int num_sms, cudaStream_t st);

// ---- inverted index (k_ivf.cu) -----------------------------------------------
// d0[q][k] = CA2 ADC of query q to centre code k (Alg. 2 L2-L5).
void launch_coarse_dist(const uint8_t *centers, int64_t K, int M, const float *q, int64_t nq, const float *cb, int D,
                        float *d0, cudaStream_t st);
// probes[q][0..P) = the P centres with the smallest (d0, k) (Alg. 2 L6), ascending k.
void launch_select_probes(const float *d0, int64_t nq, int64_t K, int64_t P, int32_t *probes, cudaStream_t st);
// probes[q][r] = id of the r-th key of the sorted per-query keys [nq][kk] (r < P).
void launch_keys_to_probes(const uint64_t *keys, int64_t nq, int kk, int64_t P, int32_t *probes, cudaStream_t st);
// probes[q][0..P) = the P nearest lists in (d0, k) order (CUB segmented sort of d0).
// Coarse ranking + top-P probes sorted by (d0, k) in one kernel (fast M, precomputed
// tables); returns false (nothing launched) when P or K exceed its shared-memory plan.
bool launch_coarse_topp(const uint8_t *centers, int64_t K, int M, const float *tables, int64_t nq, int64_t P,
                        int32_t *probes, cudaStream_t st);
void launch_sorted_probes(const float *d0, int64_t nq, int64_t K, int64_t P, int32_t *probes, cudaStream_t st);
// Alg. 2 early stop (mode B): take[q][r] = members of list probes[q][r] evaluated
// before the budget L runs out (ranks in order).
void launch_paper_takes(const int32_t *probes, int64_t nq, int64_t P, const int64_t *offsets, int64_t L,
                        int32_t *take, cudaStream_t st);
// Posting-list traversal (Alg. 2 L7-L16, mode A): out[q * ostride + i] (i < kk) keys,
// ids = local positions (ostride 0 = kk); nseg = warps sharing one (query, list) pair.
size_t ivf_smem(int M, int kk);
void launch_ivf_scan(const uint8_t *codes, int M, const float *q, int64_t nq, const float *cb, int D, int kk,
                     const int32_t *probes, int64_t P, const int64_t *offsets, const uint32_t *ids, uint64_t *out,
                     cudaStream_t st, const float *tables = nullptr, const int32_t *take = nullptr,
                     int64_t ostride = 0, int nseg = 1);
// gthr[q] = the kk-th key distance of keys[q * stride .. + kk) inflated by 1e-5 (rounded
// up), +inf when the list holds fewer than kk keys: a bound on the query's final kk-th.
void launch_rank_bound(const uint64_t *keys, int64_t nq, int64_t stride, int kk, float *gthr, cudaStream_t st);

// ---- large M (k_large.cu; M > 64, up to 256) ---------------------------------
// One query per CTA, bf16 table resident in smem, exact (CA2) rescore of pushes.
bool large_supported(int M, int kk);
// tables[nq][M][256] = CA1 entries (canonical layout).
void launch_lut_large(const float *q, int64_t nq, const float *cb, int D, int M, float *tables, cudaStream_t st);
int large_linear_chunks(int64_t nq, int64_t n_codes, int num_sms);
// out[nq][nc][kk] keys (ids = positions in codes) of Alg. 1 over n_codes codes.
void launch_large_linear(const uint8_t *codes, int64_t n_codes, int M, const float *tables, int64_t nq, int kk, int nc,
                         uint64_t *out, cudaStream_t st, int timer = TK_LINEAR);
// out[nq][kk] keys of Alg. 2 over each query's P probed lists (take: optional budget cut).
void launch_large_ivf(const uint8_t *codes, int M, const float *tables, int64_t nq, int kk, const int32_t *probes,
                      int64_t P, const int64_t *offsets, const uint32_t *ids, const int32_t *take, uint64_t *out,
                      cudaStream_t st);
// Large-M linear scan on chunked u6 oct tables (k_large_u6.cu): M > 64, M % 16 == 0.
bool large_u6_supported(int M, int kk);
int large_u6_nch(int M);  // 32-subspace chunks per code
// out[q][c][256][32] u6 entries at scale[q] = 63 (M / 4) / gthr[q] (tables: [nq][M][256] fp32)
void launch_u6_tables_large(const float *tables, const float *gthr, int64_t nq, int M, uint8_t *out, float *scale,
                            cudaStream_t st);
int large_u6_chunks(int64_t nq, int64_t n_codes, int M, int num_sms);
// out[ceil(nq/8)*8][nc][kk] exact (CA2) keys; gthr filters and is lowered (atomicMin) per CTA.
// Scans codes [base, base + n_codes) (keys = absolute positions) into slots [ci_off, ci_off + nc) of
// out[ceil(nq/8)*8][nc_out][kk].
void launch_large_u6_linear(const uint8_t *codes, int64_t base, int64_t n_codes, int M, const uint8_t *qtab8,
                            const float *qscale, const float *tables, float *gthr, int64_t nq, int kk, int nc,
                            uint64_t *out, int nc_out, int ci_off, cudaStream_t st);
bool smem_fixed_base_ok();  // dynamic shared memory starts at shared address 0x400 (probed once)
// a[i] = argmin_k d_S(codes[i], centers[k]) (CA2 SDC, ties lowest k); dist optional.
void launch_large_assign(const uint8_t *codes, int64_t n, const uint8_t *centers, int64_t K, int M, const float *T,
                         int32_t *assign, float *dist, cudaStream_t st);

// ---- OPQ (k_opq.cu) ----------------------------------------------------------
// y[n] = R x[n] with Rt = R^T (D x D), canonical order (CR: j ascending, no FMA).
void launch_rotate(const float *Rt, const float *x, int64_t n, int D, float *y, cudaStream_t st);
// y[n] = decode(codes[n]) (PQ reconstruction).
void launch_decode(const uint8_t *codes, int64_t n, int M, int D, const float *cb, float *y, cudaStream_t st);
// C (D x D, fp64) = sum_n y_n x_n^T.
void launch_cross(const float *y, const float *x, int64_t n, int D, double *C, cudaStream_t st);

// ---- build side (k_build.cu) -------------------------------------------------
void launch_encode(const float *x, int64_t n, int D, int M, const float *cb, uint8_t *codes, cudaStream_t st);
void launch_sdc_tables(const float *cb, int D, int M, float *T, cudaStream_t st);
// a[i] = argmin_k d_S(codes[i], centers[k]) (CA2, ties lowest k); dist optional.
void launch_assign(const uint8_t *codes, int64_t n, const uint8_t *centers, int64_t K, int M, const float *T,
                   int32_t *assign, float *dist, cudaStream_t st);
// k-means code-book training (O-TRAIN), all subspaces; returns status via *err (device int).
struct TrainScratch;
void run_train(const float *x, int64_t n, int D, int M, int n_iter, uint64_t seed, float *cb, int *err,
               cudaStream_t st);
// CSR of `vals` (local positions) grouped by `keys` (list ids in [0,K)), stable.
// sort.cu: stable LSD radix sort of (key, u32 value) pairs by the low `bits` key bits
// (K = uint32_t or uint64_t; outputs must not alias the inputs; n < 2^32) and an
// exclusive prefix sum (in and out may alias).
template <class K>
void radix_sort_pairs(const K *keys, const uint32_t *vals, int64_t n, int bits, K *keys_out, uint32_t *vals_out,
                      cudaStream_t st);
void exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, cudaStream_t st);
void build_csr(const int32_t *keys, const uint32_t *vals, int64_t n, int64_t K, int64_t *offsets, uint32_t *ids,
               cudaStream_t st);
// PQk-means over a sample (R9); centers out [K][M]; *err set if < K distinct codes.
void run_pqkmeans(const uint8_t *X, int64_t ns, int64_t K, int M, const float *T, int n_iter, uint8_t *centers,
                  int *err, cudaStream_t st);
// The ns smallest splitmix64(seed ^ gid) keys among n codes with global ids gid(i);
// writes their local positions in ascending key order.
void select_sample(int64_t n, const IdMap &gid, int64_t ns, uint64_t seed, uint32_t *out_pos, cudaStream_t st);
// keys[i] = splitmix64(seed ^ gid(pos[i])) for i < n.
void sample_keys_for_positions(int64_t n_local, const IdMap &gid, const uint32_t *pos, int64_t n, uint64_t seed,
                               uint64_t *keys, cudaStream_t st);
// order[0..n) = indices of keys in ascending key order (stable).
void sort_keys_with_index(const uint64_t *keys, int64_t n, uint32_t *order, cudaStream_t st);

}  // namespace rii
