/*
 * spkm.h -- C ABI of libspkm.so, the sm_100a kernels behind the accelerated
 * spherical k-means iteration loop (arXiv 2107.04074).
 *
 * Conventions:
 *   - every buffer is caller-owned DEVICE memory passed as a plain pointer;
 *     the library allocates nothing persistent;
 *   - every call is asynchronous on the given cudaStream_t (passed as void*);
 *   - return value 0 = ok, otherwise an error code; spkm_last_error() gives
 *     the message of the last failure on the calling thread;
 *   - no callbacks into the host.
 *
 * Reference boundary each entry point replaces (paths relative to
 * /root/reference/pkg/src/spkmeans/):
 *   spkm_full_assign        engine._full_sims + argmax/top-2 + bound init,
 *                           engine.py:99-100, 103-120, 249-263, 268-271
 *   spkm_hamerly_bounds     Hamerly drift update, engine.py:274, 284-303,
 *                           geometry.py:30-63 (fused with the prune test)
 *   spkm_hamerly_tighten    kernels.hamerly_scan tighten + re-test,
 *                           kernels.py:81-95
 *   spkm_hamerly_rescan     kernels.hamerly_scan full-k scan, kernels.py:96-112
 *   spkm_elkan_bounds       Elkan drift update, engine.py:274-283 (fused test)
 *   spkm_elkan_scan         kernels.elkan_scan, kernels.py:22-66
 *   spkm_elkan_heavy        kernels.elkan_scan for rows the bounds barely prune (full pass)
 *   spkm_aggregate_sums     engine._aggregate_sums, engine.py:130-139
 *   spkm_apply_moves        engine.update_centers (incremental), engine.py:174-188
 *   spkm_move_centers       engine._move_centers, engine.py:142-160
 *   spkm_center_thresholds  engine._center_thresholds, engine.py:192-198
 *   spkm_finalize           objective + convergence inputs, engine.py:326-337
 *   spkm_predict            engine.assign_full, engine.py:103-120
 *   spkm_seed_kmpp          seeding.init_kmpp, seeding.py:64-89
 *   spkm_seed_afkmc2        seeding.init_afkmc2, seeding.py:92-146
 */
#ifndef SPKM_H
#define SPKM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPKM_ABI_VERSION 3

/* variants, engine.py:22 */
enum spkm_variant {
    SPKM_STANDARD = 0,
    SPKM_ELKAN = 1,
    SPKM_SIMP_ELKAN = 2,
    SPKM_HAMERLY = 3,
    SPKM_SIMP_HAMERLY = 4,
    SPKM_YINYANG = 5            /* not in the reference: group bounds */
};

/* spkm_full_assign modes */
enum spkm_assign_mode {
    SPKM_MODE_INIT_PLAIN = 0,   /* iteration 1, no bounds (standard)          */
    SPKM_MODE_INIT_ELKAN = 1,   /* iteration 1, l + u(i,j) for every j        */
    SPKM_MODE_INIT_HAMERLY = 2, /* iteration 1, l + u = second best           */
    SPKM_MODE_LLOYD = 3,        /* iteration >= 2 of standard: reassign+moves */
    SPKM_MODE_INIT_YINYANG = 6  /* iteration 1, l + group bounds ug(i, g), g = 4 centers */
};

/* Device CSR of the (local shard of the) corpus; rows unit-normalised. */
typedef struct spkm_csr {
    int64_t n;               /* rows in this shard                        */
    int64_t d;               /* dimensionality                            */
    int64_t nnz;
    const int64_t *indptr;   /* [n+1]                                     */
    const int32_t *indices;  /* [nnz], sorted within a row                */
    const float *values;     /* [nnz]                                     */
    const float *row_eps;    /* [n] float32 similarity error bound of row i:
                                (nnz_i + 6) * 6.1e-8, rounded up           */
} spkm_csr;

/* Sparse term-major index of the centers (k > 256): for every term row t of
 * ct32, its nonzero centers as (j, value bits) pairs when there are at most
 * dense_thr of them, else the row is read densely from ct32.  desc[t] =
 * (offset into pairs << 12) | count (0xFFF: dense row).  Rebuilt from ct32 by
 * spkm_cindex_build after every center update the full pass will read.  The
 * full pass then gathers ~2.5x fewer bytes at C4 (tail term rows are ~10%
 * dense) with the same canonical FMA chain (zeros contribute nothing). */
typedef struct spkm_cindex {
    int64_t *desc;           /* [d] */
    int32_t *pairs;          /* [2 * capacity] (j, float bits) */
    int64_t *off;            /* [d] scratch: off[0] = running total of reserved pairs during a build */
    void *scratch;           /* spkm_cindex_scratch_bytes(d) bytes (unused by the one-pass build)     */
    int64_t scratch_bytes;
    int64_t capacity;        /* pairs; >= nonzeros of the centers (<= nnz of the corpus) */
    int32_t dense_thr;       /* rows with more nonzeros are read densely */
    int32_t _pad;
} spkm_cindex;

/* Replicated center state.  kp = padded k of the term-major copy. */
typedef struct spkm_centers {
    int64_t k, d, kp;
    int32_t scale_bits;      /* fixed-point sums: value = sum * 2^-scale_bits */
    int32_t _pad;
    double *cent64;          /* [k*d] unit centers, center-major, float64   */
    float *ct32;             /* [d*kp] term-major float32 copy (pad = 0)    */
    long long *sums;         /* [k*d] exact fixed-point member sums         */
    long long *counts;       /* [k]                                         */
    double *drift;           /* [k] p(j) = <c_new, c_old> = 1 - chord^2/2    */
    double *sinp;            /* [k] upper bound on sin(angle(c_new, c_old))  */
    int32_t *touched;        /* [k] cluster changed this iteration          */
    double *objc;            /* [k] <sums_j, c_j> per cluster               */
    double *part;            /* [spkm_center_scratch_doubles] partial sums  */
    double *norm;            /* [k] scratch: |sums_j|                       */
    float *cc;               /* [k*k] half-angle center cosines, rounded up */
    float *s;                /* [k]   row max of cc (diag excluded)         */
    double *hstat;           /* [8]   owner, p_min, p_min2, owner_s, smax, smax2, fuse, all-heavy */
    int32_t *tlist;          /* [k]   scratch: touched cluster list         */
    int32_t *tcount;         /* [1]   scratch: its length                   */
    long long *ctl;          /* [2]   {iterations done, converged}: every loop
                                kernel is a no-op once converged, so the
                                host may enqueue iterations ahead          */
    uint16_t *ct16;          /* [d*kp] fp16 (round to nearest) copy of ct32 for
                                the screening full pass, or NULL: the row
                                pass gathers half the bytes and re-checks
                                the near-best centers on ct32 exactly      */
    const spkm_cindex *cindex;  /* host pointer: sparse index for the full
                                   pass (k > 256), or NULL                  */
} spkm_centers;

/* Per-point bounds of the local shard. */
typedef struct spkm_bounds {
    int32_t *a;              /* [n] assignment                               */
    float *l;                /* [n] lower bound on <x_i, c_a(i)> (round down) */
    float *u;                /* [n*ku] Elkan u(i,j) or [n] Hamerly u(i)      */
    int64_t ku;              /* row stride of u (Elkan) or 1 (Hamerly)       */
} spkm_bounds;

/* Dense corpus (config C5): float32 rows and float32 centers (zero rows
 * past k, kpad a multiple of 256); the tcgen05 pass streams both with TMA and
 * splits them into tf32 hi + lo on the fly (3xTF32).  xs: [n][D] scratch the
 * Hamerly rescan compacts its survivors into (NULL if never rescanned). */
typedef struct spkm_dense {
    int64_t D;               /* dimensionality (multiple of 32)              */
    int64_t kpad;
    const float *x;          /* [n][D] rows (the spkm_csr values)            */
    float *b;                /* [kpad][D] centers, written by dense_centers  */
    float *xs;               /* [n][D] survivor scratch                      */
} spkm_dense;

/* Worklists and device-side counters. */
typedef struct spkm_work {
    int32_t *surv1;          /* [n] points failing the bound test            */
    int32_t *surv2;          /* [n] points failing after tightening          */
    int32_t *mv_i;           /* [n] moved point ids                          */
    int32_t *mv_old;         /* [n] their previous cluster                   */
    long long *ctr;          /* [8] counters, see SPKM_CTR_*                 */
    double *stats;           /* [16] per-iteration stats, see SPKM_ST_*      */
    double *stats_hist;      /* [hist_cap][16] stats of every iteration      */
    int64_t hist_cap;
    int64_t elkan_heavy;     /* > 0: spkm_elkan_bounds sends rows with at least this many unpruned
                              * centers to surv2 for spkm_elkan_heavy                     */
    int64_t allheavy_rows;   /* > 0 (= the rows this engine scans) with elkan_heavy > 0: while an iteration
                              * moves >= allheavy_rows / 256 rows, the next one skips spkm_elkan_bounds and
                              * spkm_elkan_heavy takes every row (flag in hstat[7], set by spkm_finalize);
                              * 0: never (debug hooks that read the bounds between the calls)            */
    int32_t *lightj;         /* [n][4] or NULL.  With use_cc == 0 and 0 < elkan_heavy <= 5 the bound
                              * pass lists the (< elkan_heavy) failing centers of every surv1 row here
                              * (ascending, -1 padded) and spkm_elkan_scan scans exactly those        */
} spkm_work;

enum {
    SPKM_CTR_SURV1 = 0, SPKM_CTR_SURV2 = 1, SPKM_CTR_MOVES = 2, SPKM_CTR_SIMS = 3,
    SPKM_CTR_NNZ_TIGHTEN = 4, SPKM_CTR_NNZ_RESCAN = 5, SPKM_CTR_NNZ_ELKAN = 6, SPKM_CTR_NNZ_MOVED = 7
};
enum {
    SPKM_ST_SIMS = 0, SPKM_ST_REASSIGN = 1, SPKM_ST_OBJECTIVE = 2, SPKM_ST_ALLONE = 3,
    SPKM_ST_SURV1 = 4, SPKM_ST_SURV2 = 5, SPKM_ST_TOUCHED = 6, SPKM_ST_NNZ_TIGHTEN = 7,
    SPKM_ST_NNZ_RESCAN = 8, SPKM_ST_NNZ_ELKAN = 9, SPKM_ST_ITER = 10,
    SPKM_ST_TSTAMP = 11,  /* device %globaltimer (ns) at the end of the iteration */
    SPKM_ST_T0 = 12,      /* %globaltimer at spkm_reset_counters (start of the fit) */
    SPKM_ST_NNZ_MOVED = 13, /* CSR nnz of the moved points (incremental center update) */
    SPKM_ST_COUNT = 16
};

int spkm_abi_version(void);
const char *spkm_last_error(void);
/* number of chunks the center kernels split d into (size of centers.part) */
int64_t spkm_center_chunks(int64_t d);
/* doubles of scratch the center kernels need (centers.part) */
int64_t spkm_center_scratch_doubles(int64_t k, int64_t d);
/* padded k (kp) of the term-major copy for a given k */
int64_t spkm_padded_k(int64_t k);

/* Zero counters (ctr) and stamp stats[SPKM_ST_T0] at the start of a fit. */
int spkm_reset_counters(spkm_work *w, void *stream);

/* Full pass over rows [row_begin,row_end): every <x_i, c_j> in the canonical
 * order (fp32 FMA chain over the row's nnz in CSR order), fused top-2.
 * INIT modes write a, l (and u); LLOYD reassigns with "incumbent wins exact
 * ties, otherwise lowest index" and appends moves. */
int spkm_full_assign(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W,
                     int mode, void *stream);

int spkm_hamerly_bounds(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W,
                        int use_s, int naive, void *stream);
int spkm_hamerly_tighten(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W,
                         int use_s, void *stream);
/* Yin-Yang group bounds (the reference has no
 * Yin-Yang): groups = 4 consecutive centers; B->u holds ug[n][ku] with
 * ku = ceil(k/4) rounded up to 4.  Iteration 1: spkm_full_assign with
 * SPKM_MODE_INIT_YINYANG.  Then per iteration: spkm_yy_bounds (drift update
 * of l and ug by each group's worst drift, prune test, survivor list) and
 * spkm_yy_scan (tighten s~(i, a), fetch the groups with ug + eps > s~(i, a),
 * best by the Lloyd rule, exact bounds of the fetched groups).  k <= 1024. */
int spkm_yy_bounds(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, void *stream);
int spkm_yy_scan(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, void *stream);

/* Full-k rescan of the tighten survivors.  use_s: as for spkm_hamerly_tighten
 * -- when the previous iteration's tighten pruned < 5% of the bound survivors
 * (flag in hstat[6], set by spkm_finalize) this pass takes the bound
 * survivors and applies the tighten test itself (the tighten call is then a
 * no-op): identical results and counters, one pass fewer. */
int spkm_hamerly_rescan(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int use_s,
                        void *stream);
int spkm_elkan_bounds(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W,
                      int use_cc, void *stream);
int spkm_elkan_scan(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W,
                    int use_cc, void *stream);
/* Heavy survivors (kernels.elkan_scan, kernels.py:22-66, for rows whose stored
 * bounds prune little).  With W->elkan_heavy > 0 spkm_elkan_bounds splits its
 * survivors: rows where at least W->elkan_heavy centers fail the stored-bound
 * test go to W->surv2 (count in ctr[SPKM_CTR_SURV2]), the others to W->surv1.
 * spkm_elkan_heavy takes the surv2 rows through one full pass (over the sparse
 * center index when C->cindex is attached: spkm_cindex_build first): same
 * reassignment rule as the scan (incumbent wins ties, else the lowest index),
 * l and every u(i, j) come back exact, SIMS += k per row.  Call it between
 * spkm_elkan_bounds and spkm_elkan_scan whenever W->elkan_heavy > 0.
 * spkm_elkan_heavy_threshold: the library's default for k centers (0.5% of k
 * rounded up for k > 128, SPKM_EK_HEAVY_PCT overrides; 0 = off). */
int spkm_elkan_heavy(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, void *stream);
int64_t spkm_elkan_heavy_threshold(int64_t k);
/* spkm_elkan_bounds + spkm_elkan_scan in one pass over all rows: each row's
 * drift update and prune test are done by the lanes that then scan it (same
 * results and counters as the two calls). */
int spkm_elkan_bounds_scan(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int use_cc,
                           void *stream);

/* Order a row worklist by cluster a(i) (counting sort; L2 locality of the
 * gather passes when the center table exceeds L2: rows of one cluster share
 * most of their terms).  list == NULL: rows [0, n) are ordered into `out`;
 * otherwise the first *count (device) entries of `list` are reordered in
 * place through `tmp` (n int32).  bins: 2k int32 scratch; k <= 12288.
 * Every pass's results are independent of the order rows are visited in.
 * No reference counterpart (the reference visits rows in index order,
 * kernels.py:31, 78); ctl[1] != 0 makes it a no-op like the loop kernels. */
int spkm_order_by_cluster(int64_t k, const int32_t *a, int32_t *list, const long long *count, int64_t n,
                          int32_t *tmp, int32_t *out, int32_t *bins, const long long *ctl, void *stream);

/* Center maintenance.  aggregate: sums/counts from scratch (target arrays may
 * be a delta buffer); apply_moves: sums[old] -= x, sums[new] += x for the
 * recorded moves into `sums_target`/`counts_target`, marks touched. */
int spkm_aggregate_sums(const spkm_csr *X, const spkm_centers *C, const spkm_bounds *B,
                        long long *sums_target, long long *counts_target, void *stream);
int spkm_apply_moves(const spkm_csr *X, const spkm_centers *C, const spkm_bounds *B,
                     const spkm_work *W, long long *sums_target, long long *counts_target,
                     int32_t *touched, void *stream);
/* Renormalise touched clusters (all if all_clusters), write cent64/ct32,
 * drift and per-cluster objective. */
int spkm_move_centers(const spkm_centers *C, int all_clusters, void *stream);
/* all_clusters | 4: stop after the center write; the per-cluster drift and
 * objective reduction is then spkm_center_reduce (so the next iteration's
 * spkm_center_thresholds, which needs only the new centers and the touched
 * list, can run beside it and spkm_finalize on a second stream). */
int spkm_center_reduce(const spkm_centers *C, void *stream);
/* cc(a,j) = sqrt((<c_a,c_j>+1)/2) rounded up, s(a) = max_{j!=a} cc(a,j).
 * float64 split-d Gram over the upper-triangle 32x32 tiles listed in
 * tile_pairs (from spkm_gram_tiles); gram_scratch holds
 * spkm_gram_scratch_doubles(k, d) doubles. */
int64_t spkm_gram_tiles(int64_t k, int32_t *host_pairs);
int64_t spkm_gram_scratch_doubles(int64_t k, int64_t d);
int spkm_center_thresholds(const spkm_centers *C, double *gram_scratch, const void *tile_pairs,
                           int full, void *stream);
/* The same in two halves for the multi-GPU path: spkm_gram_partial computes
 * rank's round-robin share of the (tile, d-split) Gram partials (world > 1:
 * the others are zeroed), the caller sums the spkm_gram_partial_floats(k, d)
 * floats at the start of gpart over the ranks (allreduce; exact: every
 * element is nonzero on one rank only), then spkm_gram_finish maps them to
 * cc and s.  rank 0 of world 1 == spkm_center_thresholds. */
int64_t spkm_gram_partial_floats(int64_t k, int64_t d);
/* Sparse center index (spkm_cindex): scratch size and the rebuild from ct32. */
int64_t spkm_cindex_scratch_bytes(int64_t d);
int spkm_cindex_build(const spkm_centers *C, void *stream);
int spkm_gram_partial(const spkm_centers *C, double *gpart, const void *tiles, int full, int rank, int world,
                      void *stream);
int spkm_gram_finish(const spkm_centers *C, double *gpart, int full, void *stream);
/* Objective, all-p==1 flag, Hamerly owner/p_min/p_min2, stats; clears
 * touched.  sims_extra is added to the sims counter (host-known counts). */
int spkm_finalize(const spkm_centers *C, spkm_work *W, int all_clusters, long long sims_extra,
                  void *stream);

/* predict (assign_full): a (lowest index on ties), best, second (float64). */
int spkm_predict(const spkm_csr *X, const spkm_centers *C, int32_t *a, double *best,
                 double *second, void *stream);

/* compute_objective (engine.py:123-127): Sum_j <sums_j * 2^-scale, c_j>, with
 * sums built by spkm_aggregate_sums for the given assignments. */
int spkm_objective(const spkm_centers *C, const long long *sums, double *out, void *stream);

/* Upload helper: write center-major float64 centers into cent64 and ct32. */
int spkm_load_centers(const spkm_centers *C, const double *host_or_dev_centers, void *stream);

/* Seed centers from k data rows (init_uniform, seeding.py:56-61 +
 * CentroidSet.from_data_rows, engine.py:46-58): packed CSR of the seed rows
 * (sptr[k+1], sidx, float64 values) in device memory. */
int spkm_seed_rows(const spkm_centers *C, const int64_t *sptr, const int32_t *sidx, const double *sval,
                   void *stream);

/* Dense path (config C5).  centers: cent64 -> float32 b; assign: the
 * tensor-core similarity pass (3xTF32) with fused top-2.  mode is an
 * spkm_assign_mode, 5 (predict: writes a, best, second) or 6 (Hamerly
 * tighten + full scan over work->surv1, kernels.py:81-112). */
int spkm_dense_centers(const spkm_centers *C, const spkm_dense *Dn, void *stream);
int spkm_dense_assign(const spkm_csr *X, const spkm_centers *C, const spkm_dense *Dn, spkm_bounds *B,
                      spkm_work *W, int mode, int use_s, double *best, double *second, void *stream);

/* Seeding (seeding.py:64-146): spherical k-means++ and AFK-MC2 on the
 * device, with the reference's splitmix64 stream (rng.py) and its float64
 * similarity order, so the picks equal the reference's.  The CSR is the
 * device-order corpus with float64 values; row_host maps a device row to the
 * reference's row id (row_dev is the inverse).  picks: device int64[k] of
 * reference row ids in pick order.  trace (optional, device [(k-1) * n]):
 * the kmpp weight vector of every pick (seeding.py:80-81). */
typedef struct spkm_seed {
    int64_t n, d;
    const int64_t *indptr;
    const int32_t *indices;
    const double *values;
    const int64_t *row_host;
    const int64_t *row_dev;
    double *scratch;         /* spkm_seed_scratch_doubles(n, d) doubles        */
} spkm_seed;
int64_t spkm_seed_scratch_doubles(int64_t n, int64_t d);
int spkm_seed_kmpp(const spkm_seed *S, int64_t k, double alpha, uint64_t seed, int64_t *picks,
                   double *trace, void *stream);
int spkm_seed_afkmc2(const spkm_seed *S, int64_t k, double alpha, int64_t chain_length, uint64_t seed,
                     int64_t *picks, void *stream);
/* Seed centers = data rows given by reference row id (device rows[k]),
 * gathered from the spkm_seed corpus (init_uniform + from_data_rows). */
int spkm_seed_rows_csr(const spkm_centers *C, const spkm_seed *S, const int64_t *rows, void *stream);

/* Bound auditor (validation.py:49-80) and brute-force assignment
 * (validation.py:18-29) on the device.  spkm_audit_transpose writes the
 * term-major float64 copy ct64 [d][kp] of center-major float64 centers;
 * spkm_audit computes every exact float64 similarity of the spkm_seed
 * corpus (device-order rows) and folds, with atomicMax on order-preserving
 * keys (keys[0] lower, keys[1] upper): mode 0 max(l - S[i,a]) and
 * max(S - u) over the Elkan matrix (row stride ku), 1 the Hamerly
 * max_{j != a} S[i,j] - u[i], 2 the Yin-Yang max_{j != a} S[i,j] - u[i, j/4]
 * (group bounds, row stride ku), 3 argmax per row into
 * a_out (lowest index on ties). */
int spkm_audit_transpose(int64_t k, int64_t d, int64_t kp, const double *cent64, double *ct64, void *stream);
int spkm_audit(const spkm_seed *S, int64_t k, int64_t kp, const double *ct64, const int32_t *a, const float *l,
               const float *u, int64_t ku, int mode, unsigned long long *keys, int32_t *a_out, void *stream);

/* Multi-GPU exchange (distributed.py): the corpus is replicated and the
 * scans are sharded by device-row ranges; per iteration each rank packs its
 * moves and counters into a fixed-size int32 slot of
 * spkm_move_slot_ints(cap) ints (a multiple of 4: every slot of the gathered
 * array is 16-byte aligned; cap = its shard's rows; rows are stored
 * global, p0 = the shard's first device row), the slots are allgathered
 * (NCCL), and every rank applies all ranks' moves to its replicated
 * fixed-point sums (spkm_apply_move_slots, X = the whole corpus) and takes
 * the summed counters into ctr_out. */
int64_t spkm_move_slot_ints(int64_t cap);
int spkm_pack_moves(const spkm_work *W, const spkm_bounds *B, const spkm_centers *C, int64_t p0, int64_t cap,
                    int32_t *slot, void *stream);
int spkm_apply_move_slots(const spkm_csr *X, const spkm_centers *C, const int32_t *slots, int world, int64_t slot_len,
                          int32_t *touched, long long *ctr_out, void *stream);

/* Device-driven fit loop (engine.py:239-337 without a host round trip per
 * iteration): a CUDA graph whose conditional WHILE node repeats one
 * iteration while ctl says "not converged" and ctl[0] < *limit.  begin()
 * starts capturing the body on `stream` (the caller then issues one
 * iteration's calls on it); end() closes and instantiates the graph. */
int spkm_loop_begin(const long long *ctl, const long long *limit, void *stream, void **loop_out);
int spkm_loop_end(void *loop);
int spkm_loop_launch(void *loop, void *stream);
int spkm_loop_destroy(void *loop);

/* Whole-fit graph (one launch per fit): begin() captures the prefix on
 * `stream` (seed upload, reset, iterations 1-2), loop() adds the WHILE node
 * after it and starts capturing the body on `body_stream`, spkm_loop_end()
 * closes the body, the caller captures the suffix (result downloads) on
 * `stream`, end() instantiates.  Launched and destroyed with spkm_loop_*. */
int spkm_fit_graph_begin(void *stream, void **loop_out);
int spkm_fit_graph_loop(void *loop, const long long *ctl, const long long *limit, void *body_stream);
int spkm_fit_graph_end(void *loop);
int spkm_fit_graph_abort(void *loop);     /* error path: close open captures, free */

/* out[row_perm[r]] = a[r] (int64): device-order assignments in host row order. */
int spkm_rows_to_host(int64_t n, const int64_t *row_perm, const int32_t *a, int64_t *out, void *stream);

/* Stream-ordered copies / fills (capturable; cudaMemcpyDefault). */
int spkm_memcpy_async(void *dst, const void *src, int64_t bytes, void *stream);
int spkm_memset_async(void *dst, int value, int64_t bytes, void *stream);

/* Corpus upload: write the rows of a raw CSR (ip_raw[n+1] relative offsets,
 * int32 ids, float64 values) in device order: device row r = raw row
 * perm[r] at ip_new[r], ids mapped through new_id, float32 values (round to
 * nearest), optional float64 copy (val64) and row_eps (reps) of spkm_csr. */
int spkm_permute_rows(int64_t n, const int64_t *ip_raw, const int32_t *idx_raw, const double *val_raw,
                      const int64_t *perm, const int64_t *ip_new, const int64_t *new_id, int32_t *idx, float *val,
                      double *val64, float *reps, void *stream);

/* Corpus layout on the device (replaces the host CSR build of sparse.py:136-156
 * Dataset.matrix / csr_arrays for the device copy): from the raw row offsets
 * ip_raw[n+1] (relative, ip_raw[0] = 0) -> perm[n] (device row r = raw row
 * perm[r], rows longest first, stable), pos[n] (inverse of perm, optional),
 * indptr[n+1] (device-order offsets); when order and new_id are given, also
 * the term order by document frequency over idx_raw[nnz] (descending,
 * stable): order[d] (new id -> raw id) and new_id[d] (raw id -> new id).
 * perm = NULL skips the row part.  Scratch: spkm_prepare_scratch_bytes(n, d)
 * bytes (-1: n or d >= 2^31). */
int64_t spkm_prepare_scratch_bytes(int64_t n, int64_t d);
/* Dense corpora (every row holds the D terms in order): idx[r*D + t] = t,
 * indptr[r] = r*D (n+1 entries), perm[r] = r (the stable length order is the
 * identity); indptr / perm may be NULL. */
int spkm_dense_ids(int64_t n, int64_t D, int32_t *idx, int64_t *indptr, int64_t *perm, void *stream);
int spkm_prepare_rows(int64_t n, int64_t d, int64_t nnz, const int64_t *ip_raw, const int32_t *idx_raw,
                      int64_t *perm, int64_t *pos, int64_t *indptr, int64_t *order, int64_t *new_id,
                      void *scratch, int64_t scratch_bytes, void *stream);

/* Ingestion (host, no GPU; corpus_io.py:31-131).  spkm_svml_parse parses a
 * whole SVMlight/libsvm text buffer with nthreads threads (<1: all cores);
 * on a syntax error it returns 1 with err_line (1-based) and err_msg (the
 * reference's ParseError text).  spkm_svml_fetch copies the CSR (indptr
 * [n_rows+1], int64 indices, float64 values; explicit zeros dropped) and
 * releases the result; spkm_svml_free releases it without copying.
 * spkm_host_idf: idf of every term with df > 0 (ln(n/df), or the smooth
 * variant), computed with libm log like the reference's math.log. */
typedef struct spkm_svml {
    int64_t n_rows, nnz, max_idx, err_line;
    char err_msg[256];
    void *handle;
} spkm_svml;
int spkm_svml_parse(const char *buf, int64_t len, int nthreads, spkm_svml *out);
int spkm_svml_fetch(spkm_svml *res, int64_t *indptr, int64_t *indices, double *values);
int spkm_svml_free(spkm_svml *res);
int spkm_host_idf(int64_t d, const int64_t *df, int64_t n, int smooth, double *idf);

/* Host helper (no GPU): |row| of every CSR row in the reference's np.dot
 * order (sparse.py:52), for Dataset.from_csr. */
int spkm_host_row_norms(int64_t n, const int64_t *indptr, const double *values, double *out);

/* Device geometry for tests: op 0 lower, 1 upper, 2 hamerly, 3 half-angle. */
int spkm_geometry(int op, int64_t n, const double *a, const double *b, double *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif
