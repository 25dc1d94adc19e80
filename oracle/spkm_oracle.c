/*
 * spkm_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C, float64 restatement of the reference's spherical k-means
 * iteration loop (arXiv 2107.04074 reference package `spkmeans`, mounted at
 * /root/reference/pkg/src/spkmeans).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Every function cites the reference file:line it restates.  Arithmetic is
 * kept in the reference's operation order and compiled with
 * -ffp-contract=off so that the per-pair similarity (SciPy csr_matvecs /
 * Numba _dot_row: s = 0; s += v*c, no FMA) and the elementwise numpy
 * geometry reproduce the reference bit-for-bit.  BLAS-backed reductions
 * (np.linalg.norm, np.dot, centers @ centers.T, einsum) are restated as
 * FMA chains (the form OpenBLAS's ddot tail loop takes, which reproduces
 * numpy exactly for short vectors); for long vectors they may differ from
 * OpenBLAS's blocked kernels in the last bit.
 *
 * Parity pin: tests/test_oracle.py checks this oracle against golden vectors
 * produced by running the reference itself (tests/golden/make_golden.py).
 *
 * Parallelism: OpenMP over points (the reference spec permits it,
 * SPEC.md:410-411); every per-point result and every reduction is computed
 * in a fixed order, so results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ZERO_SUM_EPS 1e-12   /* engine.py:27 */
#define SCRATCH_INTERVAL 50  /* engine.py:28 */

enum { V_STANDARD = 0, V_ELKAN = 1, V_SIMP_ELKAN = 2, V_HAMERLY = 3, V_SIMP_HAMERLY = 4 };

/* ---------------------------------------------------------------- rng.py */
/* splitmix64 transition, rng.py:39-44 */
static uint64_t sm64_next(uint64_t *state) {
    *state += 0x9E3779B97F4A7C15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void oracle_sm64_stream(uint64_t seed, int64_t count, uint64_t *out) {
    uint64_t s = seed;
    for (int64_t i = 0; i < count; ++i) out[i] = sm64_next(&s);
}

/* sample_without_replacement, rng.py:54-73 (randint = next % n, rng.py:49-52).
 * Returns 0 on success, -1 if k > n. */
int oracle_sample_without_replacement(uint64_t seed, int64_t n, int64_t k, int64_t *out) {
    if (k < 0 || k > n) return -1;
    uint64_t s = seed;
    if (2 * k < n) {
        /* rejection on randint(n); tiny k so a linear membership scan is fine,
         * but use a sorted shadow for k up to ~1e5 */
        int64_t got = 0;
        int64_t *seen = (int64_t *)malloc(sizeof(int64_t) * (size_t)(k > 0 ? k : 1));
        while (got < k) {
            int64_t v = (int64_t)(sm64_next(&s) % (uint64_t)n);
            /* binary search in seen[0..got) (kept sorted) */
            int64_t lo = 0, hi = got;
            while (lo < hi) { int64_t m = (lo + hi) / 2; if (seen[m] < v) lo = m + 1; else hi = m; }
            if (lo < got && seen[lo] == v) continue;
            memmove(seen + lo + 1, seen + lo, sizeof(int64_t) * (size_t)(got - lo));
            seen[lo] = v;
            out[got++] = v;
        }
        free(seen);
        return 0;
    }
    int64_t *pool = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) pool[i] = i;
    for (int64_t i = 0; i < k; ++i) {
        int64_t j = i + (int64_t)(sm64_next(&s) % (uint64_t)(n - i));
        int64_t t = pool[i]; pool[i] = pool[j]; pool[j] = t;
        out[i] = pool[i];
    }
    free(pool);
    return 0;
}

/* ----------------------------------------------------------- geometry.py */
static inline double clampc(double t) { return t < -1.0 ? -1.0 : (t > 1.0 ? 1.0 : t); } /* geometry.py:20-22 */
static inline double sinc_(double t) { double v = 1.0 - t * t; return sqrt(v > 0.0 ? v : 0.0); } /* 25-27 */
static inline double cos_lower(double a, double b) { return clampc(a * b - sinc_(a) * sinc_(b)); } /* 30-32 */
static inline double cos_upper(double a, double b) { return clampc(a * b + sinc_(a) * sinc_(b)); } /* 35-37 */
static inline double hamerly_upper(double u, double p) { return clampc(u + sinc_(u) * sinc_(p)); } /* 54-63 */
static inline double half_angle(double s) { double v = (s + 1.0) / 2.0; return sqrt(v > 0.0 ? v : 0.0); } /* 66-68 */

void oracle_geometry(int op, int64_t n, const double *a, const double *b, double *out) {
    for (int64_t i = 0; i < n; ++i) {
        switch (op) {
            case 0: out[i] = cos_lower(a[i], b[i]); break;
            case 1: out[i] = cos_upper(a[i], b[i]); break;
            case 2: out[i] = hamerly_upper(a[i], b[i]); break;
            case 3: out[i] = half_angle(a[i]); break;
            default: out[i] = clampc(a[i]); break;
        }
    }
}

/* ------------------------------------------------------------- kernels.py */
/* _dot_row, kernels.py:14-19: sequential, no FMA */
static inline double dot_row(const int64_t *indptr, const int32_t *indices, const double *data,
                             int64_t i, const double *c) {
    double s = 0.0;
    for (int64_t t = indptr[i]; t < indptr[i + 1]; ++t) s += data[t] * c[indices[t]];
    return s;
}

/* _full_sims, engine.py:99-100 -> SciPy csr_matvecs: y[i,:] += v * CT[idx,:]
 * with CT the C-ordered transpose (d x k); per (i,j) this is the same
 * sequential order as _dot_row.  S is n x k row-major. */
void oracle_full_sims(int64_t n, int64_t d, int64_t k, const int64_t *indptr, const int32_t *indices,
                      const double *data, const double *C, double *S) {
    double *CT = (double *)malloc(sizeof(double) * (size_t)(d * k));
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < d; ++t)
        for (int64_t j = 0; j < k; ++j) CT[t * k + j] = C[j * d + t];
    #pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        double *y = S + i * k;
        for (int64_t j = 0; j < k; ++j) y[j] = 0.0;
        for (int64_t t = indptr[i]; t < indptr[i + 1]; ++t) {
            const double v = data[t];
            const double *ct = CT + (int64_t)indices[t] * k;
            for (int64_t j = 0; j < k; ++j) y[j] += v * ct[j];
        }
    }
    free(CT);
}

/* elkan_scan, kernels.py:22-66 (per point; returns sims for the point) */
static int64_t elkan_point(const int64_t *indptr, const int32_t *indices, const double *data,
                           const double *C, int64_t d, int64_t k, int64_t i, int64_t *a, double *l,
                           double *u, const double *cc, const double *s_arr, int use_cc) {
    int64_t sims = 0;
    int64_t ai = a[i];
    double li = l[i];
    if (use_cc && li >= 0.0 && s_arr[ai] <= li) return 0;
    int tightened = 0;
    double *ui = u + i * k;
    for (int64_t j = 0; j < k; ++j) {
        if (j == ai) continue;
        if (use_cc && li >= 0.0 && cc[ai * k + j] <= li) continue;
        if (ui[j] <= li) continue;
        if (!tightened) {
            li = dot_row(indptr, indices, data, i, C + ai * d);
            sims += 1;
            l[i] = li;
            ui[ai] = li;
            tightened = 1;
            if (use_cc && li >= 0.0 && cc[ai * k + j] <= li) continue;
            if (ui[j] <= li) continue;
        }
        double sij = dot_row(indptr, indices, data, i, C + j * d);
        sims += 1;
        ui[j] = sij;
        if (sij > li) { ai = j; li = sij; a[i] = j; l[i] = sij; }
    }
    return sims;
}

/* hamerly_scan, kernels.py:69-113 (per point) */
static int64_t hamerly_point(const int64_t *indptr, const int32_t *indices, const double *data,
                             const double *C, int64_t d, int64_t k, int64_t i, int64_t *a, double *l,
                             double *u, const double *s_arr, int use_s) {
    int64_t ai = a[i];
    double li = l[i];
    if (use_s && li >= 0.0 && s_arr[ai] <= li) return 0;
    if (u[i] <= li) return 0;
    li = dot_row(indptr, indices, data, i, C + ai * d);
    int64_t sims = 1;
    l[i] = li;
    if (use_s && li >= 0.0 && s_arr[ai] <= li) return sims;
    if (u[i] <= li) return sims;
    double best = li, second = -2.0;
    int64_t best_j = ai;
    for (int64_t j = 0; j < k; ++j) {
        if (j == ai) continue;
        double sij = dot_row(indptr, indices, data, i, C + j * d);
        sims += 1;
        if (sij > best) { second = best; best = sij; best_j = j; }
        else if (sij > second) second = sij;
    }
    if (best_j != ai) { a[i] = best_j; l[i] = best; }
    u[i] = second;
    return sims;
}

int64_t oracle_elkan_scan(int64_t n, int64_t d, int64_t k, const int64_t *indptr, const int32_t *indices,
                          const double *data, const double *C, int64_t *a, double *l, double *u,
                          const double *cc, const double *s_arr, int use_cc) {
    int64_t sims = 0;
    #pragma omp parallel for schedule(dynamic, 64) reduction(+ : sims)
    for (int64_t i = 0; i < n; ++i)
        sims += elkan_point(indptr, indices, data, C, d, k, i, a, l, u, cc, s_arr, use_cc);
    return sims;
}

int64_t oracle_hamerly_scan(int64_t n, int64_t d, int64_t k, const int64_t *indptr, const int32_t *indices,
                            const double *data, const double *C, int64_t *a, double *l, double *u,
                            const double *s_arr, int use_s) {
    int64_t sims = 0;
    #pragma omp parallel for schedule(dynamic, 64) reduction(+ : sims)
    for (int64_t i = 0; i < n; ++i)
        sims += hamerly_point(indptr, indices, data, C, d, k, i, a, l, u, s_arr, use_s);
    return sims;
}

/* -------------------------------------------------------------- engine.py */
/* _aggregate_sums, engine.py:130-139: onehot(k x n) @ X -> per cluster,
 * rows accumulated in increasing row order (csr_matmat). Parallel over
 * clusters after a stable bucketing of rows, so the order is fixed. */
void oracle_aggregate_sums(int64_t n, int64_t d, int64_t k, const int64_t *indptr, const int32_t *indices,
                           const double *data, const int64_t *a, double *sums, int64_t *counts) {
    int64_t *start = (int64_t *)calloc((size_t)(k + 1), sizeof(int64_t));
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) start[a[i] + 1]++;
    for (int64_t j = 0; j < k; ++j) start[j + 1] += start[j];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    for (int64_t j = 0; j < k; ++j) fill[j] = start[j];
    for (int64_t i = 0; i < n; ++i) order[fill[a[i]]++] = i;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t j = 0; j < k; ++j) {
        double *sj = sums + j * d;
        memset(sj, 0, sizeof(double) * (size_t)d);
        for (int64_t q = start[j]; q < start[j + 1]; ++q) {
            int64_t i = order[q];
            for (int64_t t = indptr[i]; t < indptr[i + 1]; ++t) sj[indices[t]] += data[t];
        }
        counts[j] = start[j + 1] - start[j];
    }
    free(start); free(order); free(fill);
}

/* _move_centers, engine.py:142-160 over a list of changed clusters */
static void move_centers(int64_t d, double *centers, const double *sums, const int64_t *counts,
                         double *prev, double *drift, int64_t k, const int64_t *changed, int64_t nchanged) {
    for (int64_t j = 0; j < k; ++j) drift[j] = 1.0;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nchanged; ++q) {
        int64_t j = changed[q];
        double *c = centers + j * d;
        double *pj = prev + j * d;
        memcpy(pj, c, sizeof(double) * (size_t)d);
        if (counts[j] == 0) continue;
        const double *sj = sums + j * d;
        double sq = 0.0;
        for (int64_t t = 0; t < d; ++t) sq = fma(sj[t], sj[t], sq);   /* BLAS ddot tail uses FMA */
        double nrm = sqrt(sq);
        if (nrm < ZERO_SUM_EPS) continue;
        double dt = 0.0;
        for (int64_t t = 0; t < d; ++t) {
            double nv = sj[t] / nrm;
            dt = fma(nv, pj[t], dt);
            c[t] = nv;
        }
        drift[j] = clampc(dt);
    }
}

/* _center_thresholds, engine.py:192-198 */
static void center_thresholds(int64_t d, int64_t k, const double *C, double *cc, double *s_arr) {
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t a = 0; a < k; ++a) {
        for (int64_t j = 0; j < k; ++j) {
            const double *x = C + a * d, *y = C + j * d;
            double s = 0.0;
            for (int64_t t = 0; t < d; ++t) s = fma(x[t], y[t], s);   /* dgemm uses FMA */
            cc[a * k + j] = (a == j) ? -1.0 : half_angle(clampc(s));
        }
        double m = -INFINITY;
        for (int64_t j = 0; j < k; ++j) if (cc[a * k + j] > m) m = cc[a * k + j];
        s_arr[a] = m;
    }
}

static double objective_of(int64_t d, int64_t k, const double *sums, const double *C) {
    /* engine.py:326 einsum("ij,ij->", sums, centers); per-cluster partials
     * summed in cluster order */
    double tot = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        double s = 0.0;
        for (int64_t t = 0; t < d; ++t) s += sums[j * d + t] * C[j * d + t];
        tot += s;
    }
    return tot;
}

/*
 * run, engine.py:201-346.  Validation (ConfigError/InfeasibleError) and
 * seeding are done by the Python wrapper; centers[k*d] comes in seeded
 * (CentroidSet.from_data_rows, engine.py:46-58) and leaves moved.
 * Per-iteration stats are written to it_sims/it_cc/it_reassign/it_obj
 * (capacity max_iter).  Returns the number of iterations; *converged set.
 *
 * hook: optional callback invoked after the drift updates and before the
 * pruned scan (engine.py:304-309); receives the live a/l/u arrays.
 */
typedef void (*oracle_hook_t)(int64_t it, const int64_t *a, const double *l, const double *u_m,
                              const double *u, const double *centers);

int64_t oracle_run(int64_t n, int64_t d, int64_t k, const int64_t *indptr, const int32_t *indices,
                   const double *data, int variant, int64_t max_iter, int hamerly_naive,
                   double *centers, double *sums, int64_t *counts, double *drift, int64_t *a_out,
                   int64_t *it_sims, int64_t *it_cc, int64_t *it_reassign, double *it_obj,
                   int *converged, oracle_hook_t hook, double *it_t_rows, double *it_t_other) {
    const int elkan_family = (variant == V_ELKAN || variant == V_SIMP_ELKAN);
    const int hamerly_family = (variant == V_HAMERLY || variant == V_SIMP_HAMERLY);
    const int needs_cc = (variant == V_ELKAN || variant == V_HAMERLY);
    int64_t *a = a_out;
    int64_t *a_prev = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    double *l = (double *)calloc((size_t)n, sizeof(double));
    double *u_m = elkan_family ? (double *)malloc(sizeof(double) * (size_t)(n * k)) : NULL;
    double *u = hamerly_family ? (double *)malloc(sizeof(double) * (size_t)n) : NULL;
    double *S = (double *)malloc(sizeof(double) * (size_t)(n * k));
    double *prev = (double *)malloc(sizeof(double) * (size_t)(k * d));
    double *cc = needs_cc ? (double *)malloc(sizeof(double) * (size_t)(k * k)) : NULL;
    double *s_arr = needs_cc ? (double *)malloc(sizeof(double) * (size_t)k) : NULL;
    int64_t *all = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    int64_t *changed = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    unsigned char *touched = (unsigned char *)malloc((size_t)k);
    for (int64_t j = 0; j < k; ++j) all[j] = j;
    memcpy(prev, centers, sizeof(double) * (size_t)(k * d));
    for (int64_t j = 0; j < k; ++j) drift[j] = 1.0;
    for (int64_t i = 0; i < n; ++i) a[i] = 0;
    *converged = 0;
    int64_t iters = 0;

    for (int64_t it = 1; it <= max_iter; ++it) {
        int64_t cc_count = 0, sim_count = 0, reassign = 0;
        /* phase clocks (bench.py's reference arm): t_rows = work proportional
         * to the rows (sims, bounds, scans, aggregation, moves), t_other =
         * work on the k x d centers (thresholds, renormalise, objective) */
        double t_rows = 0.0, t_other = 0.0, t0 = omp_get_wtime();
        if (needs_cc) {                                   /* engine.py:242-244 */
            center_thresholds(d, k, centers, cc, s_arr);
            cc_count = k * (k - 1) / 2;
        }
        t_other += omp_get_wtime() - t0;
        t0 = omp_get_wtime();
        if (it == 1) {                                    /* engine.py:249-265 */
            oracle_full_sims(n, d, k, indptr, indices, data, centers, S);
            sim_count = n * k;
            #pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; ++i) {
                const double *y = S + i * k;
                int64_t bj = 0;
                for (int64_t j = 1; j < k; ++j) if (y[j] > y[bj]) bj = j;   /* np.argmax: first max */
                a[i] = bj;
                l[i] = y[bj];
                if (elkan_family) memcpy(u_m + i * k, y, sizeof(double) * (size_t)k);
                else if (hamerly_family) {
                    if (k == 1) u[i] = -1.0;
                    else {
                        double m = -INFINITY;
                        for (int64_t j = 0; j < k; ++j) if (j != bj && y[j] > m) m = y[j];
                        u[i] = m;
                    }
                }
            }
            reassign = n;
            oracle_aggregate_sums(n, d, k, indptr, indices, data, a, sums, counts);
            t_rows += omp_get_wtime() - t0;
            t0 = omp_get_wtime();
            move_centers(d, centers, sums, counts, prev, drift, k, all, k);
            t_other += omp_get_wtime() - t0;
        } else {
            memcpy(a_prev, a, sizeof(int64_t) * (size_t)n);
            if (variant == V_STANDARD) {                  /* engine.py:268-271 */
                oracle_full_sims(n, d, k, indptr, indices, data, centers, S);
                sim_count = n * k;
                #pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < n; ++i) {
                    const double *y = S + i * k;
                    int64_t bj = 0;
                    for (int64_t j = 1; j < k; ++j) if (y[j] > y[bj]) bj = j;
                    a[i] = bj;
                }
            } else {
                const double *p = drift;
                #pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < n; ++i) l[i] = cos_lower(l[i], p[a[i]]);   /* engine.py:274 */
                if (elkan_family) {                       /* engine.py:275-283 */
                    #pragma omp parallel for schedule(static)
                    for (int64_t i = 0; i < n; ++i)
                        for (int64_t j = 0; j < k; ++j) {
                            double v = u_m[i * k + j];
                            u_m[i * k + j] = (v <= p[j]) ? cos_upper(v, p[j]) : 1.0;
                        }
                } else {                                  /* engine.py:284-303 */
                    int64_t owner = 0;                    /* stable argsort: first index of min */
                    for (int64_t j = 1; j < k; ++j) if (p[j] < p[owner]) owner = j;
                    double p_min = p[owner], p_min2 = 1.0;
                    if (k > 1) {
                        int64_t sec = -1;                 /* order[1]: first min among the rest */
                        for (int64_t j = 0; j < k; ++j) {
                            if (j == owner) continue;
                            if (sec < 0 || p[j] < p[sec]) sec = j;
                        }
                        p_min2 = p[sec];
                    }
                    #pragma omp parallel for schedule(static)
                    for (int64_t i = 0; i < n; ++i) {
                        double worst = (a[i] == owner) ? p_min2 : p_min;
                        if (!hamerly_naive)
                            u[i] = (u[i] >= 0.0 && worst >= 0.0) ? hamerly_upper(u[i], worst) : 1.0;
                        else
                            u[i] = cos_upper(u[i], worst);
                    }
                }
                if (hook) hook(it, a, l, u_m, u, centers);  /* engine.py:304-309 */
                if (elkan_family)
                    sim_count = oracle_elkan_scan(n, d, k, indptr, indices, data, centers, a, l, u_m,
                                                  cc, s_arr, variant == V_ELKAN);
                else
                    sim_count = oracle_hamerly_scan(n, d, k, indptr, indices, data, centers, a, l, u,
                                                    s_arr, variant == V_HAMERLY);
            }
            /* engine.py:320-321 -> update_centers(prev_assignments), engine.py:174-188 */
            memset(touched, 0, (size_t)k);
            for (int64_t i = 0; i < n; ++i) {
                if (a[i] == a_prev[i]) continue;
                reassign++;
                int64_t o = a_prev[i], nw = a[i];
                for (int64_t t = indptr[i]; t < indptr[i + 1]; ++t) {
                    sums[o * d + indices[t]] -= data[t];
                    sums[nw * d + indices[t]] += data[t];
                }
                counts[o] -= 1; counts[nw] += 1;
                touched[o] = 1; touched[nw] = 1;
            }
            int64_t nch = 0;
            for (int64_t j = 0; j < k; ++j) if (touched[j]) changed[nch++] = j;
            t_rows += omp_get_wtime() - t0;
            t0 = omp_get_wtime();
            move_centers(d, centers, sums, counts, prev, drift, k, changed, nch);
            t_other += omp_get_wtime() - t0;
        }
        t0 = omp_get_wtime();
        if (it % SCRATCH_INTERVAL == 0)                   /* engine.py:323-324 */
            oracle_aggregate_sums(n, d, k, indptr, indices, data, a, sums, counts);
        t_rows += omp_get_wtime() - t0;
        t0 = omp_get_wtime();
        it_sims[it - 1] = sim_count;
        it_cc[it - 1] = cc_count;
        it_reassign[it - 1] = reassign;
        it_obj[it - 1] = objective_of(d, k, sums, centers);
        t_other += omp_get_wtime() - t0;
        if (it_t_rows) it_t_rows[it - 1] = t_rows;
        if (it_t_other) it_t_other[it - 1] = t_other;
        iters = it;
        int allone = 1;
        for (int64_t j = 0; j < k; ++j) if (drift[j] != 1.0) { allone = 0; break; }
        if (k == 1 || allone || (it >= 2 && reassign == 0)) { *converged = 1; break; }  /* 335-337 */
    }
    oracle_aggregate_sums(n, d, k, indptr, indices, data, a, sums, counts);   /* engine.py:339 */
    free(a_prev); free(l); free(u_m); free(u); free(S); free(prev); free(cc); free(s_arr);
    free(all); free(changed); free(touched);
    return iters;
}

/* assign_full, engine.py:103-120 */
void oracle_assign_full(int64_t n, int64_t d, int64_t k, const int64_t *indptr, const int32_t *indices,
                        const double *data, const double *C, int64_t *a, double *best, double *second) {
    double *S = (double *)malloc(sizeof(double) * (size_t)(n * k));
    oracle_full_sims(n, d, k, indptr, indices, data, C, S);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double *y = S + i * k;
        int64_t bj = 0;
        for (int64_t j = 1; j < k; ++j) if (y[j] > y[bj]) bj = j;
        a[i] = bj;
        best[i] = y[bj];
        if (k == 1) second[i] = -1.0;
        else {
            double m = -INFINITY;
            for (int64_t j = 0; j < k; ++j) if (j != bj && y[j] > m) m = y[j];
            second[i] = m;
        }
    }
    free(S);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* ------------------------------------------------------------ seeding.py */
/* np.dot(x, y) of two contiguous float64 vectors as numpy computes it: its
 * bundled OpenBLAS (scipy-openblas 0.3.30, a third-party dependency the
 * reference does not vendor; pyproject.toml:10-14 pins no version), ddot
 * kernel for the SkylakeX core this container reports: 32-element blocks on
 * 4 x 8 FMA accumulators, folded to 4 x 4, then one optional 16-element block
 * on the 4 x 4 accumulators, the fixed sum ((a0+a1)+a2)+a3, 256->128-bit halves
 * and hadd, then an FMA tail.  Pinned against np.dot in tests/test_oracle.py.
 * y is gathered: y[i] = c[idx[i]] (sparse.py:80-87 dot_sparse_dense). */
static double np_ddot_gather(int64_t m, const double *x, const int32_t *idx, const double *c) {
    const int64_t n32 = m & ~(int64_t)31, n1 = m & ~(int64_t)15;
    double z[32] = {0};
    for (int64_t b = 0; b < n32; b += 32)
        for (int L = 0; L < 32; ++L) z[L] = fma(x[b + L], c[idx[b + L]], z[L]);
    double a[16];
    for (int bb = 0; bb < 4; ++bb)
        for (int l = 0; l < 4; ++l) a[4 * bb + l] = z[8 * bb + l] + z[8 * bb + l + 4];
    if (n1 > n32)
        for (int q = 0; q < 16; ++q) a[q] = fma(x[n32 + q], c[idx[n32 + q]], a[q]);
    double t[4];
    for (int l = 0; l < 4; ++l) t[l] = ((a[l] + a[4 + l]) + a[8 + l]) + a[12 + l];
    double dot = (t[0] + t[2]) + (t[1] + t[3]);
    for (int64_t i = n1; i < m; ++i) dot = fma(c[idx[i]], x[i], dot);
    return dot;
}

/* np.dot(x, y), contiguous (for the order test) */
double oracle_np_ddot(int64_t m, const double *x, const double *y) {
    int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    for (int64_t i = 0; i < m; ++i) idx[i] = (int32_t)i;
    double r = np_ddot_gather(m, x, idx, y);
    free(idx);
    return r;
}

/* |row| = np.sqrt(np.dot(v, v)) for every CSR row (SparseVector.norm,
 * sparse.py:52), in the same np.dot order; lets the reference arm of
 * bench.py normalise generated rows exactly as Dataset.from_rows does
 * without touching the product library. */
void oracle_row_norms(int64_t n, const int64_t *indptr, const double *data, double *out) {
    int64_t maxlen = 0;
    for (int64_t r = 0; r < n; ++r) {
        const int64_t m = indptr[r + 1] - indptr[r];
        if (m > maxlen) maxlen = m;
    }
    #pragma omp parallel
    {
        int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(maxlen > 0 ? maxlen : 1));
        for (int64_t i = 0; i < maxlen; ++i) idx[i] = (int32_t)i;
        #pragma omp for schedule(static)
        for (int64_t r = 0; r < n; ++r) {
            const double *x = data + indptr[r];
            out[r] = sqrt(np_ddot_gather(indptr[r + 1] - indptr[r], x, idx, x));
        }
        free(idx);
    }
}

/* numpy's pairwise_sum (np.add.reduce of a contiguous float64 array) */
static double np_pairwise(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

double oracle_np_sum(const double *a, int64_t n) { return np_pairwise(a, n); }

static inline double rng_random(uint64_t *s) { return (double)(sm64_next(s) >> 11) * 0x1.0p-53; } /* rng.py:46-47 */

/* rng.weighted_index, rng.py:75-92 */
static int64_t weighted_index(uint64_t *s, const double *w, int64_t n, double *cum) {
    double c = 0.0;
    for (int64_t i = 0; i < n; ++i) { c += w[i]; cum[i] = c; }
    const double total = cum[n - 1];
    const double r = rng_random(s) * total;
    int64_t lo = 0, hi = n;          /* searchsorted(cum, r, side="right") */
    while (lo < hi) { int64_t m = (lo + hi) / 2; if (r < cum[m]) hi = m; else lo = m + 1; }
    int64_t idx = lo < n - 1 ? lo : n - 1;
    while (w[idx] == 0.0 && idx + 1 < n) ++idx;
    return idx;
}

/* _uniform_among_unchosen, seeding.py:50-52 */
static int64_t uniform_unchosen(uint64_t *s, int64_t n, const unsigned char *chosen, int64_t nchosen) {
    int64_t m = (int64_t)(sm64_next(s) % (uint64_t)(n - nchosen));
    for (int64_t i = 0; i < n; ++i)
        if (!chosen[i] && m-- == 0) return i;
    return -1;
}

/* _sims_to_center, seeding.py:45-47, c = the picked row densified */
static void sims_to_row(int64_t n, const int64_t *indptr, const int32_t *indices, const double *data,
                        const double *c, double *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        out[i] = np_ddot_gather(indptr[i + 1] - indptr[i], data + indptr[i], indices + indptr[i], c);
}

static void densify(double *c, const int64_t *indptr, const int32_t *indices, const double *data, int64_t r,
                    int set) {
    for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e) c[indices[e]] = set ? data[e] : 0.0;
}

/* init_kmpp, seeding.py:64-89.  trace (optional): (k-1) x n weight vectors. */
int oracle_seed_kmpp(int64_t n, int64_t d, const int64_t *indptr, const int32_t *indices, const double *data,
                     int64_t k, double alpha, uint64_t seed, int64_t *picks, double *trace) {
    if (k < 1 || k > n) return -1;
    uint64_t s = seed;
    double *maxsim = (double *)malloc(sizeof(double) * (size_t)n);
    double *sims = (double *)malloc(sizeof(double) * (size_t)n);
    double *w = (double *)malloc(sizeof(double) * (size_t)n);
    double *cum = (double *)malloc(sizeof(double) * (size_t)n);
    double *c = (double *)calloc((size_t)d, sizeof(double));
    unsigned char *chosen = (unsigned char *)calloc((size_t)n, 1);
    picks[0] = (int64_t)(sm64_next(&s) % (uint64_t)n);
    chosen[picks[0]] = 1;
    densify(c, indptr, indices, data, picks[0], 1);
    sims_to_row(n, indptr, indices, data, c, maxsim);
    for (int64_t t = 1; t < k; ++t) {
        int any = 0;
        for (int64_t i = 0; i < n; ++i) {
            double v = alpha - maxsim[i];
            w[i] = chosen[i] ? 0.0 : (v >= 0.0 ? v : 0.0);   /* np.maximum(alpha - maxsim, 0) */
            any |= w[i] > 0.0;
        }
        if (trace) memcpy(trace + (t - 1) * n, w, sizeof(double) * (size_t)n);
        int64_t pick = any ? weighted_index(&s, w, n, cum) : uniform_unchosen(&s, n, chosen, t);
        picks[t] = pick;
        chosen[pick] = 1;
        densify(c, indptr, indices, data, picks[t - 1], 0);
        densify(c, indptr, indices, data, pick, 1);
        sims_to_row(n, indptr, indices, data, c, sims);
        for (int64_t i = 0; i < n; ++i) maxsim[i] = maxsim[i] >= sims[i] ? maxsim[i] : sims[i];
    }
    free(maxsim); free(sims); free(w); free(cum); free(c); free(chosen);
    return 0;
}

/* bisect.bisect_right */
static int64_t bisect_right(const double *a, int64_t n, double x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t m = (lo + hi) / 2; if (x < a[m]) hi = m; else lo = m + 1; }
    return lo;
}

/* init_afkmc2, seeding.py:92-146 */
int oracle_seed_afkmc2(int64_t n, int64_t d, const int64_t *indptr, const int32_t *indices, const double *data,
                       int64_t k, double alpha, int64_t chain_length, uint64_t seed, int64_t *picks) {
    if (k < 1 || k > n || chain_length < 1) return -1;
    uint64_t s = seed;
    double *sims = (double *)malloc(sizeof(double) * (size_t)n);
    double *dd = (double *)malloc(sizeof(double) * (size_t)n);
    double *q = (double *)malloc(sizeof(double) * (size_t)n);
    double *cumq = (double *)malloc(sizeof(double) * (size_t)n);
    double *dcur = (double *)malloc(sizeof(double) * (size_t)n);
    double *cum = (double *)malloc(sizeof(double) * (size_t)n);
    double *c = (double *)calloc((size_t)d, sizeof(double));
    unsigned char *chosen = (unsigned char *)calloc((size_t)n, 1);
    const int64_t first = (int64_t)(sm64_next(&s) % (uint64_t)n);
    picks[0] = first;
    chosen[first] = 1;
    densify(c, indptr, indices, data, first, 1);
    sims_to_row(n, indptr, indices, data, c, sims);
    for (int64_t i = 0; i < n; ++i) { double v = alpha - sims[i]; dd[i] = v >= 0.0 ? v : 0.0; }
    dd[first] = 0.0;
    const double total_d = np_pairwise(dd, n);
    for (int64_t i = 0; i < n; ++i) q[i] = total_d > 0.0 ? dd[i] / (2.0 * total_d) + 0.5 / (double)n : 1.0 / (double)n;
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) { acc += q[i]; cumq[i] = acc; }
    const double qtotal = cumq[n - 1];
    memcpy(dcur, dd, sizeof(double) * (size_t)n);
    int64_t prev = first;
    for (int64_t t = 1; t < k; ++t) {
        int any = 0;
        for (int64_t i = 0; i < n; ++i) any |= dcur[i] > 0.0;
        int64_t cur;
        if (!any) {
            cur = uniform_unchosen(&s, n, chosen, t);
        } else {
            double r = rng_random(&s) * qtotal;
            cur = bisect_right(cumq, n, r);
            if (cur > n - 1) cur = n - 1;
            for (int64_t step = 1; step < chain_length; ++step) {
                r = rng_random(&s) * qtotal;
                int64_t cand = bisect_right(cumq, n, r);
                if (cand > n - 1) cand = n - 1;
                const double num = dcur[cand] * q[cur];
                const double den = dcur[cur] * q[cand];
                if (den <= 0.0) cur = cand;
                else if (rng_random(&s) * den < num) cur = cand;
            }
            if (dcur[cur] <= 0.0) cur = weighted_index(&s, dcur, n, cum);
        }
        picks[t] = cur;
        chosen[cur] = 1;
        densify(c, indptr, indices, data, prev, 0);
        densify(c, indptr, indices, data, cur, 1);
        prev = cur;
        sims_to_row(n, indptr, indices, data, c, sims);
        for (int64_t i = 0; i < n; ++i) {
            double v = alpha - sims[i];
            v = v >= 0.0 ? v : 0.0;
            dcur[i] = dcur[i] <= v ? dcur[i] : v;   /* np.minimum */
        }
        dcur[cur] = 0.0;
    }
    free(sims); free(dd); free(q); free(cumq); free(dcur); free(cum); free(c); free(chosen);
    return 0;
}
