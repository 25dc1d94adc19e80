// spkm.cu -- sm_100a kernels for the accelerated spherical k-means loop.
//
// Reference path (arXiv 2107.04074 package `spkmeans`, engine.py:201-346):
// one iteration = center thresholds -> drift update of the bounds ->
// pruned scan -> incremental center update -> renormalise -> objective.
// This file implements each phase as data-parallel CUDA over the points,
// behind the C ABI of include/spkm.h.
//
// Numerics:
//  * Similarities are float32: s~(i,j) = FMA chain over row i's nnz in CSR
//    order, starting at 0 (the canonical order).  Every kernel that computes
//    a similarity uses exactly this chain, so the full pass, the Hamerly
//    rescan, the tighten step and the Elkan pair scan agree bit-for-bit and
//    the pruned variants reproduce Lloyd exactly.
//  * Bounds are kept on the TRUE cosine <x_i, c_j> (float64 rows/centers),
//    updated in float64 and stored as float32 rounded outward.  The float32
//    similarity error is |s~ - s| <= eps_i = (m_i + 6) * 6.1e-8 (m_i = row
//    nnz; FMA-chain error bound gamma_m plus the float32 rounding of x and c).
//    A center j is pruned only if s~(i,j) <= s~(i,a) is PROVEN, i.e.
//    u + 2 eps <= l (stored bounds) or u + eps <= s~(i,a) (after tightening).
//  * Ties: "the incumbent wins exact ties, otherwise the lowest index" in
//    every variant from iteration 2; iteration 1 and
//    predict use the lowest index (numpy argmax).
//  * Center sums are exact fixed point (int64, value * 2^scale_bits), so
//    incremental == scratch and sums are independent of atomic order and of
//    the GPU count.  Renormalisation, drift and objective are float64 with
//    fixed-order reductions.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <stdint.h>
#include <stdio.h>
#include <math.h>
#include <stdlib.h>
#include <limits.h>

#include <functional>
#include <utility>
#include <vector>

#include "../../include/spkm.h"

#define FULL 0xffffffffu

// Debug build (-DSPKM_CHECKS=1, libspkm_check.so, tests/test_gpu_checks.py):
// device-side bounds checks on the indices the kernels trust, trapping with a
// message.  The pool has no compute-sanitizer; these checks
// and the bit-exact comparisons stand in for it.
#ifndef SPKM_CHECKS
#define SPKM_CHECKS 0
#endif
#if SPKM_CHECKS
#define DCHECK(cond)                                                                            \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("SPKM_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__,    \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                                   \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define DCHECK(cond) do { } while (0)
#endif

namespace {

// eps_i = (nnz_i + 6) * 6.1e-8 (>= 2^-24 * 1.02 per term) is computed on the
// host into spkm_csr.row_eps (rounded up) and read by every prune test.
constexpr double kSlack = 1e-12;            // float64 formula error of a bound update
constexpr double kCcSlack = 1e-9;           // float64 Gram error (d * 2^-53 << 1e-9 for d <= 1e6)
constexpr double kSqrt2 = 1.4142135623730951;
constexpr double kZeroSumEps = 1e-12;       // engine.py:27
constexpr int kCenterChunk = 4096;          // d-chunk of the center kernels
constexpr int kFuseFlag = 6;                // hstat slot: fused Hamerly tighten + rescan next iteration
// hstat slot: Elkan family, every row takes the full pass next iteration and the bound pass is skipped.  Set
// by k_finalize while an iteration still moves at least 1/256 of the rows: at C4 those are the iterations in
// which the bound pass sends all 4M rows to the heavy pass anyway (profiles/r02_c4_iteration_stats.txt), after
// streaming 32 GB of bounds to find that out.  A performance switch only: the full pass is exact for any row.
constexpr int kAllHeavyFlag = 7;

thread_local char g_err[512] = {0};

int fail(const char *what, cudaError_t e) {
    snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
    return (int)e ? (int)e : 1;
}
int fail_msg(const char *msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}
// Programmatic dependent launch: the loop's kernels are launched with
// programmatic stream serialization, so kernel N+1's launch and CTA
// rasterisation overlap kernel N's tail.  Every such kernel first waits for
// its predecessor grid (griddepcontrol.wait: complete, memory visible), then
// lets its own successor launch.  Outside PDL launches both are no-ops.
#define PDL_ENTRY() asm volatile("griddepcontrol.wait;" ::: "memory")
// a CTA whose main work is done lets the next kernel start launching (its
// CTAs still wait in PDL_ENTRY for this grid's completion and memory flush)
#define PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")

bool pdl_enabled() {
    static int on = -1;   // SPKM_PDL=0 turns programmatic launches off (A/B measurements)
    if (on < 0) {
        const char *e = getenv("SPKM_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}
template <typename... KArgs, typename... Args>
void pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    (void)cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);   // errors surface via CHECK_LAUNCH
}

#define CHECK_LAUNCH(name)                                          \
    do {                                                            \
        cudaError_t _e = cudaGetLastError();                        \
        if (_e != cudaSuccess) return fail(name, _e);               \
    } while (0)

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

// ------------------------------------------------------------------ geometry
// geometry.py:20-68, evaluated with explicit round-to-nearest ops (no FMA
// contraction) so the device values equal the reference's numpy values.
__device__ __forceinline__ double d_clamp(double t) { return t < -1.0 ? -1.0 : (t > 1.0 ? 1.0 : t); }
__device__ __forceinline__ double d_sin(double t) {
    double v = __dsub_rn(1.0, __dmul_rn(t, t));
    return sqrt(v > 0.0 ? v : 0.0);
}
__device__ __forceinline__ double d_cos_lower(double a, double b) {
    return d_clamp(__dsub_rn(__dmul_rn(a, b), __dmul_rn(d_sin(a), d_sin(b))));
}
__device__ __forceinline__ double d_cos_upper(double a, double b) {
    return d_clamp(__dadd_rn(__dmul_rn(a, b), __dmul_rn(d_sin(a), d_sin(b))));
}
__device__ __forceinline__ double d_hamerly_upper(double u, double p) {
    return d_clamp(__dadd_rn(u, __dmul_rn(d_sin(u), d_sin(p))));
}
__device__ __forceinline__ double d_half_angle(double s) {
    double v = __ddiv_rn(__dadd_rn(s, 1.0), 2.0);
    return sqrt(v > 0.0 ? v : 0.0);
}
// Lower-bound drift update with the theta_l + theta_p > pi guard
// (SURVEY.md §2.4 item 6): the triangle formula is only valid while
// l >= -p; past that the new cosine can be -1.
__device__ __forceinline__ double d_lower_update(double l, double p) {
    return (l < -p) ? -1.0 : d_cos_lower(l, p);
}
__device__ __forceinline__ float store_lower(double v) {
    v -= kSlack;
    if (v < -1.0) v = -1.0;
    return __double2float_rd(v);
}
__device__ __forceinline__ float store_upper(double v) {
    v += kSlack;
    if (v > 1.0) v = 1.0;
    return __double2float_ru(v);
}

// ------------------------------------------------------- canonical similarity
// s~(i,j) = float32 FMA chain over row i's nnz in CSR order, starting at 0:
//   acc = fma(val[t], ct[idx[t] * kp + j], acc)   for t = indptr[i] .. indptr[i+1]-1
// k_row_pass (per column), warp_dots (per candidate) all evaluate exactly
// this chain; only the order in which the center values are FETCHED differs.

// ------------------------------------------------------------- top-2 helpers
// Priority: larger value; on exact ties the incumbent `inc`, then lower index.
__device__ __forceinline__ bool better(float v1, int j1, float v2, int j2, int inc) {
    if (v1 != v2) return v1 > v2;
    const int p1 = (j1 == inc) ? -1 : j1;
    const int p2 = (j2 == inc) ? -1 : j2;
    return p1 < p2;
}
struct Top2 {
    float b;
    int bj;
    float s;
};
__device__ __forceinline__ void top2_push(Top2 &t, float v, int j, int inc) {
    if (better(v, j, t.b, t.bj, inc)) {
        t.s = fmaxf(t.s, t.b);
        t.b = v;
        t.bj = j;
    } else {
        t.s = fmaxf(t.s, v);
    }
}
__device__ __forceinline__ void top2_merge(Top2 &t, const Top2 &o, int inc) {
    if (better(o.b, o.bj, t.b, t.bj, inc)) {
        t.s = fmaxf(o.s, t.b);
        t.b = o.b;
        t.bj = o.bj;
    } else {
        t.s = fmaxf(t.s, o.b);
    }
}
__device__ __forceinline__ Top2 top2_shfl_down(const Top2 &t, int o) {
    Top2 r;
    r.b = __shfl_down_sync(FULL, t.b, o);
    r.bj = __shfl_down_sync(FULL, t.bj, o);
    r.s = __shfl_down_sync(FULL, t.s, o);
    return r;
}

// Warp-aggregated append of (pred ? value : nothing) to list[ctr++].
__device__ __forceinline__ void warp_append(bool pred, int32_t v0, int32_t *list0, int32_t v1, int32_t *list1,
                                            long long *ctr) {
    const unsigned m = __ballot_sync(FULL, pred);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    long long base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd((unsigned long long *)ctr, (unsigned long long)__popc(m));
    base = __shfl_sync(FULL, base, __ffs(m) - 1);
    if (pred) {
        const int r = __popc(m & ((1u << lane) - 1u));
        list0[base + r] = v0;
        if (list1) list1[base + r] = v1;
    }
}

// Block-level counter accumulation: warps add into shared memory and each
// CTA adds its totals to the 8 global counters once at the end (thousands of
// warps adding to one global address serialise at its L2 slice).
__device__ __forceinline__ void ctr_init(unsigned long long *s) {
    if (threadIdx.x < 8) s[threadIdx.x] = 0ull;
    __syncthreads();
}
__device__ __forceinline__ void ctr_add(unsigned long long *s, int slot, long long v) {
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(FULL, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(s + slot, (unsigned long long)v);
}
__device__ __forceinline__ void ctr_flush(const unsigned long long *s, long long *ctr) {
    __syncthreads();
    if (threadIdx.x < 8 && s[threadIdx.x]) atomicAdd((unsigned long long *)(ctr + threadIdx.x), s[threadIdx.x]);
}

// ------------------------------------------------------------ full row pass
// A row's (term, value) pairs are staged per 32-nnz chunk in shared memory as
// int2 {idx, value bits}, kIvStride pairs per row group: the gather loop reads
// two nnz per 16-byte broadcast load, and the 16-byte pad puts the groups of
// one warp in distinct banks (one wavefront for up to 8 groups).
constexpr int kIvStride = 34;
template <int UB>
__device__ __forceinline__ void load_iv(const int2 *p, int (&iv)[UB], float (&vv)[UB]) {
    if constexpr (UB % 2 == 0) {
#pragma unroll
        for (int b = 0; b < UB; b += 2) {
            const int4 t = *reinterpret_cast<const int4 *>(p + b);
            iv[b] = t.x;
            vv[b] = __int_as_float(t.y);
            iv[b + 1] = t.z;
            vv[b + 1] = __int_as_float(t.w);
        }
    } else {
#pragma unroll
        for (int b = 0; b < UB; ++b) {
            const int2 t = p[b];
            iv[b] = t.x;
            vv[b] = __int_as_float(t.y);
        }
    }
}

// L2 eviction priority of the center-row gathers.  Term ids are renumbered
// by document frequency, so the Zipf head is the block of term rows
// [0, hot) of ct32.  Those rows are gathered with evict_last and every other
// row with evict_first: the flood of once-per-pass topic-term rows (C4: a
// 4 GB table, ~70% of the gathers) then streams through L2 without evicting
// the head, which serves most of the remaining gathers from L2.  A hint
// only: results do not depend on it.  hot is chosen on the host (the head
// rows that fit half of L2; SPKM_HOT_MB).
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float4 ldg_hint(const float4 *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ldg_hint(const uint2 *p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float4 half4_to_float4(uint2 h) {
    const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&h.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&h.y));
    return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float ldg_hint(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// MODE_ELKAN_FULL: the Elkan family's heavy survivors (spkm_elkan_heavy) -- every similarity of the row,
// reassignment by the scan's rule (incumbent wins ties, else the lowest index), l and every u(i, j) exact
enum { MODE_RESCAN = 4, MODE_PREDICT = 5, MODE_INIT_YY = SPKM_MODE_INIT_YINYANG, MODE_ELKAN_FULL = 7 };

struct RowPassArgs {
    const int64_t *indptr;
    const int32_t *indices;
    const float *values;
    const float *reps;
    int64_t n;
    const float *ct;
    int64_t kp;
    int k, tpr, rpw, mode;
    const int32_t *rowlist;      // null = rows [0, n)
    const long long *rowcount;   // device count of rowlist
    int32_t *a;
    float *l;
    float *u;
    int64_t ku;
    int32_t *mv_i, *mv_old;
    long long *ctr;
    double *best, *second;       // predict outputs
    const long long *ctl;        // [it, done]: done -> this launch is a no-op
    // Hamerly rescan fused with the tighten (when *fuse != 0): rows come from
    // the bound survivors, and each row's s~(i, a) from the full pass decides
    // the tighten test first (k_hamerly_tighten is then a no-op)
    const double *fuse;
    const int32_t *rowlist_fused;
    const long long *rowcount_fused;
    const float *s_arr;
    int use_s;
    int64_t hot;                 // term rows [0, hot) are gathered with evict_last, the rest evict_first
    const __half *ct16;          // fp16 copy of ct for the screening pass (HALF instantiations)
    int64_t d;                   // term rows of ct (bounds checks of the debug build)
    const int64_t *ci_desc;      // sparse center index (SPARSE instantiations): per term row
    const int2 *ci_pairs;        //   (offset << 12 | count) and the (j, value bits) pairs
    const double *allheavy;      // MODE_ELKAN_FULL: != 0 -> every row [0, n), the bound pass was skipped
};

// Sparse gather (k > 256 with a center index): the row's accumulators live in
// shared memory (kp floats per warp); term by term in CSR order, a dense
// term row (more than dense_thr centers nonzero) is read from ct32 by the
// lanes that own its columns (as the register gather), a sparse one as its
// (j, value) pairs, one pair per lane.  Zeros contribute nothing to the FMA
// chain, so every s~(i, j) is the canonical chain (ties and all).  The
// epilogue streams each lane's CH columns from shared memory, one float4 at a
// time (holding them in CH registers spilled at the pass's 64 registers).
#ifndef SPKM_EK_HEAVY_PCT_DEFAULT
#define SPKM_EK_HEAVY_PCT_DEFAULT 0.5    // C4: 0.1 / 0.3 / 0.5 / 1 / 5 / 25 % -> 17.6 / 17.9 / 18.0 / 17.7 / 17.0 / 14.7 it/s (off: 13.2)
#endif
#ifndef SPKM_SP_PREFETCH
#define SPKM_SP_PREFETCH 0        // per-term bulk L2 prefetch: measured slower at C4 (2267 vs 2184 ms per fit)
#endif
// One row per warp (k > 256): lanes 0..tpr-1 own the columns (own), every
// lane loads nnz and pairs; the row's start and length come from lane 0.
template <int CH>
__device__ __forceinline__ void row_gather_sparse(const RowPassArgs &A, float *sacc, int64_t s_own,
                                                  int len_own, bool own, int lane, int j0, uint64_t pol_hot,
                                                  uint64_t pol_cold) {
    const int jstr = 4 * A.tpr;
    const int64_t s = __shfl_sync(FULL, s_own, 0);
    const int maxlen = __shfl_sync(FULL, len_own, 0);
    if (own) {
#pragma unroll
        for (int r = 0; r < CH / 4; ++r)
            *reinterpret_cast<float4 *>(sacc + j0 + r * jstr) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();
    bool last_sparse = true;
    for (int c0 = 0; c0 < maxlen; c0 += 32) {
        const int cnt = min(32, maxlen - c0);
        int id = 0;
        float v = 0.f;
        long long dsc = 0;
        if (lane < cnt) {
            id = __ldg(A.indices + s + c0 + lane);
            v = __ldg(A.values + s + c0 + lane);
            DCHECK((uint64_t)id < (uint64_t)A.d);
            dsc = __ldg(reinterpret_cast<const long long *>(A.ci_desc) + id);
#if SPKM_SP_PREFETCH
            // one bulk L2 prefetch per term of the chunk (its pair list or its
            // dense row): the per-term loads below then find them in L2
            const int n = (int)(dsc & 0xFFF);
            uintptr_t a0;
            uint32_t bytes;
            if (n == 0xFFF) {
                a0 = reinterpret_cast<uintptr_t>(A.ct + (int64_t)id * A.kp);
                bytes = (uint32_t)(A.kp * 4);
            } else {
                const uintptr_t b = reinterpret_cast<uintptr_t>(A.ci_pairs + (dsc >> 12));
                a0 = b & ~(uintptr_t)15;
                bytes = (uint32_t)(((b + (uintptr_t)n * 8 - a0) + 15) & ~(uintptr_t)15);
            }
            if (n != 0 && id >= A.hot)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(bytes) : "memory");
#endif
        }
        for (int t = 0; t < cnt; ++t) {
            const int tid = __shfl_sync(FULL, id, t);
            const float tv = __shfl_sync(FULL, v, t);
            const long long td = __shfl_sync(FULL, dsc, t);
            const int n = (int)(td & 0xFFF);
            if (n == 0xFFF) {   // dense term row: the owner lanes, float4 per column group (n, last_sparse: warp-uniform)
                if (last_sparse) __syncwarp();
                last_sparse = false;
                if (!own) continue;
                const float4 *p = reinterpret_cast<const float4 *>(A.ct + (int64_t)tid * A.kp + j0);
                const uint64_t pol = tid < A.hot ? pol_hot : pol_cold;
                // in halves of CH/8 float4: half the registers live (the kernel runs at 64)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float4 x[CH / 8];
#pragma unroll
                    for (int r = 0; r < CH / 8; ++r) x[r] = ldg_hint(p + (h * (CH / 8) + r) * A.tpr, pol);
#pragma unroll
                    for (int r = 0; r < CH / 8; ++r) {
                        float4 *ap = reinterpret_cast<float4 *>(sacc + j0 + (h * (CH / 8) + r) * jstr);
                        float4 a = *ap;
                        a.x = __fmaf_rn(tv, x[r].x, a.x);
                        a.y = __fmaf_rn(tv, x[r].y, a.y);
                        a.z = __fmaf_rn(tv, x[r].z, a.z);
                        a.w = __fmaf_rn(tv, x[r].w, a.w);
                        *ap = a;
                    }
                }
            } else if (n > 0) {   // sparse term row: its pairs, one per lane (distinct j within a row)
                const int2 *pp = A.ci_pairs + (td >> 12);
                int2 e[4];
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    if (lane + 32 * m < n) {
                        e[m] = __ldg(pp + lane + 32 * m);
                        DCHECK((uint32_t)e[m].x < (uint32_t)A.k);
                    }
                __syncwarp();   // earlier terms' updates (any lane) are visible
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    if (lane + 32 * m < n) sacc[e[m].x] = __fmaf_rn(tv, __int_as_float(e[m].y), sacc[e[m].x]);
                for (int p2 = lane + 128; p2 < n; p2 += 32) {   // rows beyond 128 pairs
                    const int2 f = __ldg(pp + p2);
                    sacc[f.x] = __fmaf_rn(tv, __int_as_float(f.y), sacc[f.x]);
                }
                last_sparse = true;
            }
        }
    }
    __syncwarp();   // the row's similarities stay in sacc: the epilogue streams them from there (acc4)
}

// One row group's gather (the canonical chain per column, CSR order): lane q
// accumulates its CH columns j0 + r * jstr + c.  H: the fp16 table (4 halves
// = 8 bytes per lane and nnz and float4 group) -- the screening values s'.
#ifndef SPKM_HINT_MINCH
#define SPKM_HINT_MINCH 16        // L2 eviction hints only where the table outgrows L2 (k > 256)
#endif
template <bool HINT>
__device__ __forceinline__ float4 ldg4(const float4 *p, uint64_t pol) {
    if constexpr (HINT) return ldg_hint(p, pol);
    else return __ldg(p);
}
template <int CH, int UB, bool H>
__device__ __forceinline__ void row_gather(float (&acc)[CH], const RowPassArgs &A, int2 *my_iv, int64_t s, int len,
                                           int maxlen, int q, int j0, uint64_t pol_hot, uint64_t pol_cold) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = 0.f;
    const float *ctj = A.ct + j0;
    const __half *chj = A.ct16 + j0;
    // Rows are staged 32 nnz at a time in shared memory (coalesced loads by
    // the row's lanes); the term-major center rows are then gathered UB
    // nnz at a time so UB * CH/4 independent loads are in flight.
    for (int c0 = 0; c0 < maxlen; c0 += 32) {
        const int cnt = max(0, min(32, len - c0));
        for (int q2 = q; q2 < cnt; q2 += A.tpr) {
            my_iv[q2] = make_int2(__ldg(A.indices + s + c0 + q2), __float_as_int(__ldg(A.values + s + c0 + q2)));
            DCHECK((uint64_t)my_iv[q2].x < (uint64_t)A.d);
        }
        __syncwarp();
        int u = 0;
        for (; u + UB <= cnt; u += UB) {
            float vv[UB];
            int iv[UB];
            load_iv<UB>(my_iv + u, iv, vv);
            if constexpr (H) {
                uint2 hv[UB][CH / 4];
#pragma unroll
                for (int b = 0; b < UB; ++b) {
                    const uint2 *p = reinterpret_cast<const uint2 *>(chj + (int64_t)iv[b] * A.kp);
                    const uint64_t pol = iv[b] < A.hot ? pol_hot : pol_cold;
#pragma unroll
                    for (int r = 0; r < CH / 4; ++r) hv[b][r] = ldg_hint(p + r * A.tpr, pol);
                }
#pragma unroll
                for (int b = 0; b < UB; ++b)
#pragma unroll
                    for (int r = 0; r < CH / 4; ++r) {
                        const float4 cv = half4_to_float4(hv[b][r]);
                        acc[4 * r + 0] = __fmaf_rn(vv[b], cv.x, acc[4 * r + 0]);
                        acc[4 * r + 1] = __fmaf_rn(vv[b], cv.y, acc[4 * r + 1]);
                        acc[4 * r + 2] = __fmaf_rn(vv[b], cv.z, acc[4 * r + 2]);
                        acc[4 * r + 3] = __fmaf_rn(vv[b], cv.w, acc[4 * r + 3]);
                    }
            } else {
                float4 cv[UB][CH / 4];
#pragma unroll
                for (int b = 0; b < UB; ++b) {
                    const float4 *p = reinterpret_cast<const float4 *>(ctj + (int64_t)iv[b] * A.kp);
                    const uint64_t pol = iv[b] < A.hot ? pol_hot : pol_cold;
#pragma unroll
                    for (int r = 0; r < CH / 4; ++r) cv[b][r] = ldg4<(CH >= SPKM_HINT_MINCH)>(p + r * A.tpr, pol);
                }
#pragma unroll
                for (int b = 0; b < UB; ++b)
#pragma unroll
                    for (int r = 0; r < CH / 4; ++r) {
                        acc[4 * r + 0] = __fmaf_rn(vv[b], cv[b][r].x, acc[4 * r + 0]);
                        acc[4 * r + 1] = __fmaf_rn(vv[b], cv[b][r].y, acc[4 * r + 1]);
                        acc[4 * r + 2] = __fmaf_rn(vv[b], cv[b][r].z, acc[4 * r + 2]);
                        acc[4 * r + 3] = __fmaf_rn(vv[b], cv[b][r].w, acc[4 * r + 3]);
                    }
            }
        }
        for (; u < cnt; ++u) {
            const int2 t = my_iv[u];
            const float v0 = __int_as_float(t.y);
            const uint64_t pol = t.x < A.hot ? pol_hot : pol_cold;
#pragma unroll
            for (int r = 0; r < CH / 4; ++r) {
                float4 cc4;
                if constexpr (H)
                    cc4 = half4_to_float4(ldg_hint(reinterpret_cast<const uint2 *>(chj + (int64_t)t.x * A.kp) + r * A.tpr, pol));
                else
                    cc4 = ldg4<(CH >= SPKM_HINT_MINCH)>(reinterpret_cast<const float4 *>(ctj + (int64_t)t.x * A.kp) + r * A.tpr, pol);
                acc[4 * r + 0] = __fmaf_rn(v0, cc4.x, acc[4 * r + 0]);
                acc[4 * r + 1] = __fmaf_rn(v0, cc4.y, acc[4 * r + 1]);
                acc[4 * r + 2] = __fmaf_rn(v0, cc4.z, acc[4 * r + 2]);
                acc[4 * r + 3] = __fmaf_rn(v0, cc4.w, acc[4 * r + 3]);
            }
        }
        __syncwarp();
    }
}

// fp16 screening (k_row_pass<.., HALF>): candidates per row whose exact value
// is re-checked on ct32; more in a row -> the warp re-gathers in fp32.
constexpr int kCand = 8;
// |s' - s~| <= E(m) for a row of m nnz: fp16 rounding of ct32 (2^-11
// relative, 2^-25 absolute below the fp16 normal range: 2^-11 |x||c| +
// 2^-25 |x|_1 <= 4.883e-4 + 2.98e-8 sqrt(m) for unit x, c) plus the two
// float32 FMA chains (2 gamma_m <= 1.2e-7 m), with margin.
__device__ __forceinline__ double screen_err(int m) { return 5.0e-4 + 1.3e-7 * m + 3.0e-8 * sqrt((double)m); }

// Thread = (row, CH centers in float4 groups tpr apart).  tpr threads cover
// one row's kp columns, rpw rows share a warp.  Per nnz: one broadcast (idx, val) load and
// CH/4 float4 loads of the term-major center row; CH independent FMA chains.
// CH <= 8: capped at 64 registers (4 CTAs of 256 per SM); CH >= 16 (k > 256):
// uncapped, the CH accumulators and loads in flight need the registers.
#ifndef SPKM_RP_SP_MINB
#define SPKM_RP_SP_MINB 4         // sparse gather: 4 CTAs/SM (C4 rescan 2282 -> 2183 ms per fit vs 3 CTAs)
#endif
#ifndef SPKM_RP_MINB
#define SPKM_RP_MINB 2        // k > 256: 128 registers, 2 CTAs per SM with UB 3 (C4 rescan 3336 -> 3281 ms per fit)
#endif
// GV: the gather variant -- 0 float32 table, 1 fp16 screening (SPKM_CT16=1),
// 2 sparse center index (k > 256)
template <int CH, int NT, int GV>
__global__ void __launch_bounds__(NT, CH <= 8 ? 1024 / NT : GV == 2 ? SPKM_RP_SP_MINB : CH == 32 ? SPKM_RP_MINB : 1)
    k_row_pass(RowPassArgs A) {
    constexpr bool HALF = GV == 1, SPARSE = GV == 2;
    PDL_ENTRY();
    // nnz per gather batch: keep ~8 float4 loads in flight per lane
#ifndef SPKM_UB_WIDE
#define SPKM_UB_WIDE 3
#endif
    // CH >= 16 (k > 256, one row per warp, one CTA per SM by registers): the
    // gathers are latency-bound, so SPKM_UB_WIDE x 8 float4 loads in flight
    // (C4: 1, 2, 3, 4 -> 8.50, 9.40, 9.70, 9.84 it/s; profiles/r02_ab_notes.txt)
    constexpr int UB = CH == 4 ? 8 : CH == 8 ? 4 : CH == 16 ? 8 : SPKM_UB_WIDE;
#ifndef SPKM_UB_HALF_MUL
#define SPKM_UB_HALF_MUL 2
#endif
    // fp16 gathers: the same registers hold twice the loads (8-byte vs 16-byte)
    constexpr int UBH = HALF ? SPKM_UB_HALF_MUL * UB : UB;
    if (A.ctl[1]) return;   // converged: later enqueued iterations are no-ops
    extern __shared__ __align__(16) int2 s_iv[];   // per row group: kIvStride staged (id, value) pairs
    const int wpb = blockDim.x >> 5;
    __shared__ unsigned long long s_ctr[8];
    __shared__ int s_cj[HALF ? NT / 32 : 1][8][kCand];     // fp16 screening: candidate columns per row group
    __shared__ float s_cv[HALF ? NT / 32 : 1][8][kCand];   // and their exact values
    __shared__ float s_cs[HALF ? NT / 32 : 1][1][HALF ? kCand * 32 : 1];   // recheck staging (HALF: k > 128, one row per warp)
    ctr_init(s_ctr);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int g = lane / A.tpr, q = lane - g * A.tpr;
    const bool lane_on = g < A.rpw;
    const bool fused = A.mode == MODE_RESCAN && A.fuse && *A.fuse != 0.0;
    const bool allrows = A.mode == MODE_ELKAN_FULL && A.allheavy && *A.allheavy != 0.0;
    const int32_t *rowlist = allrows ? nullptr : fused ? A.rowlist_fused : A.rowlist;
    const int64_t nrows = rowlist ? (fused ? *A.rowcount_fused : *A.rowcount) : A.n;
    const int64_t nslots = (nrows + A.rpw - 1) / A.rpw;
    const int o0 = A.tpr > 1 ? (1 << (31 - __clz(A.tpr - 1))) : 0;
    int2 *my_iv = s_iv + (wib * A.rpw + (lane_on ? g : 0)) * kIvStride;   // rpw row groups per warp
    for (int64_t w = (int64_t)blockIdx.x * wpb + wib; w < nslots; w += (int64_t)gridDim.x * wpb) {
        const int64_t slot = w * A.rpw + g;
        const bool valid = lane_on && slot < nrows;
        const int64_t row = valid ? (rowlist ? (int64_t)rowlist[slot] : slot) : 0;
        const int64_t s = valid ? A.indptr[row] : 0;
        const int64_t e = valid ? A.indptr[row + 1] : 0;
        const int len = (int)(e - s);
        const int maxlen = (int)__reduce_max_sync(FULL, (unsigned)len);
        // lane q holds centers j0 + r * jstr + c (r < CH/4, c < 4): for every r
        // the row's lanes read one contiguous 16 * tpr-byte span of the
        // term-major center row (one L1 wavefront per 128-byte line)
        const int j0 = q * 4;
        const int jstr = 4 * A.tpr;
        float acc[CH];
        const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
        float *sacc = nullptr;   // SPARSE: this warp's kp accumulators
        if constexpr (SPARSE) {
            sacc = reinterpret_cast<float *>(s_iv + 8 * A.rpw * kIvStride) + wib * A.kp;
            row_gather_sparse<CH>(A, sacc, s, len, lane_on, lane, j0, pol_hot, pol_cold);
        } else {
            row_gather<CH, UBH, HALF>(acc, A, my_iv, s, len, maxlen, q, j0, pol_hot, pol_cold);
        }
        // column group r of this lane: centers j0 + r * jstr .. + 3
        auto acc4 = [&](int r) -> float4 {
            if constexpr (SPARSE) return *reinterpret_cast<const float4 *>(sacc + j0 + r * jstr);
            else return make_float4(acc[4 * r], acc[4 * r + 1], acc[4 * r + 2], acc[4 * r + 3]);
        };
        const bool incumbent_mode = (A.mode == SPKM_MODE_LLOYD || A.mode == MODE_RESCAN || A.mode == MODE_ELKAN_FULL);
        const int inc = (valid && incumbent_mode) ? A.a[row] : -1;
        DCHECK(!valid || (row >= 0 && row < A.n && inc < A.k));
        if constexpr (HALF) {
            // acc holds the fp16-screened s'.  Candidates: s' >= max s' - 2E (the
            // only centers that can be the best or tie it: any other j has
            // s~_j <= s'_j + E < max - E <= s~ of the argmax of s') plus the
            // incumbent.  Their exact canonical s~ comes from one chain each on
            // ct32; every other acc becomes s' + E rounded up, an upper bound on
            // its s~ strictly below the best -- so a, l, the tie rule and the
            // tighten test are exact, and the second / u(i, j) / group bounds
            // stay valid upper bounds.
            float mx = -INFINITY;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int j = j0 + (c >> 2) * jstr + (c & 3);
                if (j < A.k) mx = fmaxf(mx, acc[c]);
            }
            for (int o = o0; o; o >>= 1) {
                const float ot = __shfl_down_sync(FULL, mx, o);
                if (q < o && q + o < A.tpr) mx = fmaxf(mx, ot);
            }
            mx = __shfl_sync(FULL, mx, lane - q);
            const double E = screen_err(len);
            const float thr = __double2float_rd((double)mx - 2.0 * E);
            const float Ef = __double2float_ru(E);
            int cnt = 0;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int j = j0 + (c >> 2) * jstr + (c & 3);
                cnt += (valid && j < A.k && (acc[c] >= thr || j == inc)) ? 1 : 0;
            }
            int x = cnt;
            for (int o = 1; o < A.tpr; o <<= 1) {
                const int v = __shfl_up_sync(FULL, x, o);
                if (q >= o) x += v;
            }
            const int tot = __shfl_sync(FULL, x, (lane - q + A.tpr - 1) & 31);
            if (__any_sync(FULL, valid && tot > kCand)) {
                // too many near-ties in some row of the warp: exact float32 gather
                row_gather<CH, UB, false>(acc, A, my_iv, s, len, maxlen, q, j0, pol_hot, pol_cold);
            } else {
                int *cj = s_cj[wib][lane_on ? g : 0];
                float *cvv = s_cv[wib][lane_on ? g : 0];
                int pos = x - cnt;
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    const int j = j0 + (c >> 2) * jstr + (c & 3);
                    if (valid && j < A.k && (acc[c] >= thr || j == inc)) cj[pos++] = j;
                }
                __syncwarp();
                // exact canonical chains of the candidates, 32 nnz at a time: the
                // row's lanes fetch every (candidate, nnz) center value of the
                // chunk at once (one round trip), then lane c < tot runs
                // candidate c's FMA chain from shared memory in CSR order
                float e = 0.f;
                float *stage = s_cs[wib][lane_on ? g : 0];
                const int mt = (int)__reduce_max_sync(FULL, (unsigned)(valid ? len : 0));
                for (int c0 = 0; c0 < mt; c0 += 32) {
                    const int cntc = valid ? max(0, min(32, len - c0)) : 0;
                    for (int q2 = q; q2 < cntc; q2 += A.tpr) {
                        const int id = __ldg(A.indices + s + c0 + q2);
                        const float *rowp = A.ct + (int64_t)id * A.kp;
                        for (int p = 0; p < tot; ++p) stage[p * 32 + q2] = __ldg(rowp + cj[p]);
                    }
                    __syncwarp();
                    if (valid && q < tot)
                        for (int t = 0; t < cntc; ++t) e = __fmaf_rn(__ldg(A.values + s + c0 + t), stage[q * 32 + t], e);
                    __syncwarp();
                }
                if (valid && q < tot) cvv[q] = e;
                __syncwarp();
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    const int j = j0 + (c >> 2) * jstr + (c & 3);
                    if (!valid || j >= A.k) continue;
                    if (acc[c] >= thr || j == inc) {
                        for (int p = 0; p < tot; ++p)
                            if (cj[p] == j) acc[c] = cvv[p];
                    } else {
                        acc[c] = __fadd_ru(acc[c], Ef);
                    }
                }
                __syncwarp();
            }
        }
        Top2 tp{-INFINITY, -2, -INFINITY};
#pragma unroll
        for (int r = 0; r < CH / 4; ++r) {
            const float4 a4 = acc4(r);
            const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int j = j0 + r * jstr + c;
                if (j < A.k) top2_push(tp, av[c], j, inc);
            }
        }
        for (int o = o0; o; o >>= 1) {
            const Top2 other = top2_shfl_down(tp, o);
            if (q < o && q + o < A.tpr) top2_merge(tp, other, inc);
        }
        const double eps = valid ? (double)A.reps[row] : 0.0;
        float sa = 0.f;   // fused rescan: s~(i, a(i)) from the lane that holds a(i)
        if (fused) {
            if constexpr (SPARSE) {
                sa = (valid && inc >= 0) ? sacc[inc] : 0.f;   // one row per warp: every lane reads the same word
            } else {
                float mine = 0.f;
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    if (j0 + (c >> 2) * jstr + (c & 3) == inc) mine = acc[c];
                const int src = (valid && inc >= 0) ? g * A.tpr + (inc % jstr) / 4 : lane;
                sa = __shfl_sync(FULL, mine, src);
            }
        }
        if (A.mode == MODE_INIT_YY) {
            // Yin-Yang group bounds: group f = the 4 consecutive centers of one
            // float4 (lane q, round r: f = q + r * tpr), ug(i, f) = the max of
            // s~ + eps over its centers j != a(i) (-1: none)
            const int bj = __shfl_sync(FULL, tp.bj, g * A.tpr);
            if (valid) {
#pragma unroll
                for (int r = 0; r < CH / 4; ++r) {
                    const int f = q + r * A.tpr;
                    if (4 * f < A.k) {
                        float m = -INFINITY;
                        const float4 a4 = acc4(r);
                        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const int j = 4 * f + c;
                            if (j < A.k && j != bj) m = fmaxf(m, av[c]);
                        }
                        A.u[row * A.ku + f] = (m == -INFINITY) ? -1.f : store_upper((double)m + eps);
                    }
                }
            }
        }
        if (A.mode == SPKM_MODE_INIT_ELKAN && valid) {
#pragma unroll
            for (int r = 0; r < CH / 4; ++r) {
                const float4 a4 = acc4(r);
                const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int j = j0 + r * jstr + c;
                    if (j < A.k) A.u[row * A.ku + j] = store_upper((double)av[c] + eps);
                }
            }
        }
        if (A.mode == MODE_ELKAN_FULL && valid) {   // every u(i, j) exact: one 16-byte store per column group (ku % 4 == 0)
            float *ur = A.u + row * A.ku;
#pragma unroll
            for (int r = 0; r < CH / 4; ++r) {
                const int j = j0 + r * jstr;
                const float4 a4 = acc4(r);
                if (j + 3 < A.k) {
                    *reinterpret_cast<float4 *>(ur + j) =
                        make_float4(store_upper((double)a4.x + eps), store_upper((double)a4.y + eps),
                                    store_upper((double)a4.z + eps), store_upper((double)a4.w + eps));
                } else {
                    const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (j + c < A.k) ur[j + c] = store_upper((double)av[c] + eps);
                }
            }
        }
        const bool leader = valid && q == 0;
        bool moved = false;
        bool tight_pruned = false;
        if (leader) {
            switch (A.mode) {
                case SPKM_MODE_INIT_PLAIN:
                case MODE_INIT_YY:
                case SPKM_MODE_INIT_ELKAN:
                case SPKM_MODE_INIT_HAMERLY:
                    A.a[row] = tp.bj;
                    A.l[row] = store_lower((double)tp.b - eps);
                    if (A.mode == SPKM_MODE_INIT_HAMERLY)
                        A.u[row] = (A.k == 1) ? -1.f : store_upper((double)tp.s + eps);
                    break;
                case SPKM_MODE_LLOYD:
                    if (tp.bj != inc) {
                        A.a[row] = tp.bj;
                        moved = true;
                    }
                    break;
                case MODE_RESCAN:
                    if (fused) {   // the tighten test of k_hamerly_tighten (kernels.py:88-95)
                        const double lbt = (double)sa - eps;
                        bool pruned = (A.use_s && lbt >= 0.0 && (double)A.s_arr[inc] + kSqrt2 * eps <= lbt);
                        if (!pruned) pruned = ((double)A.u[row] + eps <= (double)sa);
                        tight_pruned = pruned;
                        if (pruned) {
                            A.l[row] = store_lower(lbt);
                            break;
                        }
                    }
                    if (tp.bj != inc) {
                        A.a[row] = tp.bj;
                        moved = true;
                    }
                    A.l[row] = store_lower((double)tp.b - eps);
                    A.u[row] = store_upper((double)tp.s + eps);
                    break;
                case MODE_ELKAN_FULL:
                    if (tp.bj != inc) {
                        A.a[row] = tp.bj;
                        moved = true;
                    }
                    A.l[row] = store_lower((double)tp.b - eps);
                    break;
                case MODE_PREDICT:
                    A.a[row] = tp.bj;
                    A.best[row] = (double)tp.b;
                    A.second[row] = (A.k == 1) ? -1.0 : (double)tp.s;
                    break;
            }
        }
        if (A.mode == MODE_ELKAN_FULL) {
            warp_append(moved, (int32_t)row, A.mv_i, inc, A.mv_old, A.ctr + SPKM_CTR_MOVES);
            ctr_add(s_ctr, SPKM_CTR_SIMS, leader ? (long long)A.k : 0);
            ctr_add(s_ctr, SPKM_CTR_NNZ_RESCAN, leader ? (long long)(e - s) : 0);   // (the block scan counts NNZ_ELKAN)
            if (allrows) ctr_add(s_ctr, SPKM_CTR_SURV2, leader ? 1 : 0);            // (else counted by the bound pass)
        }
        if (A.mode == SPKM_MODE_LLOYD || A.mode == MODE_RESCAN) {
            warp_append(moved, (int32_t)row, A.mv_i, inc, A.mv_old, A.ctr + SPKM_CTR_MOVES);
            if (A.mode == MODE_RESCAN) {
                const bool scanned = leader && !tight_pruned;
                ctr_add(s_ctr, SPKM_CTR_SIMS, scanned ? (long long)(A.k - 1) : 0);
                ctr_add(s_ctr, SPKM_CTR_NNZ_RESCAN, scanned ? (long long)(e - s) : 0);
                if (fused) {   // the tighten's counters and its survivor count
                    ctr_add(s_ctr, SPKM_CTR_SIMS, leader ? 1 : 0);
                    ctr_add(s_ctr, SPKM_CTR_NNZ_TIGHTEN, leader ? (long long)(e - s) : 0);
                    ctr_add(s_ctr, SPKM_CTR_SURV2, scanned ? 1 : 0);
                }
            }
        }
        if constexpr (SPARSE) __syncwarp();   // every lane is done with sacc before the next row zeroes it
    }
    PDL_TRIGGER();
    if (A.ctr) ctr_flush(s_ctr, A.ctr);
}

// --------------------------------------------------------- Hamerly family
// engine.py:274 (l), 284-303 (u) fused with the kernels.py:81-87 tests.
// One CTA = a tile of kHbTile consecutive points, kHbPer per thread (strided
// by the CTA size, so every load instruction of a warp is one coalesced
// 128-byte line and the kHbPer loads of a thread are independent); the
// survivors of the tile are appended with ONE global atomic (warp ballots ->
// per-warp counts in shared memory -> one prefix), not one per warp.
// sin(acos(x)) = sqrt(1 - x^2) for a float x, rounded UP, as a double: float32 MUFU rsqrt x (1 + 2^-19) instead of
// the float64 sqrt sequence (two per point made this 96 MB stream arithmetic-bound).  Both uses below want an upper
// bound of the sine (it lowers l and raises u); the excess is < 2^-18 relative, times a sine of the drift.
__device__ __forceinline__ double f_sin_up(float x) {
    const float y = fmaxf(__fmaf_ru(-x, x, 1.0f), 1e-30f);
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
    return (double)__fmul_ru(y * r, 1.0f + 1.9073486e-6f);
}
constexpr int kHbThreads = 256, kHbPer = 4, kHbTile = kHbThreads * kHbPer;
__global__ void __launch_bounds__(kHbThreads) k_hamerly_bounds(int64_t n, const float *__restrict__ reps,
                                                        const int32_t *__restrict__ a, float *l, float *u,
                                                        const double *__restrict__ drift,
                                                        const double *__restrict__ sinp,
                                                        const float *__restrict__ s_arr,
                                                        const double *__restrict__ hstat, int use_s, int naive,
                                                        int32_t *surv1, long long *ctr, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    __shared__ int s_cnt[kHbPer][kHbThreads / 32];
    __shared__ long long s_base;
    const int owner = (int)hstat[0], owner_s = (int)hstat[3];
    const double pmin = hstat[1], pmin2 = hstat[2], smax = hstat[4], smax2 = hstat[5];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * kHbTile + threadIdx.x;
    int ai[kHbPer];
    float lo[kHbPer], uo[kHbPer], ep[kHbPer];
#pragma unroll
    for (int r = 0; r < kHbPer; ++r) {
        const int64_t i = i0 + r * kHbThreads;
        const bool in = i < n;
        ai[r] = in ? __ldg(a + i) : 0;
        lo[r] = in ? l[i] : 0.f;
        uo[r] = in ? u[i] : 0.f;
        ep[r] = in ? __ldg(reps + i) : 0.f;
    }
    unsigned surv_mask[kHbPer];
#pragma unroll
    for (int r = 0; r < kHbPer; ++r) {
        const int64_t i = i0 + r * kHbThreads;
        bool surv = false;
        if (i < n) {
            const double sa = sinp[ai[r]];
            float lf = lo[r];
            if (sa != 0.0) {   // cos(theta_l + theta_p), theta_p from the chord bound
                const double pa = drift[ai[r]];
                const double ln = (lo[r] < -pa) ? -1.0 : d_clamp((double)lo[r] * pa - f_sin_up(lo[r]) * sa);
                lf = store_lower(ln);
                l[i] = lf;
            }
            const double worst_p = (ai[r] == owner) ? pmin2 : pmin;
            const double worst_s = (ai[r] == owner_s) ? smax2 : smax;
            float uf = uo[r];
            if (naive) {       // engine.py:299-303, deliberately unsound
                if (worst_p != 1.0) {
                    uf = store_upper(d_cos_upper((double)uo[r], worst_p));
                    u[i] = uf;
                }
            } else if (!(uo[r] >= 0.f && worst_s == 0.0)) {   // engine.py:290-298
                const double un = (uo[r] >= 0.f && worst_p >= 0.0)
                                      ? d_clamp((double)uo[r] + f_sin_up(uo[r]) * worst_s)
                                      : 1.0;
                uf = store_upper(un);
                u[i] = uf;
            }
            const double eps = (double)ep[r];
            const double lb = (double)lf;
            bool pruned = (use_s && lb >= 0.0 && (double)s_arr[ai[r]] + kSqrt2 * eps <= lb);
            if (!pruned) pruned = ((double)uf + 2.0 * eps <= lb);
            surv = !pruned;
        }
        surv_mask[r] = __ballot_sync(FULL, surv);
        if (lane == 0) s_cnt[r][wib] = __popc(surv_mask[r]);
    }
    __syncthreads();
    // tile prefix over (r, warp) in the order the entries are written
    if (wib == 0) {
        constexpr int E = kHbPer * (kHbThreads / 32);   // 32 entries
        static_assert(E == 32, "one warp scans the tile counts");
        const int v = (&s_cnt[0][0])[lane];
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        const int tot = __shfl_sync(FULL, x, 31);
        long long base = 0;
        if (lane == 0 && tot) base = (long long)atomicAdd((unsigned long long *)(ctr + SPKM_CTR_SURV1),
                                                          (unsigned long long)tot);
        (&s_cnt[0][0])[lane] = x - v;
        if (lane == 0) s_base = base;
    }
    __syncthreads();
    PDL_TRIGGER();
    const long long base = s_base;
#pragma unroll
    for (int r = 0; r < kHbPer; ++r) {
        if (surv_mask[r] >> lane & 1u) {
            const int rank = __popc(surv_mask[r] & ((1u << lane) - 1u));
            surv1[base + s_cnt[r][wib] + rank] = (int32_t)(i0 + r * kHbThreads);
        }
    }
}

// kernels.py:88-95: tighten l with the exact s~(i,a), re-test.  8 lanes per
// survivor, 4 survivors per warp: per 32-nnz chunk each lane loads 4
// (idx, val) pairs and gathers the 4 center values ct[idx * kp + a(i)]
// (all independent), then the group leader runs the canonical chain.
__global__ void __launch_bounds__(256) k_hamerly_tighten(const int64_t *__restrict__ indptr,
                                                         const int32_t *__restrict__ indices,
                                                         const float *__restrict__ values,
                                                         const float *__restrict__ reps,
                                                         const float *__restrict__ ct, int64_t kp,
                                                         const int32_t *__restrict__ a, float *l,
                                                         const float *__restrict__ u,
                                                         const float *__restrict__ s_arr, int use_s,
                                                         const int32_t *__restrict__ surv1, int32_t *surv2,
                                                         long long *ctr, const double *__restrict__ fuse,
                                                         const long long *__restrict__ ctl, int64_t hot) {
    PDL_ENTRY();
    if (ctl[1] || *fuse != 0.0) return;   // converged, or the rescan does the tighten this iteration
    const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
    __shared__ __align__(16) float2 s_vc[8][4][kIvStride];   // (value, center value), padded as s_iv
    __shared__ unsigned long long s_ctr[8];
    ctr_init(s_ctr);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int g = lane >> 3, q = lane & 7;
    float2 *svc = s_vc[wib][g];
    const long long cnt = ctr[SPKM_CTR_SURV1];
    const int64_t nslots = (cnt + 3) / 4;
    const int wpb = blockDim.x >> 5;
    for (int64_t w = (int64_t)blockIdx.x * wpb + wib; w < nslots; w += (int64_t)gridDim.x * wpb) {
        const int64_t slot = w * 4 + g;
        const bool valid = slot < cnt;
        const int32_t i = valid ? surv1[slot] : 0;
        const int ai = valid ? a[i] : 0;
        const int64_t s = valid ? indptr[i] : 0, e = valid ? indptr[i + 1] : 0;
        const int len = (int)(e - s);
        const int maxlen = (int)__reduce_max_sync(FULL, (unsigned)len);
        const float *cta = ct + ai;
        float acc = 0.f;
        // software-pipelined: the next chunk's (id, value) loads are issued
        // before this chunk's center gathers and chain
        int ix[4];
        float vx[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int t = q + 8 * r;
            ix[r] = t < len ? __ldg(indices + s + t) : 0;
            vx[r] = t < len ? __ldg(values + s + t) : 0.f;
        }
        for (int c0 = 0; c0 < maxlen; c0 += 32) {
            const int cntc = max(0, min(32, len - c0));
            float cx[4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
                cx[r] = (q + 8 * r < cntc) ? ldg_hint(cta + (int64_t)ix[r] * kp, ix[r] < hot ? pol_hot : pol_cold) : 0.f;
#pragma unroll
            for (int r = 0; r < 4; ++r) svc[q + 8 * r] = make_float2(vx[r], cx[r]);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int t = c0 + 32 + q + 8 * r;
                ix[r] = t < len ? __ldg(indices + s + t) : 0;
                vx[r] = t < len ? __ldg(values + s + t) : 0.f;
            }
            __syncwarp();
            if (q == 0) {
                int t = 0;
                for (; t + 2 <= cntc; t += 2) {
                    const float4 p = *reinterpret_cast<const float4 *>(svc + t);
                    acc = __fmaf_rn(p.x, p.y, acc);
                    acc = __fmaf_rn(p.z, p.w, acc);
                }
                if (t < cntc) acc = __fmaf_rn(svc[t].x, svc[t].y, acc);
            }
            __syncwarp();
        }
        bool surv = false;
        if (valid && q == 0) {
            const double eps = (double)reps[i];
            const double lb = (double)acc - eps;
            l[i] = store_lower(lb);
            bool pruned = (use_s && lb >= 0.0 && (double)s_arr[ai] + kSqrt2 * eps <= lb);
            if (!pruned) pruned = ((double)u[i] + eps <= (double)acc);
            surv = !pruned;
        }
        warp_append(surv, i, surv2, 0, nullptr, ctr + SPKM_CTR_SURV2);
        ctr_add(s_ctr, SPKM_CTR_SIMS, (valid && q == 0) ? 1 : 0);
        ctr_add(s_ctr, SPKM_CTR_NNZ_TIGHTEN, (valid && q == 0) ? (long long)len : 0);
    }
    PDL_TRIGGER();
    ctr_flush(s_ctr, ctr);
}

// ----------------------------------------------------------- Elkan family
// engine.py:281-283, u(i,j) <- cos_upper(u(i,j), p_j) if u <= p_j else 1,
// with the chord-based sine bound sin_p (see k_finalize), evaluated in
// float32 with directed rounding: every operation rounds towards the safe
// side, so the result is an upper bound of clamp(w p + sin(w) sin_p) + 1e-12
// for the float inputs -- the float64 version's guarantee -- at float32 cost
// (n*k elements per iteration: float64 sqrt made this pass ALU-bound).
//   pd = rd(p), pu = ru(p), su = ru(sin_p) (su == 0 <=> the center did not move)
//   (double)w <= p  <=>  w <= pd, exactly (pd is the largest float <= p)
#ifndef SPKM_FAST_SQRT
#define SPKM_FAST_SQRT 1      // C4 k_elkan_bounds 430 -> 321 ms per fit with SPKM_EB_MINB 3 (r02_ab_notes)
#endif
// sqrt(x) rounded up, x in [0, 1]: the IEEE directed sqrt is a ~20-instruction
// software sequence; x * rsqrt(x) from the MUFU (<= 2 ulp + 0.5 ulp of the
// product) times (1 + 2^-19) rounded up is >= sqrt(x) at a quarter of the cost
// Branch-free: x is clamped to 1e-30 (sqrt_up(1e-30) ~ 1e-15 >= sqrt of anything smaller; the MUFU never
// sees a subnormal), rsqrt.approx (relative error < 2^-22) is one instruction.
__device__ __forceinline__ float sqrt_up(float x) {
#if SPKM_FAST_SQRT
    x = fmaxf(x, 1e-30f);
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return __fmul_ru(x * r, 1.0f + 1.9073486e-6f);
#else
    return __fsqrt_ru(x);
#endif
}
__device__ __forceinline__ float elkan_u_drift(float w, float pd, float pu, float su) {
    const float sw = sqrt_up(__fmaf_ru(-w, w, 1.0f));   // >= sin(w) (negative arguments are clamped)
    const float prod = __fmaf_ru(sw, su, 1e-12f);
    const float nv = __fmaf_ru(w, w >= 0.f ? pu : pd, prod);
    return (w <= pd) ? fminf(fmaxf(nv, -1.0f), 1.0f) : 1.0f;
}
// Prune thresholds of one row (kernels.py:35-47 with the eps margins):
//   u(i,j) + 2 eps <= l  <=>  u(i,j) <= rd(l - 2 eps)      (u a float)
//   cc(a,j) + sqrt2 eps <= l  <=>  cc(a,j) <= rd(l - sqrt2 eps)
// so the per-element tests are single float compares.
__device__ __forceinline__ float thr_u_of(double lb, double eps) { return __double2float_rd(lb - 2.0 * eps); }
__device__ __forceinline__ float thr_c_of(double lb, double eps) { return __double2float_rd(lb - kSqrt2 * eps); }

// engine.py:274-283 (l and u(i,j) drift updates) fused with the
// kernels.py:35-47 tests; a point survives if any j != a(i) is not pruned.
// Warp per point, lanes over j in 16-byte groups (u rows are contiguous,
// ku a multiple of 4); each warp takes chunks of 32 consecutive points:
// lane r prepares point r's row values (drift-updated l, thresholds), the
// warp then streams the 32 u rows (up to 8 float4 loads per lane in flight)
// and appends the chunk's survivors with one atomic.  Per-center pd/pu/su
// live in shared memory.  k <= 1024.
constexpr int kEbMaxK = 1024;
constexpr int kLightMax = 4;      // failing centers listed per light row (lightj[n][4]); needs heavy_thr <= 5
#ifndef SPKM_EB_MINB
#define SPKM_EB_MINB 3        // 80 registers, 3 CTAs per SM: the u stream needs the warps (126 -> 80 regs)
#endif
template <bool CC>   // CC: the center-center tests of elkan (simp_elkan: the per-element loop is branch-free)
__global__ void __launch_bounds__(256, SPKM_EB_MINB) k_elkan_bounds(int64_t n, int k, const float *__restrict__ reps,
                                                      const int32_t *__restrict__ a, float *l, float *u,
                                                      int64_t ku, const double *__restrict__ drift,
                                                      const double *__restrict__ sinp,
                                                      const float *__restrict__ cc,
                                                      const float *__restrict__ s_arr, int use_cc,
                                                      int32_t *surv1, long long *ctr, const long long *__restrict__ ctl,
                                                      int heavy_thr, int32_t *surv_h, int32_t *lightj,
                                                      const double *__restrict__ allheavy) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    if (heavy_thr > 0 && *allheavy != 0.0) return;   // every row takes the full pass this iteration (kAllHeavyFlag)
    __shared__ __align__(16) float s_pd[kEbMaxK], s_pu[kEbMaxK], s_su[kEbMaxK];
    const int k4 = (k + 3) >> 2;
    for (int j = threadIdx.x; j < 4 * k4; j += blockDim.x) {
        const bool in = j < k;
        const double p = in ? drift[j] : 1.0, sp = in ? sinp[j] : 0.0;
        s_pd[j] = __double2float_rd(p);
        s_pu[j] = __double2float_ru(p);
        s_su[j] = __double2float_ru(sp);
    }
    __syncthreads();
    const float4 *pd4 = reinterpret_cast<const float4 *>(s_pd), *pu4 = reinterpret_cast<const float4 *>(s_pu),
                 *su4 = reinterpret_cast<const float4 *>(s_su);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int64_t nchunks = (n + 31) >> 5;
    for (int64_t c = (int64_t)blockIdx.x * wpb + wib; c < nchunks; c += (int64_t)gridDim.x * wpb) {
        const int64_t rb = c << 5;
        const int64_t ir = rb + lane;
        int ai_r = 0;
        float thu_r = 0.f, thc_r = 0.f;
        bool pskip_r = true, ccon_r = false;
        if (ir < n) {
            ai_r = a[ir];
            const float lo = l[ir];
            float lf = lo;
            const double sa = sinp[ai_r];
            if (sa != 0.0) {
                const double pa = drift[ai_r];
                lf = store_lower((lo < -pa) ? -1.0 : d_clamp((double)lo * pa - d_sin((double)lo) * sa));
                l[ir] = lf;
            }
            const double eps = (double)reps[ir];
            const double lb = (double)lf;
            pskip_r = CC && use_cc && lb >= 0.0 && (double)s_arr[ai_r] + kSqrt2 * eps <= lb;
            ccon_r = CC && use_cc && lb >= 0.0;
            thu_r = thr_u_of(lb, eps);
            thc_r = thr_c_of(lb, eps);
        }
        const int nr = (int)min((int64_t)32, n - rb);
        unsigned smask = 0, hmask = 0;
        for (int r = 0; r < nr; ++r) {
            const int ai = __shfl_sync(FULL, ai_r, r);
            const float thu = __shfl_sync(FULL, thu_r, r), thc = __shfl_sync(FULL, thc_r, r);
            const bool pskip = __shfl_sync(FULL, (int)pskip_r, r) != 0;
            const bool ccon = __shfl_sync(FULL, (int)ccon_r, r) != 0;
            float4 *ui = reinterpret_cast<float4 *>(u + (rb + r) * ku);
            const float *cca = cc + (int64_t)ai * k;
            float4 v[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int q = lane + 32 * t;
                if (q < k4) v[t] = ui[q];
            }
            unsigned fb = 0;   // bit 4 t + cq: center 4 (lane + 32 t) + cq fails the stored-bound test
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int q = lane + 32 * t;
                if (q >= k4) break;
                const float4 su = su4[q];
                float w[4] = {v[t].x, v[t].y, v[t].z, v[t].w};
                if (su.x != 0.f || su.y != 0.f || su.z != 0.f || su.w != 0.f) {
                    const float4 pd = pd4[q], pu = pu4[q];
                    const float sa_[4] = {su.x, su.y, su.z, su.w}, pda[4] = {pd.x, pd.y, pd.z, pd.w},
                                pua[4] = {pu.x, pu.y, pu.z, pu.w};
#pragma unroll
                    for (int cq = 0; cq < 4; ++cq) {
                        const float wn = elkan_u_drift(w[cq], pda[cq], pua[cq], sa_[cq]);
                        w[cq] = sa_[cq] != 0.f ? wn : w[cq];
                    }
                    ui[q] = make_float4(w[0], w[1], w[2], w[3]);   // padding columns (j >= k) have su == 0
                }
                if (!pskip) {
#pragma unroll
                    for (int cq = 0; cq < 4; ++cq) {
                        const int j = 4 * q + cq;
                        if constexpr (CC) {
                            if (j < k && j != ai) {
                                bool skip = ccon && __ldg(cca + j) <= thc;
                                if (!skip) skip = w[cq] <= thu;
                                fb |= (skip ? 0u : 1u) << (4 * t + cq);
                            }
                        } else {
                            fb |= ((j < k && j != ai && !(w[cq] <= thu)) ? 1u : 0u) << (4 * t + cq);
                        }
                    }
                }
            }
            // heavy rows (many centers the stored bounds cannot prune) go to the
            // full pass over the sparse center index (spkm_elkan_heavy), the
            // others to the block scan; heavy_thr == 0: every survivor is light
            const int tot = __reduce_add_sync(FULL, __popc(fb));
            if (tot > 0) {
                if (heavy_thr > 0 && tot >= heavy_thr) hmask |= 1u << r;
                else smask |= 1u << r;
            }
            if constexpr (!CC) {
                // light rows (fewer than heavy_thr <= kLightMax + 1 failing centers): their ids, ascending, for
                // k_elkan_light -- decoded from the lanes' fail bits
                if (lightj != nullptr && tot > 0 && tot < heavy_thr) {
                    constexpr int NONE = 0x7fffffff;
                    int f0 = NONE, f1 = NONE, f2 = NONE, f3 = NONE;
                    unsigned lm = __ballot_sync(FULL, fb != 0);
                    while (lm) {
                        const int ln = __ffs(lm) - 1;
                        lm &= lm - 1;
                        unsigned b = __shfl_sync(FULL, fb, ln);
                        while (b) {
                            const int bit = __ffs(b) - 1;
                            b &= b - 1;
                            f3 = f2;   // (at most kLightMax entries: tot < heavy_thr <= kLightMax + 1)
                            f2 = f1;
                            f1 = f0;
                            f0 = 4 * (ln + 32 * (bit >> 2)) + (bit & 3);
                        }
                    }
                    // ascending (4-element sorting network); unused slots -> -1 at the end
                    int x;
#define SPKM_CSWAP(A_, B_) x = min(A_, B_); B_ = max(A_, B_); A_ = x;
                    SPKM_CSWAP(f0, f1) SPKM_CSWAP(f2, f3) SPKM_CSWAP(f0, f2) SPKM_CSWAP(f1, f3) SPKM_CSWAP(f1, f2)
#undef SPKM_CSWAP
                    if (lane == 0)
                        *reinterpret_cast<int4 *>(lightj + (rb + r) * kLightMax) =
                            make_int4(f0 == NONE ? -1 : f0, f1 == NONE ? -1 : f1, f2 == NONE ? -1 : f2, f3 == NONE ? -1 : f3);
                }
            }
        }
        long long base = 0;
        if (lane == 0 && smask) base = (long long)atomicAdd((unsigned long long *)(ctr + SPKM_CTR_SURV1),
                                                            (unsigned long long)__popc(smask));
        if (lane == 1 && hmask) base = (long long)atomicAdd((unsigned long long *)(ctr + SPKM_CTR_SURV2),
                                                            (unsigned long long)__popc(hmask));
        const long long base_h = __shfl_sync(FULL, base, 1);
        base = __shfl_sync(FULL, base, 0);
        if (smask >> lane & 1u) surv1[base + __popc(smask & ((1u << lane) - 1u))] = (int32_t)ir;
        if (hmask >> lane & 1u) surv_h[base_h + __popc(hmask & ((1u << lane) - 1u))] = (int32_t)ir;
    }
    PDL_TRIGGER();
}

// kernels.py:22-66 for the LIGHT survivors of a simp_elkan bound pass that
// listed their failing centers (at most kLightMax, ascending; every other
// center passed u + 2 eps <= l and so passes every later test, the running
// best only grows).  8 lanes per row, 4 rows per warp (as k_hamerly_tighten):
// per 32-nnz chunk each lane loads 4 (id, value) pairs and gathers the row's
// 1 + nF columns a(i), F of each (all independent loads), lanes 0..nF run
// one canonical chain each from shared memory in CSR order, then the leader
// replays the reference's sequential scan on those few values: tighten to
// s~(i, a), re-test each listed center against the running best, "compute"
// = take its s~, strict > reassigns.  Same results and counters as
// k_elkan_scan on these rows, without its four passes over the u row.
__global__ void __launch_bounds__(256) k_elkan_light(const int64_t *__restrict__ indptr,
                                                     const int32_t *__restrict__ indices,
                                                     const float *__restrict__ values,
                                                     const float *__restrict__ reps,
                                                     const float *__restrict__ ct, int64_t kp, int k, int32_t *a,
                                                     float *l, float *u, int64_t ku,
                                                     const int32_t *__restrict__ surv1,
                                                     const int32_t *__restrict__ lightj, int32_t *mv_i,
                                                     int32_t *mv_old, long long *ctr,
                                                     const long long *__restrict__ ctl, int64_t hot) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
    constexpr int NC = kLightMax + 1, ST = NC + 1;   // columns per row; floats staged per nnz (value + NC center values)
    __shared__ float s_st[8][4][32 * ST];
    __shared__ unsigned long long s_ctr[8];
    ctr_init(s_ctr);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int g = lane >> 3, q = lane & 7;
    float *st = s_st[wib][g];
    const long long cnt = ctr[SPKM_CTR_SURV1];
    const int64_t nslots = (cnt + 3) / 4;
    const int wpb = blockDim.x >> 5;
    for (int64_t w = (int64_t)blockIdx.x * wpb + wib; w < nslots; w += (int64_t)gridDim.x * wpb) {
        const int64_t slot = w * 4 + g;
        const bool valid = slot < cnt;
        const int32_t i = valid ? surv1[slot] : 0;
        const int ai = valid ? a[i] : 0;
        const int4 f4 = valid ? __ldg(reinterpret_cast<const int4 *>(lightj + (int64_t)i * kLightMax)) : make_int4(-1, -1, -1, -1);
        const int col[NC] = {ai, f4.x, f4.y, f4.z, f4.w};
        const int nc = 1 + (f4.x >= 0) + (f4.y >= 0) + (f4.z >= 0) + (f4.w >= 0);
        DCHECK(!valid || (f4.x >= 0 && f4.x < k && f4.w < k));
        const int64_t s = valid ? indptr[i] : 0, e = valid ? indptr[i + 1] : 0;
        const int len = (int)(e - s);
        const int maxlen = (int)__reduce_max_sync(FULL, (unsigned)len);
        float acc = 0.f;
        for (int c0 = 0; c0 < maxlen; c0 += 32) {
            const int cntc = max(0, min(32, len - c0));
            float vx[4], cx[4][NC];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int t = q + 8 * r;
                const bool on = t < cntc;
                const int id = on ? __ldg(indices + s + c0 + t) : 0;
                vx[r] = on ? __ldg(values + s + c0 + t) : 0.f;
                const float *rowp = ct + (int64_t)id * kp;
                const uint64_t pol = id < hot ? pol_hot : pol_cold;
#pragma unroll
                for (int c = 0; c < NC; ++c) cx[r][c] = (on && c < nc) ? ldg_hint(rowp + col[c], pol) : 0.f;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                float *p = st + (q + 8 * r) * ST;
                p[0] = vx[r];
#pragma unroll
                for (int c = 0; c < NC; ++c) p[1 + c] = cx[r][c];
            }
            __syncwarp();
            if (q < nc)
                for (int t = 0; t < cntc; ++t) acc = __fmaf_rn(st[t * ST], st[t * ST + 1 + q], acc);
            __syncwarp();
        }
        // the group's similarities to the leader: s~(i, a) and the listed centers'
        float sv[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) sv[c] = __shfl_sync(FULL, acc, (lane & ~7) + c);
        int cur = ai;
        long long sims = 0;
        if (valid && q == 0) {
            const double eps = (double)reps[i];
            float *ui = u + (int64_t)i * ku;
            float lcur = sv[0];
            ui[ai] = store_upper((double)lcur + eps);
            sims = 1;
#pragma unroll
            for (int c = 1; c < NC; ++c) {
                const int j = col[c];
                if (j < 0) continue;
                if ((double)ui[j] + eps <= (double)lcur) continue;
                ui[j] = store_upper((double)sv[c] + eps);
                ++sims;
                if (sv[c] > lcur) {
                    cur = j;
                    lcur = sv[c];
                }
            }
            l[i] = store_lower((double)lcur - eps);
            if (cur != ai) a[i] = cur;
        }
        const bool leader = valid && q == 0;
        warp_append(leader && cur != ai, i, mv_i, ai, mv_old, ctr + SPKM_CTR_MOVES);
        ctr_add(s_ctr, SPKM_CTR_SIMS, sims);
        ctr_add(s_ctr, SPKM_CTR_NNZ_ELKAN, leader ? (long long)len : 0);
    }
    PDL_TRIGGER();
    ctr_flush(s_ctr, ctr);
}

// Centers per lane block of k_elkan_scan: EB = 4 (one float4 of a term-major
// ct32 row per lane, so a warp's gather of one row's blocks is one load
// instruction) while the row fits one round of 32 lanes (k <= 128); EB = 8
// (two float4, one 32-byte sector) above, which halves the rounds.  Measured:
// C2 (k = 100) scan 91 -> 78 us with 4; C3 (k = 200) 2.6 -> 3.1 ms with 4.
#ifndef SPKM_EK_EB4_MAXK
#define SPKM_EK_EB4_MAXK 128
#endif
__host__ __device__ __forceinline__ int elkan_block(int64_t k) { return k <= SPKM_EK_EB4_MAXK ? 4 : 8; }
// floats of the per-warp value buffer of k_elkan_scan (EB + 1 per block)
__host__ __device__ __forceinline__ int64_t elkan_sim_stride(int64_t k) {
    const int64_t eb = elkan_block(k);
    const int64_t nb = (k + eb - 1) / eb;
    const int64_t need = nb * (eb + 1);
    const int64_t bpr = nb < 32 ? nb : 32;
    const int64_t ppw = (32 / bpr) < 8 ? (32 / bpr) : 8;
    const int64_t per = need * ppw;
    return per < 288 ? 288 : per;
}

// kernels.py:22-66 for the surviving points, in two steps:
//  1. gather pass, blocked by 16-byte float4s: centers are grouped in blocks
//     of EB = 4 (one float4 of a term-major ct32 row); a block is fetched
//     when it holds a(i) or any center failing the drift-updated u test
//     (u + 2 eps <= l).  Lane = block, bpr lanes per point, up to 8 points
//     per warp, rounds of 32 blocks for k > 128.  The canonical s~ of every
//     fetched center lands in shared memory.
//  2. the reference's sequential scan (kernels.py:35-65) replayed by the
//     group's leader lane over j = 0..k-1 on those values: tighten at the
//     first failing j, re-test against the running best (cc and u tests
//     with the eps margins), "compute" = read s~, strict > reassignment.
//     Every center the replay needs was fetched (a center passing the u
//     pre-test also passes every later u test, since the running best only
//     grows), so sim_count counts exactly what the reference's loop counts.
// FUSE: the drift update + prune test of k_elkan_bounds is done here, per
// row over all n rows (each lane updates the u(i, j) of its own blocks, the
// same lanes that later test and scan them), so the bound pass, its survivor
// list and one read of u are saved; rows that survive go straight on.
template <int EB, bool FUSE>
#ifndef SPKM_EK_MINB
#define SPKM_EK_MINB 4        // EB = 8 (k > 128): 64 registers, 4 CTAs per SM (C4 scan 3590 -> 3350 ms per fit)
#endif
#ifndef SPKM_EK4_MINB
#define SPKM_EK4_MINB 3       // EB = 4 unfused: <= 85 registers (fused and EB = 8: SPKM_EK_MINB), as the r01 build
#endif
__global__ void __launch_bounds__(256, (EB == 8 || FUSE) ? SPKM_EK_MINB : SPKM_EK4_MINB) k_elkan_scan(const int64_t *__restrict__ indptr,
                                                    const int32_t *__restrict__ indices,
                                                    const float *__restrict__ values,
                                                    const float *__restrict__ reps,
                                                    const float *__restrict__ ct, int64_t kp, int k,
                                                    int32_t *a, float *l, float *u, int64_t ku,
                                                    const float *__restrict__ cc, int use_cc,
                                                    const int32_t *__restrict__ surv1, int32_t *mv_i,
                                                    int32_t *mv_old, long long *ctr, int64_t n_rows,
                                                    const double *__restrict__ drift,
                                                    const double *__restrict__ sinp,
                                                    const float *__restrict__ s_arr,
                                                    const long long *__restrict__ ctl, int64_t hot) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
#ifndef SPKM_EK_UB
#define SPKM_EK_UB 1
#endif
    // nnz per gather batch: 8 * SPKM_EK_UB float4 loads in flight per lane
    constexpr int UB = SPKM_EK_UB * 32 / EB;
    constexpr int ES = EB + 1;    // padded per-block stride of the similarity buffer
    // staged (id, value) pairs live in dynamic shared memory after the
    // similarity buffers: ppw row groups per warp (k > 128: one), not 8

    __shared__ int s_act[8][EB == 4 && SPKM_EK_EB4_MAXK > 128 ? 256 : 128];   // per warp: the groups' active block lists
    __shared__ unsigned long long s_ctr[8];
    ctr_init(s_ctr);
    extern __shared__ float s_sim_dyn[];   // [8 warps][sim_stride]
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nb = (k + EB - 1) / EB;
    const int bpr = nb < 32 ? nb : 32;
    const int ppw = min(8, 32 / bpr);
    const int nrounds = (nb + 31) >> 5;
    const int g = lane / bpr, q = lane - g * bpr;
    const bool lane_on = g < ppw;
    const int o0 = bpr > 1 ? (1 << (31 - __clz(bpr - 1))) : 0;
    const int sim_stride = (int)elkan_sim_stride(k);  // floats per warp
    const int gstride = sim_stride / ppw;             // per-group slice (>= ES * nb)
    float *my_sim = s_sim_dyn + wib * sim_stride + (lane_on ? g : 0) * gstride;
    int2 *my_iv = reinterpret_cast<int2 *>(s_sim_dyn + 8 * sim_stride) + (wib * ppw + (lane_on ? g : 0)) * kIvStride;
    const long long cnt = FUSE ? n_rows : ctr[SPKM_CTR_SURV1];
    const int64_t nslots = (cnt + ppw - 1) / ppw;
    const int wpb = blockDim.x >> 5;
    for (int64_t w = (int64_t)blockIdx.x * wpb + wib; w < nslots; w += (int64_t)gridDim.x * wpb) {
        const int64_t slot = w * ppw + g;
        bool valid = lane_on && slot < cnt;
        const int32_t i = valid ? (FUSE ? (int32_t)slot : surv1[slot]) : 0;
        const int ai = valid ? a[i] : 0;
        float *ui = u + (int64_t)i * ku;
        const double eps = valid ? (double)reps[i] : 0.0;
        double lb;
        if constexpr (FUSE) {
            // k_elkan_bounds for this row (engine.py:274-283 + kernels.py:35-47)
            const float lo = valid ? l[i] : 0.f;
            float lf = lo;
            const double sa = valid ? sinp[ai] : 0.0;
            if (sa != 0.0) {
                const double pa = drift[ai];
                lf = store_lower((lo < -pa) ? -1.0 : d_clamp((double)lo * pa - d_sin((double)lo) * sa));
            }
            if (valid && q == 0 && lf != lo) l[i] = lf;
            lb = (double)lf;
            const bool pskip = use_cc && lb >= 0.0 && (double)s_arr[ai] + kSqrt2 * eps <= lb;
            const bool cc_on = use_cc && lb >= 0.0;
            const float thu = thr_u_of(lb, eps), thc = thr_c_of(lb, eps);
            bool surv = false;
            for (int r = 0; r < nrounds && valid; ++r) {
                const int blk = r * 32 + q;
                if (blk >= nb) break;
                for (int c2 = 0; c2 < EB; ++c2) {
                    const int j = blk * EB + c2;
                    if (j >= k) break;
                    float wv = ui[j];
                    const double sj = sinp[j];
                    if (sj != 0.0) {   // the k_elkan_bounds update, same float32 arithmetic
                        const double pj = drift[j];
                        wv = elkan_u_drift(wv, __double2float_rd(pj), __double2float_ru(pj), __double2float_ru(sj));
                        ui[j] = wv;
                    }
                    if (!pskip && j != ai) {
                        bool skip = cc_on && __ldg(cc + (int64_t)ai * k + j) <= thc;
                        if (!skip) skip = wv <= thu;
                        surv |= !skip;
                    }
                }
            }
            // the row survives if any of its lanes found a center it cannot prune
            const unsigned m = __ballot_sync(FULL, surv);
            const unsigned gmask = (bpr >= 32 ? 0xffffffffu : ((1u << bpr) - 1u)) << (lane_on ? g * bpr : 0);
            valid = valid && (m & gmask) != 0;
            ctr_add(s_ctr, SPKM_CTR_SURV1, (valid && q == 0) ? 1 : 0);
        } else {
            lb = valid ? (double)l[i] : 0.0;
        }
        const int64_t s = valid ? indptr[i] : 0, e = valid ? indptr[i + 1] : 0;
        const int len = (int)(e - s);
        const bool cc_ok = use_cc && lb >= 0.0;
        const float thu_s = thr_u_of(lb, eps), thc_s = thr_c_of(lb, eps);
        constexpr int NONE = 0x7fffffff;
        // (A) the first j failing the pre-tests (kernels.py:35-47): where the
        // reference tightens l to the exact s(i, a)
        int first_fail = NONE;
        if (valid) {
            for (int r = 0; r < nrounds && first_fail == NONE; ++r) {
                const int blk = r * 32 + q;
                if (blk >= nb) break;
                for (int c2 = 0; c2 < EB; ++c2) {
                    const int j = blk * EB + c2;
                    if (j >= k) break;
                    if (j == ai) continue;
                    if (cc_ok && cc[(int64_t)ai * k + j] <= thc_s) continue;
                    if (ui[j] <= thu_s) continue;
                    first_fail = j;
                    break;
                }
            }
        }
        for (int o = o0; o; o >>= 1) {   // group min (lanes of other groups hold their own values)
            const int other = __shfl_down_sync(FULL, first_fail, o);
            if (q < o && q + o < bpr) first_fail = min(first_fail, other);
        }
        first_fail = __shfl_sync(FULL, first_fail, lane - q);
        const bool tight = valid && first_fail != NONE;
        // (B) s~(i, a(i)) -- the canonical chain for the single center a(i),
        // as k_hamerly_tighten: the group's lanes stage (value, center value)
        // pairs of each 32-nnz chunk, the leader runs the chain in CSR order
        float lcur = 0.f;
        const int tlen = tight ? len : 0;
        const int maxt = (int)__reduce_max_sync(FULL, (unsigned)tlen);
        if (maxt > 0) {
            float acc = 0.f;
            const float *cta = ct + ai;
            for (int c0 = 0; c0 < maxt; c0 += 32) {
                const int cntc = max(0, min(32, tlen - c0));
                for (int q2 = q; q2 < cntc; q2 += bpr) {
                    const int t = __ldg(indices + s + c0 + q2);
                    const float cv = ldg_hint(cta + (int64_t)t * kp, t < hot ? pol_hot : pol_cold);
                    my_iv[q2] = make_int2(__float_as_int(__ldg(values + s + c0 + q2)), __float_as_int(cv));
                }
                __syncwarp();
                if (q == 0)
                    for (int t = 0; t < cntc; ++t)
                        acc = __fmaf_rn(__int_as_float(my_iv[t].x), __int_as_float(my_iv[t].y), acc);
                __syncwarp();
            }
            lcur = __shfl_sync(FULL, acc, lane - q);
        }
        // (C) blocks to fetch: centers j >= first_fail, j != a(i) failing the
        // u test at the tightened bound s~(i, a).  The replay below only ever
        // computes such centers: its u test u + eps <= lcur is implied by the
        // same test at s~(i, a) because the running best only grows (the cc
        // test is not used here: it refers to the current best center, which
        // changes).  Active blocks are compacted so each fetch round gives
        // every lane of the group a block that is needed.
        int *my_act = s_act[wib] + (lane_on ? g : 0) * nb;
        int nact = 0;
        {
            const double lc = (double)lcur;
            for (int r = 0; r < nrounds; ++r) {
                const int blk = r * 32 + q;
                bool act = false;
                if (tight && blk < nb) {
                    for (int c2 = 0; c2 < EB; ++c2) {
                        const int j = blk * EB + c2;
                        if (j >= k) break;
                        if (j < first_fail || j == ai) continue;
                        act |= !((double)ui[j] + eps <= lc);
                    }
                }
                const unsigned m = __ballot_sync(FULL, act);
                const unsigned gm = (m >> (lane - q)) & (bpr >= 32 ? 0xffffffffu : ((1u << bpr) - 1u));
                if (act) my_act[nact + __popc(gm & ((1u << q) - 1u))] = blk;
                nact += __popc(gm);
            }
        }
#ifndef SPKM_EK_DENSE_PCT
#define SPKM_EK_DENSE_PCT 0
#endif
#if SPKM_EK_DENSE_PCT > 0
        // most blocks active: fetch them all in block order (each warp load
        // instruction then reads one contiguous span of the center row: full
        // 128-byte lines instead of scattered sectors); the extra blocks'
        // similarities are computed but never read by the replay
        if (nact * 100 >= SPKM_EK_DENSE_PCT * nb) {
            __syncwarp();
            for (int bb = q; bb < nb; bb += bpr) my_act[bb] = bb;
            nact = nb;
        }
#endif
        __syncwarp();
        const int act_rounds = (int)__reduce_max_sync(FULL, (unsigned)((nact + bpr - 1) / bpr));
        const int maxlen = (int)__reduce_max_sync(FULL, (unsigned)(nact ? len : 0));
        for (int r = 0; r < act_rounds; ++r) {
            const int slot_b = r * bpr + q;
            const bool act = lane_on && slot_b < nact;
            const int blk = act ? my_act[slot_b] : 0;
            const int j0 = blk * EB;
            float acc[EB];
#pragma unroll
            for (int c2 = 0; c2 < EB; ++c2) acc[c2] = 0.f;
            const float4 *base4 = reinterpret_cast<const float4 *>(ct + j0);
            const int glen = nact > r * bpr ? len : 0;   // rows of the group with blocks left this round
            for (int c0 = 0; c0 < maxlen; c0 += 32) {
                const int cntc = max(0, min(32, glen - c0));
                for (int q2 = q; q2 < cntc; q2 += bpr)
                    my_iv[q2] = make_int2(__ldg(indices + s + c0 + q2), __float_as_int(__ldg(values + s + c0 + q2)));
                __syncwarp();
                if (act && EB == 8) {   // two float4 (one sector) per lane and nnz
                    int uu = 0;
                    for (; uu + UB <= cntc; uu += UB) {
                        float4 x[UB][2];
                        float vv[UB];
                        int iv[UB];
                        load_iv<UB>(my_iv + uu, iv, vv);
#pragma unroll
                        for (int b = 0; b < UB; ++b) {
                            const float4 *p = base4 + ((int64_t)iv[b] * kp >> 2);
                            const uint64_t pol = iv[b] < hot ? pol_hot : pol_cold;
                            x[b][0] = ldg_hint(p, pol);
                            x[b][1] = ldg_hint(p + 1, pol);
                        }
#pragma unroll
                        for (int b = 0; b < UB; ++b) {
                            acc[0] = __fmaf_rn(vv[b], x[b][0].x, acc[0]);
                            acc[1] = __fmaf_rn(vv[b], x[b][0].y, acc[1]);
                            acc[2] = __fmaf_rn(vv[b], x[b][0].z, acc[2]);
                            acc[3] = __fmaf_rn(vv[b], x[b][0].w, acc[3]);
                            acc[EB > 4 ? 4 : 0] = __fmaf_rn(vv[b], x[b][1].x, acc[EB > 4 ? 4 : 0]);
                            acc[EB > 4 ? 5 : 1] = __fmaf_rn(vv[b], x[b][1].y, acc[EB > 4 ? 5 : 1]);
                            acc[EB > 4 ? 6 : 2] = __fmaf_rn(vv[b], x[b][1].z, acc[EB > 4 ? 6 : 2]);
                            acc[EB > 4 ? 7 : 3] = __fmaf_rn(vv[b], x[b][1].w, acc[EB > 4 ? 7 : 3]);
                        }
                    }
                    for (; uu < cntc; ++uu) {
                        const int2 t = my_iv[uu];
                        const float v0 = __int_as_float(t.y);
                        const float4 *p = base4 + ((int64_t)t.x * kp >> 2);
                        const uint64_t pol = t.x < hot ? pol_hot : pol_cold;
                        const float4 x0 = ldg_hint(p, pol), x1 = ldg_hint(p + 1, pol);
                        acc[0] = __fmaf_rn(v0, x0.x, acc[0]);
                        acc[1] = __fmaf_rn(v0, x0.y, acc[1]);
                        acc[2] = __fmaf_rn(v0, x0.z, acc[2]);
                        acc[3] = __fmaf_rn(v0, x0.w, acc[3]);
                        acc[EB > 4 ? 4 : 0] = __fmaf_rn(v0, x1.x, acc[EB > 4 ? 4 : 0]);
                        acc[EB > 4 ? 5 : 1] = __fmaf_rn(v0, x1.y, acc[EB > 4 ? 5 : 1]);
                        acc[EB > 4 ? 6 : 2] = __fmaf_rn(v0, x1.z, acc[EB > 4 ? 6 : 2]);
                        acc[EB > 4 ? 7 : 3] = __fmaf_rn(v0, x1.w, acc[EB > 4 ? 7 : 3]);
                    }
                } else if (act) {   // EB == 4: one float4 per lane and nnz
                    int uu = 0;
                    for (; uu + UB <= cntc; uu += UB) {
                        float4 x[UB];
                        float vv[UB];
                        int iv[UB];
                        load_iv<UB>(my_iv + uu, iv, vv);
#pragma unroll
                        for (int b = 0; b < UB; ++b)
                            x[b] = ldg_hint(base4 + ((int64_t)iv[b] * kp >> 2), iv[b] < hot ? pol_hot : pol_cold);
#pragma unroll
                        for (int b = 0; b < UB; ++b) {
                            acc[0] = __fmaf_rn(vv[b], x[b].x, acc[0]);
                            acc[1] = __fmaf_rn(vv[b], x[b].y, acc[1]);
                            acc[2] = __fmaf_rn(vv[b], x[b].z, acc[2]);
                            acc[3] = __fmaf_rn(vv[b], x[b].w, acc[3]);
                        }
                    }
                    for (; uu < cntc; ++uu) {
                        const int2 t = my_iv[uu];
                        const float v0 = __int_as_float(t.y);
                        const float4 x0 = ldg_hint(base4 + ((int64_t)t.x * kp >> 2), t.x < hot ? pol_hot : pol_cold);
                        acc[0] = __fmaf_rn(v0, x0.x, acc[0]);
                        acc[1] = __fmaf_rn(v0, x0.y, acc[1]);
                        acc[2] = __fmaf_rn(v0, x0.z, acc[2]);
                        acc[3] = __fmaf_rn(v0, x0.w, acc[3]);
                    }
                }
                __syncwarp();
            }
            if (act) {
#pragma unroll
                for (int c2 = 0; c2 < EB; ++c2) my_sim[blk * ES + c2] = acc[c2];
            }
        }
        __syncwarp();
        // (D) replay of kernels.py:35-65, parallel over the group's lanes.
        // Lane q owns the centers of blocks q, q+32, ... (ascending j within
        // the lane).  With the running best (cur, lcur) every lane finds its
        // candidates and its first "event" (candidate beating lcur); the
        // earliest event of the group updates (cur, lcur) and the scan resumes
        // after it.  Between events the state is constant, so the candidate set
        // and the reassignments equal the reference's sequential loop.
        int cur = ai;
        long long sims = 0;
        if (tight && q == 0) {
            ui[ai] = store_upper((double)lcur + eps);
            sims = 1;
        }
        int start = first_fail;
        bool more = __any_sync(FULL, tight);
        bool active_g = tight;
        while (more) {
            // lane-local pass over its j >= start with the current state
            int ev = NONE;
            if (active_g) {
                const double lc = (double)lcur;
                const bool ccok2 = use_cc && lc - eps >= 0.0;
                for (int r = 0; r < nrounds && ev == NONE; ++r) {
                    const int blk = r * 32 + q;
                    if (blk >= nb) break;
                    if (blk * EB + EB - 1 < start) continue;
                    for (int c2 = 0; c2 < EB; ++c2) {
                        const int j = blk * EB + c2;
                        if (j >= k) break;
                        if (j < start || j == ai || j == cur) continue;
                        if (ccok2 && (double)cc[(int64_t)cur * k + j] + kSqrt2 * eps <= lc - eps) continue;
                        if ((double)ui[j] + eps <= lc) continue;
                        if (my_sim[blk * ES + c2] > lcur) {
                            ev = j;
                            break;
                        }
                    }
                }
            }
            int gev = ev;
            for (int o = o0; o; o >>= 1) {
                const int other = __shfl_down_sync(FULL, gev, o);
                if (q < o && q + o < bpr) gev = min(gev, other);
            }
            gev = __shfl_sync(FULL, gev, lane - q);
            // commit every candidate in [start, gev) (and the event itself)
            if (active_g) {
                const double lc = (double)lcur;
                const bool ccok2 = use_cc && lc - eps >= 0.0;
                for (int r = 0; r < nrounds; ++r) {
                    const int blk = r * 32 + q;
                    if (blk >= nb) break;
                    if (blk * EB + EB - 1 < start || blk * EB > gev) continue;
                    for (int c2 = 0; c2 < EB; ++c2) {
                        const int j = blk * EB + c2;
                        if (j >= k || j > gev) break;
                        if (j < start || j == ai || j == cur) continue;
                        if (j < gev) {
                            if (ccok2 && (double)cc[(int64_t)cur * k + j] + kSqrt2 * eps <= lc - eps) continue;
                            if ((double)ui[j] + eps <= lc) continue;
                        }
                        ui[j] = store_upper((double)my_sim[blk * ES + c2] + eps);
                        ++sims;
                    }
                }
                if (gev != NONE) {
                    cur = gev;
                    lcur = my_sim[(gev >> (EB == 4 ? 2 : 3)) * ES + (gev & (EB - 1))];
                    start = gev + 1;
                } else {
                    active_g = false;
                }
            }
            more = __any_sync(FULL, active_g);
        }
        if (valid && q == 0 && tight) {
            l[i] = store_lower((double)lcur - eps);
            if (cur != ai) a[i] = cur;
        }
        const bool leader = valid && q == 0;
        warp_append(leader && cur != ai, i, mv_i, ai, mv_old, ctr + SPKM_CTR_MOVES);
        ctr_add(s_ctr, SPKM_CTR_SIMS, sims);
        ctr_add(s_ctr, SPKM_CTR_NNZ_ELKAN, leader ? (long long)len : 0);
        __syncwarp();
    }
    PDL_TRIGGER();
    ctr_flush(s_ctr, ctr);
}

// k <= 128 (4-center blocks, one round of lanes per row): the round-1 form
// of the scan -- blocks are fetched on the drift-updated u test and the
// tightened s~(i, a) is read from the fetched a(i) block inside the replay,
// instead of a separate tighten chain + compaction (k_elkan_scan), which
// only pays off with several rounds of blocks (C4).  C2: 1.75 -> ~1.36 ms
// per step of fused bound + scan passes.  Same results and counters.
template <int EB, bool FUSE>
__global__ void __launch_bounds__(256) k_elkan_scan_r1(const int64_t *__restrict__ indptr,
                                                    const int32_t *__restrict__ indices,
                                                    const float *__restrict__ values,
                                                    const float *__restrict__ reps,
                                                    const float *__restrict__ ct, int64_t kp, int k,
                                                    int32_t *a, float *l, float *u, int64_t ku,
                                                    const float *__restrict__ cc, int use_cc,
                                                    const int32_t *__restrict__ surv1, int32_t *mv_i,
                                                    int32_t *mv_old, long long *ctr, int64_t n_rows,
                                                    const double *__restrict__ drift,
                                                    const double *__restrict__ sinp,
                                                    const float *__restrict__ s_arr,
                                                    const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    constexpr int UB = 32 / EB;   // nnz per gather batch: 8 float4 loads in flight per lane
    constexpr int ES = EB + 1;    // padded per-block stride of the similarity buffer
    __shared__ __align__(16) int2 s_iv[8][8][kIvStride];
    __shared__ unsigned long long s_ctr[8];
    ctr_init(s_ctr);
    extern __shared__ float s_sim_dyn[];   // [8 warps][sim_stride]
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nb = (k + EB - 1) / EB;
    const int bpr = nb < 32 ? nb : 32;
    const int ppw = min(8, 32 / bpr);
    const int nrounds = (nb + 31) >> 5;
    const int g = lane / bpr, q = lane - g * bpr;
    const bool lane_on = g < ppw;
    const int o0 = bpr > 1 ? (1 << (31 - __clz(bpr - 1))) : 0;
    const int sim_stride = (int)elkan_sim_stride(k);  // floats per warp
    const int gstride = sim_stride / ppw;             // per-group slice (>= ES * nb)
    float *my_sim = s_sim_dyn + wib * sim_stride + (lane_on ? g : 0) * gstride;
    int2 *my_iv = s_iv[wib][lane_on ? g : 0];
    const long long cnt = FUSE ? n_rows : ctr[SPKM_CTR_SURV1];
    const int64_t nslots = (cnt + ppw - 1) / ppw;
    const int wpb = blockDim.x >> 5;
    for (int64_t w = (int64_t)blockIdx.x * wpb + wib; w < nslots; w += (int64_t)gridDim.x * wpb) {
        const int64_t slot = w * ppw + g;
        bool valid = lane_on && slot < cnt;
        const int32_t i = valid ? (FUSE ? (int32_t)slot : surv1[slot]) : 0;
        const int ai = valid ? a[i] : 0;
        float *ui = u + (int64_t)i * ku;
        const double eps = valid ? (double)reps[i] : 0.0;
        double lb;
        if constexpr (FUSE) {
            // k_elkan_bounds for this row (engine.py:274-283 + kernels.py:35-47)
            const float lo = valid ? l[i] : 0.f;
            float lf = lo;
            const double sa = valid ? sinp[ai] : 0.0;
            if (sa != 0.0) {
                const double pa = drift[ai];
                lf = store_lower((lo < -pa) ? -1.0 : d_clamp((double)lo * pa - d_sin((double)lo) * sa));
            }
            if (valid && q == 0 && lf != lo) l[i] = lf;
            lb = (double)lf;
            const bool pskip = use_cc && lb >= 0.0 && (double)s_arr[ai] + kSqrt2 * eps <= lb;
            const bool cc_on = use_cc && lb >= 0.0;
            const float thu = thr_u_of(lb, eps), thc = thr_c_of(lb, eps);
            bool surv = false;
            for (int r = 0; r < nrounds && valid; ++r) {
                const int blk = r * 32 + q;
                if (blk >= nb) break;
                for (int c2 = 0; c2 < EB; ++c2) {
                    const int j = blk * EB + c2;
                    if (j >= k) break;
                    float wv = ui[j];
                    const double sj = sinp[j];
                    if (sj != 0.0) {   // the k_elkan_bounds update, same float32 arithmetic
                        const double pj = drift[j];
                        wv = elkan_u_drift(wv, __double2float_rd(pj), __double2float_ru(pj), __double2float_ru(sj));
                        ui[j] = wv;
                    }
                    if (!pskip && j != ai) {
                        bool skip = cc_on && __ldg(cc + (int64_t)ai * k + j) <= thc;
                        if (!skip) skip = wv <= thu;
                        surv |= !skip;
                    }
                }
            }
            // the row survives if any of its lanes found a center it cannot prune
            const unsigned m = __ballot_sync(FULL, surv);
            const unsigned gmask = (bpr >= 32 ? 0xffffffffu : ((1u << bpr) - 1u)) << (lane_on ? g * bpr : 0);
            valid = valid && (m & gmask) != 0;
            ctr_add(s_ctr, SPKM_CTR_SURV1, (valid && q == 0) ? 1 : 0);
        } else {
            lb = valid ? (double)l[i] : 0.0;
        }
        const int64_t s = valid ? indptr[i] : 0, e = valid ? indptr[i + 1] : 0;
        const int len = (int)(e - s);
        const int maxlen = (int)__reduce_max_sync(FULL, (unsigned)len);
        const bool cc_ok = use_cc && lb >= 0.0;
        for (int r = 0; r < nrounds; ++r) {
            const int blk = r * 32 + q;
            const int j0 = blk * EB;
            bool act = false;
            if (valid && blk < nb) {
                for (int c2 = 0; c2 < EB; ++c2) {
                    const int j = j0 + c2;
                    if (j >= k) break;
                    if (j == ai) {
                        act = true;
                        continue;
                    }
                    // u-test only: a center the replay may need fails it (the
                    // cc test depends on the running best, so it cannot
                    // prune the fetch)
                    act |= !((double)ui[j] + 2.0 * eps <= lb);
                }
            }
            if (!__any_sync(FULL, act)) continue;
            float acc[EB];
#pragma unroll
            for (int c2 = 0; c2 < EB; ++c2) acc[c2] = 0.f;
            const float4 *base4 = reinterpret_cast<const float4 *>(ct + j0);
            for (int c0 = 0; c0 < maxlen; c0 += 32) {
                const int cntc = max(0, min(32, len - c0));
                for (int q2 = q; q2 < cntc; q2 += bpr)
                    my_iv[q2] = make_int2(__ldg(indices + s + c0 + q2), __float_as_int(__ldg(values + s + c0 + q2)));
                __syncwarp();
                if (act && EB == 8) {   // two float4 (one sector) per lane and nnz
                    int uu = 0;
                    for (; uu + UB <= cntc; uu += UB) {
                        float4 x[UB][2];
                        float vv[UB];
                        int iv[UB];
                        load_iv<UB>(my_iv + uu, iv, vv);
#pragma unroll
                        for (int b = 0; b < UB; ++b) {
                            const float4 *p = base4 + ((int64_t)iv[b] * kp >> 2);
                            x[b][0] = __ldg(p);
                            x[b][1] = __ldg(p + 1);
                        }
#pragma unroll
                        for (int b = 0; b < UB; ++b) {
                            acc[0] = __fmaf_rn(vv[b], x[b][0].x, acc[0]);
                            acc[1] = __fmaf_rn(vv[b], x[b][0].y, acc[1]);
                            acc[2] = __fmaf_rn(vv[b], x[b][0].z, acc[2]);
                            acc[3] = __fmaf_rn(vv[b], x[b][0].w, acc[3]);
                            acc[EB > 4 ? 4 : 0] = __fmaf_rn(vv[b], x[b][1].x, acc[EB > 4 ? 4 : 0]);
                            acc[EB > 4 ? 5 : 1] = __fmaf_rn(vv[b], x[b][1].y, acc[EB > 4 ? 5 : 1]);
                            acc[EB > 4 ? 6 : 2] = __fmaf_rn(vv[b], x[b][1].z, acc[EB > 4 ? 6 : 2]);
                            acc[EB > 4 ? 7 : 3] = __fmaf_rn(vv[b], x[b][1].w, acc[EB > 4 ? 7 : 3]);
                        }
                    }
                    for (; uu < cntc; ++uu) {
                        const int2 t = my_iv[uu];
                        const float v0 = __int_as_float(t.y);
                        const float4 *p = base4 + ((int64_t)t.x * kp >> 2);
                        const float4 x0 = __ldg(p), x1 = __ldg(p + 1);
                        acc[0] = __fmaf_rn(v0, x0.x, acc[0]);
                        acc[1] = __fmaf_rn(v0, x0.y, acc[1]);
                        acc[2] = __fmaf_rn(v0, x0.z, acc[2]);
                        acc[3] = __fmaf_rn(v0, x0.w, acc[3]);
                        acc[EB > 4 ? 4 : 0] = __fmaf_rn(v0, x1.x, acc[EB > 4 ? 4 : 0]);
                        acc[EB > 4 ? 5 : 1] = __fmaf_rn(v0, x1.y, acc[EB > 4 ? 5 : 1]);
                        acc[EB > 4 ? 6 : 2] = __fmaf_rn(v0, x1.z, acc[EB > 4 ? 6 : 2]);
                        acc[EB > 4 ? 7 : 3] = __fmaf_rn(v0, x1.w, acc[EB > 4 ? 7 : 3]);
                    }
                } else if (act) {   // EB == 4: one float4 per lane and nnz
                    int uu = 0;
                    for (; uu + UB <= cntc; uu += UB) {
                        float4 x[UB];
                        float vv[UB];
                        int iv[UB];
                        load_iv<UB>(my_iv + uu, iv, vv);
#pragma unroll
                        for (int b = 0; b < UB; ++b) x[b] = __ldg(base4 + ((int64_t)iv[b] * kp >> 2));
#pragma unroll
                        for (int b = 0; b < UB; ++b) {
                            acc[0] = __fmaf_rn(vv[b], x[b].x, acc[0]);
                            acc[1] = __fmaf_rn(vv[b], x[b].y, acc[1]);
                            acc[2] = __fmaf_rn(vv[b], x[b].z, acc[2]);
                            acc[3] = __fmaf_rn(vv[b], x[b].w, acc[3]);
                        }
                    }
                    for (; uu < cntc; ++uu) {
                        const int2 t = my_iv[uu];
                        const float v0 = __int_as_float(t.y);
                        const float4 x0 = __ldg(base4 + ((int64_t)t.x * kp >> 2));
                        acc[0] = __fmaf_rn(v0, x0.x, acc[0]);
                        acc[1] = __fmaf_rn(v0, x0.y, acc[1]);
                        acc[2] = __fmaf_rn(v0, x0.z, acc[2]);
                        acc[3] = __fmaf_rn(v0, x0.w, acc[3]);
                    }
                }
                __syncwarp();
            }
            if (act) {
#pragma unroll
                for (int c2 = 0; c2 < EB; ++c2) my_sim[blk * ES + c2] = acc[c2];
            }
        }
        __syncwarp();
        // replay of kernels.py:35-65, parallel over the group's lanes.  Lane q
        // owns the centers of blocks q, q+32, ... (ascending j within the
        // lane).  (A) tighten at the first j failing the pre-tests; (B) with
        // the running best (cur, lcur) every lane finds its candidates and
        // its first "event" (candidate beating lcur); the earliest event of
        // the group updates (cur, lcur) and the scan resumes after it.
        // Between events the state is constant, so the candidate set and the
        // reassignments equal the reference's sequential loop.
        int cur = ai;
        float lcur = 0.f;
        long long sims = 0;
        constexpr int NONE = 0x7fffffff;
        int first_fail = NONE;
        if (valid) {
            for (int r = 0; r < nrounds && first_fail == NONE; ++r) {
                const int blk = r * 32 + q;
                if (blk >= nb) break;
                for (int c2 = 0; c2 < EB; ++c2) {
                    const int j = blk * EB + c2;
                    if (j >= k) break;
                    if (j == ai) continue;
                    if (cc_ok && (double)cc[(int64_t)ai * k + j] + kSqrt2 * eps <= lb) continue;
                    if ((double)ui[j] + 2.0 * eps <= lb) continue;
                    first_fail = j;
                    break;
                }
            }
        }
        // group min (lanes of other groups hold their own values)
        for (int o = o0; o; o >>= 1) {
            const int other = __shfl_down_sync(FULL, first_fail, o);
            if (q < o && q + o < bpr) first_fail = min(first_fail, other);
        }
        first_fail = __shfl_sync(FULL, first_fail, lane - q);
        const bool tight = valid && first_fail != NONE;
        if (tight) {
            lcur = my_sim[(ai >> (EB == 4 ? 2 : 3)) * ES + (ai & (EB - 1))];
            if (q == 0) {
                ui[ai] = store_upper((double)lcur + eps);
                sims = 1;
            }
        }
        int start = first_fail;
        bool more = __any_sync(FULL, tight);
        bool active_g = tight;
        while (more) {
            // lane-local pass over its j >= start with the current state
            int ev = NONE;
            if (active_g) {
                const double lc = (double)lcur;
                const bool ccok2 = use_cc && lc - eps >= 0.0;
                for (int r = 0; r < nrounds && ev == NONE; ++r) {
                    const int blk = r * 32 + q;
                    if (blk >= nb) break;
                    if (blk * EB + EB - 1 < start) continue;
                    for (int c2 = 0; c2 < EB; ++c2) {
                        const int j = blk * EB + c2;
                        if (j >= k) break;
                        if (j < start || j == ai || j == cur) continue;
                        if (ccok2 && (double)cc[(int64_t)cur * k + j] + kSqrt2 * eps <= lc - eps) continue;
                        if ((double)ui[j] + eps <= lc) continue;
                        if (my_sim[blk * ES + c2] > lcur) {
                            ev = j;
                            break;
                        }
                    }
                }
            }
            int gev = ev;
            for (int o = o0; o; o >>= 1) {
                const int other = __shfl_down_sync(FULL, gev, o);
                if (q < o && q + o < bpr) gev = min(gev, other);
            }
            gev = __shfl_sync(FULL, gev, lane - q);
            // commit every candidate in [start, gev) (and the event itself)
            if (active_g) {
                const double lc = (double)lcur;
                const bool ccok2 = use_cc && lc - eps >= 0.0;
                for (int r = 0; r < nrounds; ++r) {
                    const int blk = r * 32 + q;
                    if (blk >= nb) break;
                    if (blk * EB + EB - 1 < start || blk * EB > gev) continue;
                    for (int c2 = 0; c2 < EB; ++c2) {
                        const int j = blk * EB + c2;
                        if (j >= k || j > gev) break;
                        if (j < start || j == ai || j == cur) continue;
                        if (j < gev) {
                            if (ccok2 && (double)cc[(int64_t)cur * k + j] + kSqrt2 * eps <= lc - eps) continue;
                            if ((double)ui[j] + eps <= lc) continue;
                        }
                        ui[j] = store_upper((double)my_sim[blk * ES + c2] + eps);
                        ++sims;
                    }
                }
                if (gev != NONE) {
                    cur = gev;
                    lcur = my_sim[(gev >> (EB == 4 ? 2 : 3)) * ES + (gev & (EB - 1))];
                    start = gev + 1;
                } else {
                    active_g = false;
                }
            }
            more = __any_sync(FULL, active_g);
        }
        if (valid && q == 0 && tight) {
            l[i] = store_lower((double)lcur - eps);
            if (cur != ai) a[i] = cur;
        }
        const bool leader = valid && q == 0;
        warp_append(leader && cur != ai, i, mv_i, ai, mv_old, ctr + SPKM_CTR_MOVES);
        ctr_add(s_ctr, SPKM_CTR_SIMS, sims);
        ctr_add(s_ctr, SPKM_CTR_NNZ_ELKAN, leader ? (long long)len : 0);
        __syncwarp();
    }
    PDL_TRIGGER();
    ctr_flush(s_ctr, ctr);
}


// ------------------------------------------------ sparse center index
// spkm_cindex_build, one pass over ct32: a CTA takes 8 term rows per round
// (warp per row, float4 per lane, 128 columns per step).  Each warp counts its
// row's nonzero centers; the CTA reserves the pairs of its sparse rows (count
// <= thr) with ONE atomic on the running total; each warp then re-reads its
// row (4 KB, still in L1) and writes its (j, value) pairs in j order and
// desc[t] = offset << 12 | count (0xFFF: dense row).  Where a row's pairs
// land depends on the atomic order; the row's pairs, their order and so every
// result do not.  (A count kernel + CUB scan + fill kernel read the 4 GB
// table twice: 1.8 ms per build at C4 against 0.7.)
__global__ void __launch_bounds__(256) k_ci_build(int64_t d, int64_t kp, int k, const float *__restrict__ ct, int thr,
                                                  unsigned long long *total, int64_t *desc, int2 *pairs,
                                                  const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;
    __shared__ int s_c[8];
    __shared__ int s_off[8];
    __shared__ long long s_base;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int64_t t0 = (int64_t)blockIdx.x * 8; t0 < d; t0 += (int64_t)gridDim.x * 8) {
        const int64_t t = t0 + wib;
        const float *row = ct + t * kp;
        int c = 0;
        if (t < d) {
            for (int j0 = 4 * lane; j0 < k; j0 += 128) {
                const float4 v = __ldg(reinterpret_cast<const float4 *>(row + j0));
                c += (v.x != 0.f) + (j0 + 1 < k && v.y != 0.f) + (j0 + 2 < k && v.z != 0.f) + (j0 + 3 < k && v.w != 0.f);
            }
        }
        c = (int)__reduce_add_sync(FULL, (unsigned)c);
        const bool sparse = t < d && c <= thr;
        if (lane == 0) s_c[wib] = sparse ? c : 0;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                s_off[w] = tot;
                tot += s_c[w];
            }
            s_base = tot ? (long long)atomicAdd(total, (unsigned long long)tot) : 0;
        }
        __syncthreads();
        const int64_t base = s_base + s_off[wib];
        if (t >= d) continue;           // (every warp still reaches the barriers of the next round: t0 is CTA-uniform)
        if (!sparse) {
            if (lane == 0) desc[t] = 0xFFF;
            continue;
        }
        int pos = 0;
        for (int j0 = 4 * lane, jb = 0; jb < k; j0 += 128, jb += 128) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (j0 < k) v = __ldg(reinterpret_cast<const float4 *>(row + j0));
            const float vv[4] = {v.x, v.y, v.z, v.w};
            int m = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) m += (j0 + q < k && vv[q] != 0.f);
            int x = m;   // inclusive prefix over the lanes
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, x, o);
                if (lane >= o) x += y;
            }
            int w = pos + x - m;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (j0 + q < k && vv[q] != 0.f) pairs[base + w++] = make_int2(j0 + q, __float_as_int(vv[q]));
            pos += __shfl_sync(FULL, x, 31);
        }
        DCHECK(pos == c);
        if (lane == 0) desc[t] = (base << 12) | (int64_t)c;
    }
    PDL_TRIGGER();
}

// ------------------------------------------------------ Yin-Yang family
// Group bounds (Ding et al., ICML 2015, carried over to cosine similarities
// as the paper says its bounds transfer: PAPER.md:409-414, 667-671) with the
// groups = blocks of 4 consecutive centers (one float4 of a term-major ct32
// row, the gather unit of the scans).  Per point: a(i), l(i) <= <x_i, c_a>,
// ug(i, g) >= max over j in g, j != a(i) of <x_i, c_j>  (n x ceil(k/4)
// floats: a quarter of Elkan's n x k).  Per iteration:
//   * drift update: l by a(i)'s own drift (engine.py:274), ug(i, g) by the
//     group's worst drift (min p_j, max sin_p over the group; Eq. 9 as the
//     Elkan u update, kernels.py:35-47 via engine.py:281-283);
//   * a point survives if some group may beat l: ug + 2 eps > l;
//   * survivors: tighten s~(i, a), fetch every group with ug + eps >
//     s~(i, a) (its 4 canonical similarities), take the best (strict >
//     beats the incumbent, ties to the lowest index: the Lloyd rule), and
//     recompute the bounds of the fetched groups exactly.
// Skips only what is provably <= s~(i, a) with the same eps margins as the
// Elkan kernels, so every fit equals the GPU Lloyd bit for bit.
constexpr int kYyMaxGroups = 256;   // k <= 1024
__global__ void __launch_bounds__(256) k_yy_bounds(int64_t n, int k, const float *__restrict__ reps,
                                                   const int32_t *__restrict__ a, float *l, float *ug, int64_t gp,
                                                   const double *__restrict__ drift,
                                                   const double *__restrict__ sinp, int32_t *surv1, long long *ctr,
                                                   const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    __shared__ __align__(16) float s_pd[kYyMaxGroups], s_pu[kYyMaxGroups], s_su[kYyMaxGroups];
    const int ng = (k + 3) >> 2;
    const int g4 = (ng + 3) >> 2;
    for (int g = threadIdx.x; g < 4 * g4; g += blockDim.x) {
        double pmin = 1.0, smax = 0.0;
        for (int c = 0; c < 4; ++c) {
            const int j = 4 * g + c;
            if (g < ng && j < k) {
                pmin = fmin(pmin, drift[j]);
                smax = fmax(smax, sinp[j]);
            }
        }
        s_pd[g] = __double2float_rd(pmin);
        s_pu[g] = __double2float_ru(pmin);
        s_su[g] = __double2float_ru(smax);
    }
    __syncthreads();
    const float4 *pd4 = reinterpret_cast<const float4 *>(s_pd), *pu4 = reinterpret_cast<const float4 *>(s_pu),
                 *su4 = reinterpret_cast<const float4 *>(s_su);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int64_t nchunks = (n + 31) >> 5;
    __shared__ int s_cnt[8];
    __shared__ long long s_base;
    for (int64_t c0 = (int64_t)blockIdx.x * wpb; c0 < nchunks; c0 += (int64_t)gridDim.x * wpb) {
        const int64_t c = c0 + wib;
        const int64_t rb = c << 5;
        const int64_t ir = rb + lane;
        float thu_r = 0.f;
        if (c < nchunks && ir < n) {
            const int ai = a[ir];
            const float lo = l[ir];
            float lf = lo;
            const double sa = sinp[ai];
            if (sa != 0.0) {
                const double pa = drift[ai];
                lf = store_lower((lo < -pa) ? -1.0 : d_clamp((double)lo * pa - d_sin((double)lo) * sa));
                l[ir] = lf;
            }
            thu_r = thr_u_of((double)lf, (double)reps[ir]);
        }
        const int nr = c < nchunks ? (int)min((int64_t)32, n - rb) : 0;
        unsigned smask = 0;
        for (int r = 0; r < nr; ++r) {
            const float thu = __shfl_sync(FULL, thu_r, r);
            float4 *gi = reinterpret_cast<float4 *>(ug + (rb + r) * gp);
            bool any = false;
            for (int q = lane; q < g4; q += 32) {
                float4 v = gi[q];
                const float4 su = su4[q];
                if (su.x != 0.f || su.y != 0.f || su.z != 0.f || su.w != 0.f) {
                    const float4 pd = pd4[q], pu = pu4[q];
                    v.x = su.x != 0.f ? elkan_u_drift(v.x, pd.x, pu.x, su.x) : v.x;
                    v.y = su.y != 0.f ? elkan_u_drift(v.y, pd.y, pu.y, su.y) : v.y;
                    v.z = su.z != 0.f ? elkan_u_drift(v.z, pd.z, pu.z, su.z) : v.z;
                    v.w = su.w != 0.f ? elkan_u_drift(v.w, pd.w, pu.w, su.w) : v.w;
                    gi[q] = v;        // padding groups (g >= ng) have su == 0: never rewritten
                }
                const int gb = 4 * q;
                any |= (gb + 0 < ng && v.x > thu) || (gb + 1 < ng && v.y > thu) || (gb + 2 < ng && v.z > thu) ||
                       (gb + 3 < ng && v.w > thu);
            }
            if (__any_sync(FULL, any)) smask |= 1u << r;
        }
        // one global atomic per CTA round: warp counts -> shared prefix
        if (lane == 0) s_cnt[wib] = __popc(smask);
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < wpb; ++w) {
                const int t = s_cnt[w];
                s_cnt[w] = tot;
                tot += t;
            }
            s_base = tot ? (long long)atomicAdd((unsigned long long *)(ctr + SPKM_CTR_SURV1), (unsigned long long)tot)
                         : 0ll;
        }
        __syncthreads();
        if (smask >> lane & 1u) surv1[s_base + s_cnt[wib] + __popc(smask & ((1u << lane) - 1u))] = (int32_t)ir;
        __syncthreads();
    }
    PDL_TRIGGER();
}

// floats of the per-warp similarity buffer of k_yy_scan: 4 per group and point
__host__ __device__ __forceinline__ int yy_sim_stride(int64_t k) {
    const int ng = (int)((k + 3) / 4);
    const int bpr = ng < 32 ? ng : 32;
    const int ppw = (32 / bpr) < 8 ? (32 / bpr) : 8;
    return 4 * ng * ppw;
}
// Survivor scan: lanes = groups (bpr lanes per point, up to 8 points per
// warp, rounds of 32 groups), the gather machinery of k_elkan_scan<4>.
#ifndef SPKM_YY_MINB
#define SPKM_YY_MINB 4        // 64 registers (C4 yy_scan 2492 -> 2423 ms per fit)
#endif
__global__ void __launch_bounds__(256, SPKM_YY_MINB) k_yy_scan(const int64_t *__restrict__ indptr,
                                                 const int32_t *__restrict__ indices,
                                                 const float *__restrict__ values, const float *__restrict__ reps,
                                                 const float *__restrict__ ct, int64_t kp, int k, int32_t *a,
                                                 float *l, float *ug, int64_t gp,
                                                 const int32_t *__restrict__ surv1, int32_t *mv_i, int32_t *mv_old,
                                                 long long *ctr, const long long *__restrict__ ctl, int64_t hot) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
    constexpr int UB = 8;     // nnz per gather batch: 8 float4 loads in flight per lane
    __shared__ int s_act[8][kYyMaxGroups];
    extern __shared__ float s_sim_yy[];    // [8 warps][yy_sim_stride(k)]
    __shared__ unsigned long long s_ctr[8];
    ctr_init(s_ctr);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int ng = (k + 3) >> 2;
    const int bpr = ng < 32 ? ng : 32;
    const int ppw = min(8, 32 / bpr);
    const int nrounds = (ng + 31) >> 5;
    const int g = lane / bpr, q = lane - g * bpr;
    const bool lane_on = g < ppw;
    const int o0 = bpr > 1 ? (1 << (31 - __clz(bpr - 1))) : 0;
    float *my_sim = s_sim_yy + wib * yy_sim_stride(k) + (lane_on ? g : 0) * 4 * ng;   // 4 per group and point
    int *my_act = s_act[wib] + (lane_on ? g : 0) * (kYyMaxGroups / ppw);
    // staged (id, value) pairs after the similarity buffers: ppw row groups per warp
    int2 *my_iv = reinterpret_cast<int2 *>(s_sim_yy + 8 * yy_sim_stride(k)) + (wib * ppw + (lane_on ? g : 0)) * kIvStride;
    const long long cnt = ctr[SPKM_CTR_SURV1];
    const int64_t nslots = (cnt + ppw - 1) / ppw;
    const int wpb = blockDim.x >> 5;
    const unsigned gmask_lo = bpr >= 32 ? 0xffffffffu : ((1u << bpr) - 1u);
    for (int64_t w = (int64_t)blockIdx.x * wpb + wib; w < nslots; w += (int64_t)gridDim.x * wpb) {
        const int64_t slot = w * ppw + g;
        const bool valid = lane_on && slot < cnt;
        const int32_t i = valid ? surv1[slot] : 0;
        const int ai = valid ? a[i] : 0;
        float *gi = ug + (int64_t)i * gp;
        const double eps = valid ? (double)reps[i] : 0.0;
        const int64_t s = valid ? indptr[i] : 0, e = valid ? indptr[i + 1] : 0;
        const int len = (int)(e - s);
        // (A) tighten: s~(i, a(i)), the canonical chain for the single center a(i)
        float lcur = 0.f;
        {
            const int maxt = (int)__reduce_max_sync(FULL, (unsigned)len);
            float acc = 0.f;
            const float *cta = ct + ai;
            for (int c0 = 0; c0 < maxt; c0 += 32) {
                const int cntc = max(0, min(32, len - c0));
                for (int q2 = q; q2 < cntc; q2 += bpr) {
                    const int t = __ldg(indices + s + c0 + q2);
                    const float cv = ldg_hint(cta + (int64_t)t * kp, t < hot ? pol_hot : pol_cold);
                    my_iv[q2] = make_int2(__float_as_int(__ldg(values + s + c0 + q2)), __float_as_int(cv));
                }
                __syncwarp();
                if (q == 0)
                    for (int t = 0; t < cntc; ++t)
                        acc = __fmaf_rn(__int_as_float(my_iv[t].x), __int_as_float(my_iv[t].y), acc);
                __syncwarp();
            }
            lcur = __shfl_sync(FULL, acc, lane - q);
        }
        // (B) groups to fetch: ug + eps > s~(i, a), compacted per point
        int nact = 0;
        {
            const double lc = (double)lcur;
            for (int r = 0; r < nrounds; ++r) {
                const int gr = r * 32 + q;
                const bool act = valid && gr < ng && !((double)gi[gr] + eps <= lc);
                const unsigned m = __ballot_sync(FULL, act);
                const unsigned gm = (m >> (lane - q)) & gmask_lo;
                if (act) my_act[nact + __popc(gm & ((1u << q) - 1u))] = gr;
                nact += __popc(gm);
            }
        }
        DCHECK(nact <= ng);
        __syncwarp();
        // (C) the 4 canonical similarities of every active group
        const int act_rounds = (int)__reduce_max_sync(FULL, (unsigned)((nact + bpr - 1) / bpr));
        const int maxlen = (int)__reduce_max_sync(FULL, (unsigned)(nact ? len : 0));
        const float4 *base4 = reinterpret_cast<const float4 *>(ct);
        for (int r = 0; r < act_rounds; ++r) {
            const int sb = r * bpr + q;
            const bool act = lane_on && sb < nact;
            const int gr = act ? my_act[sb] : 0;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            const int glen = nact > r * bpr ? len : 0;
            for (int c0 = 0; c0 < maxlen; c0 += 32) {
                const int cntc = max(0, min(32, glen - c0));
                for (int q2 = q; q2 < cntc; q2 += bpr)
                    my_iv[q2] = make_int2(__ldg(indices + s + c0 + q2), __float_as_int(__ldg(values + s + c0 + q2)));
                __syncwarp();
                if (act) {
                    int uu = 0;
                    for (; uu + UB <= cntc; uu += UB) {
                        float4 x[UB];
                        float vv[UB];
                        int iv[UB];
                        load_iv<UB>(my_iv + uu, iv, vv);
#pragma unroll
                        for (int b = 0; b < UB; ++b)
                            x[b] = ldg_hint(base4 + (((int64_t)iv[b] * kp) >> 2) + gr, iv[b] < hot ? pol_hot : pol_cold);
#pragma unroll
                        for (int b = 0; b < UB; ++b) {
                            acc[0] = __fmaf_rn(vv[b], x[b].x, acc[0]);
                            acc[1] = __fmaf_rn(vv[b], x[b].y, acc[1]);
                            acc[2] = __fmaf_rn(vv[b], x[b].z, acc[2]);
                            acc[3] = __fmaf_rn(vv[b], x[b].w, acc[3]);
                        }
                    }
                    for (; uu < cntc; ++uu) {
                        const int2 t = my_iv[uu];
                        const float v0 = __int_as_float(t.y);
                        const float4 x0 = ldg_hint(base4 + (((int64_t)t.x * kp) >> 2) + gr, t.x < hot ? pol_hot : pol_cold);
                        acc[0] = __fmaf_rn(v0, x0.x, acc[0]);
                        acc[1] = __fmaf_rn(v0, x0.y, acc[1]);
                        acc[2] = __fmaf_rn(v0, x0.z, acc[2]);
                        acc[3] = __fmaf_rn(v0, x0.w, acc[3]);
                    }
                }
                __syncwarp();
            }
            if (act) {
#pragma unroll
                for (int c = 0; c < 4; ++c) my_sim[4 * sb + c] = acc[c];
            }
        }
        __syncwarp();
        // (D) the best candidate (larger value, ties to the lower index), then
        // the incumbent rule: strictly greater than s~(i, a) to move
        float bs = -INFINITY;
        int bj = 0x7fffffff;
        long long sims = 0;
        for (int sb = q; sb < nact; sb += bpr) {
            const int gr = my_act[sb];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int j = 4 * gr + c;
                if (j >= k || j == ai) continue;
                ++sims;
                const float v = my_sim[4 * sb + c];
                if (v > bs || (v == bs && j < bj)) {
                    bs = v;
                    bj = j;
                }
            }
        }
        for (int o = o0; o; o >>= 1) {
            const float ov = __shfl_down_sync(FULL, bs, o);
            const int oj = __shfl_down_sync(FULL, bj, o);
            if (q < o && q + o < bpr && (ov > bs || (ov == bs && oj < bj))) {
                bs = ov;
                bj = oj;
            }
        }
        bs = __shfl_sync(FULL, bs, lane - q);
        bj = __shfl_sync(FULL, bj, lane - q);
        const int b = (valid && bs > lcur) ? bj : ai;
        const float sb_val = b == ai ? lcur : bs;
        // (E) bounds: fetched groups exactly (max over j != b), a(i)'s group
        // when it was not fetched and a(i) lost the point gains s~(i, a)
        for (int sb = q; sb < nact; sb += bpr) {
            const int gr = my_act[sb];
            float m = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int j = 4 * gr + c;
                if (j < k && j != b) m = fmaxf(m, my_sim[4 * sb + c]);
            }
            gi[gr] = (m == -INFINITY) ? -1.f : store_upper((double)m + eps);
        }
        const bool leader = valid && q == 0;
        if (leader) {
            l[i] = store_lower((double)sb_val - eps);
            if (b != ai) {
                a[i] = b;
                const int ga = ai >> 2;
                bool fetched = false;
                for (int sb = 0; sb < nact; ++sb) fetched |= my_act[sb] == ga;
                if (!fetched) gi[ga] = fmaxf(gi[ga], store_upper((double)lcur + eps));
            }
        }
        warp_append(leader && b != ai, i, mv_i, ai, mv_old, ctr + SPKM_CTR_MOVES);
        ctr_add(s_ctr, SPKM_CTR_SIMS, sims + (leader ? 1 : 0));
        ctr_add(s_ctr, SPKM_CTR_NNZ_ELKAN, leader ? (long long)len : 0);
        __syncwarp();
    }
    PDL_TRIGGER();
    ctr_flush(s_ctr, ctr);
}

// --------------------------------------------------------- center updates
__device__ __forceinline__ long long to_fixed(float v, double scale) { return __double2ll_rn((double)v * scale); }

// engine._aggregate_sums (engine.py:130-139): warp per row, lanes over nnz.
__global__ void __launch_bounds__(256) k_aggregate(int64_t n, int64_t d, const int64_t *__restrict__ indptr,
                                                   const int32_t *__restrict__ indices,
                                                   const float *__restrict__ values,
                                                   const int32_t *__restrict__ a, long long *sums,
                                                   long long *counts, double scale, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    for (int64_t i = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); i < n; i += (int64_t)gridDim.x * wpb) {
        const int ai = a[i];
        long long *sj = sums + (int64_t)ai * d;
        for (int64_t t = indptr[i] + lane; t < indptr[i + 1]; t += 32) {
            DCHECK((uint64_t)__ldg(indices + t) < (uint64_t)d);
            atomicAdd((unsigned long long *)(sj + __ldg(indices + t)), (unsigned long long)to_fixed(__ldg(values + t), scale));
        }
        if (lane == 0) atomicAdd((unsigned long long *)(counts + ai), 1ull);
    }
}

// engine.update_centers incremental branch (engine.py:174-188).
__global__ void __launch_bounds__(256) k_apply_moves(int64_t d, const int64_t *__restrict__ indptr,
                                                     const int32_t *__restrict__ indices,
                                                     const float *__restrict__ values,
                                                     const int32_t *__restrict__ a,
                                                     const int32_t *__restrict__ mv_i,
                                                     const int32_t *__restrict__ mv_old,
                                                     long long *ctr, long long *sums,
                                                     long long *counts, int32_t *touched, double scale, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const long long cnt = ctr[SPKM_CTR_MOVES];
    long long nnz_moved = 0;   // one atomic per warp at the end
    for (int64_t w = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); w < cnt; w += (int64_t)gridDim.x * wpb) {
        const int32_t i = mv_i[w];
        const int o = mv_old[w], nw = a[i];
        long long *so = sums + (int64_t)o * d;
        long long *sn = sums + (int64_t)nw * d;
        for (int64_t t = indptr[i] + lane; t < indptr[i + 1]; t += 32) {
            const int c = __ldg(indices + t);
            DCHECK((uint64_t)c < (uint64_t)d && o >= 0 && nw >= 0);
            const long long q = to_fixed(__ldg(values + t), scale);
            atomicAdd((unsigned long long *)(so + c), (unsigned long long)(-q));
            atomicAdd((unsigned long long *)(sn + c), (unsigned long long)q);
        }
        if (lane == 0) {
            atomicAdd((unsigned long long *)(counts + o), (unsigned long long)(-1ll));
            atomicAdd((unsigned long long *)(counts + nw), 1ull);
            touched[o] = 1;
            touched[nw] = 1;
        }
        nnz_moved += indptr[i + 1] - indptr[i];
    }
    if (lane == 0 && nnz_moved) atomicAdd((unsigned long long *)(ctr + SPKM_CTR_NNZ_MOVED), (unsigned long long)nnz_moved);
}

// Fixed-shape block sum (deterministic for a given blockDim).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh) {
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(FULL, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = (threadIdx.x < NT / 32) ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) r += __shfl_down_sync(FULL, r, o);
    }
    return r;  // valid in thread 0
}

// ---------------------------------------------------- _move_centers pipeline
// engine.py:142-160 for the touched clusters T (all clusters in iteration 1):
//   list -> |sum_j|^2 partials -> norm_j -> write c_j (cent64 + term-major
//   ct32 through a shared-memory transpose) with partial chord^2 and
//   objective -> per-cluster reduction -> drift.
// The drift is carried as (p_j, sinp_j): p_j = 1 - |c_new - c_old|^2 / 2
// (exactly 1 for a bit-identical center) and sinp_j an UPPER bound on the
// sine of the rotation angle computed from the chord (no cancellation near
// p = 1, where sqrt(1 - p^2) would amplify float64 rounding).
constexpr int kTileT = 256;          // terms per write tile
constexpr int kTileJ = 32;           // clusters per write tile
constexpr double kChordPad = 4e-10;  // |1 - |c|| <= d * 2^-53 for d <= 1e6, twice

__global__ void k_touched_list(int64_t k, const int32_t *__restrict__ touched, int all, int32_t *tlist,
                               int32_t *tcount, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    __shared__ int wsum[32];
    __shared__ int base_s;
    if (threadIdx.x == 0) base_s = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t j0 = 0; j0 < k; j0 += blockDim.x) {
        const int64_t j = j0 + threadIdx.x;
        const int f = (j < k) && (all || touched[j]);
        const unsigned m = __ballot_sync(FULL, f);
        if (lane == 0) wsum[w] = __popc(m);
        __syncthreads();
        int off = base_s;
        for (int q = 0; q < w; ++q) off += wsum[q];
        if (f) tlist[off + __popc(m & ((1u << lane) - 1u))] = (int32_t)j;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int q = 0; q < nw; ++q) t += wsum[q];
            base_s += t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *tcount = base_s;
}

constexpr int kListInline = 2048;   // k up to this: the norm-part CTAs build the touched list themselves

// build_list: every CTA derives the touched list from the flags (k <= kListInline,
// a few flag loads per thread), takes its own entry, and the x == 0 column
// publishes it for the later kernels -- one launch (k_touched_list) less.
__global__ void __launch_bounds__(256) k_center_norm_part(int64_t d, int64_t nchunk,
                                                          const long long *__restrict__ sums,
                                                          int32_t *tlist, int32_t *tcount, double inv_scale,
                                                          double *part, int build_list, int64_t k,
                                                          const int32_t *__restrict__ touched, int all,
                                                          const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    __shared__ double sh[8];
    const int64_t y = blockIdx.y, c = blockIdx.x;
    int64_t j;
    if (build_list) {
        __shared__ int s_list[kListInline];
        __shared__ int wsum[8];
        __shared__ int base_s;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        if (threadIdx.x == 0) base_s = 0;
        __syncthreads();
        for (int64_t j0 = 0; j0 < k; j0 += blockDim.x) {
            const int64_t jj = j0 + threadIdx.x;
            const int f = (jj < k) && (all || touched[jj]);
            const unsigned m = __ballot_sync(FULL, f);
            if (lane == 0) wsum[w] = __popc(m);
            __syncthreads();
            int off = base_s;
            for (int q = 0; q < w; ++q) off += wsum[q];
            if (f) s_list[off + __popc(m & ((1u << lane) - 1u))] = (int)jj;
            __syncthreads();
            if (threadIdx.x == 0)
                for (int q = 0; q < 8; ++q) base_s += wsum[q];
            __syncthreads();
        }
        const int cnt = base_s;
        if (c == 0 && y == 0 && threadIdx.x == 0) *tcount = cnt;
        if (y >= cnt) return;
        j = s_list[y];
        if (c == 0 && threadIdx.x == 0) tlist[y] = (int32_t)j;
    } else {
        if (y >= *tcount) return;
        j = tlist[y];
    }
    const int64_t t0 = c * kCenterChunk, t1 = min(d, t0 + kCenterChunk);
    const long long *sj = sums + j * d;
    double acc = 0.0;
    for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        const long long q = sj[t];
        if (q) {
            const double v = (double)q * inv_scale;
            acc = fma(v, v, acc);
        }
    }
    const double r = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) part[y * nchunk + c] = r;
}

// norm_j = sqrt(sum of partials, fixed order); -1 = keep the old center
// (empty cluster or |sum| < 1e-12, engine.py:153-157).
__global__ void __launch_bounds__(256) k_center_norm_final(int64_t nchunk, const long long *__restrict__ counts,
                                                           const int32_t *__restrict__ tlist,
                                                           const int32_t *__restrict__ tcount,
                                                           const double *__restrict__ part, double *norm, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    __shared__ double sh[8];
    const int64_t y = blockIdx.x;
    if (y >= *tcount) return;
    double acc = 0.0;
    for (int64_t c = threadIdx.x; c < nchunk; c += blockDim.x) acc += part[y * nchunk + c];
    const double sq = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) {
        const int j = tlist[y];
        const double nrm = sqrt(sq);
        norm[j] = (counts[j] == 0 || nrm < kZeroSumEps) ? -1.0 : nrm;
    }
}

// Write tile: kTileJ listed clusters x kTileT terms.  Warp w owns clusters
// 4w..4w+3 of the tile; lanes stride the terms (coalesced int64/float64
// rows).  The float32 values are transposed through shared memory so each
// ct32 row segment (kTileJ consecutive clusters) is one coalesced store.
#define kKeep __int_as_float(0x7fc00abc)   // NaN payload no center value has
__global__ void __launch_bounds__(256) k_center_write(int64_t d, int64_t kp, int64_t ntile,
                                                      const long long *__restrict__ sums,
                                                      const int32_t *__restrict__ tlist,
                                                      const int32_t *__restrict__ tcount, double inv_scale,
                                                      const double *__restrict__ norm, double *cent64, float *ct32,
                                                      __half *ct16, double *part, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    __shared__ float tile[kTileT][kTileJ + 1];
    __shared__ int js[kTileJ];
    const int64_t nT = *tcount;
    const int64_t y0 = (int64_t)blockIdx.y * kTileJ;
    if (y0 >= nT) return;
    const int64_t t0 = (int64_t)blockIdx.x * kTileT;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x < kTileJ) js[threadIdx.x] = (y0 + threadIdx.x < nT) ? tlist[y0 + threadIdx.x] : -1;
    __syncthreads();
    constexpr int QN = kTileT / 32;   // terms per lane per cluster
#pragma unroll 1
    for (int r = 0; r < 4; ++r) {
        const int jr = w * 4 + r;
        const int j = js[jr];
        double ch = 0.0, ob = 0.0;
        if (j >= 0) {
            const double nrm = norm[j];
            const double inv_nrm = 1.0 / nrm;
            const long long *sj = sums + (int64_t)j * d;
            double *cj = cent64 + (int64_t)j * d;
            // all loads of this cluster's slice first (QN sums + QN old values
            // in flight per lane), then the arithmetic and the stores
            long long sv[QN];
            double ov[QN];
#pragma unroll
            for (int qi = 0; qi < QN; ++qi) {
                const int64_t t = t0 + lane + 32 * qi;
                sv[qi] = t < d ? __ldg(sj + t) : 0;
                ov[qi] = t < d ? cj[t] : 0.0;
            }
#pragma unroll
            for (int qi = 0; qi < QN; ++qi) {
                const int q = lane + 32 * qi;
                const int64_t t = t0 + q;
                // kKeep: the entry did not change (92% of a C4 center row is zero and stays zero), so the
                // term-major copies keep their value too and are not rewritten
                float f = kKeep;
                if (t < d) {
                    const double v = (double)sv[qi] * inv_scale;
                    const double old = ov[qi];
                    if (nrm < 0.0) {
                        ob = fma(v, old, ob);
                    } else {
                        const double nv = v * inv_nrm;
                        const double df = nv - old;
                        ch = fma(df, df, ch);
                        ob = fma(v, nv, ob);
                        if (nv != old) {
                            cj[t] = nv;
                            f = (float)nv;
                        }
                    }
                }
                tile[q][jr] = f;
            }
        } else {
            for (int q = lane; q < kTileT; q += 32) tile[q][jr] = kKeep;
        }
        for (int o = 16; o; o >>= 1) {
            ch += __shfl_down_sync(FULL, ch, o);
            ob += __shfl_down_sync(FULL, ob, o);
        }
        if (lane == 0 && j >= 0) {
            part[((y0 + jr) * ntile + blockIdx.x) * 2] = ch;
            part[((y0 + jr) * ntile + blockIdx.x) * 2 + 1] = ob;
        }
    }
    __syncthreads();
    // transpose out: warp w handles terms w, w+8, ...; lane = cluster slot
    const int j = js[lane];
    for (int q = w; q < kTileT; q += 8) {
        const int64_t t = t0 + q;
        if (t < d && j >= 0) {
            const float f = tile[q][lane];
            if (__float_as_int(f) != __float_as_int(kKeep)) {
                ct32[t * kp + j] = f;
                if (ct16) ct16[t * kp + j] = __float2half_rn(f);
            }
        }
    }
}

// per touched cluster: chord^2 -> (p, sin bound), objective term.
__global__ void __launch_bounds__(256) k_center_reduce(int64_t ntile, const int32_t *__restrict__ tlist,
                                                       const int32_t *__restrict__ tcount,
                                                       const double *__restrict__ part,
                                                       const double *__restrict__ norm, double *drift,
                                                       double *sinp, double *objc, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    __shared__ double sh[8];
    const int64_t y = blockIdx.x;
    if (y >= *tcount) return;
    double ch = 0.0, ob = 0.0;
    for (int64_t c = threadIdx.x; c < ntile; c += blockDim.x) {
        ch += part[(y * ntile + c) * 2];
        ob += part[(y * ntile + c) * 2 + 1];
    }
    const double rch = block_sum<256>(ch, sh);
    const double rob = block_sum<256>(ob, sh);
    if (threadIdx.x == 0) {
        const int j = tlist[y];
        objc[j] = rob;
        if (norm[j] < 0.0 || rch == 0.0) {
            drift[j] = 1.0;
            sinp[j] = 0.0;
        } else {
            const double chord = sqrt(rch);
            drift[j] = d_clamp(1.0 - 0.5 * rch);
            const double s = chord * sqrt(fmax(0.0, 1.0 - 0.25 * rch));
            sinp[j] = fmin(1.0, s * (1.0 + 1e-12) + kChordPad);
        }
    }
}

// Sum_j <sums_j, c_j> partials (compute_objective, engine.py:123-127).
__global__ void __launch_bounds__(256) k_objective_part(int64_t d, int64_t nchunk, const long long *__restrict__ sums,
                                                        const double *__restrict__ cent64, double inv_scale,
                                                        double *part) {
    __shared__ double sh[8];
    const int64_t j = blockIdx.y, c = blockIdx.x;
    const int64_t t0 = c * kCenterChunk, t1 = min(d, t0 + kCenterChunk);
    double ob = 0.0;
    for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x)
        ob = fma((double)sums[j * d + t] * inv_scale, cent64[j * d + t], ob);
    const double r = block_sum<256>(ob, sh);
    if (threadIdx.x == 0) part[(j * nchunk + c) * 2 + 1] = r;
}

__global__ void k_objective_final(int64_t k, int64_t nchunk, const double *__restrict__ part, double *out) {
    if (threadIdx.x != 0) return;
    double tot = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        double ob = 0.0;
        for (int64_t c = 0; c < nchunk; ++c) ob += part[(j * nchunk + c) * 2 + 1];
        tot += ob;
    }
    *out = tot;
}

// ------------------------------------------------------------ finalize
// drift of untouched clusters = 1 (engine.py:149), objective
// (engine.py:326), convergence inputs (engine.py:335-337), Hamerly
// aggregation (engine.py:285-289): owner = first argmin p, p_min, p_min2,
// plus the sine bounds smax = max_j sinp_j and smax2 = max over j != owner_s
// (owner_s = first argmax sinp).  hstat = {owner, p_min, p_min2, owner_s,
// smax, smax2}.
// Two smallest (value, index) pairs, ties broken by the lower index (the
// stable argsort order of engine.py:285).
struct Low2 {
    double v1;
    int i1;
    double v2;
    int i2;
};
__device__ __forceinline__ bool lt_vi(double v, int i, double w, int j) { return v < w || (v == w && i < j); }
__device__ __forceinline__ void low2_push(Low2 &t, double v, int i) {
    if (lt_vi(v, i, t.v1, t.i1)) {
        t.v2 = t.v1;
        t.i2 = t.i1;
        t.v1 = v;
        t.i1 = i;
    } else if (lt_vi(v, i, t.v2, t.i2)) {
        t.v2 = v;
        t.i2 = i;
    }
}
__device__ __forceinline__ void low2_merge(Low2 &t, const Low2 &o) {
    low2_push(t, o.v1, o.i1);
    low2_push(t, o.v2, o.i2);
}
__device__ __forceinline__ Low2 low2_shfl(const Low2 &t, int o) {
    return Low2{__shfl_down_sync(FULL, t.v1, o), __shfl_down_sync(FULL, t.i1, o), __shfl_down_sync(FULL, t.v2, o),
                __shfl_down_sync(FULL, t.i2, o)};
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// zero the counters and stamp the start of a fit (stats[ST_T0])
__global__ void k_reset(long long *ctr, double *stats) {
    PDL_ENTRY();
    if (threadIdx.x < 8) ctr[threadIdx.x] = 0;
    if (threadIdx.x == 0) stats[SPKM_ST_T0] = (double)globaltimer_ns();
}

// Condition of the device-driven fit loop: run another iteration while not
// converged and fewer than *limit iterations are done (engine.py:239, 335-337).
// Assignments of device row order -> host row order as int64 (the result's
// layout), so the fit's one D2H is the final array.
__global__ void k_rows_to_host(int64_t n, const int64_t *__restrict__ row_perm, const int32_t *__restrict__ a,
                               int64_t *out) {
    PDL_ENTRY();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) out[row_perm[r]] = a[r];
}

__global__ void k_loop_cond(cudaGraphConditionalHandle h, const long long *ctl, const long long *limit) {
    cudaGraphSetConditional(h, (ctl[1] == 0 && ctl[0] < *limit) ? 1u : 0u);
}

// centers = data rows (CentroidSet.from_data_rows, engine.py:46-58) gathered
// from the device CSR: one CTA per center
__global__ void k_seed_rows_csr(int64_t d, int64_t kp, const int64_t *__restrict__ indptr,
                                const int32_t *__restrict__ indices, const double *__restrict__ v64,
                                const int64_t *__restrict__ row_dev, const int64_t *__restrict__ rows,
                                double *cent64, float *ct32, __half *ct16) {
    PDL_ENTRY();
    const int64_t j = blockIdx.x;
    const int64_t r = row_dev[rows[j]];
    for (int64_t e = indptr[r] + threadIdx.x; e < indptr[r + 1]; e += blockDim.x) {
        const int c = indices[e];
        const double v = v64[e];
        cent64[j * d + c] = v;
        ct32[(int64_t)c * kp + j] = (float)v;
        if (ct16) ct16[(int64_t)c * kp + j] = __float2half_rn((float)v);
    }
}

// corpus upload: raw CSR rows -> device order (longest first), term ids
// renumbered, float32 values (round to nearest), optional float64 copy and
// row_eps = (nnz + 6) * 6.1e-8 rounded up (spkm_csr.row_eps); warp per row
__global__ void __launch_bounds__(256) k_permute_rows(int64_t n, const int64_t *__restrict__ ip_raw,
                                                      const int32_t *__restrict__ idx_raw,
                                                      const double *__restrict__ val_raw,
                                                      const int64_t *__restrict__ perm,
                                                      const int64_t *__restrict__ ip_new,
                                                      const int64_t *__restrict__ new_id, int32_t *idx, float *val,
                                                      double *val64, float *reps) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
        const int64_t src = perm[r];
        const int64_t s0 = ip_raw[src], len = ip_raw[src + 1] - s0, d0 = ip_new[r];
        for (int64_t q = lane; q < len; q += 32) {
            const double v = val_raw[s0 + q];
            idx[d0 + q] = (int32_t)new_id[idx_raw[s0 + q]];
            val[d0 + q] = __double2float_rn(v);
            if (val64) val64[d0 + q] = v;
        }
        if (lane == 0 && reps) reps[r] = __double2float_ru(((double)len + 6.0) * 6.1e-8);
    }
}

constexpr int kFinThreads = 256;
__global__ void __launch_bounds__(kFinThreads) k_finalize(int64_t k, int32_t *touched,
                                                          const int32_t *__restrict__ tcount, double *drift,
                                                          double *sinp, const double *__restrict__ objc,
                                                          double *hstat, long long *ctr, double *stats,
                                                          long long sims_extra, int all, double *stats_hist,
                                                          int64_t hist_cap, int fuse_policy, long long *ctl,
                                                          long long allheavy_rows) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    __shared__ double s_ob[kFinThreads / 32];
    __shared__ int s_no[kFinThreads / 32];
    __shared__ Low2 s_p[kFinThreads / 32], s_s[kFinThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double ob = 0.0;
    int notone = 0;
    Low2 pm{INFINITY, 0x7fffffff, INFINITY, 0x7fffffff}, sm = pm;
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
        double p = 1.0, sp = 0.0;
        if (all || touched[j]) {           // set by k_center_reduce this iteration
            p = drift[j];
            sp = sinp[j];
        } else {                           // engine.py:149: untouched -> p = 1
            drift[j] = 1.0;
            sinp[j] = 0.0;
        }
        touched[j] = 0;
        ob += objc[j];
        notone |= (p != 1.0);
        low2_push(pm, p, (int)j);
        low2_push(sm, -sp, (int)j);
    }
    for (int o = 16; o; o >>= 1) {
        ob += __shfl_down_sync(FULL, ob, o);
        notone |= __shfl_down_sync(FULL, notone, o);
        Low2 x = low2_shfl(pm, o), y = low2_shfl(sm, o);
        low2_merge(pm, x);
        low2_merge(sm, y);
    }
    if (lane == 0) {
        s_ob[w] = ob;
        s_no[w] = notone;
        s_p[w] = pm;
        s_s[w] = sm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        int no = 0;
        Low2 P = s_p[0], Sx = s_s[0];
        for (int q = 0; q < kFinThreads / 32; ++q) {
            tot += s_ob[q];
            no |= s_no[q];
            if (q) {
                low2_merge(P, s_p[q]);
                low2_merge(Sx, s_s[q]);
            }
        }
        // every global read first (independent loads in flight together), the
        // stats row assembled in registers, then the stores
        long long cv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cv[q] = ctr[q];
        double sv[SPKM_ST_COUNT];
#pragma unroll
        for (int q = 0; q < SPKM_ST_COUNT; ++q) sv[q] = stats[q];
        const long long it = ctl[0];
        const int tc = *tcount;
        hstat[0] = (double)P.i1;
        hstat[1] = P.v1;
        hstat[2] = (k > 1) ? P.v2 : 1.0;
        hstat[3] = (double)Sx.i1;
        hstat[4] = -Sx.v1;
        hstat[5] = (k > 1) ? -Sx.v2 : 0.0;
        // Hamerly: when the tighten pruned < 5% of the bound survivors this
        // iteration, the next rescan runs over the bound survivors and does
        // the tighten test itself (same results and counters, one pass less)
        const bool fuse_auto = 20 * cv[SPKM_CTR_SURV2] >= 19 * cv[SPKM_CTR_SURV1];
        hstat[kFuseFlag] = (cv[SPKM_CTR_SURV1] > 0 && (fuse_policy == 1 || (fuse_policy == 2 && fuse_auto))) ? 1.0 : 0.0;
        hstat[kAllHeavyFlag] = (allheavy_rows > 0 && 256 * cv[SPKM_CTR_MOVES] >= allheavy_rows) ? 1.0 : 0.0;
        sv[SPKM_ST_OBJECTIVE] = tot;
        sv[SPKM_ST_ALLONE] = no ? 0.0 : 1.0;
        sv[SPKM_ST_TOUCHED] = (double)tc;
        sv[SPKM_ST_SIMS] = (double)(cv[SPKM_CTR_SIMS] + sims_extra);
        sv[SPKM_ST_REASSIGN] = (double)cv[SPKM_CTR_MOVES];
        sv[SPKM_ST_SURV1] = (double)cv[SPKM_CTR_SURV1];
        sv[SPKM_ST_SURV2] = (double)cv[SPKM_CTR_SURV2];
        sv[SPKM_ST_NNZ_TIGHTEN] = (double)cv[SPKM_CTR_NNZ_TIGHTEN];
        sv[SPKM_ST_NNZ_RESCAN] = (double)cv[SPKM_CTR_NNZ_RESCAN];
        sv[SPKM_ST_NNZ_ELKAN] = (double)cv[SPKM_CTR_NNZ_ELKAN];
        sv[SPKM_ST_NNZ_MOVED] = (double)cv[SPKM_CTR_NNZ_MOVED];
        // iteration bookkeeping and the convergence test (engine.py:335-337),
        // evaluated on the device so the host can enqueue iterations ahead
        sv[SPKM_ST_ITER] = (double)(it + 1);
        sv[SPKM_ST_TSTAMP] = (double)globaltimer_ns();
#pragma unroll
        for (int q = 0; q < SPKM_ST_COUNT; ++q) stats[q] = sv[q];
        if (it < hist_cap)
#pragma unroll
            for (int q = 0; q < SPKM_ST_COUNT; ++q) stats_hist[it * SPKM_ST_COUNT + q] = sv[q];
        const bool conv = (k == 1) || (no == 0) || (it >= 1 && cv[SPKM_CTR_MOVES] == 0);
        ctl[0] = it + 1;
        ctl[1] = conv ? 1 : 0;
        for (int q = 0; q < 8; ++q) ctr[q] = 0;
    }
}

// ---------------------------------------------------------- center thresholds
// engine._center_thresholds (engine.py:192-198): Gram G = C C^T on the 5th-gen
// tensor cores (tcgen05.mma kind::tf32, accumulator in TMEM), 3xTF32
// (x = hi + lo, G ~ lo.hi + hi.lo + hi.hi).  One CTA = one 128 x 128 output
// tile (upper triangle of 128-tiles) over one d-split, read from the
// term-major float32 copy ct32 by TMA (k_gram_mn below); a tile is skipped
// when none of its clusters moved since the last call.  The per-split fp32
// tiles are written as float32 and summed in float64 by k_gram_final.
// Error bound per entry: products of tf32 values are exact; the fp32 TMEM
// accumulation over 3L/8 MMA steps adds <= (3L/8 + 8) 2^-22 sum|a b| (even
// with truncating adds); the float32 copy and the hi/lo split add < 2e-6.
constexpr int GT = 128;
constexpr int GKC = 32;                       // terms per stage
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// InstrDescriptor: c_format F32 (1) [4,6), a/b format TF32 (2) [7,10)/[10,13),
// a/b major bits 15/16 (set by kGramIdescMN), N>>3 [17,23), M>>4 [24,29)
constexpr uint32_t kGramIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(GT >> 3) << 17) |
                                ((uint32_t)(GT >> 4) << 24);

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    long long spins = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (!done && ++spins > (1ll << 28)) __trap();   // never hang the GPU on a logic error
    }
}


// cc = half-angle of the Gram entry plus the error bound, rounded up.  8
// lanes per (a, j): lane r sums splits y = r, r+8, ... then a fixed shuffle
// tree, so the result does not depend on scheduling.
__global__ void k_gram_final(int64_t k, int64_t dsplit, const float *__restrict__ gpart, int full, double gdelta,
                             float *cc, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t e = gt >> 3;
    const int r = threadIdx.x & 7;
    const bool in = e < k * k;
    const int64_t a = in ? e / k : 0, j = in ? e % k : 0;
    bool work = in && a < j;
    if (work && !full) {   // the tile's dirty flag (written by k_gram_mn)
        const int64_t tk = (k + GT - 1) / GT, ta = a / GT, tj = j / GT;
        work = reinterpret_cast<const int *>(gpart + dsplit * k * k)[ta * tk - ta * (ta - 1) / 2 + (tj - ta)] != 0;
    }
    double g = 0.0;
    if (work)
        for (int64_t y = r; y < dsplit; y += 8) g += (double)gpart[(y * k + a) * k + j];
    g += __shfl_down_sync(FULL, g, 4, 8);
    g += __shfl_down_sync(FULL, g, 2, 8);
    g += __shfl_down_sync(FULL, g, 1, 8);
    if (r == 0 && in) {
        if (a == j) {
            cc[e] = -1.f;
        } else if (work) {
            double h = d_half_angle(d_clamp(g + gdelta)) + kCcSlack;
            if (h > 1.0) h = 1.0;
            const float f = __double2float_ru(h);
            cc[a * k + j] = f;
            cc[j * k + a] = f;
        }
    }
}

// s(a) = max_{j != a} cc(a, j); warp per row.
__global__ void k_row_max(int64_t k, const float *__restrict__ cc, float *s, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    const int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (a >= k) return;
    float m = -INFINITY;
    for (int64_t j = lane; j < k; j += 32)
        if (j != a) m = fmaxf(m, cc[a * k + j]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_down_sync(FULL, m, o));
    if (lane == 0) s[a] = (k > 1) ? m : -1.f;
}


// ============================================================== dense rows
// Config C5 (dense unit vectors): every similarity of the dense corpus is
// computed by this tensor-core pass, so all variants share one canonical
// value (the 3xTF32 tcgen05 result) and pruned == Lloyd holds exactly.
//   * rows (float32, [n][D]; Hamerly survivors first compacted into a
//     contiguous block) and centers (float32, [kpad][D]) are streamed by TMA
//     in stages of 16 dims (64-byte rows, 64-byte swizzle = the K-major
//     SWIZZLE_64B layout tcgen05 reads); one thread issues 2 box loads per
//     stage;
//   * warp roles (512 threads): w0 issues the MMAs, w1 the TMA loads, w2-7
//     write the lo parts, w8-15 run the epilogue (thread = row, two warps
//     per TMEM lane quarter, each folding half of every pass's columns);
//   * CTA = 128 rows (TMEM lanes) x 256 centers (TMEM columns) per pass,
//     ceil(k/256) passes into two TMEM accumulators (the epilogue of one pass
//     overlaps the MMAs of the next), 4 stages in flight, 3 MMAs per 8-dim
//     group (lo.hi, hi.lo, hi.hi); the epilogue folds each 32-column TMEM
//     load into a running top-2 (tie rule) with a 5-level merge tree;
//   * split: hi = the float32 word read as tf32 (the tensor core truncates to
//     tf32), lo = x - trunc_tf32(x) (exact), truncated again by the MMA; the
//     residual of each operand is below 2^-20 |x|;
//   * error: (3D/8 + 8) 2^-22 (fp32 TMEM accumulation, truncation assumed)
//     + 4e-6 (split residuals of rows and centers and the dropped lo.lo
//     product, 3 x 2^-20, plus float32 rounding of rows and centers
//     2 x 2^-24, times sum|x c| <= 1) -> row eps (host).
constexpr int DN_M = 128;                         // rows per tile (TMEM lanes)
constexpr int DN_N = 256;                         // centers per pass (TMEM columns per accumulator)
constexpr int DN_KC = 16;                         // dims per pipeline stage
constexpr int DN_STAGES = 4;                      // stages: raw float32 (= tf32 hi operand) + lo
constexpr int DN_THREADS = 512;                   // w0 MMA, w1 TMA, w2-7 converters, w8-15 epilogue
constexpr int DN_CONV = 192;                      // converter threads
// K-major no-swizzle core matrices, unpadded so that a TMA box of 4 dims x
constexpr int DN_OPA = DN_M * DN_KC * 4;          // one stage, one part (float32 or lo) of A: 64-byte rows
constexpr int DN_OPB = DN_N * DN_KC * 4;
constexpr int DN_RAWST = DN_OPA + DN_OPB;          // float32 A, B of one stage (TMA); read as the hi operand
constexpr int DN_STAGE = 2 * DN_RAWST;             // + the lo parts written by the converters
constexpr uint32_t kDenseIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(DN_N >> 3) << 17) |
                                 ((uint32_t)(DN_M >> 4) << 24);
enum { DMODE_RESCAN_H = 6 };

// SmemDescriptor for K-major SWIZZLE_64B operands: rows of 64 bytes, 8-row
// atoms 512 bytes apart (SBO), LBO unused (1), layout type 4 at bits [61,64)
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((512 >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}


struct DenseArgs {
    CUtensorMap tm_x, tm_b;          // TMA maps: rows [rows][D] and centers [kpad][D], float32
    int64_t n, D, k, kpad, ku;
    const float *reps;
    const int32_t *rowmap;           // null: row = slot; else slot -> row (compacted survivors)
    const long long *rowcount;       // null: n rows; else device count
    int mode, use_s;
    int dbg;                         // experiments only (SPKM_DN_DBG): 1 skip epilogue math, 2 skip MMAs
    int32_t *a;
    float *l, *u;
    const float *s_arr;
    int32_t *mv_i, *mv_old, *surv2;
    long long *ctr;
    double *best, *second;
    const long long *ctl;
};

// Warp-specialised tcgen05 pipeline.  Work items are (tile, pass, stage) in
// a fixed order; producers fill stage buffers with 16-byte cp.async copies
// (tf32 hi/lo parts prepared on upload / per move) and signal `full`; the
// MMA thread waits, issues 6 MMAs (2 8-dim groups x 3xTF32) into the
// accumulator of the pass (two TMEM buffers of 256 columns, so the epilogue
// of pass p overlaps the MMAs of pass p+1) and commits to `empty`; after
// the last stage of a pass it commits to `accf`; the epilogue warps (one
// thread per row) read the 256 columns, fold them into a running top-2 and
// release the buffer through `acce`.
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(DN_THREADS, 1) k_dense_pass(const __grid_constant__ DenseArgs P) {
    PDL_ENTRY();
    if (P.ctl[1]) return;
    extern __shared__ __align__(1024) uint8_t dsm[];
    // stage s: [A f32 | B f32] (TMA; the tensor core reads these float32 words
    // as tf32 = the hi parts, truncated) [A lo | B lo] (converters)
    __shared__ __align__(8) uint64_t full_b[DN_STAGES], lo_full[DN_STAGES], empty_b[DN_STAGES], accf[2], acce[2];
    __shared__ uint32_t tmem_base_s;
    __shared__ unsigned long long s_ctr[8];
    __shared__ float4 s_ep[DN_M];   // epilogue: the second half's top-2 (and incumbent value) per row
    __shared__ int s_epf[DN_M];
    if (threadIdx.x < 8) s_ctr[threadIdx.x] = 0ull;   // made visible by the setup __syncthreads
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nrows = P.rowcount ? *P.rowcount : P.n;
    const int64_t ntiles = (nrows + DN_M - 1) / DN_M;
    const int nks = (int)(P.D / DN_KC);
    const int npass = (int)(P.kpad / DN_N);
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_s)),
                     "r"(2 * DN_N)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < DN_STAGES; ++s) {
            mbar_init(&full_b[s], 1);
            mbar_init(&lo_full[s], DN_CONV);
            mbar_init(&empty_b[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accf[b], 1);
            mbar_init(&acce[b], 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    auto stage_ptr = [&](int s) { return dsm + (size_t)s * DN_STAGE; };
    const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t total_stages = (uint32_t)(my_tiles * npass * nks);

    if (w == 1) {
        // ---------------- TMA producer: one box of rows + one of centers per stage
        if (lane == 0) {
            uint32_t it = 0;
            for (int64_t ti = 0; ti < my_tiles; ++ti) {
                const int row0 = (int)((blockIdx.x + ti * gridDim.x) * DN_M);
                for (int pass = 0; pass < npass; ++pass) {
                    for (int ks = 0; ks < nks; ++ks, ++it) {
                        const int s = it % DN_STAGES;
                        if (it >= DN_STAGES) mbar_wait(smem_u32(&empty_b[s]), ((it / DN_STAGES) - 1) & 1);
                        const uint32_t ra = smem_u32(stage_ptr(s)), rb = ra + DN_OPA;
                        const int k0 = ks * DN_KC;
                        if (P.dbg & 8) {
                            mbar_arrive(&full_b[s]);
                        } else {
                            mbar_expect_tx(&full_b[s], (uint32_t)DN_RAWST);
                            tma_load_2d(ra, &P.tm_x, k0, row0, smem_u32(&full_b[s]));
                            tma_load_2d(rb, &P.tm_b, k0, pass * DN_N, smem_u32(&full_b[s]));
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (w >= 2 && w < 2 + DN_CONV / 32) {
        // ---------------- converters: lo = x - trunc_tf32(x) (exact in float32;
        // the tensor core truncates it to tf32 in turn), an elementwise map
        // because the lo parts share the raw layout byte for byte
        const int ct = threadIdx.x - 64;
        for (uint32_t it = 0; it < total_stages; ++it) {
            const int s = it % DN_STAGES;
            mbar_wait(smem_u32(&full_b[s]), (it / DN_STAGES) & 1);
            const uint8_t *ra = stage_ptr(s);
            uint8_t *lo = stage_ptr(s) + DN_RAWST;
            if (!(P.dbg & 4)) {
                constexpr int NV = DN_RAWST / 16 / DN_CONV;
                static_assert(NV * DN_CONV * 16 == DN_RAWST, "converter split");
                float4 x[NV];
#pragma unroll
                for (int u = 0; u < NV; ++u) x[u] = *reinterpret_cast<const float4 *>(ra + (ct + u * DN_CONV) * 16);
#pragma unroll
                for (int u = 0; u < NV; ++u) {
                    const float4 v = x[u];
                    const float4 l = make_float4(v.x - __uint_as_float(__float_as_uint(v.x) & 0xffffe000u),
                                                 v.y - __uint_as_float(__float_as_uint(v.y) & 0xffffe000u),
                                                 v.z - __uint_as_float(__float_as_uint(v.z) & 0xffffe000u),
                                                 v.w - __uint_as_float(__float_as_uint(v.w) & 0xffffe000u));
                    *reinterpret_cast<float4 *>(lo + (ct + u * DN_CONV) * 16) = l;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic writes -> async proxy
            mbar_arrive(&lo_full[s]);
        }
    } else if (w == 0) {
        // ---------------- MMA issuer
        if (lane == 0) {
            uint32_t it = 0, pcount = 0;
            for (int64_t ti = 0; ti < my_tiles; ++ti) {
                for (int pass = 0; pass < npass; ++pass, ++pcount) {
                    const int b = pcount & 1;
                    if (pcount >= 2) mbar_wait(smem_u32(&acce[b]), ((pcount >> 1) - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    const uint32_t dt = tmem + (uint32_t)(b * DN_N);
                    for (int ks = 0; ks < nks; ++ks, ++it) {
                        const int s = it % DN_STAGES;
                        mbar_wait(smem_u32(&lo_full[s]), (it / DN_STAGES) & 1);   // implies the TMA data landed
                        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                        const uint32_t ahi = smem_u32(stage_ptr(s)), bhi = ahi + DN_OPA, alo = ahi + DN_RAWST,
                                       blo = alo + DN_OPA;
#pragma unroll
                        for (int g = 0; g < DN_KC / 8; ++g) {
                            if (P.dbg & 2) break;
                            // K-major SWIZZLE_64B: 8 dims (32 B) per MMA -> +32 B within the 64-byte rows
                            const uint64_t dah = umma_desc_sw64(ahi + 32 * g);
                            const uint64_t dal = umma_desc_sw64(alo + 32 * g);
                            const uint64_t dbh = umma_desc_sw64(bhi + 32 * g);
                            const uint64_t dbl = umma_desc_sw64(blo + 32 * g);
                            const uint32_t acc0 = (ks > 0 || g > 0) ? 1u : 0u;
                            asm volatile(
                                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
                                "l"(dal), "l"(dbh), "r"(kDenseIdesc), "r"(acc0)
                                : "memory");
                            asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(dt),
                                         "l"(dah), "l"(dbl), "r"(kDenseIdesc)
                                         : "memory");
                            asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(dt),
                                         "l"(dah), "l"(dbh), "r"(kDenseIdesc)
                                         : "memory");
                        }
                        asm volatile(
                            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                smem_u32(&empty_b[s]))
                            : "memory");
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                     smem_u32(&accf[b]))
                                 : "memory");
                }
            }
        }
        __syncwarp();
    } else if (w >= 8) {
        // ---------------- epilogue: thread = row; two warps per TMEM lane
        // quarter (w % 4), half hf folds columns [128 hf, 128 hf + 128) of
        // every 256-column pass; the halves merge once per tile in smem
        const int qd = w & 3, hf = (w - 8) >> 2;
        const int m = qd * 32 + lane;
        uint32_t pcount = 0;
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            const int64_t tile = blockIdx.x + ti * gridDim.x;
            const int64_t slot = tile * DN_M + m;
            const int32_t my_row = slot < nrows ? (P.rowmap ? P.rowmap[slot] : (int32_t)slot) : -1;
            const int inc = (my_row >= 0 && (P.mode == SPKM_MODE_LLOYD || P.mode == DMODE_RESCAN_H)) ? P.a[my_row] : -1;
            Top2 tp{-INFINITY, -2, -INFINITY};
            float s_inc = 0.f;
            int has_inc = 0;
            for (int pass = 0; pass < npass; ++pass, ++pcount) {
                const int b = pcount & 1;
                mbar_wait(smem_u32(&accf[b]), (pcount >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll 1
                for (int cb = 0; cb < DN_N / 32 / 2; ++cb) {
                    uint32_t r[16];
                    const int col0 = hf * (DN_N / 2) + cb * 32;
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const uint32_t taddr = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(b * DN_N + col0 + 16 * hh);
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                            "%15}, [%16];\n"
                            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                              "=r"(r[14]), "=r"(r[15])
                            : "r"(taddr));
                        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                        if (my_row >= 0 && !(P.dbg & 1)) {
                            // top-2 of 16 columns as a 4-level merge tree (order-free under
                            // the tie rule), then into the running top-2
                            const int jb = pass * DN_N + col0 + 16 * hh;
                            Top2 t[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const int j0 = jb + 2 * q, j1 = j0 + 1;
                                const float v0 = j0 < P.k ? __uint_as_float(r[2 * q]) : -INFINITY;
                                const float v1 = j1 < P.k ? __uint_as_float(r[2 * q + 1]) : -INFINITY;
                                t[q] = better(v1, j1, v0, j0, inc) ? Top2{v1, j1, v0} : Top2{v0, j0, v1};
                            }
#pragma unroll
                            for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
                                for (int q = 0; q < h; ++q) top2_merge(t[q], t[q + h], inc);
                            top2_merge(tp, t[0], inc);
#pragma unroll
                            for (int q = 0; q < 16; ++q)
                                if (jb + q == inc) {
                                    s_inc = __uint_as_float(r[q]);
                                    has_inc = 1;
                                }
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                mbar_arrive(&acce[b]);
            }
            // merge the two halves of the row: hf 1 hands its top-2 to hf 0
            if (hf == 1) {
                s_ep[m] = make_float4(tp.b, __int_as_float(tp.bj), tp.s, has_inc ? s_inc : -INFINITY);
                s_epf[m] = has_inc;
            }
            asm volatile("bar.sync %0, 64;\n" ::"r"(1 + qd) : "memory");
            if (hf == 0) {
                const float4 o4 = s_ep[m];
                const Top2 o{o4.x, __float_as_int(o4.y), o4.z};
                top2_merge(tp, o, inc);
                if (s_epf[m]) s_inc = o4.w;
            }
            asm volatile("bar.sync %0, 64;\n" ::"r"(1 + qd) : "memory");
            if (hf == 1) continue;
            const double eps = my_row >= 0 ? (double)P.reps[my_row] : 0.0;
            bool moved = false, surv = false;
            long long sims = 0;
            if (my_row >= 0) {
                switch (P.mode) {
                    case SPKM_MODE_INIT_PLAIN:
                    case SPKM_MODE_INIT_ELKAN:
                    case SPKM_MODE_INIT_HAMERLY:
                        P.a[my_row] = tp.bj;
                        P.l[my_row] = store_lower((double)tp.b - eps);
                        if (P.mode == SPKM_MODE_INIT_HAMERLY)
                            P.u[my_row] = (P.k == 1) ? -1.f : store_upper((double)tp.s + eps);
                        break;
                    case SPKM_MODE_LLOYD:
                        if (tp.bj != inc) {
                            P.a[my_row] = tp.bj;
                            moved = true;
                        }
                        break;
                    case DMODE_RESCAN_H: {
                        // kernels.py:88-112 on the canonical values: tighten, re-test, full scan
                        const double lb = (double)s_inc - eps;
                        sims = 1;
                        bool pruned = (P.use_s && lb >= 0.0 && (double)P.s_arr[inc] + kSqrt2 * eps <= lb);
                        if (!pruned) pruned = ((double)P.u[my_row] + eps <= (double)s_inc);
                        if (pruned) {
                            P.l[my_row] = store_lower(lb);
                        } else {
                            surv = true;
                            sims += P.k - 1;
                            if (tp.bj != inc) {
                                P.a[my_row] = tp.bj;
                                moved = true;
                            }
                            P.l[my_row] = store_lower((double)tp.b - eps);
                            P.u[my_row] = store_upper((double)tp.s + eps);
                        }
                        break;
                    }
                    case MODE_PREDICT:
                        P.a[my_row] = tp.bj;
                        P.best[my_row] = (double)tp.b;
                        P.second[my_row] = (P.k == 1) ? -1.0 : (double)tp.s;
                        break;
                }
            }
            if (P.mode == SPKM_MODE_LLOYD || P.mode == DMODE_RESCAN_H)
                warp_append(moved, my_row, P.mv_i, inc, P.mv_old, P.ctr + SPKM_CTR_MOVES);
            if (P.mode == DMODE_RESCAN_H) {
                warp_append(surv, my_row, P.surv2, 0, nullptr, P.ctr + SPKM_CTR_SURV2);
                ctr_add(s_ctr, SPKM_CTR_SIMS, sims);
                ctr_add(s_ctr, SPKM_CTR_NNZ_RESCAN, my_row >= 0 ? P.D : 0);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 8 && s_ctr[threadIdx.x] && P.ctr)
        atomicAdd((unsigned long long *)(P.ctr + threadIdx.x), s_ctr[threadIdx.x]);
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * DN_N) : "memory");
}


// MN-major Gram tile (the default): the term-major float32 centers are
// already the MN-major operand layout tcgen05 reads (centers contiguous), so
// TMA drops 32-center x 32-term boxes straight into the canonical swizzled
// MN-major atoms and the tensor core reads the raw float32 words as
// the truncated tf32 hi part.  Converter warps only write lo = x - trunc(x)
// elementwise at the same (swizzled) offsets -- no transpose.  DIAG stages
// A alone (6 stages of 32 KB), other tiles A and B (3 stages of 64 KB).
constexpr int GM_THREADS = 384;
constexpr int GM_CONV = 320;                 // warps 2-11
constexpr int GM_BLK = 32 * GKC * 4;         // 4 KB: one TMA box (32 centers x 32 terms)
constexpr int GM_OP = 4 * GM_BLK;            // 16 KB: 128 centers x 32 terms
// MN-major tf32 operands use the 128-byte swizzle with 32-byte atoms
// (SWIZZLE_128B_BASE32B, layout type 1 at bits [61,64)): 32-byte chunks of a
// 128-byte row XOR row % 4, 4-row K atoms 512 B apart (SBO), 32-center
// blocks GM_BLK apart (LBO).  (The 16-byte-atom SWIZZLE_128B reads back as
// zeros for tf32 MN-major; measured with tools/mn_probe.cu.)
__device__ __forceinline__ uint64_t umma_desc_mn128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((GM_BLK >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((512 >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;
    return d;
}
constexpr uint32_t kGramIdescMN = kGramIdesc | (1u << 15) | (1u << 16);
template <bool DIAG> struct GmCfg {
    static constexpr int ST = DIAG ? 6 : 3;
    static constexpr int NOP = DIAG ? 1 : 2;                 // operands staged per stage
    static constexpr int STAGE = 2 * NOP * GM_OP;            // [raw A | raw B | lo A | lo B]
    static constexpr size_t SMEM = (size_t)ST * STAGE + 1024;
};

// gpart: [dsplit][k][k] float32 partial Grams, then one dirty flag per tile.
template <bool DIAG>
__global__ void __launch_bounds__(GM_THREADS, 1) k_gram_mn(const __grid_constant__ CUtensorMap tm, int64_t k, int64_t d,
                                                          int64_t dsplit, const int2 *__restrict__ tiles,
                                                          const int32_t *__restrict__ tlist,
                                                          const int32_t *__restrict__ tcount, int full, float *gpart,
                                                          const long long *__restrict__ ctl, int rank, int world) {
    PDL_ENTRY();
    using G = GmCfg<DIAG>;
    if (ctl[1]) return;   // converged: later enqueued iterations are no-ops
    extern __shared__ uint8_t gsm_raw[];
    uint8_t *gsm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full_b[G::ST], lo_b[G::ST], empty_b[G::ST], done_b;
    __shared__ uint32_t tmem_base_s;
    const int2 tl = DIAG ? make_int2(0, 0) : tiles[blockIdx.x];
    const int64_t a0 = (int64_t)tl.x * GT, j0 = (int64_t)tl.y * GT;
    // the tile is recomputed only if one of its clusters was touched by this
    // iteration's center update (the touched list of spkm_move_centers)
    int mine = full;
    if (!mine) {
        const int tc = *tcount;
        for (int t = threadIdx.x; t < tc; t += blockDim.x) {
            const int64_t j = tlist[t];
            mine |= (j >= a0 && j < a0 + GT) || (j >= j0 && j < j0 + GT);
        }
    }
    const int dirty = __syncthreads_or(mine);
    if (blockIdx.y == 0 && threadIdx.x == 0) reinterpret_cast<int *>(gpart + dsplit * k * k)[blockIdx.x] = dirty;
    // multi-GPU: the (tile, split) CTAs are dealt round-robin to the ranks;
    // every rank still writes every tile's dirty flag (above), its own
    // partials only (the others are zero and summed in by an allreduce)
    if (!dirty || (int)(((int64_t)blockIdx.x * gridDim.y + blockIdx.y) % world) != rank) return;
    const int64_t per = ((d + dsplit - 1) / dsplit + GKC - 1) / GKC * GKC;
    const int64_t t0 = blockIdx.y * per, t1 = min(d, t0 + per);
    const int nch = t1 > t0 ? (int)((t1 - t0 + GKC - 1) / GKC) : 0;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_s)),
                     "r"(GT)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < G::ST; ++q) {
            mbar_init(&full_b[q], 1);
            mbar_init(&lo_b[q], GM_CONV);
            mbar_init(&empty_b[q], 1);
        }
        mbar_init(&done_b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    auto stage = [&](int st) { return gsm + (size_t)st * G::STAGE; };   // raw operands, then lo operands
    if (w == 1) {
        if (lane == 0) {
            for (int c = 0; c < nch; ++c) {
                const int st = c % G::ST;
                if (c >= G::ST) mbar_wait(smem_u32(&empty_b[st]), ((c / G::ST) - 1) & 1);
                mbar_expect_tx(&full_b[st], (uint32_t)(G::NOP * GM_OP));
                const int trow = (int)(t0 + (int64_t)c * GKC);
                const uint32_t dst = smem_u32(stage(st));
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    tma_load_2d(dst + b * GM_BLK, &tm, (int)(a0 + 32 * b), trow, smem_u32(&full_b[st]));
                    if (!DIAG) tma_load_2d(dst + GM_OP + b * GM_BLK, &tm, (int)(j0 + 32 * b), trow, smem_u32(&full_b[st]));
                }
            }
        }
        __syncwarp();
    } else if (w >= 2) {
        const int ct = threadIdx.x - 64;
        constexpr int N16 = G::NOP * GM_OP / 16;   // 16-byte chunks of raw operands per stage
        for (int c = 0; c < nch; ++c) {
            const int st = c % G::ST;
            mbar_wait(smem_u32(&full_b[st]), (c / G::ST) & 1);
            const uint4 *raw = reinterpret_cast<const uint4 *>(stage(st));
            uint4 *lo = reinterpret_cast<uint4 *>(stage(st) + G::NOP * GM_OP);
            for (int e = ct; e < N16; e += GM_CONV) {
                const uint4 x = raw[e];
                uint4 y;
                y.x = __float_as_uint(__uint_as_float(x.x) - __uint_as_float(x.x & 0xffffe000u));
                y.y = __float_as_uint(__uint_as_float(x.y) - __uint_as_float(x.y & 0xffffe000u));
                y.z = __float_as_uint(__uint_as_float(x.z) - __uint_as_float(x.z & 0xffffe000u));
                y.w = __float_as_uint(__uint_as_float(x.w) - __uint_as_float(x.w & 0xffffe000u));
                lo[e] = y;
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_arrive(&lo_b[st]);
        }
    } else if (lane == 0) {   // w == 0: MMA issuer
        for (int c = 0; c < nch; ++c) {
            const int st = c % G::ST;
            mbar_wait(smem_u32(&lo_b[st]), (c / G::ST) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t ahi = smem_u32(stage(st));
            const uint32_t bhi = DIAG ? ahi : ahi + GM_OP;
            const uint32_t alo = ahi + G::NOP * GM_OP, blo = bhi + G::NOP * GM_OP;
#pragma unroll
            for (int g = 0; g < GKC / 8; ++g) {
                const uint32_t off = g * 1024;   // next 8-term K group
                const uint64_t dah = umma_desc_mn128(ahi + off), dal = umma_desc_mn128(alo + off);
                const uint64_t dbh = umma_desc_mn128(bhi + off), dbl = umma_desc_mn128(blo + off);
                const uint32_t acc0 = (c > 0 || g > 0) ? 1u : 0u;
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(dal), "l"(dbh), "r"(kGramIdescMN), "r"(acc0)
                    : "memory");
                asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(tmem), "l"(dah),
                             "l"(dbl), "r"(kGramIdescMN)
                             : "memory");
                asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(tmem), "l"(dah),
                             "l"(dbh), "r"(kGramIdescMN)
                             : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_u32(&empty_b[st]))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&done_b))
                     : "memory");
    }
    __syncwarp();
    // epilogue: warps 0-3 read their TMEM lane quarters into the split's partial Gram
    if (w < 4) {
        if (nch > 0) mbar_wait(smem_u32(&done_b), 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const int64_t row = a0 + w * 32 + lane;
#pragma unroll 1
        for (int cb = 0; cb < GT / 32; ++cb) {
            uint32_t r[32];
            const uint32_t taddr = tmem + ((uint32_t)(w * 32) << 16) + (uint32_t)(cb * 32);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                  "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                  "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (row < k) {
                float *out = gpart + ((int64_t)blockIdx.y * k + row) * k;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const int64_t col = j0 + cb * 32 + q;
                    if (col < k) out[col] = nch > 0 ? __uint_as_float(r[q]) : 0.f;
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(GT) : "memory");
}

// centers (float64, [k][D]) -> float32 rows padded with zeros to kpad; the
// dense pass splits them into tf32 hi + lo on the fly
__global__ void k_dense_centers(int64_t k, int64_t kpad, int64_t D, const double *__restrict__ C, float *b,
                                const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < kpad * D;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / D;
        b[e] = j < k ? (float)C[e] : 0.f;
    }
}

// survivors' float32 rows -> a contiguous block (slot order) for the dense rescan
__global__ void k_gather_rows(const float *__restrict__ x, int64_t D, const int32_t *__restrict__ list,
                              const long long *__restrict__ count, float *out, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;
    const int64_t per = D / 4, tot = *count * per;
    const float4 *src = reinterpret_cast<const float4 *>(x);
    float4 *dst = reinterpret_cast<float4 *>(out);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = e / per, c = e - slot * per;
        dst[e] = __ldg(src + (int64_t)list[slot] * per + c);
    }
}

// ---------------------------------------------------------------- misc
__global__ void k_load_centers(int64_t k, int64_t d, int64_t kp, const double *__restrict__ src, double *cent64,
                               float *ct32, __half *ct16) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= k * d) return;
    const int64_t j = e / d, t = e % d;
    const double v = src[e];
    cent64[e] = v;
    ct32[t * kp + j] = (float)v;
    if (ct16) ct16[t * kp + j] = __float2half_rn((float)v);
}

// CentroidSet.from_data_rows (engine.py:46-58) on the device: k packed seed
// rows (float64 values) scattered into zeroed cent64 / ct32.
__global__ void k_seed_rows(int64_t d, int64_t kp, const int64_t *__restrict__ sptr, const int32_t *__restrict__ sidx,
                            const double *__restrict__ sval, double *cent64, float *ct32, __half *ct16) {
    const int64_t j = blockIdx.x;
    for (int64_t t = sptr[j] + threadIdx.x; t < sptr[j + 1]; t += blockDim.x) {
        const int c = sidx[t];
        const double v = sval[t];
        cent64[j * d + c] = v;
        ct32[(int64_t)c * kp + j] = (float)v;
        if (ct16) ct16[(int64_t)c * kp + j] = __float2half_rn((float)v);
    }
}

__global__ void k_geometry(int op, int64_t n, const double *a, const double *b, double *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    switch (op) {
        case 0: out[i] = d_cos_lower(a[i], b[i]); break;
        case 1: out[i] = d_cos_upper(a[i], b[i]); break;
        case 2: out[i] = d_hamerly_upper(a[i], b[i]); break;
        case 3: out[i] = d_half_angle(a[i]); break;
        case 4: out[i] = d_lower_update(a[i], b[i]); break;
        default: out[i] = d_clamp(a[i]); break;
    }
}

// ------------------------------------------------------------- host glue
struct ColPlan {
    int ch, tpr, rpw;
};
ColPlan col_plan(int64_t k) {
    int ch = 4;
    while (ch < 32 && (k + ch - 1) / ch > 32) ch *= 2;
    ColPlan p;
    p.ch = ch;
    p.tpr = (int)((k + ch - 1) / ch);
    if (p.tpr > 32) p.tpr = 32;
    p.rpw = 32 / p.tpr;
    if (p.rpw > 8) p.rpw = 8;   // k_row_pass stages at most 8 rows per warp
    return p;
}

int grid_for(int64_t work_items, int per_block) {
    const int64_t need = (work_items + per_block - 1) / per_block;
    const int64_t cap = (int64_t)num_sms() * 16;
    int64_t g = need < cap ? need : cap;
    return (int)(g < 1 ? 1 : g);
}

template <int CH, int NT, int GV>
int launch_rp(RowPassArgs &A, int grid, size_t smem, cudaStream_t st) {
    if (GV == 2) {   // + kp floats of accumulators per warp
        smem += (size_t)(NT / 32) * A.kp * sizeof(float);
        const cudaError_t e = cudaFuncSetAttribute(k_row_pass<CH, NT, GV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)smem);
        if (e != cudaSuccess) return fail("row_pass smem attribute", e);
    }
    pdl_launch(k_row_pass<CH, NT, GV>, dim3(grid), dim3(NT), smem, st, A);
    CHECK_LAUNCH("row_pass");
    return 0;
}

// (A persistent 1024-thread variant that served the Zipf head of ct32 from a
// shared-memory table was 1.2x slower on C2 than these L1-cached 256-thread
// CTAs and was removed: profiles/r01_rowpass_hot_vs_plain.txt.)
int launch_row_pass(RowPassArgs &A, int64_t k, cudaStream_t st, int64_t max_rows) {
    const ColPlan p = col_plan(k);
    A.tpr = p.tpr;
    A.rpw = p.rpw;
    A.k = (int)k;
    const int64_t slots = (max_rows + p.rpw - 1) / p.rpw;
    const int grid = grid_for(slots, 8);
    // staging for rpw row groups per warp (k > 256: one) -- the rest of the
    // shared-memory carve-out stays L1 (C4 Elkan scan: -20% from this alone)
#ifndef SPKM_RP_SMEM_GROUPS
#define SPKM_RP_SMEM_GROUPS 0     // > 0: reserve this many row groups per warp (A/B of the L1 carve-out)
#endif
    const size_t smem = (size_t)(256 / 32) * (SPKM_RP_SMEM_GROUPS > p.rpw ? SPKM_RP_SMEM_GROUPS : p.rpw) * kIvStride * 8;
    // fp16 screening for every full pass but predict, when the table exists (k > 128)
    const bool half = A.ct16 != nullptr && A.mode != MODE_PREDICT && p.ch >= 8;
    // sparse center index for every full pass but predict, when built (k > 256)
    const bool sparse = A.ci_desc != nullptr && A.mode != MODE_PREDICT && p.ch >= 16;
    if (p.ch == 4) return launch_rp<4, 256, 0>(A, grid, smem, st);
    if (p.ch == 8) return half ? launch_rp<8, 256, 1>(A, grid, smem, st) : launch_rp<8, 256, 0>(A, grid, smem, st);
    if (p.ch == 16)
        return sparse ? launch_rp<16, 256, 2>(A, grid, smem, st)
                      : half ? launch_rp<16, 256, 1>(A, grid, smem, st) : launch_rp<16, 256, 0>(A, grid, smem, st);
    return sparse ? launch_rp<32, 256, 2>(A, grid, smem, st)
                  : half ? launch_rp<32, 256, 1>(A, grid, smem, st) : launch_rp<32, 256, 0>(A, grid, smem, st);
}

// Term rows of the Zipf head kept in L2 by the gathers' eviction hints:
// as many as fit SPKM_HOT_MB (default 64 MB, about half of L2).
int64_t hot_terms(const spkm_centers *C) {
    static int64_t mb = -1;
    if (mb < 0) {
        const char *e = getenv("SPKM_HOT_MB");
        mb = e ? atoll(e) : 64;
    }
    const int64_t rows = (mb << 20) / (C->kp * 4 > 0 ? C->kp * 4 : 1);
    return rows < C->d ? rows : C->d;
}

// Elkan family, k > 128: rows with at least this many centers failing the
// stored-bound test take the full pass (spkm_elkan_heavy).
// SPKM_EK_HEAVY_PCT: percent of k (0 = off).
int64_t elkan_heavy_default(int64_t k) {
    const char *e = getenv("SPKM_EK_HEAVY_PCT");
    const double pct = e ? atof(e) : (double)SPKM_EK_HEAVY_PCT_DEFAULT;
    // smallest k with a heavy-row pass: 129 (k <= 128 keeps the fused bound + scan pass: C2, k = 100, is 6% slower
    // with heavy rows; C3, k = 200: 221 -> 305 it/s with every bound survivor heavy); SPKM_EK_HEAVY_MINK overrides
    const char *m = getenv("SPKM_EK_HEAVY_MINK");
    const int64_t mink = m ? atoll(m) : 129;
    if (k < mink || !(pct > 0.0)) return 0;
    const int64_t t = (int64_t)ceil((double)k * pct / 100.0 - 1e-9);
    return t < 1 ? 1 : t;
}

// simp_elkan with a heavy threshold of at most kLightMax + 1: the bound pass lists the failing centers of
// every light row (W->lightj) and k_elkan_light scans just those (instead of k_elkan_scan)
bool light_lists(const spkm_work *W, int use_cc) {
    return !use_cc && W->lightj != nullptr && W->elkan_heavy > 0 && W->elkan_heavy <= kLightMax + 1;
}

RowPassArgs row_args(const spkm_csr *X, const spkm_centers *C) {
    RowPassArgs A{};
    A.ctl = C->ctl;
    A.indptr = X->indptr;
    A.indices = X->indices;
    A.values = X->values;
    A.reps = X->row_eps;
    A.n = X->n;
    A.ct = C->ct32;
    A.kp = C->kp;
    A.hot = hot_terms(C);
    A.ct16 = reinterpret_cast<const __half *>(C->ct16);
    A.d = X->d;
    if (C->cindex) {
        A.ci_desc = C->cindex->desc;
        A.ci_pairs = reinterpret_cast<const int2 *>(C->cindex->pairs);
    }
    return A;
}


// ------------------------------------------------------------ bound auditor
// validation.py:49-80 on the device: exact float64 similarities of every row
// to every center (FMA chain over the row's nnz, |error| ~ 1e-16 << the
// auditor's 1e-9 tolerance) from a term-major float64 copy of the centers,
// checked against the stored bounds.  mode 0: Elkan u(i,j) matrix, 1:
// Hamerly single u (max over j != a(i)), 2: lower bound only, 3: argmax
// (brute_force_assign, lowest index on ties) into a_out.  Maxima are
// accumulated as order-preserving 64-bit keys with atomicMax.
__device__ __forceinline__ unsigned long long dkey(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
constexpr int kAuditCols = 4;   // columns per lane per block (128 per warp)

__global__ void __launch_bounds__(256) k_audit(int64_t n, int64_t k, int64_t kp, const int64_t *__restrict__ indptr,
                                               const int32_t *__restrict__ indices, const double *__restrict__ v64,
                                               const double *__restrict__ ct64, const int32_t *__restrict__ a,
                                               const float *__restrict__ l, const float *__restrict__ u, int64_t ku,
                                               int mode, unsigned long long *keys, int32_t *a_out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
        const int64_t s = indptr[i], e = indptr[i + 1];
        const int ai = (mode == 3) ? -1 : a[i];
        double own = -INFINITY, up = -INFINITY, best = -INFINITY;
        int bj = 0x7fffffff;
        for (int64_t j0 = 0; j0 < k; j0 += 32 * kAuditCols) {
            double acc[kAuditCols];
#pragma unroll
            for (int c = 0; c < kAuditCols; ++c) acc[c] = 0.0;
            for (int64_t t = s; t < e; ++t) {
                const double x = v64[t];
                const double *row = ct64 + (int64_t)indices[t] * kp;
#pragma unroll
                for (int c = 0; c < kAuditCols; ++c) {
                    const int64_t j = j0 + c * 32 + lane;
                    if (j < k) acc[c] = fma(x, row[j], acc[c]);
                }
            }
#pragma unroll
            for (int c = 0; c < kAuditCols; ++c) {
                const int64_t j = j0 + c * 32 + lane;
                if (j >= k) continue;
                const double S = acc[c];
                if (j == ai) own = S;
                if (mode == 0) up = fmax(up, S - (double)u[i * ku + j]);
                if (mode == 1 && j != ai) up = fmax(up, S);
                if (mode == 2 && j != ai) up = fmax(up, S - (double)u[i * ku + (j >> 2)]);   // Yin-Yang groups
                if (mode == 3 && (S > best || (S == best && j < bj))) {
                    best = S;
                    bj = (int)j;
                }
            }
        }
        for (int o = 16; o; o >>= 1) {
            own = fmax(own, __shfl_xor_sync(FULL, own, o));
            up = fmax(up, __shfl_xor_sync(FULL, up, o));
            const double ob = __shfl_xor_sync(FULL, best, o);
            const int oj = __shfl_xor_sync(FULL, bj, o);
            if (ob > best || (ob == best && oj < bj)) {
                best = ob;
                bj = oj;
            }
        }
        if (lane == 0) {
            if (mode == 3) {
                a_out[i] = bj;
            } else {
                atomicMax(keys, dkey((double)l[i] - own));
                if (mode == 0 || (mode == 2 && k > 1)) atomicMax(keys + 1, dkey(up));
                if (mode == 1 && k > 1) atomicMax(keys + 1, dkey(up - (double)u[i]));
            }
        }
    }
}

// center-major float64 [k][d] -> term-major [d][kp] (zero padding columns)
__global__ void k_transpose_centers(int64_t k, int64_t d, int64_t kp, const double *__restrict__ c64, double *ct64) {
    __shared__ double tile[32][33];
    const int64_t t0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + r, t = t0 + threadIdx.x;
        tile[r][threadIdx.x] = (j < k && t < d) ? c64[j * d + t] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t t = t0 + r, j = j0 + threadIdx.x;
        if (t < d && j < kp) ct64[t * kp + j] = tile[threadIdx.x][r];
    }
}


// ------------------------------------------------------ multi-GPU exchange
// Corpus replicated on every rank, scans sharded by device-row ranges; the
// only per-iteration collective is an allgather of fixed-size move slots:
//   slot (int32) = [count, 0, ctr as 8 x int64, (row, old, new) x cap]
// Every rank then applies ALL moves to its replicated fixed-point sums, so
// the sums (integers, order-free atomics) are identical on every rank.
constexpr int kSlotHead = 2 + 16;

__global__ void k_pack_moves(const int32_t *__restrict__ mv_i, const int32_t *__restrict__ mv_old,
                             const int32_t *__restrict__ a, const long long *__restrict__ ctr, int64_t p0,
                             int64_t cap, int32_t *slot, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;
    const long long cnt = ctr[SPKM_CTR_MOVES];
    DCHECK(cnt <= cap);
    const long long c = cnt < cap ? cnt : cap;   // cap = shard rows >= moves
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        slot[0] = (int32_t)c;
        slot[1] = 0;
        long long *h = reinterpret_cast<long long *>(slot + 2);
        for (int q = 0; q < 8; ++q) h[q] = ctr[q];
    }
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < c; m += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = mv_i[m];
        int32_t *t = slot + kSlotHead + 3 * m;
        t[0] = (int32_t)(p0 + i);
        t[1] = mv_old[m];
        t[2] = a[i];
    }
}

// all ranks' moves -> sums/counts/touched (warp per move); block 0 also
// writes the summed counters of all ranks into ctr_out
__global__ void __launch_bounds__(256) k_apply_move_slots(const int32_t *__restrict__ slots, int world,
                                                          int64_t slot_len, int64_t d,
                                                          const int64_t *__restrict__ indptr,
                                                          const int32_t *__restrict__ indices,
                                                          const float *__restrict__ values, long long *sums,
                                                          long long *counts, int32_t *touched, double scale,
                                                          long long *ctr_out, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl[1]) return;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int q = 0; q < world; ++q) {
        const int32_t *sl = slots + (int64_t)q * slot_len;
        const int64_t cnt = sl[0];
        for (int64_t m = wid; m < cnt; m += warps) {
            const int32_t *t = sl + kSlotHead + 3 * m;
            const int64_t i = t[0];
            const int o = t[1], nw = t[2];
            long long *so = sums + (int64_t)o * d;
            long long *sn = sums + (int64_t)nw * d;
            for (int64_t e = indptr[i] + lane; e < indptr[i + 1]; e += 32) {
                const int c = __ldg(indices + e);
                const long long v = to_fixed(__ldg(values + e), scale);
                atomicAdd((unsigned long long *)(so + c), (unsigned long long)(-v));
                atomicAdd((unsigned long long *)(sn + c), (unsigned long long)v);
            }
            if (lane == 0) {
                atomicAdd((unsigned long long *)(counts + o), (unsigned long long)(-1ll));
                atomicAdd((unsigned long long *)(counts + nw), 1ull);
                touched[o] = 1;
                touched[nw] = 1;
            }
        }
        wid = (wid + warps - (cnt % warps)) % warps;   // rotate so ranks' tails spread over warps
    }
    if (blockIdx.x == 0 && threadIdx.x < 8) {
        long long tot = 0;
        for (int q = 0; q < world; ++q) tot += reinterpret_cast<const long long *>(slots + (int64_t)q * slot_len + 2)[threadIdx.x];
        ctr_out[threadIdx.x] = tot;
    }
}

// ------------------------------------------------------ cluster-ordered worklists
// The gather passes (Hamerly rescan, Elkan survivor scan, Lloyd pass) read,
// per nnz, a term row of the center table.  When the table does not fit L2
// (C4: ct32 = 4 GB) and rows arrive in storage order, every topic-term
// gather misses L2.  Rows of one cluster share most of their terms (one
// topic), so a worklist ordered by a(i) keeps the CTAs in flight on a few
// clusters' term rows at a time: the gathers become L2 hits.  Results do not
// depend on the order in which rows are visited (per-row outputs, integer
// counters, int64 fixed-point sums), so this is a pure locality change.
//
// Counting sort by a(i) in tiles of kOrdTile list entries: k_order_hist adds
// each tile's bin counts to a global histogram, k_order_scan turns it into
// bin starts, k_order_scatter reserves a range per (tile, bin) with one
// global atomic and writes each entry at its shared-memory rank.  Within a
// bin the order is the tiles' reservation order (not stable; any order is
// valid).
constexpr int kOrdThreads = 256, kOrdPer = 8, kOrdTile = kOrdThreads * kOrdPer;

__device__ __forceinline__ int64_t ord_count(const long long *count, int64_t n) {
    return count ? (int64_t)*count : n;
}

__global__ void __launch_bounds__(kOrdThreads) k_order_hist(int64_t k, const int32_t *__restrict__ a,
                                                          const int32_t *__restrict__ list,
                                                          const long long *__restrict__ count, int64_t n,
                                                          int32_t *bins, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl && ctl[1]) return;
    extern __shared__ int32_t s_h[];
    const int64_t cnt = ord_count(count, n);
    const int64_t ntile = (cnt + kOrdTile - 1) / kOrdTile;
    for (int j = threadIdx.x; j < k; j += blockDim.x) s_h[j] = 0;
    __syncthreads();
    for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
#pragma unroll
        for (int r = 0; r < kOrdPer; ++r) {
            const int64_t p = t * kOrdTile + r * kOrdThreads + threadIdx.x;
            if (p < cnt) atomicAdd(s_h + a[list ? list[p] : p], 1);
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x)
        if (s_h[j]) atomicAdd(bins + j, s_h[j]);
}

// bins[0..k) counts -> bins[k..2k) exclusive starts (one CTA)
__global__ void __launch_bounds__(1024) k_order_scan(int64_t k, int32_t *bins, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl && ctl[1]) return;
    __shared__ int32_t s_w[32];
    __shared__ int32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t j0 = 0; j0 < k; j0 += blockDim.x) {
        const int64_t j = j0 + threadIdx.x;
        const int32_t v = j < k ? bins[j] : 0;
        int32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[w] = x;
        __syncthreads();
        if (w == 0) {
            int32_t z = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(FULL, z, o);
                if (lane >= o) z += y;
            }
            s_w[lane] = z;
        }
        __syncthreads();
        const int32_t excl = s_carry + (w ? s_w[w - 1] : 0) + x - v;
        if (j < k) bins[k + j] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kOrdThreads) k_order_scatter(int64_t k, const int32_t *__restrict__ a,
                                                             const int32_t *__restrict__ list,
                                                             const long long *__restrict__ count, int64_t n,
                                                             int32_t *cursor, int32_t *out,
                                                             const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl && ctl[1]) return;
    extern __shared__ int32_t s_h[];   // [k] tile counts, then the tile's base per bin
    const int64_t cnt = ord_count(count, n);
    const int64_t ntile = (cnt + kOrdTile - 1) / kOrdTile;
    for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
        for (int j = threadIdx.x; j < k; j += blockDim.x) s_h[j] = 0;
        __syncthreads();
        int32_t row[kOrdPer], bin[kOrdPer], rank[kOrdPer];
#pragma unroll
        for (int r = 0; r < kOrdPer; ++r) {
            const int64_t p = t * kOrdTile + r * kOrdThreads + threadIdx.x;
            row[r] = -1;
            if (p < cnt) {
                row[r] = list ? list[p] : (int32_t)p;
                bin[r] = a[row[r]];
                rank[r] = atomicAdd(s_h + bin[r], 1);
            }
        }
        __syncthreads();
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
            const int32_t c = s_h[j];
            if (c) s_h[j] = atomicAdd(cursor + j, c);
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kOrdPer; ++r)
            if (row[r] >= 0) out[s_h[bin[r]] + rank[r]] = row[r];
        __syncthreads();
    }
}

__global__ void k_copy_list(const int32_t *__restrict__ src, int32_t *dst, const long long *__restrict__ count,
                            int64_t n, const long long *__restrict__ ctl) {
    PDL_ENTRY();
    if (ctl && ctl[1]) return;
    const int64_t cnt = ord_count(count, n);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src ? src[i] : (int32_t)i;
}


// TMA descriptor of a row-major float32 [rows][D] operand: box = one stage
// (16 dims = 64 bytes) x box_rows rows, 64-byte swizzle (the K-major
// SWIZZLE_64B layout tcgen05 reads), zero fill past the last row.
// cuTensorMapEncodeTiled comes from the driver entry point.
int encode_dense_map(CUtensorMap *map, const float *base, int64_t rows, int64_t D, int box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return fail_msg("cuTensorMapEncodeTiled unavailable");
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)(rows > 0 ? rows : 1)};
    const cuuint64_t strides[1] = {(cuuint64_t)D * 4};
    const cuuint32_t box[2] = {(cuuint32_t)DN_KC, (cuuint32_t)box_rows};   // one stage: 64-byte rows
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail_msg("cuTensorMapEncodeTiled failed");
    return 0;
}

// TMA descriptor of the term-major float32 centers ct32 [d][kp]: box = 32
// centers x 32 terms with the 128-byte / 32-byte-atom swizzle (the MN-major
// tf32 operand layout of k_gram_mn), zero fill past kp and d.
int encode_gram_map(CUtensorMap *map, const float *base, int64_t kp, int64_t d) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return fail_msg("cuTensorMapEncodeTiled unavailable");
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)d};
    const cuuint64_t strides[1] = {(cuuint64_t)kp * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)GKC};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail_msg("cuTensorMapEncodeTiled (gram) failed");
    return 0;
}

#include "seed.cuh"
#include "prepare.cuh"

}  // namespace

extern "C" {

int spkm_abi_version(void) { return SPKM_ABI_VERSION; }
const char *spkm_last_error(void) { return g_err; }
int64_t spkm_center_chunks(int64_t d) { return (d + kCenterChunk - 1) / kCenterChunk; }
int64_t spkm_padded_k(int64_t k) {
    // a multiple of 8 (one 32-byte sector per 8-center block) covering the
    // row pass's tpr * ch columns
    const ColPlan p = col_plan(k);
    if (k > 32 * 32) return ((k + 1023) / 1024) * 1024;
    const int64_t c = (int64_t)p.tpr * p.ch;
    return (c + 7) / 8 * 8;
}

int spkm_reset_counters(spkm_work *W, void *stream) {
    pdl_launch(k_reset, dim3(1), dim3(32), (size_t)(0), S(stream), W->ctr, W->stats);
    CHECK_LAUNCH("reset_counters");
    return 0;
}

int spkm_full_assign(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int mode,
                     void *stream) {
    if (C->k > 1024) return fail_msg("k > 1024 not supported by this build");
    if (X->n == 0) return 0;
    RowPassArgs A = row_args(X, C);
    A.mode = mode;
    A.a = B->a;
    A.l = B->l;
    A.u = B->u;
    A.ku = B->ku;
    A.mv_i = W->mv_i;
    A.mv_old = W->mv_old;
    A.ctr = W->ctr;
    return launch_row_pass(A, C->k, S(stream), X->n);
}

int spkm_hamerly_bounds(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int use_s,
                        int naive, void *stream) {
    if (X->n == 0) return 0;
    const int64_t tiles = (X->n + kHbTile - 1) / kHbTile;
    if (tiles > INT_MAX) return fail_msg("hamerly_bounds: n too large");
    const int grid = (int)tiles;
    pdl_launch(k_hamerly_bounds, dim3(grid), dim3(kHbThreads), (size_t)(0), S(stream), X->n, X->row_eps, B->a, B->l, B->u, C->drift, C->sinp, C->s,
                                                  C->hstat,
                                                  use_s, naive, W->surv1, W->ctr, C->ctl);
    CHECK_LAUNCH("hamerly_bounds");
    return 0;
}

int spkm_hamerly_tighten(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int use_s,
                         void *stream) {
    if (X->n == 0) return 0;
    const int grid = grid_for((X->n + 3) / 4, 8);
    pdl_launch(k_hamerly_tighten, dim3(grid), dim3(256), (size_t)(0), S(stream), X->indptr, X->indices, X->values, X->row_eps, C->ct32, C->kp,
                                                   B->a, B->l, B->u, C->s, use_s, W->surv1, W->surv2, W->ctr,
                                                   (const double *)(C->hstat + kFuseFlag), C->ctl, hot_terms(C));
    CHECK_LAUNCH("hamerly_tighten");
    return 0;
}

int spkm_hamerly_rescan(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int use_s,
                        void *stream) {
    if (C->k > 1024) return fail_msg("k > 1024 not supported by this build");
    if (X->n == 0) return 0;
    RowPassArgs A = row_args(X, C);
    A.mode = MODE_RESCAN;
    A.rowlist = W->surv2;
    A.rowcount = W->ctr + SPKM_CTR_SURV2;
    A.fuse = C->hstat + kFuseFlag;
    A.rowlist_fused = W->surv1;
    A.rowcount_fused = W->ctr + SPKM_CTR_SURV1;
    A.s_arr = C->s;
    A.use_s = use_s;
    A.a = B->a;
    A.l = B->l;
    A.u = B->u;
    A.ku = 1;
    A.mv_i = W->mv_i;
    A.mv_old = W->mv_old;
    A.ctr = W->ctr;
    return launch_row_pass(A, C->k, S(stream), X->n);
}

int spkm_yy_bounds(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, void *stream) {
    if (X->n == 0) return 0;
    if (C->k > 4 * kYyMaxGroups) return fail_msg("yy_bounds: k > 1024 not supported by this build");
    if (B->ku < (C->k + 3) / 4 || B->ku % 4) return fail_msg("yy_bounds: ku must be ceil(k/4) rounded up to 4");
    const int grid = grid_for((X->n + 31) / 32, 8);
    pdl_launch(k_yy_bounds, dim3(grid), dim3(256), (size_t)(0), S(stream), X->n, (int)C->k, X->row_eps, B->a, B->l,
               B->u, B->ku, C->drift, C->sinp, W->surv1, W->ctr, C->ctl);
    CHECK_LAUNCH("yy_bounds");
    return 0;
}

int spkm_yy_scan(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, void *stream) {
    if (X->n == 0) return 0;
    if (C->k > 4 * kYyMaxGroups) return fail_msg("yy_scan: k > 1024 not supported by this build");
    const int grid = grid_for(X->n, 8);
    const int64_t ngk = (C->k + 3) / 4, ppw_k = (32 / (ngk < 32 ? ngk : 32)) < 8 ? (32 / (ngk < 32 ? ngk : 32)) : 8;
    const size_t dyn = (size_t)8 * yy_sim_stride(C->k) * sizeof(float) + (size_t)8 * ppw_k * kIvStride * sizeof(int2);
    const cudaError_t attr = cudaFuncSetAttribute(k_yy_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (attr != cudaSuccess) return fail("yy_scan smem", attr);
    pdl_launch(k_yy_scan, dim3(grid), dim3(256), dyn, S(stream), X->indptr, X->indices, X->values, X->row_eps,
               C->ct32, C->kp, (int)C->k, B->a, B->l, B->u, B->ku, W->surv1, W->mv_i, W->mv_old, W->ctr, C->ctl,
               hot_terms(C));
    CHECK_LAUNCH("yy_scan");
    return 0;
}

int spkm_elkan_bounds(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int use_cc,
                      void *stream) {
    if (X->n == 0) return 0;
    if (C->k > kEbMaxK) return fail_msg("elkan_bounds: k > 1024 not supported by this build");
    const int grid = grid_for((X->n + 31) / 32, 8);
    if (use_cc)
        pdl_launch(k_elkan_bounds<true>, dim3(grid), dim3(256), (size_t)(0), S(stream), X->n, (int)C->k, X->row_eps, B->a, B->l,
                   B->u, B->ku, C->drift, C->sinp, C->cc, C->s, use_cc, W->surv1, W->ctr, C->ctl, (int)W->elkan_heavy,
                   W->surv2, (int32_t *)nullptr, (const double *)(C->hstat + kAllHeavyFlag));
    else
        pdl_launch(k_elkan_bounds<false>, dim3(grid), dim3(256), (size_t)(0), S(stream), X->n, (int)C->k, X->row_eps, B->a, B->l,
                   B->u, B->ku, C->drift, C->sinp, C->cc, C->s, use_cc, W->surv1, W->ctr, C->ctl, (int)W->elkan_heavy,
                   W->surv2, light_lists(W, use_cc) ? W->lightj : (int32_t *)nullptr,
                   (const double *)(C->hstat + kAllHeavyFlag));
    CHECK_LAUNCH("elkan_bounds");
    return 0;
}

// The heavy survivors of spkm_elkan_bounds (rows where at least
// W->elkan_heavy centers fail the stored-bound test): one full
// pass over the sparse center index instead of the tighten chain + block
// gathers of spkm_elkan_scan -- at C4 a row with > ~1/4 of its centers
// unpruned gathers fewer bytes that way (1.5 KB per nnz against 32 B per
// active 8-center block), and every u(i, j) comes back exact.  Same
// assignments as the scan (both are the Lloyd argmax on the canonical s~).
// With a center index attached, spkm_cindex_build comes before the call; a
// no-op when W->elkan_heavy is 0.
int spkm_elkan_heavy(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, void *stream) {
    if (X->n == 0 || W->elkan_heavy <= 0) return 0;
    if (C->k > 1024) return fail_msg("elkan_heavy: k > 1024 not supported by this build");
    RowPassArgs A = row_args(X, C);
    A.mode = MODE_ELKAN_FULL;
    A.rowlist = W->surv2;
    A.rowcount = W->ctr + SPKM_CTR_SURV2;
    A.allheavy = C->hstat + kAllHeavyFlag;
    A.a = B->a;
    A.l = B->l;
    A.u = B->u;
    A.ku = B->ku;
    A.mv_i = W->mv_i;
    A.mv_old = W->mv_old;
    A.ctr = W->ctr;
    return launch_row_pass(A, C->k, S(stream), X->n);
}

int64_t spkm_elkan_heavy_threshold(int64_t k) { return elkan_heavy_default(k); }

static int elkan_scan_launch(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int use_cc,
                             bool fuse, void *stream) {
    if (X->n == 0) return 0;
    if (C->k > 1024) return fail_msg("elkan_scan: k > 1024 not supported by this build");
    if (!fuse && light_lists(W, use_cc)) {   // the bound pass listed every light row's failing centers
        pdl_launch(k_elkan_light, dim3(grid_for((X->n + 3) / 4, 8)), dim3(256), (size_t)0, S(stream), X->indptr, X->indices,
                   X->values, X->row_eps, C->ct32, C->kp, (int)C->k, B->a, B->l, B->u, B->ku, W->surv1, W->lightj,
                   W->mv_i, W->mv_old, W->ctr, C->ctl, hot_terms(C));
        CHECK_LAUNCH("elkan_light");
        return 0;
    }
    const int grid = grid_for(X->n, 8);
    const int64_t eb = elkan_block(C->k), nbk = (C->k + eb - 1) / eb;
    const int64_t ppw_k = (32 / (nbk < 32 ? nbk : 32)) < 8 ? (32 / (nbk < 32 ? nbk : 32)) : 8;
#ifndef SPKM_EK_SMEM_PAD
#define SPKM_EK_SMEM_PAD 0        // extra bytes of dynamic shared memory (A/B of the L1 carve-out)
#endif
    const size_t dyn = (size_t)8 * elkan_sim_stride(C->k) * sizeof(float) + (size_t)8 * ppw_k * kIvStride * sizeof(int2) +
                       SPKM_EK_SMEM_PAD;
    cudaError_t attr = cudaSuccess;
    auto launch = [&](auto kern) {
        // static smem (staging + active lists) + dyn must fit the opt-in
        // limit; set per launch (cheap), so it holds for every instantiation
        // and device
        attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (attr != cudaSuccess) return;
        pdl_launch(kern, dim3(grid), dim3(256), dyn, S(stream), X->indptr, X->indices, X->values, X->row_eps, C->ct32,
                   C->kp, (int)C->k, B->a, B->l, B->u, B->ku, C->cc, use_cc, W->surv1, W->mv_i, W->mv_old, W->ctr,
                   X->n, C->drift, C->sinp, C->s, C->ctl, hot_terms(C));
    };
    auto launch_r1 = [&](auto kern) {   // k <= 128: the round-1 scan (no `hot` argument)
        attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (attr != cudaSuccess) return;
        pdl_launch(kern, dim3(grid), dim3(256), dyn, S(stream), X->indptr, X->indices, X->values, X->row_eps, C->ct32,
                   C->kp, (int)C->k, B->a, B->l, B->u, B->ku, C->cc, use_cc, W->surv1, W->mv_i, W->mv_old, W->ctr,
                   X->n, C->drift, C->sinp, C->s, C->ctl);
    };
#ifndef SPKM_EK_SMALL_R1
#define SPKM_EK_SMALL_R1 1
#endif
    const bool eb4 = elkan_block(C->k) == 4;
    if (fuse) {
        if (eb4) SPKM_EK_SMALL_R1 ? launch_r1(k_elkan_scan_r1<4, true>) : launch(k_elkan_scan<4, true>);
        else launch(k_elkan_scan<8, true>);
    } else {
        if (eb4) SPKM_EK_SMALL_R1 ? launch_r1(k_elkan_scan_r1<4, false>) : launch(k_elkan_scan<4, false>);
        else launch(k_elkan_scan<8, false>);
    }
    if (attr != cudaSuccess) return fail("elkan_scan smem attribute", attr);
    CHECK_LAUNCH("elkan_scan");
    return 0;
}

int spkm_elkan_scan(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int use_cc,
                    void *stream) {
    return elkan_scan_launch(X, C, B, W, use_cc, false, stream);
}

int spkm_elkan_bounds_scan(const spkm_csr *X, const spkm_centers *C, spkm_bounds *B, spkm_work *W, int use_cc,
                           void *stream) {
    return elkan_scan_launch(X, C, B, W, use_cc, true, stream);
}

// Order a row list by cluster (see "cluster-ordered worklists" above).
// list == NULL: the rows [0, n) are ordered into `out`.  Otherwise the
// first *count (device) entries of `list` are ordered in place through
// `tmp` (n int32).  bins: 2k int32 scratch.  k <= 12288.
int spkm_order_by_cluster(int64_t k, const int32_t *a, int32_t *list, const long long *count, int64_t n,
                          int32_t *tmp, int32_t *out, int32_t *bins, const long long *ctl, void *stream) {
    if (n <= 0 || k <= 1) {
        if (!list && n > 0) {   // identity order
            pdl_launch(k_copy_list, dim3(grid_for(n, 256 * 4)), dim3(256), (size_t)0, S(stream),
                       (const int32_t *)nullptr, out, (const long long *)nullptr, n, ctl);
        }
        return 0;
    }
    if (k > 12288) return fail_msg("order_by_cluster: k > 12288");
    cudaStream_t st = S(stream);
    const size_t smem = (size_t)k * sizeof(int32_t);
    cudaError_t e = cudaMemsetAsync(bins, 0, (size_t)k * sizeof(int32_t), st);
    if (e != cudaSuccess) return fail("order memset", e);
    const int64_t ntile = (n + kOrdTile - 1) / kOrdTile;
    const int64_t cap = (int64_t)num_sms() * 4;
    const int ghist = (int)(ntile < cap ? (ntile < 1 ? 1 : ntile) : cap);
    const int gscat = (int)(ntile < (int64_t)num_sms() * 8 ? (ntile < 1 ? 1 : ntile) : (int64_t)num_sms() * 8);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(k_order_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_order_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    pdl_launch(k_order_hist, dim3(ghist), dim3(kOrdThreads), smem, st, k, a, (const int32_t *)list, count, n,
               bins, ctl);
    CHECK_LAUNCH("order_hist");
    pdl_launch(k_order_scan, dim3(1), dim3(1024), (size_t)0, st, k, bins, ctl);
    CHECK_LAUNCH("order_scan");
    int32_t *dst = list ? tmp : out;
    pdl_launch(k_order_scatter, dim3(gscat), dim3(kOrdThreads), smem, st, k, a, (const int32_t *)list, count, n,
               bins + k, dst, ctl);
    CHECK_LAUNCH("order_scatter");
    if (list) {
        pdl_launch(k_copy_list, dim3(grid_for(n, 256 * 4)), dim3(256), (size_t)0, st, (const int32_t *)tmp, list,
                   count, n, ctl);
        CHECK_LAUNCH("order_copy");
    }
    return 0;
}

int spkm_aggregate_sums(const spkm_csr *X, const spkm_centers *C, const spkm_bounds *B, long long *sums_target,
                        long long *counts_target, void *stream) {
    cudaStream_t st = S(stream);
    cudaError_t e = cudaMemsetAsync(sums_target, 0, sizeof(long long) * C->k * C->d, st);
    if (e != cudaSuccess) return fail("aggregate memset", e);
    e = cudaMemsetAsync(counts_target, 0, sizeof(long long) * C->k, st);
    if (e != cudaSuccess) return fail("aggregate memset", e);
    if (X->n == 0) return 0;
    const int grid = grid_for(X->n, 8);
    pdl_launch(k_aggregate, dim3(grid), dim3(256), (size_t)(0), st, X->n, C->d, X->indptr, X->indices, X->values, B->a, sums_target,
                                      counts_target, ldexp(1.0, C->scale_bits), C->ctl);
    CHECK_LAUNCH("aggregate");
    return 0;
}

int spkm_apply_moves(const spkm_csr *X, const spkm_centers *C, const spkm_bounds *B, const spkm_work *W,
                     long long *sums_target, long long *counts_target, int32_t *touched, void *stream) {
    if (X->n == 0) return 0;
    const int grid = grid_for(X->n, 8);
    pdl_launch(k_apply_moves, dim3(grid), dim3(256), (size_t)(0), S(stream), C->d, X->indptr, X->indices, X->values, B->a, W->mv_i, W->mv_old,
                                               W->ctr, sums_target, counts_target, touched,
                                               ldexp(1.0, C->scale_bits), C->ctl);
    CHECK_LAUNCH("apply_moves");
    return 0;
}

int64_t spkm_center_scratch_doubles(int64_t k, int64_t d) {
    const int64_t nch = spkm_center_chunks(d), ntile = (d + kTileT - 1) / kTileT;
    return k * (nch > 2 * ntile ? nch : 2 * ntile);
}

int spkm_center_reduce(const spkm_centers *C, void *stream);

int spkm_move_centers(const spkm_centers *C, int all_clusters, void *stream) {
    cudaStream_t st = S(stream);
    const int64_t nch = spkm_center_chunks(C->d);
    const int64_t ntile = (C->d + kTileT - 1) / kTileT;
    const double inv = ldexp(1.0, -C->scale_bits);
    const bool defer_reduce = (all_clusters & 4) != 0;   // spkm_center_reduce is issued separately
    all_clusters &= 1;
    // the norm-part CTAs build the touched list themselves only while the
    // grid is small: each of the nch x k CTAs scans all k flags (C4: 245k
    // CTAs x 1000 flags, 73% issue-bound) -- else one k_touched_list launch
    const int build = C->k <= kListInline && nch * C->k <= 65536;
    if (!build) {
        pdl_launch(k_touched_list, dim3(1), dim3(1024), (size_t)(0), st, C->k, C->touched, all_clusters, C->tlist,
                   C->tcount, C->ctl);
        CHECK_LAUNCH("touched_list");
    }
    pdl_launch(k_center_norm_part, dim3(dim3((unsigned)nch, (unsigned)C->k)), dim3(256), (size_t)(0), st, C->d, nch,
               C->sums, C->tlist, C->tcount, inv, C->part, build, C->k, (const int32_t *)C->touched, all_clusters, C->ctl);
    CHECK_LAUNCH("center_norm_part");
    pdl_launch(k_center_norm_final, dim3((unsigned)C->k), dim3(256), (size_t)(0), st, nch, C->counts, C->tlist, C->tcount, C->part, C->norm, C->ctl);
    CHECK_LAUNCH("center_norm_final");
    pdl_launch(k_center_write, dim3(dim3((unsigned)ntile, (unsigned)((C->k + kTileJ - 1) / kTileJ))), dim3(256), (size_t)(0), st, 
        C->d, C->kp, ntile, C->sums, C->tlist, C->tcount, inv, C->norm, C->cent64, C->ct32,
        reinterpret_cast<__half *>(C->ct16), C->part, C->ctl);
    CHECK_LAUNCH("center_write");
    return defer_reduce ? 0 : spkm_center_reduce(C, stream);
}

int spkm_center_reduce(const spkm_centers *C, void *stream) {
    const int64_t ntile = (C->d + kTileT - 1) / kTileT;
    pdl_launch(k_center_reduce, dim3((unsigned)C->k), dim3(256), (size_t)0, S(stream), ntile, C->tlist, C->tcount, C->part,
               C->norm, C->drift, C->sinp, C->objc, C->ctl);
    CHECK_LAUNCH("center_reduce");
    return 0;
}

// SPKM_HAMERLY_FUSE: 0 = never fuse the tighten into the rescan, 1 = always,
// unset / 2 = when the last tighten pruned < 5% (read at every call, so the
// eager loop can be switched for A/B tests; a captured graph keeps its value)
static int hamerly_fuse_policy() {
    const char *e = getenv("SPKM_HAMERLY_FUSE");
    const int v = e ? atoi(e) : 2;
    return (v >= 0 && v <= 2) ? v : 2;
}

int spkm_finalize(const spkm_centers *C, spkm_work *W, int all_clusters, long long sims_extra, void *stream) {
    pdl_launch(k_finalize, dim3(1), dim3(kFinThreads), (size_t)(0), S(stream), C->k, C->touched, C->tcount, C->drift, C->sinp, C->objc, C->hstat,
                                                 W->ctr, W->stats, sims_extra, all_clusters, W->stats_hist,
                                                 W->hist_cap, hamerly_fuse_policy(), C->ctl,
                                                 (long long)(W->elkan_heavy > 0 ? W->allheavy_rows : 0));
    CHECK_LAUNCH("finalize");
    return 0;
}

int64_t spkm_gram_dsplit(int64_t k, int64_t d) {
    // one wave: one CTA per SM (k_gram_mn stages ~192 KB); at least 256
    // terms per CTA
    const int64_t tk = (k + GT - 1) / GT;
    const int64_t tiles = tk * (tk + 1) / 2;
    const int64_t per_sm = 1;
    int64_t ds = (int64_t)num_sms() * per_sm / tiles;
    const int64_t maxds = (d + 255) / 256;
    if (ds > maxds) ds = maxds;
    if (ds < 1) ds = 1;
    return ds;
}

int64_t spkm_gram_scratch_doubles(int64_t k, int64_t d) { return spkm_gram_dsplit(k, d) * k * k; }

int spkm_gram_partial(const spkm_centers *C, double *gpart, const void *tiles_ptr, int full, int rank, int world,
                      void *stream);
int spkm_gram_finish(const spkm_centers *C, double *gpart, int full, void *stream);

int spkm_center_thresholds(const spkm_centers *C, double *gpart, const void *tiles_ptr, int full, void *stream) {
    const int rc = spkm_gram_partial(C, gpart, tiles_ptr, full, 0, 1, stream);
    return rc ? rc : spkm_gram_finish(C, gpart, full, stream);
}

int64_t spkm_gram_partial_floats(int64_t k, int64_t d) { return spkm_gram_dsplit(k, d) * k * k; }

int spkm_gram_partial(const spkm_centers *C, double *gpart, const void *tiles_ptr, int full, int rank, int world,
                      void *stream) {
    if (world < 1 || rank < 0 || rank >= world) return fail_msg("gram_partial: bad rank / world");
    const int2 *tiles_dev = static_cast<const int2 *>(tiles_ptr);
    cudaStream_t st = S(stream);
    const int64_t tk = (C->k + GT - 1) / GT;
    const int64_t ntiles = tk * (tk + 1) / 2;
    const int64_t ds = spkm_gram_dsplit(C->k, C->d);
    // float32 partials [ds][k][k], then one dirty flag per tile (fits the double-sized scratch)
    float *gp = reinterpret_cast<float *>(gpart);
    CUtensorMap tm;
    int rc = encode_gram_map(&tm, C->ct32, C->kp, C->d);
    if (rc) return rc;
    // set on every call (cheap; the opt-in is per device, a process-wide
    // "done" flag would miss a second device)
    cudaError_t ae = tk == 1 ? cudaFuncSetAttribute(k_gram_mn<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)GmCfg<true>::SMEM)
                             : cudaFuncSetAttribute(k_gram_mn<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)GmCfg<false>::SMEM);
    if (ae != cudaSuccess) return fail("gram_mn smem attribute", ae);
    if (world > 1) {   // this rank's share of the partials; the others are zeroed and summed in by the caller
        const cudaError_t me = cudaMemsetAsync(gp, 0, sizeof(float) * ds * C->k * C->k, st);
        if (me != cudaSuccess) return fail("gram_partial memset", me);
    }
    if (tk == 1)
        pdl_launch(k_gram_mn<true>, dim3(1, (unsigned)ds), dim3(GM_THREADS), GmCfg<true>::SMEM, st, tm, C->k, C->d, ds,
                   tiles_dev, C->tlist, C->tcount, full, gp, C->ctl, rank, world);
    else
        pdl_launch(k_gram_mn<false>, dim3((unsigned)ntiles, (unsigned)ds), dim3(GM_THREADS), GmCfg<false>::SMEM, st, tm,
                   C->k, C->d, ds, tiles_dev, C->tlist, C->tcount, full, gp, C->ctl, rank, world);
    CHECK_LAUNCH("gram_mn");
    return 0;
}

int spkm_gram_finish(const spkm_centers *C, double *gpart, int full, void *stream) {
    cudaStream_t st = S(stream);
    const int64_t ds = spkm_gram_dsplit(C->k, C->d);
    const int64_t per = ((C->d + ds - 1) / ds + GKC - 1) / GKC * GKC;
    const double gdelta = (3.0 * (double)per / 8.0 + 8.0) * ldexp(1.0, -22) + 2e-6;
    float *gp = reinterpret_cast<float *>(gpart);
    pdl_launch(k_gram_final, dim3((unsigned)((C->k * C->k * 8 + 255) / 256)), dim3(256), (size_t)0, st, C->k, ds, gp,
               full, gdelta, C->cc, C->ctl);
    CHECK_LAUNCH("gram_final");
    pdl_launch(k_row_max, dim3((unsigned)((C->k * 32 + 255) / 256)), dim3(256), (size_t)(0), st, C->k, C->cc, C->s, C->ctl);
    CHECK_LAUNCH("row_max");
    return 0;
}

// Fill the upper-triangle tile list used by the Gram kernel.
int64_t spkm_gram_tiles(int64_t k, int32_t *host_pairs /* [2*ntiles] */) {
    const int64_t tk = (k + GT - 1) / GT;
    int64_t q = 0;
    for (int64_t a = 0; a < tk; ++a)
        for (int64_t j = a; j < tk; ++j) {
            if (host_pairs) {
                host_pairs[2 * q] = (int32_t)a;
                host_pairs[2 * q + 1] = (int32_t)j;
            }
            ++q;
        }
    return q;
}

int spkm_predict(const spkm_csr *X, const spkm_centers *C, int32_t *a, double *best, double *second,
                 void *stream) {
    if (C->k > 1024) return fail_msg("k > 1024 not supported by this build");
    if (X->n == 0) return 0;
    RowPassArgs A = row_args(X, C);
    A.mode = MODE_PREDICT;
    A.a = a;
    A.best = best;
    A.second = second;
    return launch_row_pass(A, C->k, S(stream), X->n);
}


int spkm_dense_centers(const spkm_centers *C, const spkm_dense *Dn, void *stream) {
    pdl_launch(k_dense_centers, dim3(grid_for(Dn->kpad * Dn->D, 256)), dim3(256), (size_t)(0), S(stream), C->k, Dn->kpad, Dn->D, C->cent64,
                                                                           Dn->b, C->ctl);
    CHECK_LAUNCH("dense_centers");
    return 0;
}

int spkm_dense_assign(const spkm_csr *X, const spkm_centers *C, const spkm_dense *Dn, spkm_bounds *B,
                      spkm_work *W, int mode, int use_s, double *best, double *second, void *stream) {
    if (X->n == 0) return 0;
    if (Dn->D % 32 != 0) return fail_msg("dense dimension must be a multiple of 32");
    if (Dn->kpad % DN_N != 0 || Dn->kpad < C->k) return fail_msg("dense kpad must cover k in multiples of 256");
    cudaStream_t st = S(stream);
    DenseArgs P{};
    P.n = X->n;
    P.D = Dn->D;
    P.k = C->k;
    P.kpad = Dn->kpad;
    P.ku = B ? B->ku : 1;
    P.reps = X->row_eps;
    P.mode = mode;
    P.use_s = use_s;
    P.a = B->a;
    P.l = B->l;
    P.u = B->u;
    P.s_arr = C->s;
    P.ctl = C->ctl;
    if (W) {
        P.mv_i = W->mv_i;
        P.mv_old = W->mv_old;
        P.surv2 = W->surv2;
        P.ctr = W->ctr;
    }
    P.best = best;
    P.second = second;
    const float *rows = Dn->x;
    if (mode == DMODE_RESCAN_H) {
        // survivors are compacted into a contiguous float32 block so the
        // pass streams them with TMA exactly like a full pass
        if (!Dn->xs) return fail_msg("dense rescan needs the survivor scratch (spkm_dense.xs)");
        P.rowmap = W->surv1;
        P.rowcount = W->ctr + SPKM_CTR_SURV1;
        pdl_launch(k_gather_rows, dim3(grid_for(X->n * (Dn->D / 4), 256)), dim3(256), (size_t)(0), st, Dn->x, Dn->D, W->surv1, P.rowcount, Dn->xs,
                                                                          C->ctl);
        CHECK_LAUNCH("dense_gather");
        rows = Dn->xs;
    }
    int rc = encode_dense_map(&P.tm_x, rows, X->n, Dn->D, DN_M);
    if (!rc) rc = encode_dense_map(&P.tm_b, Dn->b, Dn->kpad, Dn->D, DN_N);
    if (rc) return rc;
    {
        static int dbg = -1;
        if (dbg < 0) {
            const char *e = getenv("SPKM_DN_DBG");
            dbg = e ? atoi(e) : 0;
        }
        P.dbg = dbg;
    }
    const size_t smem = (size_t)DN_STAGES * DN_STAGE;
    const cudaError_t ae = cudaFuncSetAttribute(k_dense_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ae != cudaSuccess) return fail("dense_pass smem attribute", ae);
    int64_t tiles = (X->n + DN_M - 1) / DN_M;
    int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    if (grid < 1) grid = 1;
    pdl_launch(k_dense_pass, dim3(grid), dim3(DN_THREADS), (size_t)(smem), st, P);
    CHECK_LAUNCH("dense_pass");
    return 0;
}

int spkm_objective(const spkm_centers *C, const long long *sums, double *out, void *stream) {
    cudaStream_t st = S(stream);
    const int64_t nch = spkm_center_chunks(C->d);
    dim3 grid((unsigned)nch, (unsigned)C->k);
    k_objective_part<<<grid, 256, 0, st>>>(C->d, nch, sums, C->cent64, ldexp(1.0, -C->scale_bits), C->part);
    CHECK_LAUNCH("objective_part");
    k_objective_final<<<1, 32, 0, st>>>(C->k, nch, C->part, out);
    CHECK_LAUNCH("objective_final");
    return 0;
}

int spkm_load_centers(const spkm_centers *C, const double *src, void *stream) {
    const int64_t tot = C->k * C->d;
    k_load_centers<<<(unsigned)((tot + 255) / 256), 256, 0, S(stream)>>>(C->k, C->d, C->kp, src, C->cent64,
                                                                         C->ct32, reinterpret_cast<__half *>(C->ct16));
    CHECK_LAUNCH("load_centers");
    return 0;
}

int spkm_seed_rows(const spkm_centers *C, const int64_t *sptr, const int32_t *sidx, const double *sval,
                   void *stream) {
    cudaStream_t st = S(stream);
    cudaError_t e = cudaMemsetAsync(C->cent64, 0, sizeof(double) * C->k * C->d, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(C->ct32, 0, sizeof(float) * C->kp * C->d, st);
    if (e == cudaSuccess && C->ct16) e = cudaMemsetAsync(C->ct16, 0, sizeof(uint16_t) * C->kp * C->d, st);
    if (e != cudaSuccess) return fail("seed_rows memset", e);
    k_seed_rows<<<(unsigned)C->k, 128, 0, st>>>(C->d, C->kp, sptr, sidx, sval, C->cent64, C->ct32,
                                                reinterpret_cast<__half *>(C->ct16));
    CHECK_LAUNCH("seed_rows");
    return 0;
}

int spkm_geometry(int op, int64_t n, const double *a, const double *b, double *out, void *stream) {
    if (n == 0) return 0;
    k_geometry<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(op, n, a, b, out);
    CHECK_LAUNCH("geometry");
    return 0;
}

// ------------------------------------------------------------------ seeding
int64_t spkm_seed_scratch_doubles(int64_t n, int64_t d) { return seed::scratch_doubles(n, d); }

static int seed_init(const seed::Args &A, uint64_t seed_value, cudaStream_t st) {
    seed::Ctl c{};
    c.rng = seed_value;
    const char *fs = getenv("SPKM_SEED_EXACT");   // test hook (see seed.cuh)
    c.force_seq = (fs && atoi(fs)) ? 1 : 0;
    cudaError_t e = cudaMemsetAsync(A.chosen, 0, (size_t)A.n, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(A.cden, 0, sizeof(double) * (size_t)A.d, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(A.ctl, &c, sizeof c, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);   // c lives on this stack frame
    return e == cudaSuccess ? 0 : fail("seed init", e);
}

int spkm_seed_kmpp(const spkm_seed *Sd, int64_t k, double alpha, uint64_t seed_value, int64_t *picks,
                   double *trace, void *stream) {
    if (k < 1 || k > Sd->n) return fail_msg("seed_kmpp: k must be in [1, n]");
    cudaStream_t st = S(stream);
    const seed::Args A = seed::carve(Sd, picks);
    if (int rc = seed_init(A, seed_value, st)) return rc;
    const int gs = grid_for(A.n, 8);
    seed::k_select<<<1, seed::kSelThreads, 0, st>>>(A, seed::SEL_FIRST, 0, 0);
    for (int64_t t = 0; t + 1 < k; ++t) {
        seed::k_scatter<<<1, 256, 0, st>>>(A, t);
        seed::k_sims<<<gs, 256, 0, st>>>(A, seed::SIM_KMPP, t, alpha);
        seed::k_partials<<<(unsigned)A.nb, 256, 0, st>>>(A.w, A.n, A.part);
        if (trace) {
            cudaError_t e = cudaMemcpyAsync(trace + t * A.n, A.w, sizeof(double) * A.n, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return fail("seed_kmpp trace", e);
        }
        seed::k_select<<<1, seed::kSelThreads, 0, st>>>(A, seed::SEL_KMPP, t + 1, 0);
    }
    CHECK_LAUNCH("seed_kmpp");
    return 0;
}

int spkm_seed_afkmc2(const spkm_seed *Sd, int64_t k, double alpha, int64_t chain_length, uint64_t seed_value,
                     int64_t *picks, void *stream) {
    if (k < 1 || k > Sd->n) return fail_msg("seed_afkmc2: k must be in [1, n]");
    if (chain_length < 1) return fail_msg("seed_afkmc2: chain_length must be >= 1");
    cudaStream_t st = S(stream);
    const seed::Args A = seed::carve(Sd, picks);
    if (int rc = seed_init(A, seed_value, st)) return rc;
    const int gs = grid_for(A.n, 8);
    seed::k_select<<<1, seed::kSelThreads, 0, st>>>(A, seed::SEL_FIRST, 0, 0);
    seed::k_scatter<<<1, 256, 0, st>>>(A, 0);
    seed::k_sims<<<gs, 256, 0, st>>>(A, seed::SIM_AFK_INIT, 0, alpha);
    // sum(d) in numpy's pairwise order: plan (integers) on the host, sums on the device
    seed::PwPlan P;
    seed::pw_plan(A.n, P);
    const int64_t L = (int64_t)P.leaf_off.size() - 1;
    const int H = (int)P.lvl.size() - 1;
    if (L > seed::max_leaves(A.n) || H > 62) return fail_msg("seed_afkmc2: pairwise plan exceeds scratch");
    cudaError_t e = cudaMemcpyAsync(A.leaf_off, P.leaf_off.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && !P.node_lr.empty())
        e = cudaMemcpyAsync(A.node_lr, P.node_lr.data(), sizeof(int64_t) * P.node_lr.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(A.lvl, P.lvl.data(), sizeof(int64_t) * P.lvl.size(), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail("seed_afkmc2 plan upload", e);
    seed::k_pw_leaves<<<(unsigned)((L + 255) / 256), 256, 0, st>>>(A, L);
    seed::k_pw_tree<<<1, 1024, 0, st>>>(A, A.lvl, H, L);
    seed::k_afk_q<<<(unsigned)((A.n + 255) / 256), 256, 0, st>>>(A);
    seed::k_afk_cumq<<<1, 32, 0, st>>>(A);
    for (int64_t t = 1; t < k; ++t) {
        seed::k_partials<<<(unsigned)A.nb, 256, 0, st>>>(A.ms, A.n, A.part);
        seed::k_select<<<1, seed::kSelThreads, 0, st>>>(A, seed::SEL_AFK, t, chain_length);
        if (t + 1 < k) {
            seed::k_scatter<<<1, 256, 0, st>>>(A, t);
            seed::k_sims<<<gs, 256, 0, st>>>(A, seed::SIM_AFK_UPDATE, t, alpha);
        }
    }
    CHECK_LAUNCH("seed_afkmc2");
    // the host plan vectors are freed on return: wait for the uploads
    e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? 0 : fail("seed_afkmc2", e);
}

// SparseVector.norm (sparse.py:52) for every CSR row on the host, in the
// reference's np.dot order (the ddot order of seed::warp_ddot): lets
// Dataset.from_csr normalise rows bit-identically to Dataset.from_rows.
int spkm_host_row_norms(int64_t n, const int64_t *indptr, const double *values, double *out) {
    for (int64_t r = 0; r < n; ++r) {
        const double *x = values + indptr[r];
        const int64_t m = indptr[r + 1] - indptr[r];
        const int64_t n32 = m & ~int64_t(31), n1 = m & ~int64_t(15);
        double z[32] = {0};
        for (int64_t b = 0; b < n32; b += 32)
            for (int L = 0; L < 32; ++L) z[L] = fma(x[b + L], x[b + L], z[L]);
        double a[16];
        for (int bb = 0; bb < 4; ++bb)
            for (int l = 0; l < 4; ++l) a[4 * bb + l] = z[8 * bb + l] + z[8 * bb + l + 4];
        if (n1 > n32)
            for (int mm = 0; mm < 16; ++mm) a[mm] = fma(x[n32 + mm], x[n32 + mm], a[mm]);
        double t[4];
        for (int l = 0; l < 4; ++l) t[l] = ((a[l] + a[4 + l]) + a[8 + l]) + a[12 + l];
        const double h0 = t[0] + t[2], h1 = t[1] + t[3];
        double dot = h0 + h1;
        for (int64_t i = n1; i < m; ++i) dot = fma(x[i], x[i], dot);
        out[r] = sqrt(dot);
    }
    return 0;
}


int spkm_seed_rows_csr(const spkm_centers *C, const spkm_seed *Sd, const int64_t *rows, void *stream) {
    cudaStream_t st = S(stream);
    cudaError_t e = cudaMemsetAsync(C->cent64, 0, sizeof(double) * C->k * C->d, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(C->ct32, 0, sizeof(float) * C->kp * C->d, st);
    if (e == cudaSuccess && C->ct16) e = cudaMemsetAsync(C->ct16, 0, sizeof(uint16_t) * C->kp * C->d, st);
    if (e != cudaSuccess) return fail("seed_rows_csr memset", e);
    pdl_launch(k_seed_rows_csr, dim3((unsigned)C->k), dim3(128), (size_t)(0), st, C->d, C->kp, Sd->indptr, Sd->indices, Sd->values, Sd->row_dev,
                                                     rows, C->cent64, C->ct32, reinterpret_cast<__half *>(C->ct16));
    CHECK_LAUNCH("seed_rows_csr");
    return 0;
}

int spkm_permute_rows(int64_t n, const int64_t *ip_raw, const int32_t *idx_raw, const double *val_raw,
                      const int64_t *perm, const int64_t *ip_new, const int64_t *new_id, int32_t *idx, float *val,
                      double *val64, float *reps, void *stream) {
    if (n == 0) return 0;
    k_permute_rows<<<grid_for(n, 8), 256, 0, S(stream)>>>(n, ip_raw, idx_raw, val_raw, perm, ip_new, new_id, idx, val,
                                                         val64, reps);
    CHECK_LAUNCH("permute_rows");
    return 0;
}


int64_t spkm_cindex_scratch_bytes(int64_t d) {
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, (const int64_t *)nullptr, (int64_t *)nullptr, (int)(d > 0 ? d : 1));
    return (int64_t)t;
}

int spkm_cindex_build(const spkm_centers *C, void *stream) {
    const spkm_cindex *I = C->cindex;
    if (!I) return fail_msg("cindex_build: no index attached");
    if (C->k > 2047) return fail_msg("cindex_build: k > 2047");
    cudaStream_t st = S(stream);
    const int grid = grid_for((C->d + 7) / 8, 1);
    // the running total of reserved pairs lives in off[0] (the scan scratch of the two-pass build is unused)
    if (cudaMemsetAsync(I->off, 0, sizeof(int64_t), st) != cudaSuccess) return fail_msg("cindex_build: memset failed");
    pdl_launch(k_ci_build, dim3(grid), dim3(256), (size_t)0, st, C->d, C->kp, (int)C->k, C->ct32, I->dense_thr,
               reinterpret_cast<unsigned long long *>(I->off), I->desc, reinterpret_cast<int2 *>(I->pairs), C->ctl);
    CHECK_LAUNCH("ci_build");
    return 0;
}

// ------------------------------------------------- corpus layout (prepare.cuh)
int64_t spkm_prepare_scratch_bytes(int64_t n, int64_t d) {
    if (n < 0 || d < 0 || n > INT32_MAX || d > INT32_MAX) return -1;
    return (int64_t)prep_plan(n, d).total;
}

int spkm_prepare_rows(int64_t n, int64_t d, int64_t nnz, const int64_t *ip_raw, const int32_t *idx_raw,
                      int64_t *perm, int64_t *pos, int64_t *indptr, int64_t *order, int64_t *new_id,
                      void *scratch, int64_t scratch_bytes, void *stream) {
    if (n < 0 || d < 0 || n > INT32_MAX || d > INT32_MAX) return fail_msg("prepare_rows: n and d must be < 2^31");
    const PrepPlan p = prep_plan(n, d);
    if (scratch_bytes < (int64_t)p.total || (!scratch && p.total)) return fail_msg("prepare_rows: scratch too small");
    cudaStream_t st = (cudaStream_t)stream;
    char *s = (char *)scratch;
    uint32_t *rk = (uint32_t *)s;
    int64_t *rv = (int64_t *)(s + p.rows_key);
    void *rt = s + p.rows_key + p.rows_val;
    int64_t *lens = (int64_t *)(s + p.rows_key + p.rows_val + p.rows_tmp);
    char *s2 = s + p.rows_key + p.rows_val + p.rows_tmp + p.rows_lens;
    uint32_t *tk = (uint32_t *)s2;
    int64_t *tv = (int64_t *)(s2 + p.terms_key);
    void *tt = s2 + p.terms_key + p.terms_val;
    if (perm && n > 0) {
        // rows: stable sort by length, descending -> perm
        k_row_keys<<<grid1(n), 256, 0, st>>>(n, ip_raw, rk, rv);
        size_t tb = p.rows_tmp;
        if (cub::DeviceRadixSort::SortPairsDescending(rt, tb, rk, rk + n, rv, perm, (int)n, 0, 32, st) != cudaSuccess)
            return fail_msg("prepare_rows: CUB sort/scan failed");
        k_perm_lens<<<grid1(n), 256, 0, st>>>(n, ip_raw, perm, lens, pos, indptr);
        tb = p.rows_tmp;
        if (cub::DeviceScan::InclusiveSum(rt, tb, lens, indptr + 1, (int)n, st) != cudaSuccess) return fail_msg("prepare_rows: CUB sort/scan failed");
    } else if (perm) {
        cudaMemsetAsync(indptr, 0, sizeof(int64_t), st);
    }
    if (order && new_id && d > 0) {
        // terms: stable sort by document frequency, descending -> order; new_id = order^-1
        cudaMemsetAsync(tk, 0, (size_t)d * sizeof(uint32_t), st);
        if (nnz > 0) k_term_df<<<grid1(nnz), 256, 0, st>>>(nnz, idx_raw, tk);
        k_iota<<<grid1(d), 256, 0, st>>>(d, tv);
        size_t tb = p.terms_tmp;
        if (cub::DeviceRadixSort::SortPairsDescending(tt, tb, tk, tk + d, tv, order, (int)d, 0, 32, st) != cudaSuccess)
            return fail_msg("prepare_rows: CUB sort/scan failed");
        k_invert<<<grid1(d), 256, 0, st>>>(d, order, new_id);
    }
    CHECK_LAUNCH("prepare_rows");
    return 0;
}


int spkm_dense_ids(int64_t n, int64_t D, int32_t *idx, int64_t *indptr, int64_t *perm, void *stream) {
    if (n <= 0 || D <= 0) return 0;
    k_dense_ids<<<grid1(n * D), 256, 0, S(stream)>>>(n, D, idx, indptr, perm);
    CHECK_LAUNCH("dense_ids");
    return 0;
}


// ------------------------------------------------------------ bound auditor
int spkm_audit_transpose(int64_t k, int64_t d, int64_t kp, const double *cent64, double *ct64, void *stream) {
    dim3 grid((unsigned)((d + 31) / 32), (unsigned)((kp + 31) / 32));
    k_transpose_centers<<<grid, dim3(32, 8), 0, S(stream)>>>(k, d, kp, cent64, ct64);
    CHECK_LAUNCH("audit_transpose");
    return 0;
}

int spkm_audit(const spkm_seed *Sd, int64_t k, int64_t kp, const double *ct64, const int32_t *a, const float *l,
               const float *u, int64_t ku, int mode, unsigned long long *keys, int32_t *a_out, void *stream) {
    if (Sd->n == 0) return 0;
    k_audit<<<grid_for(Sd->n, 8), 256, 0, S(stream)>>>(Sd->n, k, kp, Sd->indptr, Sd->indices, Sd->values, ct64, a, l,
                                                       u, ku, mode, keys, a_out);
    CHECK_LAUNCH("audit");
    return 0;
}


// ------------------------------------------------------ multi-GPU exchange
// rounded up to 4 ints: every slot of the allgathered array starts 16-byte
// aligned, so its int64 counter head is an aligned load for every rank q
// (an odd slot length put rank 1's head on a 4-byte boundary: misaligned
// address at world 3, found by tests/test_gpu_loopback.py)
int64_t spkm_move_slot_ints(int64_t cap) { return (kSlotHead + 3 * cap + 3) / 4 * 4; }

int spkm_pack_moves(const spkm_work *W, const spkm_bounds *B, const spkm_centers *C, int64_t p0, int64_t cap,
                    int32_t *slot, void *stream) {
    pdl_launch(k_pack_moves, dim3(grid_for(cap > 0 ? cap : 1, 256)), dim3(256), (size_t)(0), S(stream), W->mv_i, W->mv_old, B->a, W->ctr, p0, cap,
                                                                        slot, C->ctl);
    CHECK_LAUNCH("pack_moves");
    return 0;
}

int spkm_apply_move_slots(const spkm_csr *X, const spkm_centers *C, const int32_t *slots, int world, int64_t slot_len,
                          int32_t *touched, long long *ctr_out, void *stream) {
    pdl_launch(k_apply_move_slots, dim3(grid_for(X->n > 0 ? X->n : 1, 8)), dim3(256), (size_t)(0), S(stream), 
        slots, world, slot_len, C->d, X->indptr, X->indices, X->values, C->sums, C->counts, touched,
        ldexp(1.0, C->scale_bits), ctr_out, C->ctl);
    CHECK_LAUNCH("apply_move_slots");
    return 0;
}

// ---------------------------------------------------- device-driven fit loop
// One CUDA graph per engine: [k_loop_cond] -> WHILE(cond) { one iteration's
// kernels (captured from the host's own calls) ; k_loop_cond }.  A fit is
// then iteration 1 + one graph launch, with no host round trip per iteration.
struct spkm_loop {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle handle = 0;
    const long long *ctl = nullptr;
    const long long *limit = nullptr;
    cudaStream_t stream = nullptr;        // body capture stream
    cudaStream_t outer = nullptr;         // whole-fit graph: the prefix / suffix capture stream
    cudaGraphNode_t loop_node = nullptr;
};

int spkm_loop_begin(const long long *ctl, const long long *limit, void *stream, void **out) {
    spkm_loop *L = new spkm_loop();
    L->ctl = ctl;
    L->limit = limit;
    L->stream = S(stream);
    cudaError_t e = cudaGraphCreate(&L->graph, 0);
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&L->handle, L->graph, 0, 0);
    cudaGraphNode_t pre = nullptr, loop = nullptr;
    if (e == cudaSuccess) {
        cudaKernelNodeParams kp = {};
        void *args[] = {&L->handle, &L->ctl, &L->limit};
        kp.func = (void *)k_loop_cond;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = args;
        e = cudaGraphAddKernelNode(&pre, L->graph, nullptr, 0, &kp);
    }
    cudaGraph_t body = nullptr;
    if (e == cudaSuccess) {
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = L->handle;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        e = cudaGraphAddNode(&loop, L->graph, &pre, 1, &np);
        if (e == cudaSuccess) body = np.conditional.phGraph_out[0];
    }
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(L->stream, body, nullptr, nullptr, 0,
                                                            cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        if (L->graph) cudaGraphDestroy(L->graph);
        delete L;
        return fail("loop_begin", e);
    }
    *out = L;
    return 0;
}

int spkm_loop_end(void *loop) {
    spkm_loop *L = static_cast<spkm_loop *>(loop);
    k_loop_cond<<<1, 1, 0, L->stream>>>(L->handle, L->ctl, L->limit);
    cudaError_t e0 = cudaGetLastError();
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(L->stream, &g);
    if (e0 != cudaSuccess) return fail("loop_end cond", e0);
    if (e != cudaSuccess) return fail("loop_end capture", e);
    if (L->outer) return 0;   // whole-fit graph: the suffix follows on the outer stream
    e = cudaGraphInstantiate(&L->exec, L->graph, 0);
    return e == cudaSuccess ? 0 : fail("loop_end instantiate", e);
}

// Whole-fit graph: prefix (seed upload, iterations 1-2) captured on `stream`,
// then the WHILE node, then the suffix (result downloads) on `stream` again.
int spkm_fit_graph_begin(void *stream, void **out) {
    spkm_loop *L = new spkm_loop();
    L->outer = S(stream);
    cudaError_t e = cudaGraphCreate(&L->graph, 0);
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(L->outer, L->graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        if (L->graph) cudaGraphDestroy(L->graph);
        delete L;
        return fail("fit_graph_begin", e);
    }
    *out = L;
    return 0;
}

int spkm_fit_graph_loop(void *loop, const long long *ctl, const long long *limit, void *body_stream) {
    spkm_loop *L = static_cast<spkm_loop *>(loop);
    L->ctl = ctl;
    L->limit = limit;
    L->stream = S(body_stream);
    cudaError_t e = cudaGraphConditionalHandleCreate(&L->handle, L->graph, 0, 0);
    if (e != cudaSuccess) return fail("fit_graph_loop handle", e);
    k_loop_cond<<<1, 1, 0, L->outer>>>(L->handle, L->ctl, L->limit);   // sets the first condition value
    e = cudaGetLastError();
    cudaStreamCaptureStatus cs;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t ndeps = 0;
    if (e == cudaSuccess) e = cudaStreamGetCaptureInfo(L->outer, &cs, nullptr, &g, &deps, &ndeps);
    cudaGraph_t body = nullptr;
    if (e == cudaSuccess) {
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = L->handle;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        e = cudaGraphAddNode(&L->loop_node, g, deps, ndeps, &np);
        if (e == cudaSuccess) body = np.conditional.phGraph_out[0];
    }
    if (e == cudaSuccess)
        e = cudaStreamUpdateCaptureDependencies(L->outer, &L->loop_node, 1, cudaStreamSetCaptureDependencies);
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(L->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    return e == cudaSuccess ? 0 : fail("fit_graph_loop", e);
}

int spkm_fit_graph_end(void *loop) {
    spkm_loop *L = static_cast<spkm_loop *>(loop);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(L->outer, &g);
    if (e != cudaSuccess) return fail("fit_graph_end capture", e);
    e = cudaGraphInstantiate(&L->exec, L->graph, 0);
    return e == cudaSuccess ? 0 : fail("fit_graph_end instantiate", e);
}

// Error path of a whole-fit capture: close whatever capture is still open
// (body and outer stream) so the streams are usable again, drop the graph.
int spkm_fit_graph_abort(void *loop) {
    spkm_loop *L = static_cast<spkm_loop *>(loop);
    if (!L) return 0;
    for (cudaStream_t st : {L->stream, L->outer}) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (st && cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(st, &g);
        }
    }
    cudaGetLastError();
    // the graph is left to the driver: after an invalidated capture its state
    // is undefined, and destroying it has crashed (a one-off leak on an error path)
    delete L;
    return 0;
}

int spkm_rows_to_host(int64_t n, const int64_t *row_perm, const int32_t *a, int64_t *out, void *stream) {
    if (n <= 0) return 0;
    pdl_launch(k_rows_to_host, dim3((unsigned)((n + 255) / 256)), dim3(256), (size_t)(0), S(stream), n, row_perm, a, out);
    CHECK_LAUNCH("rows_to_host");
    return 0;
}

int spkm_memcpy_async(void *dst, const void *src, int64_t bytes, void *stream) {
    if (bytes <= 0) return 0;
    cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, S(stream));
    return e == cudaSuccess ? 0 : fail("memcpy_async", e);
}

int spkm_memset_async(void *dst, int value, int64_t bytes, void *stream) {
    if (bytes <= 0) return 0;
    cudaError_t e = cudaMemsetAsync(dst, value, (size_t)bytes, S(stream));
    return e == cudaSuccess ? 0 : fail("memset_async", e);
}

int spkm_loop_launch(void *loop, void *stream) {
    spkm_loop *L = static_cast<spkm_loop *>(loop);
    cudaError_t e = cudaGraphLaunch(L->exec, S(stream));
    return e == cudaSuccess ? 0 : fail("loop_launch", e);
}

int spkm_loop_destroy(void *loop) {
    spkm_loop *L = static_cast<spkm_loop *>(loop);
    if (!L) return 0;
    if (L->exec) cudaGraphExecDestroy(L->exec);
    if (L->graph) cudaGraphDestroy(L->graph);
    delete L;
    return 0;
}

}  // extern "C"
