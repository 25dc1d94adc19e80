// seed.cuh -- spherical k-means++ and AFK-MC2 seeding on the device
// (reference seeding.py:64-146), included by spkm.cu inside its anonymous
// namespace.
//
// Exactness contract: the picks equal the reference's picks.
//  * Similarities to the picked row are float64 in the order of the
//    reference's np.dot(x.values, c[x.indices]) (sparse.py:80-87), i.e. the
//    OpenBLAS 0.3.30 SkylakeX ddot kernel numpy ships with (32-wide blocks on
//    32 FMA accumulators folded 8->4 wide, one optional 16-wide block on the
//    4x4 accumulators, a fixed horizontal sum, then an FMA tail); one warp per
//    row, lane L = accumulator L.  Pinned bit-for-bit against np.dot in
//    tests/test_seeding.py.
//  * The splitmix64 stream (rng.py:39-73) runs on the device.
//  * weighted_index (rng.py:75-92) inverts a SEQUENTIAL float64 cumsum.  The
//    device finds the index from a parallel prefix sum and accepts it only
//    if r stays more than delta = 8 (n + 2) 2^-53 * total away from both
//    neighbouring prefix values; every computed prefix is within
//    gamma_n * total of the exact one (sequential or tree order alike), so
//    the accepted index is the one the sequential cumsum gives.  Otherwise
//    one warp replays the sequential cumsum exactly (rare: probability about
//    16 n^2 2^-53 per pick).
//  * AFK-MC2's sum(d) is numpy's pairwise summation (leaves of <= 128 on 8
//    accumulators, split at n/2 rounded down to a multiple of 8); the tree is
//    planned on the host (integers only) and evaluated level by level.
//    np.cumsum(q) is replayed sequentially by one warp.

namespace seed {

constexpr int kBlock = 2048;       // weights per partial sum
constexpr int kSelThreads = 1024;  // the one-CTA select kernel
enum { SEL_FIRST = 0, SEL_KMPP = 1, SEL_AFK = 2 };
enum { SIM_KMPP = 0, SIM_AFK_INIT = 1, SIM_AFK_UPDATE = 2 };

struct Ctl {
    unsigned long long rng;   // splitmix64 state (rng.py:36)
    long long fallbacks;      // sequential cumsum replays (diagnostic)
    long long uniform_picks;  // _uniform_among_unchosen calls
    long long force_seq;      // test hook: always replay the sequential cumsum
    double qtotal;            // cumq[-1]
    double total_d;           // AFK-MC2 sum(d), numpy pairwise order
    double pad1, pad2;
};

struct Args {
    int64_t n, d, nb;
    const int64_t *indptr;
    const int32_t *indices;
    const double *values;
    const int64_t *row_host;
    const int64_t *row_dev;
    double *w;        // [n] kmpp weights | AFK-MC2 d (host row order)
    double *ms;       // [n] kmpp running max similarity | AFK-MC2 dcur
    double *q;        // [n] AFK-MC2 proposal q
    double *cumq;     // [n] np.cumsum(q)
    double *cden;     // [d] the picked row, densified (device term ids)
    double *part;     // [nb] block sums of the weights in use
    double *excl;     // [nb + 1] exclusive prefix of part, excl[nb] = total
    unsigned char *chosen;   // [n]
    Ctl *ctl;
    int64_t *leaf_off;       // pairwise-sum plan (AFK-MC2)
    int64_t *node_lr;        // [2 * nodes] children of each internal node
    double *pw_val;          // [leaves + nodes]
    int64_t *lvl;            // [64] level offsets of the internal nodes
    int64_t *picks;          // [k] host row ids, in pick order
};

inline int64_t num_blocks(int64_t n) { return (n + kBlock - 1) / kBlock; }
inline int64_t max_leaves(int64_t n) { return n / 32 + 4; }

inline int64_t scratch_doubles(int64_t n, int64_t d) {
    const int64_t nb = num_blocks(n), L = max_leaves(n);
    return 4 * n + d + nb + (nb + 1) + (n + 7) / 8 + (int64_t)(sizeof(Ctl) / 8) + (L + 1) + 2 * L + 2 * L + 64 + 8;
}

inline Args carve(const spkm_seed *Sd, int64_t *picks) {
    Args A;
    A.n = Sd->n;
    A.d = Sd->d;
    A.nb = num_blocks(Sd->n);
    A.indptr = Sd->indptr;
    A.indices = Sd->indices;
    A.values = Sd->values;
    A.row_host = Sd->row_host;
    A.row_dev = Sd->row_dev;
    double *p = Sd->scratch;
    const int64_t n = A.n, L = max_leaves(n);
    A.w = p; p += n;
    A.ms = p; p += n;
    A.q = p; p += n;
    A.cumq = p; p += n;
    A.cden = p; p += A.d;
    A.part = p; p += A.nb;
    A.excl = p; p += A.nb + 1;
    A.ctl = reinterpret_cast<Ctl *>(p); p += sizeof(Ctl) / 8;
    A.leaf_off = reinterpret_cast<int64_t *>(p); p += L + 1;
    A.node_lr = reinterpret_cast<int64_t *>(p); p += 2 * L;
    A.pw_val = p; p += 2 * L;
    A.lvl = reinterpret_cast<int64_t *>(p); p += 64;
    A.chosen = reinterpret_cast<unsigned char *>(p);
    A.picks = picks;
    return A;
}

// ----------------------------------------------------------- splitmix64
__device__ __forceinline__ unsigned long long sm_next(unsigned long long &s) {
    s += 0x9E3779B97F4A7C15ull;
    unsigned long long z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double sm_random(unsigned long long &s) {
    return (double)(sm_next(s) >> 11) * 0x1.0p-53;
}

// ---------------------------------------------- densify the picked row
// cden holds exactly one row: the previous pick's terms are cleared first.
__global__ void k_scatter(Args A, int64_t t) {
    if (t > 0) {
        const int64_t r = A.row_dev[A.picks[t - 1]];
        for (int64_t e = A.indptr[r] + threadIdx.x; e < A.indptr[r + 1]; e += blockDim.x) A.cden[A.indices[e]] = 0.0;
        __syncthreads();
    }
    const int64_t r = A.row_dev[A.picks[t]];
    for (int64_t e = A.indptr[r] + threadIdx.x; e < A.indptr[r + 1]; e += blockDim.x)
        A.cden[A.indices[e]] = A.values[e];
}

// ----------------------------------------------- similarity to the pick
// np.dot(x.values, c[x.indices]) in the OpenBLAS SkylakeX ddot order.
__device__ __forceinline__ double warp_ddot(const Args &A, int64_t s, int64_t e, int lane) {
    const int64_t m = e - s;
    const int64_t n32 = m & ~int64_t(31), n1 = m & ~int64_t(15);
    double z = 0.0;   // accumulator z[b][l] of the 4 x 8-wide AVX-512 loop, lane = 8b + l
    for (int64_t base = 0; base < n32; base += 32) {
        const int64_t i = s + base + lane;
        z = fma(A.values[i], A.cden[A.indices[i]], z);
    }
    // fold 8 -> 4 wide: a[b][l] = z[b][l] + z[b][l+4] (lanes 8b + l, l < 4)
    double a = __dadd_rn(z, __shfl_down_sync(FULL, z, 4));
    if (n1 > n32 && (lane & 7) < 4) {   // one 16-wide step on the 4 x 4-wide accumulators
        const int64_t i = s + n32 + (lane >> 3) * 4 + (lane & 7);
        a = fma(A.values[i], A.cden[A.indices[i]], a);
    }
    const int l4 = lane & 3;
    const double a0 = __shfl_sync(FULL, a, l4), a1 = __shfl_sync(FULL, a, 8 + l4);
    const double a2 = __shfl_sync(FULL, a, 16 + l4), a3 = __shfl_sync(FULL, a, 24 + l4);
    const double tl = __dadd_rn(__dadd_rn(__dadd_rn(a0, a1), a2), a3);   // accum_0+accum_1+accum_2+accum_3
    const double t0 = __shfl_sync(FULL, tl, 0), t1 = __shfl_sync(FULL, tl, 1);
    const double t2 = __shfl_sync(FULL, tl, 2), t3 = __shfl_sync(FULL, tl, 3);
    double dot = __dadd_rn(__dadd_rn(t0, t2), __dadd_rn(t1, t3));        // 256 -> 128 bit, then hadd
    for (int64_t i = s + n1; i < e; ++i) dot = fma(A.cden[A.indices[i]], A.values[i], dot);   // tail
    return dot;
}

// kmpp: ms = max(ms, sim) (seeding.py:88), w = max(alpha - ms, 0), w[chosen] = 0 (78-79)
// AFK init: d = max(alpha - sim, 0), d[first] = 0 (seeding.py:113-114); dcur = d
// AFK update: dcur = min(dcur, max(alpha - sim, 0)), dcur[cur] = 0 (seeding.py:144-145)
__global__ void __launch_bounds__(256) k_sims(Args A, int mode, int64_t t, double alpha) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t pick = A.picks[t];
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < A.n; r += warps) {
        const double sim = warp_ddot(A, A.indptr[r], A.indptr[r + 1], lane);
        if (lane != 0) continue;
        const int64_t h = A.row_host[r];
        const double dis = fmax(__dsub_rn(alpha, sim), 0.0);
        if (mode == SIM_KMPP) {
            const double m0 = A.ms[h];
            const double m = (t == 0 || sim > m0) ? sim : m0;
            A.ms[h] = m;
            A.w[h] = A.chosen[h] ? 0.0 : fmax(__dsub_rn(alpha, m), 0.0);
        } else if (mode == SIM_AFK_INIT) {
            const double v = (h == pick) ? 0.0 : dis;
            A.w[h] = v;
            A.ms[h] = v;
        } else {
            const double c0 = A.ms[h];
            A.ms[h] = (h == pick) ? 0.0 : (c0 <= dis ? c0 : dis);
        }
    }
}

// block sums of v (any fixed order: only used to locate, see the header)
__global__ void __launch_bounds__(256) k_partials(const double *__restrict__ v, int64_t n, double *part) {
    __shared__ double sh[8];
    const int64_t b0 = (int64_t)blockIdx.x * kBlock;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kBlock / 256; ++j) {
        const int64_t i = b0 + j * 256 + threadIdx.x;
        if (i < n) s += v[i];
    }
    for (int o = 16; o; o >>= 1) s += __shfl_down_sync(FULL, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
}

// ---------------------------------------------------------- CTA helpers
// exclusive scan of one value per thread (1024 threads); returns the
// exclusive prefix, *total = sum over the CTA
__device__ double cta_excl_scan(double v, double *sh, double *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x = y + x;
    }
    double ex = __shfl_up_sync(FULL, x, 1);
    if (lane == 0) ex = 0.0;
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        double s = sh[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(FULL, s, o);
            if (lane >= o) s = y + s;
        }
        sh[32 + lane] = s;   // inclusive warp-total prefix
    }
    __syncthreads();
    const double base = wid ? sh[32 + wid - 1] : 0.0;
    *total = sh[32 + 31];
    __syncthreads();
    return base + ex;
}

// excl[b] = sum part[0..b), excl[nb] = total
__device__ void cta_prefix_partials(const Args &A, double *sh) {
    double carry = 0.0;
    for (int64_t c0 = 0; c0 < A.nb; c0 += kSelThreads) {
        const int64_t b = c0 + threadIdx.x;
        const double v = b < A.nb ? A.part[b] : 0.0;
        double tot;
        const double ex = cta_excl_scan(v, sh, &tot);
        if (b < A.nb) A.excl[b] = carry + ex;
        carry = carry + tot;
    }
    if (threadIdx.x == 0) A.excl[A.nb] = carry;
    __syncthreads();
}

// One warp replays np.cumsum(w) exactly (sequential float64): every lane
// runs the same chain on shuffled values.  mode 0: return the total;
// mode 1: first index with cumsum > r (n if none); mode 2: also store the
// cumsum into out[].
__device__ double warp_seq_cumsum(const double *w, int64_t n, int mode, double r, int64_t *idx, double *out) {
    const int lane = threadIdx.x & 31;
    double c = 0.0;
    for (int64_t base = 0; base < n; base += 32) {
        const int64_t i = base + lane;
        const double v = i < n ? w[i] : 0.0;
        double mine = 0.0;
        const int cnt = (int)((n - base) < 32 ? (n - base) : 32);
        for (int j = 0; j < cnt; ++j) {
            c = __dadd_rn(c, __shfl_sync(FULL, v, j));
            if (j == lane) mine = c;
            if (mode == 1 && c > r) {
                *idx = base + j;
                return c;
            }
        }
        if (mode == 2 && i < n) out[i] = mine;
    }
    if (mode == 1) *idx = n;
    return c;
}

// rng.weighted_index(w) (rng.py:75-92) with the CTA; excl must hold the
// prefix of w's block sums.  All threads return the index.
__device__ int64_t cta_weighted_index(const Args &A, const double *w, double *sh, long long *shl) {
    const int64_t n = A.n;
    const double total = A.excl[A.nb];
    __shared__ double s_u;
    if (threadIdx.x == 0) s_u = sm_random(A.ctl->rng);
    if (threadIdx.x == 0) {
        shl[0] = -1;
        shl[1] = LLONG_MAX;
        shl[2] = 0;
    }
    __syncthreads();
    const double U = s_u;
    const double r = U * total;
    for (int64_t b = threadIdx.x; b < A.nb; b += kSelThreads)
        if (A.excl[b] <= r && r < A.excl[b + 1]) shl[0] = b;
    __syncthreads();
    const long long blk = shl[0];
    const double delta = 8.0 * (double)(n + 2) * 0x1.0p-53 * total;
    if (blk >= 0) {
        const int64_t i0 = blk * kBlock + 2 * threadIdx.x;
        const double v0 = i0 < n ? w[i0] : 0.0, v1 = i0 + 1 < n ? w[i0 + 1] : 0.0;
        double tot;
        const double ex = cta_excl_scan(v0 + v1, sh, &tot);
        const double base = A.excl[blk];
        const double p_prev = base + ex;
        const double c0 = base + (ex + v0);
        const double c1 = base + ((ex + v0) + v1);
        long long cand = LLONG_MAX;
        if (i0 < n && c0 > r) cand = i0;
        else if (i0 + 1 < n && c1 > r) cand = i0 + 1;
        if (cand != LLONG_MAX) atomicMin(&shl[1], cand);
        __syncthreads();
        if (cand != LLONG_MAX && cand == shl[1]) {
            const double hi = (cand == i0) ? c0 : c1;
            const double lo = (cand == i0) ? p_prev : c0;
            const bool first_overall = (cand == 0);
            const bool ok = (hi - r > delta) && (first_overall || r - lo >= delta);
            shl[2] = ok ? 1 : 0;
        }
        __syncthreads();
    }
    int64_t idx;
    if (blk < 0 || shl[1] == LLONG_MAX || shl[2] == 0 || A.ctl->force_seq) {
        // replay the reference exactly: total = cumsum[-1], r = U * total,
        // searchsorted(cum, r, 'right')
        if (threadIdx.x < 32) {
            int64_t dummy;
            const double tseq = warp_seq_cumsum(w, n, 0, 0.0, &dummy, nullptr);
            int64_t j;
            warp_seq_cumsum(w, n, 1, U * tseq, &j, nullptr);
            if (threadIdx.x == 0) {
                shl[1] = j;
                A.ctl->fallbacks += 1;
            }
        }
        __syncthreads();
    }
    idx = shl[1];
    if (idx > n - 1) idx = n - 1;
    // skip zero-weight cells at floating-point edges (rng.py:89-91)
    if (threadIdx.x == 0) {
        while (w[idx] == 0.0 && idx + 1 < n) ++idx;
        shl[3] = idx;
    }
    __syncthreads();
    idx = shl[3];
    __syncthreads();
    return idx;
}

// _uniform_among_unchosen (seeding.py:50-52): the m-th unchosen row, m = randint(n - chosen)
__device__ int64_t cta_uniform_unchosen(const Args &A, int64_t nchosen, long long *shl) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ int s_wc[32];
    if (threadIdx.x == 0) {
        const unsigned long long bound = (unsigned long long)(A.n - nchosen);
        shl[0] = (long long)(sm_next(A.ctl->rng) % bound);
        shl[1] = -1;
        A.ctl->uniform_picks += 1;
    }
    __syncthreads();
    long long m = shl[0];
    for (int64_t c0 = 0; c0 < A.n; c0 += kSelThreads) {
        const int64_t i = c0 + threadIdx.x;
        const bool f = i < A.n && !A.chosen[i];
        const unsigned bal = __ballot_sync(FULL, f);
        if (lane == 0) s_wc[wid] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
        for (int w2 = 0; w2 < 32; ++w2) {
            if (w2 < wid) before += s_wc[w2];
            tot += s_wc[w2];
        }
        if (m < tot) {
            const int rank = before + __popc(bal & ((1u << lane) - 1u));
            if (f && rank == m) shl[1] = i;
            __syncthreads();
            break;
        }
        m -= tot;
        __syncthreads();
    }
    __syncthreads();
    return shl[1];
}

// bisect.bisect_right(cumq, r) by one warp (32-ary search)
__device__ int64_t warp_bisect_right(const double *cum, int64_t n, double r) {
    const int lane = threadIdx.x & 31;
    int64_t lo = 0, hi = n;   // cum[< lo] <= r, cum[>= hi] > r
    while (lo < hi) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t p = lo + lane * step;
        const bool pred = p < hi && cum[p] <= r;
        const int c = __popc(__ballot_sync(FULL, pred));
        if (c == 0) {
            hi = lo;
        } else {
            const int64_t pl = lo + (int64_t)(c - 1) * step;
            const int64_t pc = lo + (int64_t)c * step;
            lo = pl + 1;
            if (c < 32 && pc < hi) hi = pc;
        }
    }
    return lo;
}

// One CTA: the next pick (seeding.py:74-89 kmpp, 107-146 AFK-MC2).
__global__ void __launch_bounds__(kSelThreads) k_select(Args A, int mode, int64_t t, int64_t chain_length) {
    __shared__ double sh[64];
    __shared__ long long shl[4];
    __shared__ long long s_pick;
    const int64_t n = A.n;
    if (mode == SEL_FIRST) {
        if (threadIdx.x == 0) {
            const int64_t p = (int64_t)(sm_next(A.ctl->rng) % (unsigned long long)n);
            A.picks[0] = p;
            A.chosen[p] = 1;
        }
        return;
    }
    cta_prefix_partials(A, sh);
    const double total = A.excl[A.nb];
    int64_t pick;
    if (!(total > 0.0)) {
        pick = cta_uniform_unchosen(A, t, shl);
    } else if (mode == SEL_KMPP) {
        pick = cta_weighted_index(A, A.w, sh, shl);
    } else {
        // Metropolis-Hastings chain over q (seeding.py:128-141), one warp
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            unsigned long long st = A.ctl->rng;
            const double qtotal = A.ctl->qtotal;
            double u = 0.0;
            if (lane == 0) u = sm_random(st);
            int64_t cur = warp_bisect_right(A.cumq, n, __shfl_sync(FULL, u, 0) * qtotal);
            if (cur > n - 1) cur = n - 1;
            for (int64_t step = 1; step < chain_length; ++step) {
                if (lane == 0) u = sm_random(st);
                int64_t cand = warp_bisect_right(A.cumq, n, __shfl_sync(FULL, u, 0) * qtotal);
                if (cand > n - 1) cand = n - 1;
                const double num = A.ms[cand] * A.q[cur];
                const double den = A.ms[cur] * A.q[cand];
                if (den <= 0.0) {
                    cur = cand;
                } else {
                    if (lane == 0) u = sm_random(st);
                    if (__shfl_sync(FULL, u, 0) * den < num) cur = cand;
                }
            }
            if (lane == 0) {
                A.ctl->rng = st;
                s_pick = cur;
            }
        }
        __syncthreads();
        pick = s_pick;
        if (!(A.ms[pick] > 0.0)) pick = cta_weighted_index(A, A.ms, sh, shl);   // seeding.py:139-140
    }
    if (threadIdx.x == 0) {
        A.picks[t] = pick;
        A.chosen[pick] = 1;
    }
}

// ----------------------------------------------- AFK-MC2 proposal setup
// pairwise-sum leaves (numpy pairwise_sum, n in [8, 128]: 8 accumulators)
__device__ double np_leaf_sum(const double *a, int64_t m) {
    if (m < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < m; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < m - (m % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < m; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

__global__ void k_pw_leaves(Args A, int64_t nleaves) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nleaves) return;
    const int64_t o = A.leaf_off[j], m = A.leaf_off[j + 1] - o;
    A.pw_val[j] = np_leaf_sum(A.w + o, m);
}

// internal nodes are numbered nleaves.. in order of height; level h spans
// [lvl[h], lvl[h+1])
__global__ void __launch_bounds__(1024) k_pw_tree(Args A, const int64_t *lvl, int nlevels, int64_t nleaves) {
    for (int h = 0; h < nlevels; ++h) {
        for (int64_t q = lvl[h] + threadIdx.x; q < lvl[h + 1]; q += blockDim.x) {
            const int64_t l = A.node_lr[2 * q], r = A.node_lr[2 * q + 1];
            A.pw_val[nleaves + q] = __dadd_rn(A.pw_val[l], A.pw_val[r]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int64_t root = nlevels ? nleaves + lvl[nlevels] - 1 : 0;
        A.ctl->total_d = A.pw_val[root];
    }
}

// q = d / (2 sum d) + 0.5 / n, or 1/n if sum d == 0 (seeding.py:115-118)
__global__ void k_afk_q(Args A) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const double td = A.ctl->total_d;
    A.q[i] = td > 0.0 ? __dadd_rn(__ddiv_rn(A.w[i], __dmul_rn(2.0, td)), __ddiv_rn(0.5, (double)A.n))
                      : __ddiv_rn(1.0, (double)A.n);
}

// cumq = np.cumsum(q) (sequential), qtotal = cumq[-1]
__global__ void k_afk_cumq(Args A) {
    int64_t dummy;
    const double c = warp_seq_cumsum(A.q, A.n, 2, 0.0, &dummy, A.cumq);
    if (threadIdx.x == 0) A.ctl->qtotal = c;
}

// numpy pairwise_sum tree over n elements: leaves (offsets) and internal
// nodes grouped by height.  Integers only; no data.
struct PwPlan {
    std::vector<int64_t> leaf_off;          // nleaves + 1
    std::vector<int64_t> node_lr;           // 2 per internal node, by height
    std::vector<int64_t> lvl;               // level offsets
};

inline void pw_plan(int64_t n, PwPlan &P) {
    struct Node { int64_t l, r; int h; };
    std::vector<Node> nodes;
    std::vector<int64_t> offs;
    // returns (id, height); leaves get ids 0.., internal nodes are encoded
    // as -(index + 1) until renumbered (recursion depth ~ log2(n / 64))
    struct Ret { int64_t id; int h; };
    std::function<Ret(int64_t, int64_t)> rec = [&](int64_t off, int64_t m) -> Ret {
        if (m <= 128) {
            offs.push_back(off);
            return Ret{(int64_t)offs.size() - 1, 0};
        }
        int64_t m2 = m / 2;
        m2 -= m2 % 8;
        const Ret a = rec(off, m2);
        const Ret b = rec(off + m2, m - m2);
        const int h = (a.h > b.h ? a.h : b.h) + 1;
        nodes.push_back(Node{a.id, b.id, h});
        return Ret{-(int64_t)nodes.size(), h};
    };
    rec(0, n);
    const int64_t L = (int64_t)offs.size();
    offs.push_back(n);
    int H = 0;
    for (const Node &x : nodes) H = x.h > H ? x.h : H;
    // renumber internal nodes by height (stable), ids >= L
    std::vector<int64_t> newid(nodes.size());
    P.lvl.assign(H + 1, 0);
    std::vector<int64_t> cnt(H + 2, 0);
    for (const Node &x : nodes) cnt[x.h]++;
    int64_t acc = 0;
    for (int h = 1; h <= H; ++h) {
        P.lvl[h - 1] = acc;
        acc += cnt[h];
    }
    P.lvl[H] = acc;
    std::vector<int64_t> fill(P.lvl.begin(), P.lvl.end());
    for (size_t q = 0; q < nodes.size(); ++q) newid[q] = fill[nodes[q].h - 1]++;
    P.node_lr.assign(2 * nodes.size(), 0);
    auto map = [&](int64_t id) { return id >= 0 ? id : L + newid[(size_t)(-id - 1)]; };
    for (size_t q = 0; q < nodes.size(); ++q) {
        P.node_lr[2 * newid[q]] = map(nodes[q].l);
        P.node_lr[2 * newid[q] + 1] = map(nodes[q].r);
    }
    P.leaf_off = std::move(offs);
}

}  // namespace seed
