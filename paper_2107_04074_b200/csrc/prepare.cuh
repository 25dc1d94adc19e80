// Device layout of an uploaded corpus, built on the GPU (the reference builds
// its CSR on the host: sparse.py:136-156 Dataset.matrix / csr_arrays).
//
//   rows longest first (stable)       -> perm, pos (inverse), indptr
//   term ids by document frequency    -> order (new id -> raw id), new_id (raw id -> new id)
//
// Both orders are stable descending sorts: CUB's LSD radix sort (stable by
// construction) over 32-bit keys with int64 payloads; the row offsets are one
// inclusive scan.  Scratch comes from the caller (spkm_prepare_scratch_bytes).
// The row order is what k_row_pass et al. rely on for load balance (long rows
// first); the term order puts the Zipf head in the first rows
// of the term-major center table (the L2 evict_last block).
// Included by spkm.cu inside its anonymous namespace (shares fail/fail_msg);
// the C ABI wrappers spkm_prepare_* are in spkm.cu.


__global__ void k_row_keys(int64_t n, const int64_t *__restrict__ ip, uint32_t *key, int64_t *val) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = ip[i + 1] - ip[i];
        key[i] = len > 0xffffffffll ? 0xffffffffu : (uint32_t)len;
        val[i] = i;
    }
}

__global__ void k_perm_lens(int64_t n, const int64_t *__restrict__ ip, const int64_t *__restrict__ perm,
                            int64_t *lens, int64_t *pos, int64_t *indptr0) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = perm[r];
        lens[r] = ip[src + 1] - ip[src];
        if (pos) pos[src] = r;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *indptr0 = 0;
}

__global__ void k_term_df(int64_t nnz, const int32_t *__restrict__ idx, uint32_t *df) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(df + idx[t], 1u);
}

__global__ void k_iota(int64_t m, int64_t *v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = i;
}

__global__ void k_invert(int64_t m, const int64_t *__restrict__ order, int64_t *inv) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        inv[order[i]] = i;
}

inline unsigned grid1(int64_t m) {
    const int64_t b = (m + 255) / 256;
    return (unsigned)(b < 1 ? 1 : b > 148 * 16 ? 148 * 16 : b);
}

inline size_t al(size_t b) { return (b + 255) & ~size_t(255); }

struct PrepPlan {
    size_t rows_key, rows_val, rows_tmp, rows_lens, terms_key, terms_val, terms_tmp, total;
};

PrepPlan prep_plan(int64_t n, int64_t d) {
    PrepPlan p{};
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, t1, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                              (const int64_t *)nullptr, (int64_t *)nullptr, (int)(n > 0 ? n : 1));
    cub::DeviceScan::InclusiveSum(nullptr, t2, (const int64_t *)nullptr, (int64_t *)nullptr, (int)(n > 0 ? n : 1));
    cub::DeviceRadixSort::SortPairsDescending(nullptr, t3, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                              (const int64_t *)nullptr, (int64_t *)nullptr, (int)(d > 0 ? d : 1));
    const size_t nn = (size_t)(n > 0 ? n : 1), dd = (size_t)(d > 0 ? d : 1);
    p.rows_key = al(2 * nn * sizeof(uint32_t));
    p.rows_val = al(nn * sizeof(int64_t));
    p.rows_tmp = al(t1 > t2 ? t1 : t2);
    p.rows_lens = al(nn * sizeof(int64_t));
    p.terms_key = al(2 * dd * sizeof(uint32_t));
    p.terms_val = al(dd * sizeof(int64_t));
    p.terms_tmp = al(t3);
    p.total = p.rows_key + p.rows_val + p.rows_tmp + p.rows_lens + p.terms_key + p.terms_val + p.terms_tmp;
    return p;
}

// dense corpora (every row holds the D terms 0..D-1): the device term ids,
// the row offsets r * D and the (identity) row order
__global__ void k_dense_ids(int64_t n, int64_t D, int32_t *idx, int64_t *indptr, int64_t *perm) {
    const int64_t tot = n * D;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += stride) idx[i] = (int32_t)(i % D);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= n; r += stride) {
        if (indptr) indptr[r] = r * D;
        if (perm && r < n) perm[r] = r;
    }
}
