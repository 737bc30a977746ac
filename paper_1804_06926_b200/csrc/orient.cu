// orient.cu -- steps a1-a3 of the hot path:
//   a1 clean: arcs -> 64-bit undirected keys (min << b | max), radix sort,
//      unique (Table 1 caption P:604-606: "treated as undirected ... de-duplicate");
//   a2 degree d(v) of the cleaned graph;
//   a3 orientation filter + compaction ("Form_Filtered_Edge_List", Alg. 2
//      P:336-343; Advance + Filter + segmented reduction, §4.2.1):
//      keep (u,v) iff rank(u) < rank(v), rank = (d, id), ties by smaller id
//      (P:521-522); direction low -> high rank (DESIGN reading R2).
// Dirty input: the unique pair list is sorted by (a, b); a STABLE radix sort of
// the oriented pairs by source then yields every N+(u) ascending (the a4 sort
// is subsumed: N+(x) = [a < x in increasing order] ++ [b > x in increasing order]).
// Clean input: the compaction is stable, so rows stay sorted iff the input rows
// were; otherwise a4 (segmented_sort) runs.
#include "block_scan.cuh"
#include "tc_internal.cuh"

namespace tc {

__device__ __forceinline__ bool rank_less(const uint32_t *__restrict__ deg, uint32_t u,
                                          uint32_t v) {
    uint32_t du = deg[u], dv = deg[v];
    return du < dv || (du == dv && u < v);
}

static int id_bits(uint64_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) b++;
    return b;
}

// ------------------------------------------------------------------ a1: keys
__global__ void __launch_bounds__(kTileThreads)
    k_clean_keys(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col, uint64_t n,
                 uint64_t M, int b, uint64_t *__restrict__ keys) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
    tile_rows(rowptr, n, t0, len, s_row, s_scan);
    for (uint32_t i = threadIdx.x; i < len; i += kTileThreads) {
        uint64_t u = s_row[i], v = col[t0 + i];
        uint64_t key = ~0ull;  // self-loop: invalid, sorts last on the low 2b bits
        if (u != v) {
            uint64_t a = u < v ? u : v, c = u < v ? v : u;
            key = (a << b) | c;
        }
        keys[t0 + i] = key;
    }
}

// ------------------------------------------------------------------ a1: unique
__device__ __forceinline__ bool unique_flag(const uint64_t *__restrict__ keys, uint64_t i) {
    uint64_t k = keys[i];
    return k != ~0ull && (i == 0 || keys[i - 1] != k);
}

__global__ void __launch_bounds__(kTileThreads)
    k_unique_count(const uint64_t *__restrict__ keys, uint64_t M, uint32_t *__restrict__ counts) {
    __shared__ uint64_t s_red[kTileThreads / 32];
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    uint64_t c = 0;
    for (int k = 0; k < kItemsPerThread; k++) {
        uint64_t i = t0 + (uint64_t)k * kTileThreads + threadIdx.x;
        if (i < M) c += unique_flag(keys, i);
    }
    c = block_sum_u64(c, s_red);
    if (threadIdx.x == 0) counts[blockIdx.x] = (uint32_t)c;
}

__global__ void __launch_bounds__(kTileThreads)
    k_unique_scatter(const uint64_t *__restrict__ keys, uint64_t M,
                     const uint64_t *__restrict__ offs, uint64_t *__restrict__ out) {
    __shared__ uint32_t s_scan[kTileThreads / 32];
    uint64_t base = (uint64_t)blockIdx.x * kTileItems + (uint64_t)threadIdx.x * kItemsPerThread;
    uint32_t f[kItemsPerThread];
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        uint64_t i = base + k;
        f[k] = i < M ? unique_flag(keys, i) : 0u;
        c += f[k];
    }
    uint32_t pos = block_exclusive_scan<SumOp>(c, s_scan);
    uint64_t o = offs[blockIdx.x] + pos;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++)
        if (f[k]) out[o++] = keys[base + k];
}

// ------------------------------------------------------------------ a2/a3 from pairs
__global__ void k_deg_pairs(const uint64_t *__restrict__ E, const uint64_t *__restrict__ m_dev,
                            int b, uint32_t *__restrict__ deg) {
    uint64_t m = *m_dev, mask = (1ull << b) - 1;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t k = E[i];
        atomicAdd(&deg[k >> b], 1u);
        atomicAdd(&deg[k & mask], 1u);
    }
}

__global__ void k_orient_pairs(const uint64_t *__restrict__ E, const uint64_t *__restrict__ m_dev,
                               int b, const uint32_t *__restrict__ deg, uint32_t *__restrict__ okey,
                               uint32_t *__restrict__ oval, uint32_t *__restrict__ dplus) {
    uint64_t m = *m_dev, mask = (1ull << b) - 1;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t k = E[i];
        uint32_t a = (uint32_t)(k >> b), c = (uint32_t)(k & mask);
        bool fwd = rank_less(deg, a, c);
        uint32_t s = fwd ? a : c, d = fwd ? c : a;
        okey[i] = s;
        oval[i] = d;
        atomicAdd(&dplus[s], 1u);
    }
}

void orient_dirty(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
                  Oriented &out, Timer *tm) {
    int b = id_bits(n);
    uint32_t tiles = (uint32_t)((M + kTileItems - 1) / kTileItems);
    if (tm) tm->begin(kClean);
    uint64_t *keys = ctx.alloc<uint64_t>(M);
    uint64_t *keys_alt = ctx.alloc<uint64_t>(M);
    k_clean_keys<<<tiles, kTileThreads, 0, ctx.stream>>>(rowptr, col, n, M, b, keys);
    TC_LAUNCHED(ctx);
    bool alt = radix_sort(ctx, keys, keys_alt, M, nullptr, 2 * b);
    uint64_t *sorted = alt ? keys_alt : keys, *E = alt ? keys : keys_alt;
    uint32_t *counts = ctx.alloc<uint32_t>(tiles);
    uint64_t *offs = ctx.alloc<uint64_t>(tiles + 1);
    k_unique_count<<<tiles, kTileThreads, 0, ctx.stream>>>(sorted, M, counts);
    TC_LAUNCHED(ctx);
    scan_exclusive(ctx, counts, offs, tiles);
    k_unique_scatter<<<tiles, kTileThreads, 0, ctx.stream>>>(sorted, M, offs, E);
    TC_LAUNCHED(ctx);
    uint64_t *m_dev = offs + tiles;
    if (tm) tm->end(kClean);

    if (tm) tm->begin(kOrient);
    uint32_t *deg = ctx.alloc<uint32_t>(n);
    uint32_t *dplus = ctx.alloc<uint32_t>(n + 1);
    TC_CUDA(cudaMemsetAsync(deg, 0, n * sizeof(uint32_t), ctx.stream));
    TC_CUDA(cudaMemsetAsync(dplus, 0, (n + 1) * sizeof(uint32_t), ctx.stream));
    int grid = ctx.persistent_grid(8);
    k_deg_pairs<<<grid, 256, 0, ctx.stream>>>(E, m_dev, b, deg);
    TC_LAUNCHED(ctx);
    uint32_t *okey = ctx.alloc<uint32_t>(M), *oval = ctx.alloc<uint32_t>(M);
    uint32_t *okey2 = ctx.alloc<uint32_t>(M), *oval2 = ctx.alloc<uint32_t>(M);
    k_orient_pairs<<<grid, 256, 0, ctx.stream>>>(E, m_dev, b, deg, okey, oval, dplus);
    TC_LAUNCHED(ctx);
    bool alt2 = radix_sort_pairs(ctx, okey, okey2, oval, oval2, M, m_dev, b);
    uint64_t *off = ctx.alloc<uint64_t>(n + 1);
    scan_exclusive(ctx, dplus, off, n);
    if (tm) tm->end(kOrient);
    out.n = n;
    out.off = off;
    out.col = alt2 ? oval2 : oval;
    out.dplus = dplus;
    out.m_dev = m_dev;
    out.m_cap = M;
}

// ------------------------------------------------------------------ clean input
__global__ void k_deg_rowptr(const uint64_t *__restrict__ rowptr, uint64_t n,
                             uint32_t *__restrict__ deg) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x)
        deg[u] = (uint32_t)(rowptr[u + 1] - rowptr[u]);
}

__global__ void __launch_bounds__(kTileThreads)
    k_orient_count(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col,
                   uint64_t n, uint64_t M, const uint32_t *__restrict__ deg,
                   uint32_t *__restrict__ counts) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    __shared__ uint64_t s_red[kTileThreads / 32];
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
    tile_rows(rowptr, n, t0, len, s_row, s_scan);
    uint64_t c = 0;
    for (uint32_t i = threadIdx.x; i < len; i += kTileThreads)
        c += rank_less(deg, s_row[i], col[t0 + i]);
    c = block_sum_u64(c, s_red);
    if (threadIdx.x == 0) counts[blockIdx.x] = (uint32_t)c;
}

__global__ void __launch_bounds__(kTileThreads)
    k_orient_scatter(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col,
                     uint64_t n, uint64_t M, const uint32_t *__restrict__ deg,
                     const uint64_t *__restrict__ offs, uint32_t *__restrict__ col_plus,
                     uint64_t *__restrict__ off_plus) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_excl[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    __shared__ uint64_t s_bounds[2];
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
    tile_rows(rowptr, n, t0, len, s_row, s_scan);
    uint32_t i0 = threadIdx.x * kItemsPerThread;
    uint32_t f[kItemsPerThread], v[kItemsPerThread], c = 0;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        uint32_t i = i0 + k;
        v[k] = i < len ? col[t0 + i] : 0u;
        f[k] = i < len ? (uint32_t)rank_less(deg, s_row[i], v[k]) : 0u;
        c += f[k];
    }
    uint32_t pos = block_exclusive_scan<SumOp>(c, s_scan);
    uint64_t base = offs[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        s_excl[i0 + k] = pos;
        if (f[k]) col_plus[base + pos] = v[k];
        pos += f[k];
    }
    if (threadIdx.x == 0) {
        s_bounds[0] = lower_bound_u64(rowptr, n + 1, t0);
        s_bounds[1] = lower_bound_u64(rowptr, n + 1, t0 + len);
    }
    __syncthreads();
    for (uint64_t u = s_bounds[0] + threadIdx.x; u < s_bounds[1]; u += kTileThreads)
        off_plus[u] = base + s_excl[rowptr[u] - t0];
}

// Rows starting at M (trailing empty rows, and u = n) get off+ = m.
__global__ void k_orient_tail(const uint64_t *__restrict__ rowptr, uint64_t n, uint64_t M,
                              const uint64_t *__restrict__ m_dev, uint64_t *__restrict__ off_plus) {
    uint64_t m = *m_dev;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= n;
         u += (uint64_t)gridDim.x * blockDim.x)
        if (rowptr[u] >= M) off_plus[u] = m;
}

__global__ void k_dplus(const uint64_t *__restrict__ off, uint64_t n, uint32_t *__restrict__ dplus) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x)
        dplus[u] = (uint32_t)(off[u + 1] - off[u]);
}

void orient_clean(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
                  bool sorted, uint32_t segsort_block_max, Oriented &out, Timer *tm) {
    uint32_t tiles = (uint32_t)((M + kTileItems - 1) / kTileItems);
    int grid = ctx.persistent_grid(8);
    if (tm) tm->begin(kOrient);
    uint32_t *deg = ctx.alloc<uint32_t>(n);
    k_deg_rowptr<<<grid, 256, 0, ctx.stream>>>(rowptr, n, deg);
    TC_LAUNCHED(ctx);
    uint32_t *counts = ctx.alloc<uint32_t>(tiles);
    uint64_t *offs = ctx.alloc<uint64_t>(tiles + 1);
    k_orient_count<<<tiles, kTileThreads, 0, ctx.stream>>>(rowptr, col, n, M, deg, counts);
    TC_LAUNCHED(ctx);
    scan_exclusive(ctx, counts, offs, tiles);
    uint64_t m_cap = M / 2 + 1;
    uint32_t *col_plus = ctx.alloc<uint32_t>(m_cap);
    uint64_t *off_plus = ctx.alloc<uint64_t>(n + 1);
    k_orient_scatter<<<tiles, kTileThreads, 0, ctx.stream>>>(rowptr, col, n, M, deg, offs,
                                                             col_plus, off_plus);
    TC_LAUNCHED(ctx);
    k_orient_tail<<<grid, 256, 0, ctx.stream>>>(rowptr, n, M, offs + tiles, off_plus);
    TC_LAUNCHED(ctx);
    uint32_t *dplus = ctx.alloc<uint32_t>(n + 1);
    k_dplus<<<grid, 256, 0, ctx.stream>>>(off_plus, n, dplus);
    TC_LAUNCHED(ctx);
    if (tm) tm->end(kOrient);
    if (!sorted) {
        if (tm) tm->begin(kSort);
        segmented_sort(ctx, n, off_plus, col_plus, m_cap, segsort_block_max);
        if (tm) tm->end(kSort);
    }
    out.n = n;
    out.off = off_plus;
    out.col = col_plus;
    out.dplus = dplus;
    out.m_dev = offs + tiles;
    out.m_cap = m_cap;
}

}  // namespace tc
