// orient.cu -- steps a1-a4 of the hot path:
//   a1 clean: arcs -> 64-bit undirected keys (min << b | max), radix sort,
//      unique (Table 1 caption P:604-606: "treated as undirected ... de-duplicate");
//   a2 degree d(v) of the cleaned graph;
//   a3 orientation filter + compaction ("Form_Filtered_Edge_List", Alg. 2
//      P:336-343; Advance + Filter + segmented reduction, §4.2.1):
//      keep (u,v) iff rank(u) < rank(v), rank = (d, id), ties by smaller id
//      (P:521-522); direction low -> high rank (DESIGN reading R2).
// Vertices are RELABELLED by rank: a stable radix sort of (d, id) gives
// order[i] = the vertex of rank position i and newid[order[i]] = i, so
// rank(u) < rank(v) <=> newid[u] < newid[v].  The oriented CSR is built in the
// new id space (sources by a stable radix sort of the oriented pairs), so a
// hub's N+ lies in the short id range above it (bitmap staging in a6) and the
// hot lists are contiguous at the end of col+.  Every row comes out ascending (a4):
// the two-key LSD sort (target, then source) that builds the CSR also sorts its rows.
#include <algorithm>

#include "block_scan.cuh"
#include "tc_internal.cuh"

namespace tc {

// Also the TC_PRUNE survival test: a pruned-away vertex has degree 0 (prune.cu), and
// without pruning every arc's endpoints have degree >= 1.
__device__ __forceinline__ bool rank_less(const uint32_t *__restrict__ deg, uint32_t u,
                                          uint32_t v) {
    uint32_t du = deg[u], dv = deg[v];
    return du != 0 && (du < dv || (du == dv && u < v));
}

static int id_bits(uint64_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) b++;
    return b;
}

// ------------------------------------------------------------------ a1: keys
// Round 2: the a1 radix sort orders the keys by (min, h-bit hash of max) only, not by the
// full (min, max): the key (min << b) | max is re-laid out BIJECTIVELY as
//     [ high b - h bits of mix(max) | min (b bits) | low h bits of mix(max) ]
// (mix = an invertible xorshift-multiply-xorshift on b bits) and the sort takes its low
// b + h bits.  Equal edges stay equal and land in one RUN of equal (min, hash) -- the unique
// step compares each key with the earlier keys of its run (runs of one min group of D arcs
// average D / 2^h keys) -- and the output stays grouped by min (the degree atomics of the
// min side aggregate per run, k_orient_pairs keeps its locality).  b + h is a multiple of 8
// with h >= 11: 4 passes instead of 6 at s21 (b = 21), 5 instead of 6 at s24 and on the road
// mesh.  h = 0: plain (min, max) order (tc_options.clean_method = 1, the round-1 sort).
constexpr uint64_t kMixOdd = 0x9E3779B97F4A7C15ull;
__device__ __forceinline__ uint64_t mix_inv_odd() {   // kMixOdd^-1 mod 2^64 (Newton)
    uint64_t x = kMixOdd;
#pragma unroll
    for (int i = 0; i < 5; i++) x *= 2 - kMixOdd * x;
    return x;
}
__device__ __forceinline__ uint64_t key_enc(uint64_t key, int b, int h) {
    if (h == 0) return key;
    const uint64_t mb = (1ull << b) - 1, s = (uint64_t)(b + 1) / 2;
    uint64_t x = key & mb;
    x ^= x >> s;
    x = (x * kMixOdd) & mb;
    x ^= x >> s;
    const uint64_t mn = key >> b;
    return ((x >> h) << (b + h)) | (mn << h) | (x & ((1ull << h) - 1));
}
__device__ __forceinline__ uint64_t key_dec(uint64_t k, int b, int h) {
    if (h == 0) return k;
    const uint64_t mb = (1ull << b) - 1, s = (uint64_t)(b + 1) / 2, mh = (1ull << h) - 1;
    uint64_t x = ((k >> (b + h)) << h) | (k & mh);
    x ^= x >> s;
    x = (x * mix_inv_odd()) & mb;
    x ^= x >> s;
    return (((k >> h) & mb) << b) | x;
}

// Hash bits h of the a1 sort (0 = full order); the sort then takes b + h bits.
static int clean_hash_bits(int b, uint32_t method) {
    if (method != 0) return 0;
    const int S = (b + 11 + 7) / 8 * 8, full = 2 * b;
    const int dbf = radix_digit_bits(full), pf = (full + dbf - 1) / dbf;
    return S < full && S / 8 < pf ? S - b : 0;
}

// (Fusing the radix digit histograms in here was measured slower than the separate
// histogram pass: +0.13 ms against -0.09 ms at s21.)
__global__ void __launch_bounds__(kTileThreads)
    k_clean_keys(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col, uint64_t n,
                 uint64_t M, int b, int hb, uint64_t *__restrict__ keys, const uint2 *__restrict__ tb) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
    tile_rows_tb(rowptr, n, blockIdx.x, t0, len, tb, s_row, s_scan);
    for (uint32_t i = threadIdx.x; i < len; i += kTileThreads) {
        uint64_t u = s_row[i], v = col[t0 + i];
        uint64_t key = ~0ull;  // self-loop: invalid, sorts last on the low 2b bits
        if (u != v) {
            uint64_t a = u < v ? u : v, c = u < v ? v : u;
            key = key_enc((a << b) | c, b, hb);
        }
        keys[t0 + i] = key;
    }
}

// tc_clean_shard: only the arcs whose undirected edge belongs to this rank (min endpoint
// mod world == rank: every copy of an edge lands on one rank, and the ranks get about equal
// shares), compacted -- one atomic per tile, order free (the keys are sorted next).
__global__ void __launch_bounds__(kTileThreads)
    k_clean_keys_shard(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col,
                       uint64_t n, uint64_t M, int b, int hb, uint32_t rank, uint32_t world,
                       uint64_t *__restrict__ keys, uint64_t *__restrict__ count) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    __shared__ uint64_t s_base;
    const uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    const uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
    tile_rows(rowptr, n, t0, len, s_row, s_scan);
    const uint32_t i0 = threadIdx.x * kItemsPerThread;
    uint64_t kk[kItemsPerThread];
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        const uint32_t i = i0 + k;
        kk[k] = ~0ull;
        if (i < len) {
            const uint64_t u = s_row[i], v = col[t0 + i];
            const uint64_t a = u < v ? u : v, d = u < v ? v : u;
            if (u != v && a % world == rank) {
                kk[k] = key_enc((a << b) | d, b, hb);
                c++;
            }
        }
    }
    uint32_t total;
    const uint32_t pos = block_exclusive_scan<SumOp>(c, s_scan, &total);
    if (threadIdx.x == 0) s_base = atomicAdd((unsigned long long *)count, (unsigned long long)total);
    __syncthreads();
    uint64_t o = s_base + pos;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++)
        if (kk[k] != ~0ull) keys[o++] = kk[k];
}

// ------------------------------------------------------------------ a1: unique
// One pass: a key is unique iff no EARLIER key of its run (equal sort bits, i.e. equal
// (min, hash) -- or equal keys in the full order) is equal to it.  The output order is free
// (every consumer of E -- orientation, pruning, tc_clean_shard -- takes any order), so each
// tile takes its output offset with ONE atomic (round 2; round 1 kept the sorted order with a
// decoupled look-back, whose chain made every tile wait for the slowest predecessor).
// Also a2 (fused): the degrees of the cleaned graph.  A thread's unique keys are grouped by
// min (the sort order), so the min side takes one atomic per run of equal mins, the max side
// one per key.
// TC_UNIQUE_SMEM: the tile's keys are read with coalesced (striped) loads into shared memory
// and each thread takes its kItemsPerThread consecutive keys from there (padded rows: no bank
// conflicts), and the unique keys are staged in shared memory and written out coalesced --
// instead of per-thread runs of 64 bytes at a 64-byte lane stride on both sides.
#ifndef TC_UNIQUE_SMEM
#define TC_UNIQUE_SMEM 1
#endif
constexpr int kUqPad = kItemsPerThread + 1;   // shared row of a thread's keys, padded
__global__ void __launch_bounds__(kTileThreads)
    k_unique_scatter(const uint64_t *__restrict__ keys, uint64_t M, const uint64_t *__restrict__ count_dev,
                     uint64_t *__restrict__ m_out, uint64_t *__restrict__ out, int b, int hb,
                     uint32_t *__restrict__ deg) {
    __shared__ uint32_t s_scan[kTileThreads / 32];
    __shared__ uint64_t s_base;
#if TC_UNIQUE_SMEM
    __shared__ uint64_t s_k[kTileThreads * kUqPad];
#endif
    if (count_dev) {   // the keys are a compacted prefix (tc_clean_shard): tiles past it exit
        const uint64_t c = *count_dev;
        M = c < M ? c : M;
    }
    const uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    if (t0 >= M) return;
    const uint64_t base = t0 + (uint64_t)threadIdx.x * kItemsPerThread;
    uint64_t kk[kItemsPerThread];
    bool dup[kItemsPerThread];
#if TC_UNIQUE_SMEM
    const uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {   // striped global -> padded rows
        const uint32_t i = k * kTileThreads + threadIdx.x;
        s_k[(i / kItemsPerThread) * kUqPad + i % kItemsPerThread] = i < len ? keys[t0 + i] : ~0ull;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) kk[k] = s_k[threadIdx.x * kUqPad + k];
    // the key before this thread's first one: the previous row's last (the previous tile's
    // last key for thread 0)
    const uint64_t before = threadIdx.x ? s_k[(threadIdx.x - 1) * kUqPad + kItemsPerThread - 1]
                                        : (t0 ? keys[t0 - 1] : ~0ull);
#else
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        const uint64_t i = base + k;
        kk[k] = i < M ? keys[i] : ~0ull;
    }
    const uint64_t before = base > 0 && base < M ? keys[base - 1] : ~0ull;
#endif
    const uint64_t lowm = hb == 0 ? ~0ull : (1ull << (b + hb)) - 1;
    // earlier keys of the same run among the thread's own items ...
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        dup[k] = false;
#pragma unroll
        for (int q = 0; q < k; q++) dup[k] |= kk[q] == kk[k];
    }
    // ... and before them: ONE backward walk over the run of item 0 (if it began earlier),
    // compared with every item of that run
    if (base > 0 && base < M && ((before ^ kk[0]) & lowm) == 0) {
        for (uint64_t j = base; j-- > 0;) {
            const uint64_t pk = j + 1 == base ? before : keys[j];
            if (((pk ^ kk[0]) & lowm) != 0) break;
#pragma unroll
            for (int k = 0; k < kItemsPerThread; k++) dup[k] |= pk == kk[k];
        }
    }
    uint32_t f[kItemsPerThread], c = 0;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        f[k] = base + k < M && kk[k] != ~0ull && !dup[k];
        c += f[k];
        kk[k] = key_dec(kk[k], b, hb);   // (min << b) | max
    }
    uint32_t total;
    const uint32_t pos = block_exclusive_scan<SumOp>(c, s_scan, &total);   // ends with a barrier
    if (threadIdx.x == 0) s_base = atomicAdd((unsigned long long *)m_out, (unsigned long long)total);
    const uint64_t mask = (1ull << b) - 1;
    uint32_t run_a = 0, run_n = 0;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++)
        if (f[k]) {
            const uint32_t a = (uint32_t)(kk[k] >> b);
            atomicAdd(&deg[kk[k] & mask], 1u);
            if (run_n && a == run_a) {
                run_n++;
            } else {
                if (run_n) atomicAdd(&deg[run_a], run_n);
                run_a = a;
                run_n = 1;
            }
        }
    if (run_n) atomicAdd(&deg[run_a], run_n);
#if TC_UNIQUE_SMEM
    {   // stage the unique keys (the scan's barrier ordered every read of s_k before this)
        uint32_t o = pos;
#pragma unroll
        for (int k = 0; k < kItemsPerThread; k++)
            if (f[k]) s_k[o++] = kk[k];
    }
    __syncthreads();
    const uint64_t ob = s_base;
    for (uint32_t i = threadIdx.x; i < total; i += kTileThreads) out[ob + i] = s_k[i];
#else
    __syncthreads();
    uint64_t o = s_base + pos;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++)
        if (f[k]) out[o++] = kk[k];
#endif
}

// ------------------------------------------------------------------ a3 from pairs
// Also counts the digit histograms of both radix sorts that follow (fused k_rs_hist):
// hist_val for the sort by target (keys oval), hist_key for the sort by source (its keys
// are the okey values in another order: the same histogram).
__global__ void k_orient_pairs(const uint64_t *__restrict__ E, const uint64_t *__restrict__ m_dev,
                               int b, const uint32_t *__restrict__ newid, uint32_t *__restrict__ okey,
                               uint32_t *__restrict__ oval, uint32_t *__restrict__ dplus,
                               uint32_t *__restrict__ hist_key, uint32_t *__restrict__ hist_val,
                               int passes, int db) {
    __shared__ RsHist<4> s_hk, s_hv;
    s_hk.clear();
    s_hv.clear();
    __syncthreads();
    uint64_t m = *m_dev, mask = (1ull << b) - 1;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < m; i0 += stride) {
        uint64_t i = i0 + threadIdx.x;
        bool ok = i < m;
        uint32_t s = 0xffffffffu;
        if (ok) {
            uint64_t k = E[i];
            uint32_t a = newid[k >> b], c = newid[k & mask];
            s = min(a, c);   // low -> high rank
            okey[i] = s;
            oval[i] = max(a, c);
            s_hk.add(s, passes, db);
            s_hv.add(max(a, c), passes, db);
        }
        // runs of one min often keep the same (low-rank) source: aggregate per warp
        uint32_t peers = __match_any_sync(0xffffffffu, s);
        if (ok && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&dplus[s], (uint32_t)__popc(peers));
    }
    __syncthreads();
    s_hk.flush(hist_key, passes);
    s_hv.flush(hist_val, passes);
}

// ------------------------------------------------------------------ rank relabelling
// TC_ID_ORDER (Alg. 3 without its row permutation, the order of Fig. mm): the rank
// key is [d(v) > 0], so every non-isolated vertex ranks by id alone (isolated and
// pruned-away vertices, key 0, keep failing the rank filter).
__global__ void k_id_order_key(const uint32_t *__restrict__ deg, uint64_t n, uint32_t *__restrict__ key) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        key[i] = deg[i] ? 1u : 0u;
}

static const uint32_t *rank_key(Ctx &ctx, uint64_t n, const uint32_t *deg, bool id_order) {
    if (!id_order) return deg;
    uint32_t *key = ctx.alloc<uint32_t>(n);
    k_id_order_key<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(deg, n, key);
    TC_LAUNCHED(ctx);
    return key;
}

// order[i] = vertex with the i-th smallest (d, id); newid = inverse.  `deg` is kept.
static void rank_permutation(Ctx &ctx, uint64_t n, const uint32_t *deg, Oriented &out) {
    int b = id_bits(n);
    int grid = ctx.persistent_grid(8);
    uint32_t *kA = ctx.alloc<uint32_t>(n), *kB = ctx.alloc<uint32_t>(n);
    uint32_t *vA = ctx.alloc<uint32_t>(n), *vB = ctx.alloc<uint32_t>(n);
    // stable sort by degree (< n <= 2^b) of the ids 0..n-1 (generated by the first pass,
    // ascending), so ties stay ordered by id
    uint32_t *rk, *rv;
    out.newid = ctx.alloc<uint32_t>(n);   // written by the last pass (fused inverse)
    radix_sort_pairs_from(ctx, deg, nullptr, kA, kB, vA, vB, n, nullptr, b, &rk, &rv, nullptr,
                          nullptr, nullptr, out.newid);
    out.order = rv;
    (void)grid;
}

void rank_relabel(Ctx &ctx, uint64_t n, const uint32_t *deg, bool id_order, uint32_t *newid_out) {
    Oriented o;
    rank_permutation(ctx, n, rank_key(ctx, n, deg, id_order), o);
    TC_CUDA(cudaMemcpyAsync(newid_out, o.newid, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx.stream));
}

// d-(x) = d(x) - d+(x), in rank ids.
// Also sum_v d-(v) d+(v) (stats: SURVEY 8(d)'s B_stage) into *stage, one atomic per warp.
__global__ void k_dminus(const uint32_t *__restrict__ deg, const uint32_t *__restrict__ newid,
                         const uint32_t *__restrict__ dplus, uint64_t n, uint32_t *__restrict__ dminus,
                         uint64_t *__restrict__ stage) {
    uint64_t acc = 0;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x = newid[v], dp = dplus[x], dm = deg[v] - dp;
        dminus[x] = dm;
        acc += (uint64_t)dm * dp;
    }
    acc = warp_sum_u64(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd((unsigned long long *)stage, (unsigned long long)acc);
}

// Oriented pairs (okey = source, oval = target, new ids; m_dev of them) -> CSR with
// ascending rows (a4) by an LSD radix sort on (source, target): a stable pass set
// over the target gives the transposed CSR T (in-lists N-(x), in edge-list order),
// then a stable pass set over the source of T's index p.  So pidx[e] = the in-list
// slot of CSR edge e, col+[e] = T's target at pidx[e], and no edge ever has to be
// searched for.  dplus / dminus already counted.

// hist_src / hist_tgt (optional): digit histograms of okey / oval (fused by the producer).
// d-(x) = length of x's run in the target-sorted pairs (clean input: counted from the pairs
// actually written, so in_off stays consistent with them even under a false TC_CLEAN claim).
// Two atomics per run: +end at its last element, -start at its first.
__global__ void k_runs_dminus(const uint32_t *__restrict__ tgt, const uint64_t *__restrict__ m_dev,
                              uint32_t *__restrict__ dminus) {
    const uint64_t m = *m_dev;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = tgt[i];
        if (i + 1 == m || tgt[i + 1] != x) atomicAdd(&dminus[x], (uint32_t)(i + 1));
        if (i == 0 || tgt[i - 1] != x) atomicSub(&dminus[x], (uint32_t)i);
    }
}

// sum_x d-(x) d+(x) (stats: SURVEY 8(d)'s B_stage), rank ids, one atomic per warp.
__global__ void k_stage_work(const uint32_t *__restrict__ dplus, const uint32_t *__restrict__ dminus,
                             uint64_t n, uint64_t *__restrict__ stage) {
    uint64_t acc = 0;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (uint64_t)gridDim.x * blockDim.x)
        acc += (uint64_t)dminus[x] * dplus[x];
    acc = warp_sum_u64(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd((unsigned long long *)stage, (unsigned long long)acc);
}

static void pairs_to_csr(Ctx &ctx, uint64_t n, uint64_t cap, uint32_t *okey, uint32_t *oval,
                         uint32_t *dplus, uint32_t *dminus, uint64_t *m_dev, Oriented &out,
                         Timer *tm, const uint32_t *hist_src = nullptr,
                         const uint32_t *hist_tgt = nullptr, bool count_dminus = false) {
    int b = id_bits(n);
    int grid = ctx.persistent_grid(8);
    uint32_t *okey2 = ctx.alloc<uint32_t>(cap), *oval2 = ctx.alloc<uint32_t>(cap);
    // 1) by target (keys = oval, values = okey): T = (targets, sources) = transposed CSR
    bool a1 = radix_sort_pairs(ctx, oval, oval2, okey, okey2, cap, m_dev, b, hist_tgt);
    uint32_t *t_tgt = a1 ? oval2 : oval, *t_src = a1 ? okey2 : okey;
    if (count_dminus) {
        k_runs_dminus<<<grid, 256, 0, ctx.stream>>>(t_tgt, m_dev, dminus);
        TC_LAUNCHED(ctx);
        k_stage_work<<<grid, 256, 0, ctx.stream>>>(dplus, dminus, n, out.stage_work);
        TC_LAUNCHED(ctx);
    }
    uint32_t *f_key = a1 ? oval : oval2, *f_val = a1 ? okey : okey2;   // free pair
    // 2) stable by source of T's index p (values = p, generated by the first pass),
    // reading T without modifying it; the last pass also gathers col+[e] = T.target[p]
    uint32_t *g_key = ctx.alloc<uint32_t>(cap), *g_val = ctx.alloc<uint32_t>(cap);
    // col+ is read by the a6 probes in aligned 8-element slots (two 16-byte loads): pad the
    // allocation to whole slots so the last slot never reads past it (compute-sanitizer)
    uint32_t *col = ctx.alloc<uint32_t>((cap + 7) / 8 * 8);
    uint32_t *rk, *rv;
    radix_sort_pairs_from(ctx, t_src, nullptr, f_key, g_key, f_val, g_val, cap, m_dev, b, &rk, &rv,
                          t_tgt, col, hist_src);
    (void)grid;
    uint64_t *off = ctx.alloc<uint64_t>(n + 1), *in_off = ctx.alloc<uint64_t>(n + 1);
    scan_exclusive(ctx, dplus, off, n);
    scan_exclusive(ctx, dminus, in_off, n);
    out.n = n;
    out.off = off;
    out.col = col;
    out.dplus = dplus;
    out.in_off = in_off;
    out.in_src = t_src;
    out.pidx = rv;
    out.m_dev = m_dev;
    out.m_cap = cap;
    phase_end(tm, kOrient);
}

// a1 on all arcs, or (world > 1, tc_clean_shard) on this rank's share: the unique undirected
// edges as sorted keys (min << b) | max in E (m_dev of them; E = one of keys / keys_alt),
// and the degrees they give both endpoints added into deg (zeroed by the caller).
static void clean_arcs(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
                       int rank, int world, uint64_t *keys, uint64_t *keys_alt, uint64_t *&E,
                       uint64_t *&m_dev, uint32_t *deg, uint32_t method) {
    const int b = id_bits(n);
    const int hb = clean_hash_bits(b, method), sb = hb ? b + hb : 2 * b;
    const uint32_t tiles = (uint32_t)((M + kTileItems - 1) / kTileItems);
    // m (the unique-edge count), the key count (sharded)
    uint64_t *uq = ctx.alloc<uint64_t>(2);
    TC_CUDA(cudaMemsetAsync(uq, 0, 2 * sizeof(uint64_t), ctx.stream));
    m_dev = uq;
    uint64_t mk = M;   // keys to sort
    if (world > 1) {
        k_clean_keys_shard<<<tiles, kTileThreads, 0, ctx.stream>>>(rowptr, col, n, M, b, hb, (uint32_t)rank,
                                                                   (uint32_t)world, keys, uq + 1);
        TC_LAUNCHED(ctx);
        // this rank's share of the keys, read back so the sort and the unique step launch exactly
        // its tiles (a capacity-M launch spent ~0.4 ms per radix pass at s24, world 8, on tail
        // tiles that only exit); tc_clean_shard is synchronous anyway
        TC_CUDA(cudaMemcpyAsync(&mk, uq + 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
        TC_CUDA(cudaStreamSynchronize(ctx.stream));
    } else {
        uint2 *tb = nullptr;
        if (TC_TILE_BOUNDS) {
            tb = ctx.alloc<uint2>(tiles + 1);
            tile_bounds(ctx, rowptr, n, M, nullptr, tb);
        }
        k_clean_keys<<<tiles, kTileThreads, 0, ctx.stream>>>(rowptr, col, n, M, b, hb, keys, tb);
        TC_LAUNCHED(ctx);
    }
    bool alt = radix_sort(ctx, keys, keys_alt, mk, nullptr, sb);
    uint64_t *sorted = alt ? keys_alt : keys;
    E = alt ? keys : keys_alt;
    const uint32_t utiles = (uint32_t)((mk + kTileItems - 1) / kTileItems);
    if (utiles) {
        k_unique_scatter<<<utiles, kTileThreads, 0, ctx.stream>>>(sorted, mk, nullptr, m_dev, E, b, hb, deg);
        TC_LAUNCHED(ctx);
    }
}

void clean_shard(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
                 int rank, int world, uint64_t *edges, uint32_t *deg, uint64_t *m_dev_out,
                 uint32_t method) {
    uint64_t *alt = ctx.alloc<uint64_t>(M), *E = nullptr, *m_dev = nullptr;
    // keys are sorted in `edges` / `alt`; the unique edges end up in the other one
    clean_arcs(ctx, n, M, rowptr, col, rank, world, edges, alt, E, m_dev, deg, method);
    if (E != edges) {
        uint64_t m = 0;
        TC_CUDA(cudaMemcpyAsync(&m, m_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
        TC_CUDA(cudaStreamSynchronize(ctx.stream));
        if (m) TC_CUDA(cudaMemcpyAsync(edges, E, m * sizeof(uint64_t), cudaMemcpyDeviceToDevice, ctx.stream));
    }
    TC_CUDA(cudaMemcpyAsync(m_dev_out, m_dev, sizeof(uint64_t), cudaMemcpyDeviceToDevice, ctx.stream));
}

void orient_dirty(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
                  Oriented &out, Timer *tm,
                  PruneInfo &prune, bool id_order, uint32_t method) {
    phase_begin(tm, kClean);
    uint64_t *keys = ctx.alloc<uint64_t>(M);
    uint64_t *keys_alt = ctx.alloc<uint64_t>(M);
    uint32_t *deg = ctx.alloc<uint32_t>(n);
    TC_CUDA(cudaMemsetAsync(deg, 0, n * sizeof(uint32_t), ctx.stream));
    uint64_t *E = nullptr, *m_dev = nullptr;
    clean_arcs(ctx, n, M, rowptr, col, 0, 1, keys, keys_alt, E, m_dev, deg, method);
    phase_end(tm, kClean);
    orient_edges(ctx, n, M, E, m_dev, deg, out, tm, prune, id_order, keys, keys_alt);
}

// a2-a4 from the unique undirected edges E (keys (min << b) | max; any order) and the degrees
// of the graph they form.  free0 / free1: workspace blocks that are dead once the oriented
// pairs exist (the a1 key buffers), given back to the pool before the CSR build.
void orient_edges(Ctx &ctx, uint64_t n, uint64_t M, uint64_t *E, uint64_t *m_dev, uint32_t *deg,
                  Oriented &out, Timer *tm, PruneInfo &prune, bool id_order, void *free0,
                  void *free1) {
    const int b = id_bits(n);
    phase_begin(tm, kOrient);
    uint32_t *dplus = ctx.alloc<uint32_t>(n + 1), *dminus = ctx.alloc<uint32_t>(n + 1);
    TC_CUDA(cudaMemsetAsync(dplus, 0, (n + 1) * sizeof(uint32_t), ctx.stream));
    TC_CUDA(cudaMemsetAsync(dminus, 0, (n + 1) * sizeof(uint32_t), ctx.stream));
    int grid = ctx.persistent_grid(8);
    if (prune.enabled) {
        phase_begin(tm, kPrune);
        prune_pairs(ctx, n, b, prune.rounds_wanted, E, m_dev, deg, M, prune);
        phase_end(tm, kPrune);
    }
    rank_permutation(ctx, n, rank_key(ctx, n, deg, id_order), out);
    uint32_t *okey = ctx.alloc<uint32_t>(M), *oval = ctx.alloc<uint32_t>(M);
    const int pdb = radix_digit_bits(b), ppasses = (b + pdb - 1) / pdb;
    uint32_t *phist = ctx.alloc<uint32_t>(2 * ppasses * kHistDigits);
    TC_CUDA(cudaMemsetAsync(phist, 0, 2 * ppasses * kHistDigits * sizeof(uint32_t), ctx.stream));
    k_orient_pairs<<<grid, 256, 0, ctx.stream>>>(E, m_dev, b, out.newid, okey, oval, dplus, phist,
                                                 phist + ppasses * kHistDigits, ppasses, pdb);
    TC_LAUNCHED(ctx);
    out.stage_work = ctx.alloc<uint64_t>(1);
    TC_CUDA(cudaMemsetAsync(out.stage_work, 0, sizeof(uint64_t), ctx.stream));
    k_dminus<<<grid, 256, 0, ctx.stream>>>(deg, out.newid, dplus, n, dminus, out.stage_work);
    TC_LAUNCHED(ctx);
    // the 64-bit keys (E and its sort buffer) are dead: give 16 B per raw arc back to the
    // pool before the CSR build (peak device memory at s26: -17 GB)
    if (free0) ctx.free_now(free0);
    if (free1) ctx.free_now(free1);
    pairs_to_csr(ctx, n, M, okey, oval, dplus, dminus, m_dev, out, tm, phist,
                 phist + ppasses * kHistDigits);
}

// ------------------------------------------------------------------ clean input
__global__ void k_deg_rowptr(const uint64_t *__restrict__ rowptr, uint64_t n,
                             uint32_t *__restrict__ deg) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x)
        deg[u] = (uint32_t)(rowptr[u + 1] - rowptr[u]);
}

// Clean input: one persistent pass.  Tiles of arcs keep the arcs with u < v (ids; each edge of
// a simple symmetric CSR once) and write them as oriented pairs (lower rank, higher rank) in rank ids at a tile offset taken by ONE atomic per tile (the
// pair order is free: the two-key sort that follows fixes the CSR order), count d+ (one atomic
// per run of equal sources) and the digit histograms of both radix sorts that follow (flushed
// once per block).  (A decoupled look-back for an order-preserving offset measured 1.07 ms at
// s21 against this.)  Writes stop at cap: a false TC_CLEAN claim is reported, never written
// out of bounds.
#ifndef TC_EMIT_MINB
#define TC_EMIT_MINB 1
#endif
__global__ void __launch_bounds__(kTileThreads, TC_EMIT_MINB)
    k_orient_emit(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col,
                  uint64_t n, uint64_t M, const uint32_t *__restrict__ deg,
                  const uint32_t *__restrict__ newid, uint64_t *__restrict__ m_out,
                  uint32_t *__restrict__ okey, uint32_t *__restrict__ oval,
                  uint32_t *__restrict__ dplus, uint32_t *__restrict__ hist_key,
                  uint32_t *__restrict__ hist_val, int passes, int db, uint64_t cap,
                  uint32_t *__restrict__ claim_err, const uint2 *__restrict__ tb, bool pruned) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    __shared__ uint64_t s_base;
    __shared__ RsHist<4> s_hk, s_hv;
    s_hk.clear();
    s_hv.clear();
    const uint64_t tiles = (M + kTileItems - 1) / kTileItems;
    for (uint64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        __syncthreads();   // s_row / s_base of the previous tile are no longer read
        const uint64_t t0 = tile * kTileItems;
        const uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
        tile_rows_b(rowptr, t0, len, tb[tile], s_row, s_scan);
        const uint32_t i0 = threadIdx.x * kItemsPerThread;
        // a symmetric input holds every edge twice: keep the arc with u < v (ids, no gather
        // needed to decide) and orient it by rank, rank(u) < rank(v) <=> newid[u] < newid[v]
        // (round 2: half the random newid gathers of filtering every arc by rank); deg = 0
        // marks a pruned vertex (TC_PRUNE only)
        uint32_t f[kItemsPerThread], nu[kItemsPerThread], nv[kItemsPerThread], c = 0;
#pragma unroll
        for (int k = 0; k < kItemsPerThread; k++) {
            const uint32_t i = i0 + k;
            const uint32_t u = i < len ? s_row[i] : 0u, v = i < len ? col[t0 + i] : 0u;
            f[k] = i < len && u < v && (!pruned || (deg[u] != 0 && deg[v] != 0));
            const uint32_t a = newid[u], b = f[k] ? newid[v] : 0u;
            nu[k] = min(a, b);
            nv[k] = max(a, b);
            c += f[k];
        }
        uint32_t total;
        const uint32_t pos = block_exclusive_scan<SumOp>(c, s_scan, &total);
        if (threadIdx.x == 0) s_base = atomicAdd((unsigned long long *)m_out, (unsigned long long)total);
        __syncthreads();
        uint64_t base = s_base + pos;
        uint32_t run_s = 0, run_n = 0;
#pragma unroll
        for (int k = 0; k < kItemsPerThread; k++) {
            if (f[k] && base < cap) {
                const uint32_t sv = nu[k], tv = nv[k];
                okey[base] = sv;
                oval[base] = tv;
                s_hk.add(sv, passes, db);
                s_hv.add(tv, passes, db);
                base++;
                if (run_n && sv == run_s) {
                    run_n++;
                } else {
                    if (run_n) atomicAdd(&dplus[run_s], run_n);
                    run_s = sv;
                    run_n = 1;
                }
            }
        }
        if (run_n) atomicAdd(&dplus[run_s], run_n);
    }
    __syncthreads();
    s_hk.flush(hist_key, passes);
    s_hv.flush(hist_val, passes);
}

// A simple symmetric graph keeps exactly one arc per edge (M/2 < cap); more means a false
// TC_CLEAN claim: clamp m to what was written and flag it (TC_EGRAPH at the end of the call).
__global__ void k_emit_clamp(uint64_t *__restrict__ m, uint64_t cap, uint32_t *__restrict__ claim_err) {
    if (*m >= cap) {
        *claim_err = 1u;
        *m = cap;
    }
}

void orient_clean(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
                  Oriented &out, Timer *tm,
                  PruneInfo &prune, bool id_order) {
    uint32_t tiles = (uint32_t)((M + kTileItems - 1) / kTileItems);
    int grid = ctx.persistent_grid(8);
    phase_begin(tm, kOrient);
    uint32_t *deg = ctx.alloc<uint32_t>(n);
    k_deg_rowptr<<<grid, 256, 0, ctx.stream>>>(rowptr, n, deg);
    TC_LAUNCHED(ctx);
    if (prune.enabled) {
        phase_begin(tm, kPrune);
        prune.m_before_host = M / 2;
        prune_csr(ctx, n, M, rowptr, col, prune.rounds_wanted, deg, prune);
        phase_end(tm, kPrune);
    }
    const uint32_t *key = rank_key(ctx, n, deg, id_order);
    rank_permutation(ctx, n, key, out);
    // m and the false-claim flag; the digit histograms of both pair sorts
    uint64_t *st = ctx.alloc<uint64_t>(2);   // m, the false-claim flag
    TC_CUDA(cudaMemsetAsync(st, 0, 2 * sizeof(uint64_t), ctx.stream));
    uint64_t *m_dev = st;
    out.claim_err = (uint32_t *)(st + 1);
    const int b = id_bits(n), pdb = radix_digit_bits(b), ppasses = (b + pdb - 1) / pdb;
    uint32_t *phist = ctx.alloc<uint32_t>(2 * ppasses * kHistDigits);
    TC_CUDA(cudaMemsetAsync(phist, 0, 2 * ppasses * kHistDigits * sizeof(uint32_t), ctx.stream));
    uint64_t cap = M / 2 + 1;
    uint32_t *okey = ctx.alloc<uint32_t>(cap), *oval = ctx.alloc<uint32_t>(cap);
    uint32_t *dplus = ctx.alloc<uint32_t>(n + 1), *dminus = ctx.alloc<uint32_t>(n + 1);
    TC_CUDA(cudaMemsetAsync(dplus, 0, (n + 1) * sizeof(uint32_t), ctx.stream));
    TC_CUDA(cudaMemsetAsync(dminus, 0, (n + 1) * sizeof(uint32_t), ctx.stream));
#ifndef TC_EMIT_PER_SM
#define TC_EMIT_PER_SM 4   // swept 4 / 6 / 8: clean-input orient 2.53 / 2.77 / 2.65 ms (s21)
#endif
    uint32_t egrid = (uint32_t)std::min<uint64_t>(tiles, (uint64_t)ctx.persistent_grid(TC_EMIT_PER_SM));
    uint2 *tb = ctx.alloc<uint2>(tiles + 1);
    tile_bounds(ctx, rowptr, n, M, nullptr, tb);
    k_orient_emit<<<egrid, kTileThreads, 0, ctx.stream>>>(rowptr, col, n, M, key, out.newid, m_dev,
                                                          okey, oval, dplus, phist,
                                                          phist + ppasses * kHistDigits, ppasses,
                                                          pdb, cap, out.claim_err, tb, prune.enabled);
    TC_LAUNCHED(ctx);
    k_emit_clamp<<<1, 1, 0, ctx.stream>>>(m_dev, cap, out.claim_err);
    TC_LAUNCHED(ctx);
    out.stage_work = ctx.alloc<uint64_t>(1);
    TC_CUDA(cudaMemsetAsync(out.stage_work, 0, sizeof(uint64_t), ctx.stream));
    // d-(x) is counted from the written pairs (not d(x) - d+(x)), so a false TC_CLEAN claim
    // cannot make the transposed CSR disagree with them
    pairs_to_csr(ctx, n, cap, okey, oval, dplus, dminus, m_dev, out, tm, phist,
                 phist + ppasses * kHistDigits, true);
}

// ------------------------------------------------------------------ back to original ids
__global__ void __launch_bounds__(kTileThreads)
    k_pairs_original(const uint64_t *__restrict__ off, const uint32_t *__restrict__ colp, uint64_t n,
                     const uint64_t *__restrict__ m_dev, const uint32_t *__restrict__ order,
                     uint32_t *__restrict__ src, uint32_t *__restrict__ dst,
                     uint32_t *__restrict__ idx, uint32_t *__restrict__ dcount) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    uint64_t m = *m_dev;
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    if (t0 >= m) return;
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, m - t0);
    tile_rows(off, n, t0, len, s_row, s_scan);
    for (uint32_t i = threadIdx.x; i < len; i += kTileThreads) {
        uint32_t a = order[s_row[i]], c = order[colp[t0 + i]];
        src[t0 + i] = a;
        dst[t0 + i] = c;
        idx[t0 + i] = (uint32_t)(t0 + i);
        atomicAdd(&dcount[a], 1u);
    }
}

// out[k] = in[perm[k]] for k < *m_dev.
__global__ void k_permute(const uint32_t *__restrict__ in, const uint32_t *__restrict__ perm,
                          const uint64_t *__restrict__ m_dev, uint32_t *__restrict__ out) {
    uint64_t m = *m_dev;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = in[perm[k]];
}

void to_original(Ctx &ctx, const Oriented &g, uint64_t *off_out, uint32_t *col_out,
                 const uint32_t *pay_in, uint32_t *pay_out) {
    uint64_t cap = g.m_cap, n = g.n;
    int b = id_bits(n);
    int grid = ctx.persistent_grid(8);
    uint32_t *src = ctx.alloc<uint32_t>(cap), *dst = ctx.alloc<uint32_t>(cap);
    uint32_t *kA = ctx.alloc<uint32_t>(cap), *kB = ctx.alloc<uint32_t>(cap);
    uint32_t *kC = ctx.alloc<uint32_t>(cap);
    uint32_t *vA = ctx.alloc<uint32_t>(cap), *vB = ctx.alloc<uint32_t>(cap);
    uint32_t *vC = ctx.alloc<uint32_t>(cap), *vD = ctx.alloc<uint32_t>(cap);
    uint32_t *cnt = ctx.alloc<uint32_t>(n + 1);
    TC_CUDA(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(uint32_t), ctx.stream));
    uint32_t tiles = (uint32_t)((cap + kTileItems - 1) / kTileItems);
    k_pairs_original<<<tiles, kTileThreads, 0, ctx.stream>>>(g.off, g.col, n, g.m_dev, g.order, src,
                                                             dst, vA, cnt);
    TC_LAUNCHED(ctx);
    // rows ascending: the edge index (vA) sorted stably by target, then by source
    uint32_t *k1, *p1, *k2, *p2;
    radix_sort_pairs_from(ctx, dst, vA, kA, kB, vB, vC, cap, g.m_dev, b, &k1, &p1);
    uint32_t *s1 = (k1 == kA) ? kB : kA;
    k_permute<<<grid, 256, 0, ctx.stream>>>(src, p1, g.m_dev, s1);
    TC_LAUNCHED(ctx);
    radix_sort_pairs_from(ctx, s1, p1, k1, kC, vA, vD, cap, g.m_dev, b, &k2, &p2);
    (void)k2;
    scan_exclusive(ctx, cnt, off_out, n);
    k_permute<<<grid, 256, 0, ctx.stream>>>(dst, p2, g.m_dev, col_out);
    TC_LAUNCHED(ctx);
    if (pay_in) {
        k_permute<<<grid, 256, 0, ctx.stream>>>(pay_in, p2, g.m_dev, pay_out);
        TC_LAUNCHED(ctx);
    }
}

__global__ void k_pv_original(const uint64_t *__restrict__ pv_new, const uint32_t *__restrict__ newid,
                              uint64_t n, uint64_t *__restrict__ pv_out) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        pv_out[v] = pv_new[newid[v]];
}

void per_vertex_to_original(Ctx &ctx, const Oriented &g, const uint64_t *pv_new, uint64_t *pv_out) {
    k_pv_original<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(pv_new, g.newid, g.n, pv_out);
    TC_LAUNCHED(ctx);
}

}  // namespace tc
