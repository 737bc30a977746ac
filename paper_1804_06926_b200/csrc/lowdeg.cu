// lowdeg.cu -- the bounded-degree path (round 2): graphs on which every vertex has at most
// L <= 32 arc incidences (road networks, meshes: BASELINE configs[3]).
//
// The paper flags this regime: on road networks the filtering step's "overhead causes a
// slowdown" because there is little intersection work to amortise it.  The general
// pipeline spends 3.3 ms on the 14 M-vertex road mesh, 97 % of it in a1-a5 (rank sort, two-key
// pair sort, in-lists, binning) for 0.09 ms of intersection.  When no vertex has more than L
// incidences, every list fits in one thread's registers / local memory and none of that
// machinery is needed -- the method is unchanged, only its data layout is:
//   a1 clean      (Table 1 caption; DESIGN R1)  each vertex gathers its incidences
//                 (its out-arcs plus its in-arcs, scattered by one counting pass), drops
//                 self-loops, sorts and de-duplicates them in a thread: N(v) ascending, d(v);
//   a2 degree     (R3)  d(v) = |N(v)| after cleaning;
//   a3 filter     (Alg. 2, R2)  N+(u) = {x in N(u) : (d(u), u) < (d(x), x)} is taken
//                 on the fly from N(u) and d(.), in the thread that owns u (no relabelling: the
//                 rank test is a comparison, as in tiny.cu);
//   a4 sort       rows are ascending by id (the cleaning sorted them), so N+(u) is too;
//   a6 intersect  (Alg. 2, "TwoSmall" P:533)  for each x in N+(u) a two-pointer merge
//                 of N+(u) with N(x), counting common w with rank(w) > rank(x), i.e. w in
//                 N+(x): |N+(u) & N+(x)| exactly as P:315-321 (each triangle once, at its
//                 lowest-ranked vertex u and middle vertex x);
//   a7 reduce  per-thread u64 -> warp shuffle -> shared memory -> one atomicAdd.
// Per-vertex counts credit u, x and w.  Eligibility is decided on the device (a row longer than
// L, or a vertex with more than L incidences, sets a flag) and read once by the host; a graph
// that fails takes the general pipeline (tc_api.cu).
#include "tc_internal.cuh"
#include "block_scan.cuh"

namespace tc {

constexpr uint32_t kLdThreads = 256;
// TC_BOUNDS_CHECK=1 (scripts/build_variant.py; the pool's compute-sanitizer is closed): every
// index into the rows, the slot bytes and the per-thread lists is asserted (trap on violation)
#ifndef TC_BOUNDS_CHECK
#define TC_BOUNDS_CHECK 0
#endif
#define LD_CHECK(c)                          \
    do {                                     \
        if (TC_BOUNDS_CHECK && !(c)) __trap(); \
    } while (0)

__device__ __forceinline__ bool ld_rank_less(uint32_t du, uint32_t u, uint32_t dv, uint32_t v) {
    return du < dv || (du == dv && u < v);
}

__device__ __forceinline__ uint64_t ld_block_sum(uint64_t x, uint64_t *s_red) {
    x = __reduce_add_sync(0xffffffffu, (uint32_t)x) + ((uint64_t)__reduce_add_sync(0xffffffffu, (uint32_t)(x >> 32)) << 32);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) s_red[warp] = x;
    __syncthreads();
    uint64_t s = 0;
    if (threadIdx.x == 0)
        for (uint32_t w = 0; w < kLdThreads / 32; w++) s += s_red[w];
    return s;   // valid in thread 0
}

#define LD_FOR_VERTICES(v, n)                                                                  \
    for (uint64_t v = (uint64_t)blockIdx.x * kLdThreads + threadIdx.x; v < (n);               \
         v += (uint64_t)gridDim.x * kLdThreads)

// Rows of at most kLdReg entries (all of them on road meshes) are held in registers: static
// indices only (a sorting network, membership masks); longer rows use local-memory arrays.
constexpr uint32_t kLdReg = 8;
constexpr uint32_t kLdNone = 0xffffffffu;   // padding: above every vertex id
// pk[v] = d(v) << 40 | offset of v's row in adj (offsets < 2^33: 2M < 2^33 arcs): the count
// kernel's gather of a neighbour x yields its degree AND its row in one 8-byte load.
__device__ __forceinline__ uint64_t ld_pack(uint32_t d, uint64_t off) { return ((uint64_t)d << 40) | off; }
__device__ __forceinline__ uint32_t ld_pk_deg(uint64_t p) { return (uint32_t)(p >> 40); }
__device__ __forceinline__ uint64_t ld_pk_off(uint64_t p) { return p & ((1ull << 40) - 1); }
__device__ __forceinline__ void ld_cswap(uint32_t &a, uint32_t &b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}
__device__ __forceinline__ void ld_sort8(uint32_t (&a)[8]) {   // Batcher's 19-comparator network
    ld_cswap(a[0], a[1]); ld_cswap(a[2], a[3]); ld_cswap(a[4], a[5]); ld_cswap(a[6], a[7]);
    ld_cswap(a[0], a[2]); ld_cswap(a[1], a[3]); ld_cswap(a[4], a[6]); ld_cswap(a[5], a[7]);
    ld_cswap(a[1], a[2]); ld_cswap(a[5], a[6]); ld_cswap(a[0], a[4]); ld_cswap(a[3], a[7]);
    ld_cswap(a[1], a[5]); ld_cswap(a[2], a[6]); ld_cswap(a[1], a[4]); ld_cswap(a[3], a[6]);
    ld_cswap(a[2], a[4]); ld_cswap(a[3], a[5]); ld_cswap(a[3], a[4]);
}

// Dirty input, pass 1: in-arc counts cin[v]; each arc keeps the slot its atomic returned
// (slot8[k], one byte: slots < L <= 32); flag a row longer than L or a count above L.
__global__ void __launch_bounds__(kLdThreads)
    k_ld_in(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col, uint64_t n,
            uint32_t L, uint32_t *__restrict__ cin, uint8_t *__restrict__ slot8, uint32_t *__restrict__ flag) {
    LD_FOR_VERTICES(u, n) {
        const uint64_t b = rowptr[u], e = rowptr[u + 1];
        if (e - b > L) {
            *flag = 1u;
            continue;
        }
        for (uint64_t k = b; k < e; k++) {
            const uint32_t v = col[k];
            if (v == (uint32_t)u) continue;
            const uint32_t old = atomicAdd(&cin[v], 1u);
            slot8[k] = (uint8_t)min(old, 255u);
            if (old == L) *flag = 1u;
        }
    }
}

// Pass 2: inc[v] = in-arcs + out-arcs (flag inc > L) and the row offsets aoff[v]: a block scan
// of inc plus ONE atomic per block on *next (rows are contiguous per block of vertices, blocks
// in any order: no device-wide scan).  inc overwrites cin.
__global__ void __launch_bounds__(kLdThreads)
    k_ld_offsets(const uint64_t *__restrict__ rowptr, uint64_t n, uint32_t L, uint32_t *__restrict__ inc,
                 uint64_t *__restrict__ aoff, unsigned long long *__restrict__ next, uint32_t *__restrict__ flag) {
    __shared__ uint32_t s_scan[kLdThreads / 32];
    __shared__ uint64_t s_base;
    for (uint64_t v0 = (uint64_t)blockIdx.x * kLdThreads; v0 < n; v0 += (uint64_t)gridDim.x * kLdThreads) {
        const uint64_t v = v0 + threadIdx.x;
        uint32_t x = 0;
        if (v < n) {
            const uint64_t c = (rowptr[v + 1] - rowptr[v]) + inc[v];
            if (c > L) *flag = 1u;
            x = (uint32_t)min(c, (uint64_t)kLowDegMax + 1);   // (rows of a flagged graph are never read)
            inc[v] = x;
        }
        uint32_t total;
        const uint32_t pre = block_exclusive_scan<SumOp>(x, s_scan, &total);
        if (threadIdx.x == 0) s_base = atomicAdd(next, (unsigned long long)total);
        __syncthreads();
        if (v < n) aoff[v] = s_base + pre;
        __syncthreads();
    }
}

// Pass 3: every incidence into its vertex's row: the in-arc u of v at aoff[v] + slot8, row u's
// out-arcs after its in-arcs at aoff[u] + cin(u).
__global__ void __launch_bounds__(kLdThreads)
    k_ld_scatter(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col, uint64_t n,
                 const uint64_t *__restrict__ aoff, const uint32_t *__restrict__ inc,
                 const uint8_t *__restrict__ slot8, uint32_t *__restrict__ adj, uint64_t cap,
                 const uint32_t *__restrict__ flag) {
    if (*flag) return;   // not eligible: the call is re-run on the general pipeline
    LD_FOR_VERTICES(u, n) {
        const uint64_t b = rowptr[u], e = rowptr[u + 1];
        if (b == e) continue;
        const uint64_t s = aoff[u] + (inc[u] - (uint32_t)(e - b));
        for (uint64_t k = b; k < e; k++) {
            const uint32_t v = col[k];
            LD_CHECK(v < n && s + (k - b) < cap && (k - b) < inc[u]);
            adj[s + (k - b)] = v;
            if (v != (uint32_t)u) {
                LD_CHECK(slot8[k] < inc[v] && aoff[v] + slot8[k] < cap);
                adj[aoff[v] + slot8[k]] = (uint32_t)u;
            }
        }
    }
}

// Pass 4 (a1 + a2): each vertex sorts its incidences, drops self-loops and duplicates, and
// writes N(v) ascending back to the front of its row; d(v); Sum d(v) = 2m into *m2.
__global__ void __launch_bounds__(kLdThreads)
    k_ld_clean(const uint64_t *__restrict__ aoff, const uint32_t *__restrict__ inc, uint64_t n,
               uint32_t *__restrict__ adj, uint64_t *__restrict__ pk, unsigned long long *__restrict__ m2,
               const uint32_t *__restrict__ flag) {
    __shared__ uint64_t s_red[kLdThreads / 32];
    if (*flag) return;   // (uniform: the flag is final before this kernel starts)
    uint64_t sum = 0;
    LD_FOR_VERTICES(v, n) {
        const uint64_t s = aoff[v];
        const uint32_t c = inc[v];
        LD_CHECK(c <= kLowDegMax);
        uint32_t d = 0;
        if (c <= kLdReg) {   // registers: pad, sort (network), unique
            uint32_t r[8];
#pragma unroll
            for (uint32_t i = 0; i < 8; i++) {
                const uint32_t x = i < c ? adj[s + i] : kLdNone;
                r[i] = x == (uint32_t)v ? kLdNone : x;
            }
            ld_sort8(r);
#pragma unroll
            for (uint32_t i = 0; i < 8; i++)
                if (r[i] != kLdNone && (i == 0 || r[i] != r[i - 1])) adj[s + d++] = r[i];
        } else {
            uint32_t a[32];
            uint32_t k = 0;
            for (uint32_t i = 0; i < c && i < 32; i++) {   // insertion sort, self-loops dropped
                const uint32_t x = adj[s + i];
                if (x == (uint32_t)v) continue;
                uint32_t j = k++;
                while (j > 0 && a[j - 1] > x) {
                    a[j] = a[j - 1];
                    j--;
                }
                a[j] = x;
            }
            for (uint32_t i = 0; i < k; i++)
                if (i == 0 || a[i] != a[i - 1]) adj[s + d++] = a[i];
        }
        pk[v] = ld_pack(d, s);
        sum += d;
    }
    sum = ld_block_sum(sum, s_red);
    if (threadIdx.x == 0 && sum) atomicAdd(m2, (unsigned long long)sum);
}

// Clean input (TC_CLEAN): d(v) = row length; flag a row longer than L; rows not promised
// sorted are sorted into adj (same offsets).
__global__ void __launch_bounds__(kLdThreads)
    k_ld_clean_rows(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col, uint64_t n,
                    uint32_t L, bool sort, uint32_t *__restrict__ adj, uint64_t *__restrict__ pk,
                    uint32_t *__restrict__ flag) {
    LD_FOR_VERTICES(v, n) {
        const uint64_t b = rowptr[v], c = rowptr[v + 1] - b;
        if (c > L) {
            *flag = 1u;
            continue;
        }
        pk[v] = ld_pack((uint32_t)c, b);
        if (!sort) continue;
        uint32_t a[32];
        for (uint32_t i = 0; i < (uint32_t)c; i++) {
            const uint32_t x = col[b + i];
            uint32_t j = i;
            while (j > 0 && a[j - 1] > x) {
                a[j] = a[j - 1];
                j--;
            }
            a[j] = x;
        }
        for (uint32_t i = 0; i < (uint32_t)c; i++) adj[b + i] = a[i];
    }
}

// a3 + a6 + a7: one thread per vertex u.  out[]: 0 = W, 1 = probe work, 2 = max d+,
// 3 = Sum d-(v) d+(v), 4 = skipped edges, 5 = Sum d+ (arcs passing the rank filter).
template <bool STATS>
__global__ void __launch_bounds__(kLdThreads, 8)   // 8 CTAs / SM: occupancy hides the gathers
    k_ld_count(const uint32_t *__restrict__ adj, uint64_t cap, const uint64_t *__restrict__ pk, uint64_t n,
               unsigned long long *__restrict__ total, unsigned long long *__restrict__ pv,
               unsigned long long *__restrict__ out, const uint32_t *__restrict__ flag) {
    __shared__ uint64_t s_red[kLdThreads / 32];
    if (*flag) return;   // not eligible: nothing is counted, the call is re-run
    uint64_t tri = 0, npsum = 0, W = 0, probe = 0, stage = 0, skipped = 0, maxdp = 0;
    LD_FOR_VERTICES(u, n) {
        const uint64_t pu = pk[u];   // one 8-byte load: d(u) and the row's offset
        const uint32_t du = ld_pk_deg(pu);
        const uint64_t s = ld_pk_off(pu);
        uint32_t pid[32];
        uint64_t ppk[32];
        uint32_t np = 0;
        LD_CHECK(du <= kLowDegMax && s + du <= cap);
        for (uint32_t i = 0; i < du; i++) {   // N+(u), ascending by id
            const uint32_t x = adj[s + i];
            LD_CHECK(x < n && (i == 0 || adj[s + i - 1] < x));
            const uint64_t px = pk[x];
            if (ld_rank_less(du, (uint32_t)u, ld_pk_deg(px), x)) {
                pid[np] = x;
                ppk[np] = px;
                np++;
            }
        }
        npsum += np;
        uint64_t tu = 0;
        for (uint32_t j = 0; j < np; j++) {
            const uint32_t x = pid[j], dx = ld_pk_deg(ppk[j]);
            const uint64_t sx = ld_pk_off(ppk[j]);
            LD_CHECK(dx <= kLowDegMax && sx + dx <= cap);
            uint32_t i = 0, k = 0;
            while (i < dx && k < np) {   // N(x) merged with N+(u): common w with rank(w) > rank(x)
                const uint32_t w = adj[sx + i], y = pid[k];
                if (w < y) i++;
                else if (y < w) k++;
                else {
                    if (ld_rank_less(dx, x, ld_pk_deg(ppk[k]), w)) {
                        tu++;
                        if (pv) {
                            atomicAdd(&pv[x], 1ull);
                            atomicAdd(&pv[w], 1ull);
                        }
                    }
                    i++;
                    k++;
                }
            }
            if (STATS) {   // d+(x), |N+(u) after x| (rank order): W, probe work, skipped edges
                uint32_t dpx = 0;
                for (uint32_t t = 0; t < dx; t++) {
                    const uint32_t w = adj[sx + t];
                    dpx += ld_rank_less(dx, x, ld_pk_deg(pk[w]), w);
                }
                uint32_t after = 0;
                for (uint32_t t = 0; t < np; t++) after += ld_rank_less(dx, x, ld_pk_deg(ppk[t]), pid[t]);
                W += np + dpx;
                probe += min(after, dpx);
                skipped += (after == 0 || dpx == 0);
            }
        }
        if (pv && tu) atomicAdd(&pv[u], (unsigned long long)tu);
        tri += tu;
        if (STATS) {
            stage += (uint64_t)(du - np) * np;
            maxdp = max(maxdp, (uint64_t)np);
        }
    }
    tri = ld_block_sum(tri, s_red);
    if (threadIdx.x == 0 && tri) atomicAdd(total, (unsigned long long)tri);
    npsum = ld_block_sum(npsum, s_red);
    if (threadIdx.x == 0 && npsum) atomicAdd(&out[5], (unsigned long long)npsum);
    if (STATS) {
        W = ld_block_sum(W, s_red);
        probe = ld_block_sum(probe, s_red);
        stage = ld_block_sum(stage, s_red);
        skipped = ld_block_sum(skipped, s_red);
        if (threadIdx.x == 0) {
            atomicAdd(&out[0], (unsigned long long)W);
            atomicAdd(&out[1], (unsigned long long)probe);
            atomicAdd(&out[3], (unsigned long long)stage);
            atomicAdd(&out[4], (unsigned long long)skipped);
        }
        if (maxdp) atomicMax(&out[2], (unsigned long long)maxdp);
    }
}

static uint32_t ld_grid(const Ctx &ctx, uint64_t n) {
    return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + kLdThreads - 1) / kLdThreads,
                                                              (uint64_t)ctx.persistent_grid(8)));
}

void lowdeg_prepare(Ctx &ctx, LowDeg &ld, uint64_t n, uint64_t M, const uint64_t *rowptr,
                    const uint32_t *col, bool clean, bool sorted, uint32_t L, uint32_t *flag_dev) {
    L = std::min<uint32_t>(L, kLowDegMax);
    const uint32_t grid = ld_grid(ctx, n);
    ld.n = n;
    ld.flag = flag_dev;
    ld.pk = ctx.alloc<uint64_t>(n);
    if (clean) {
        ld.aoff = rowptr;
        ld.adj = sorted ? col : ctx.alloc<uint32_t>(M);
        k_ld_clean_rows<<<grid, kLdThreads, 0, ctx.stream>>>(rowptr, col, n, L, !sorted,
                                                            const_cast<uint32_t *>(ld.adj), ld.pk, flag_dev);
        TC_LAUNCHED(ctx);
        ld.m2_host = M;
        ld.adj_cap = M;
        return;
    }
    // dirty: in-counts (+ each arc's slot), slot counts and row offsets; the scatter and
    // k_ld_clean run in lowdeg_count
    ld.m2 = ctx.alloc<uint64_t>(2);
    TC_CUDA(cudaMemsetAsync(ld.m2, 0, 2 * sizeof(uint64_t), ctx.stream));   // [0] Sum d, [1] next row
    uint32_t *inc = ctx.alloc<uint32_t>(n);
    TC_CUDA(cudaMemsetAsync(inc, 0, n * sizeof(uint32_t), ctx.stream));
    ld.slot8 = ctx.alloc<uint8_t>(M);
    k_ld_in<<<grid, kLdThreads, 0, ctx.stream>>>(rowptr, col, n, L, inc, ld.slot8, flag_dev);
    TC_LAUNCHED(ctx);
    uint64_t *aoff = ctx.alloc<uint64_t>(n);
    k_ld_offsets<<<grid, kLdThreads, 0, ctx.stream>>>(rowptr, n, L, inc, aoff,
                                                     (unsigned long long *)(ld.m2 + 1), flag_dev);
    TC_LAUNCHED(ctx);
    ld.inc = inc;
    ld.aoff = aoff;
    ld.rowptr = rowptr;
    ld.col = col;
}

void lowdeg_count(Ctx &ctx, LowDeg &ld, uint64_t M, Timer *tm, uint64_t *total_dev, uint64_t *pv_dev,
                  uint64_t *out_dev, bool stats) {
    const uint64_t n = ld.n;
    const uint32_t grid = ld_grid(ctx, n);
    if (ld.inc) {   // dirty input: finish a1 + a2
        uint32_t *adj = ctx.alloc<uint32_t>(2 * M);
        k_ld_scatter<<<grid, kLdThreads, 0, ctx.stream>>>(ld.rowptr, ld.col, n, ld.aoff, ld.inc, ld.slot8,
                                                         adj, 2 * M, ld.flag);
        TC_LAUNCHED(ctx);
        k_ld_clean<<<grid, kLdThreads, 0, ctx.stream>>>(ld.aoff, ld.inc, n, adj, ld.pk,
                                                       (unsigned long long *)ld.m2, ld.flag);
        TC_LAUNCHED(ctx);
        ld.adj = adj;
        ld.adj_cap = 2 * M;
    }
    phase_end(tm, kClean);
    phase_begin(tm, kIntersect);
    if (stats)
        k_ld_count<true><<<grid, kLdThreads, 0, ctx.stream>>>(
            ld.adj, ld.adj_cap, ld.pk, n, (unsigned long long *)total_dev, (unsigned long long *)pv_dev,
            (unsigned long long *)out_dev, ld.flag);
    else
        k_ld_count<false><<<grid, kLdThreads, 0, ctx.stream>>>(
            ld.adj, ld.adj_cap, ld.pk, n, (unsigned long long *)total_dev, (unsigned long long *)pv_dev,
            (unsigned long long *)out_dev, ld.flag);
    TC_LAUNCHED(ctx);
    phase_end(tm, kIntersect);
}

}  // namespace tc
