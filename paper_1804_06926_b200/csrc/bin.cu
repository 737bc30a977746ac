// bin.cu -- a5: work estimation and binning (§4.2.2 P:527-542 "dynamic
// grouping ... divide the edge lists into groups"; third kernel P:704-708).
// Per oriented edge (u,v): a = min(d+u, d+v), b = max.  Edges that cannot close
// a triangle (d+(u) < 2 or d+(v) = 0) are skipped.  AUTO policy:
//   b <= short_max            -> SHORT   (thread per edge)
//   skew_ratio && b >= r * a  -> SEARCH  (binary search of the short list)
//   otherwise                 -> HASH    (shorter list probed into a shared-memory
//                                         hash of the longer one, grouped by owner)
// force_variant routes every edge to one variant instead.
// HASH edges are regrouped into an owner CSR (counting sort by owner with
// atomics; order inside a group is irrelevant to the count).  Owners with
// d+ >= hub_min (or too long for a warp table) go to the CTA kernel.
// Multi-GPU: sources are split into `world` groups by an exclusive
// prefix of per-source work w(u) = sum_{v in N+(u)} (1 + min(d+u, d+v)); a rank keeps
// only its group's edges.  The split needs no communication.
#include "block_scan.cuh"
#include "tc_internal.cuh"

namespace tc {

// Rank owning source u: floor(prefix[u] / ceil(W/world)), clamped.
__device__ __forceinline__ int owner_of(const uint64_t *__restrict__ prefix, uint64_t chunk,
                                        uint32_t u, int world) {
    if (world <= 1 || chunk == 0) return 0;
    uint64_t r = prefix[u] / chunk;
    return r >= (uint64_t)world ? world - 1 : (int)r;
}

__device__ __forceinline__ void warp_append(bool take, uint64_t *counter, uint2 *out, uint2 item) {
    uint32_t mask = __ballot_sync(0xffffffffu, take);
    if (!mask) return;
    int lane = threadIdx.x & 31;
    int leader = __ffs(mask) - 1;
    uint64_t base = 0;
    if (lane == leader) base = atomicAdd((unsigned long long *)counter, (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (take) out[base + __popc(mask & ((1u << lane) - 1u))] = item;
}

__global__ void __launch_bounds__(kTileThreads)
    k_bin(const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
          const uint32_t *__restrict__ dplus, uint64_t n, const uint64_t *__restrict__ m_dev,
          BinParams p, uint2 *__restrict__ b_short, uint2 *__restrict__ b_merge,
          uint2 *__restrict__ b_search, uint2 *__restrict__ b_hash, uint32_t *__restrict__ pcnt,
          uint64_t *__restrict__ counts) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    __shared__ uint64_t s_red[kTileThreads / 32];
    uint64_t m = *m_dev;
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    if (t0 >= m) return;
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, m - t0);
    tile_rows(off, n, t0, len, s_row, s_scan);
    uint64_t chunk = 0;
    if (p.world > 1) chunk = (p.work_prefix[n] + p.world - 1) / p.world;
    uint64_t W = 0, probe = 0, skipped = 0;
    // striped over the tile so each warp handles 32 consecutive edges per round
    for (uint32_t base = 0; base < kTileItems; base += kTileThreads) {
        uint32_t i = base + threadIdx.x;
        bool valid = i < len;
        uint32_t u = 0, v = 0, du = 0, dv = 0;
        if (valid) {
            u = s_row[i];
            v = col[t0 + i];
            du = dplus[u];
            dv = dplus[v];
            W += du + dv;
            probe += min(du, dv);
        }
        int bin = -1;
        uint2 item = make_uint2(u, v);
        if (valid && owner_of(p.work_prefix, chunk, u, p.world) == p.rank) {
            uint32_t a = min(du, dv), b = max(du, dv);
            if (du < 2 || dv == 0) {
                skipped++;
            } else if (p.force >= 0) {
                bin = p.force;
            } else if (b <= p.short_max) {
                bin = TC_VARIANT_SHORT;
            } else if (p.skew_ratio && (uint64_t)b >= (uint64_t)p.skew_ratio * a) {
                bin = TC_VARIANT_SEARCH;
            } else {
                bin = TC_VARIANT_HASH;
            }
            if (bin == TC_VARIANT_HASH) {
                if (dv > du) item = make_uint2(v, u);   // owner = longer list (ties: source)
                atomicAdd(&pcnt[item.x], 1u);
            }
        }
        warp_append(bin == TC_VARIANT_SHORT, &counts[0], b_short, item);
        warp_append(bin == TC_VARIANT_MERGE, &counts[1], b_merge, item);
        warp_append(bin == TC_VARIANT_SEARCH, &counts[2], b_search, item);
        warp_append(bin == TC_VARIANT_HASH, &counts[3], b_hash, item);
    }
    W = block_sum_u64(W, s_red);
    probe = block_sum_u64(probe, s_red);
    skipped = block_sum_u64(skipped, s_red);
    if (threadIdx.x == 0) {
        atomicAdd((unsigned long long *)&counts[4], (unsigned long long)W);
        atomicAdd((unsigned long long *)&counts[5], (unsigned long long)probe);
        atomicAdd((unsigned long long *)&counts[6], (unsigned long long)skipped);
    }
}

// Scatter HASH pairs into the owner CSR (poff = exclusive scan of pcnt).
__global__ void k_group(const uint2 *__restrict__ b_hash, const uint64_t *__restrict__ counts,
                        const uint64_t *__restrict__ poff, uint32_t *__restrict__ cursor,
                        uint32_t *__restrict__ plist) {
    uint64_t ne = counts[3];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint2 e = b_hash[i];
        plist[poff[e.x] + atomicAdd(&cursor[e.x], 1u)] = e.y;
    }
}

// Owner lists and max d+: warp owners (d+ < cta_min), CTA bitmap owners (rank span
// n-1-x <= kCtaBitmapBits) and CTA hash owners (the rest).
__global__ void k_owners(const uint32_t *__restrict__ dplus, const uint32_t *__restrict__ pcnt,
                         uint64_t n, uint32_t cta_min, uint32_t *__restrict__ owners_warp,
                         uint32_t *__restrict__ owners_cta, uint32_t *__restrict__ owners_bitmap,
                         uint64_t *__restrict__ counts) {
    uint32_t local_max = 0;
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t end = (n + 31) & ~31ull;  // whole warps stay in the loop (warp-aggregated appends)
    int lane = threadIdx.x & 31;
    uint32_t lt = (1u << lane) - 1u;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < end; u += stride) {
        int kind = -1;
        if (u < n) {
            uint32_t du = dplus[u];
            local_max = max(local_max, du);
            if (pcnt[u]) kind = du < cta_min ? 0 : (n - 1 - u <= kCtaBitmapBits ? 2 : 1);
        }
        uint32_t *dst[3] = {owners_warp, owners_cta, owners_bitmap};
#pragma unroll
        for (int k = 0; k < 3; k++) {
            uint32_t mk = __ballot_sync(0xffffffffu, kind == k);
            uint64_t base = 0;
            if (lane == 0 && mk)
                base = atomicAdd((unsigned long long *)&counts[8 + k], (unsigned long long)__popc(mk));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (kind == k) dst[k][base + __popc(mk & lt)] = (uint32_t)u;
        }
    }
    local_max = __reduce_max_sync(0xffffffffu, local_max);
    if (lane == 0) atomicMax((unsigned long long *)&counts[7], (unsigned long long)local_max);
}

// Tasks: owner i of `owners` (i < *ocount) gets ceil(pcnt / L) tasks.
__global__ void k_task_count(const uint32_t *__restrict__ owners, const uint64_t *__restrict__ ocount,
                             const uint32_t *__restrict__ pcnt, uint64_t n, uint32_t L,
                             uint32_t *__restrict__ tcnt) {
    uint64_t no = *ocount;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        tcnt[i] = i < no ? (pcnt[owners[i]] + L - 1) / L : 0u;
}

__global__ void k_task_expand(const uint32_t *__restrict__ owners, const uint64_t *__restrict__ ocount,
                              const uint32_t *__restrict__ tcnt, const uint64_t *__restrict__ toff,
                              uint2 *__restrict__ tasks) {
    uint64_t no = *ocount;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < no;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x = owners[i], c = tcnt[i];
        uint64_t o = toff[i];
        for (uint32_t k = 0; k < c; k++) tasks[o + k] = make_uint2(x, k);
    }
}

static void make_tasks(Ctx &ctx, uint64_t n, uint64_t cap, const uint32_t *owners,
                       const uint64_t *ocount, const uint32_t *pcnt, uint32_t L, uint2 *&tasks,
                       uint64_t *&ntasks) {
    uint32_t *tcnt = ctx.alloc<uint32_t>(n);
    uint64_t *toff = ctx.alloc<uint64_t>(n + 1);
    int grid = ctx.persistent_grid(4);
    k_task_count<<<grid, 256, 0, ctx.stream>>>(owners, ocount, pcnt, n, L, tcnt);
    TC_LAUNCHED(ctx);
    scan_exclusive(ctx, tcnt, toff, n);
    tasks = ctx.alloc<uint2>(cap / L + n + 1);
    k_task_expand<<<grid, 256, 0, ctx.stream>>>(owners, ocount, tcnt, toff, tasks);
    TC_LAUNCHED(ctx);
    ntasks = toff + n;
}

void bin_edges(Ctx &ctx, const Oriented &g, const BinParams &p, Bins &bins) {
    uint64_t cap = g.m_cap;
    bins.cap = cap;
    bins.count = ctx.alloc<uint64_t>(16);
    TC_CUDA(cudaMemsetAsync(bins.count, 0, 16 * sizeof(uint64_t), ctx.stream));
    for (int k = 0; k < 4; k++) bins.edges[k] = ctx.alloc<uint2>(cap);
    bins.pcnt = ctx.alloc<uint32_t>(g.n + 1);
    uint32_t *cursor = ctx.alloc<uint32_t>(g.n + 1);
    TC_CUDA(cudaMemsetAsync(bins.pcnt, 0, (g.n + 1) * sizeof(uint32_t), ctx.stream));
    TC_CUDA(cudaMemsetAsync(cursor, 0, (g.n + 1) * sizeof(uint32_t), ctx.stream));
    uint32_t tiles = (uint32_t)((cap + kTileItems - 1) / kTileItems);
    if (tiles) {
        k_bin<<<tiles, kTileThreads, 0, ctx.stream>>>(g.off, g.col, g.dplus, g.n, g.m_dev, p,
                                                      bins.edges[0], bins.edges[1], bins.edges[2],
                                                      bins.edges[3], bins.pcnt, bins.count);
        TC_LAUNCHED(ctx);
    }
    bins.poff = ctx.alloc<uint64_t>(g.n + 1);
    scan_exclusive(ctx, bins.pcnt, bins.poff, g.n);
    bins.plist = ctx.alloc<uint32_t>(cap);
    k_group<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(bins.edges[3], bins.count, bins.poff,
                                                            cursor, bins.plist);
    TC_LAUNCHED(ctx);
    bins.owners_warp = ctx.alloc<uint32_t>(g.n);
    bins.owners_cta = ctx.alloc<uint32_t>(g.n);
    bins.owners_bitmap = ctx.alloc<uint32_t>(g.n);
    uint32_t cta_min = p.hub_min < kWarpTableSlots / 4 + 1 ? p.hub_min : kWarpTableSlots / 4 + 1;
    k_owners<<<ctx.persistent_grid(4), 256, 0, ctx.stream>>>(g.dplus, bins.pcnt, g.n, cta_min,
                                                             bins.owners_warp, bins.owners_cta,
                                                             bins.owners_bitmap, bins.count);
    TC_LAUNCHED(ctx);
    make_tasks(ctx, g.n, cap, bins.owners_warp, bins.count + 8, bins.pcnt, kWarpTaskLists,
               bins.tasks_warp, bins.ntasks_warp);
    make_tasks(ctx, g.n, cap, bins.owners_cta, bins.count + 9, bins.pcnt, kCtaTaskLists,
               bins.tasks_cta, bins.ntasks_cta);
    make_tasks(ctx, g.n, cap, bins.owners_bitmap, bins.count + 10, bins.pcnt, kCtaTaskLists,
               bins.tasks_bitmap, bins.ntasks_bitmap);
}

// Per-source work estimate w(u) = sum_{v in N+(u)} (1 + min(d+u, d+v)) -- the
// probe count of the HASH kernel plus one per edge -- then exclusive prefix.
__global__ void k_work(const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
                       const uint32_t *__restrict__ dplus, uint64_t n, uint64_t *__restrict__ work) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t b = off[u], e = off[u + 1];
        uint32_t du = (uint32_t)(e - b);
        uint64_t w = 0;
        for (uint64_t k = b; k < e; k++) w += 1 + min(du, dplus[col[k]]);
        work[u] = w;
    }
}

void work_prefix(Ctx &ctx, const Oriented &g, uint64_t *prefix) {
    uint64_t *work = ctx.alloc<uint64_t>(g.n);
    k_work<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(g.off, g.col, g.dplus, g.n, work);
    TC_LAUNCHED(ctx);
    scan_exclusive(ctx, work, prefix, g.n);
}

}  // namespace tc
