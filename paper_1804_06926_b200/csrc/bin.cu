// bin.cu -- a5: work estimation and binning (§4.2.2 P:527-542 "dynamic
// grouping ... divide the edge lists into groups"; third kernel P:704-708).
// Per oriented edge (u,v): a = min(d+u, d+v), b = max.  Edges that cannot close
// a triangle (d+(u) < 2 or d+(v) = 0) are skipped.  Sources with
// d+(u) >= hub_min go whole to the HASH kernel; other edges go to
// SHORT (b <= short_max), SEARCH (b >= skew_ratio * a) or MERGE.
// Multi-GPU: sources are split into `world` groups by an exclusive
// prefix of per-source work w(u) = sum_{v in N+(u)} (d+u + d+v); a rank keeps
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
          uint2 *__restrict__ b_search, uint64_t *__restrict__ counts) {
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
    uint64_t W = 0, probe = 0, skipped = 0, hashed = 0;
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
            probe += dv;
        }
        int bin = -1;
        if (valid && owner_of(p.work_prefix, chunk, u, p.world) == p.rank) {
            if (du < 2 || dv == 0) {
                skipped++;
            } else if (p.force == TC_VARIANT_HASH || (p.force < 0 && du >= p.hub_min)) {
                hashed++;
            } else if (p.force >= 0) {
                bin = p.force;
            } else {
                uint32_t a = min(du, dv), b = max(du, dv);
                if (b <= p.short_max) bin = 0;
                else if ((uint64_t)b >= (uint64_t)p.skew_ratio * a) bin = 2;
                else bin = 1;
            }
        }
        uint2 item = make_uint2(u, v);
        warp_append(bin == 0, &counts[0], b_short, item);
        warp_append(bin == 1, &counts[1], b_merge, item);
        warp_append(bin == 2, &counts[2], b_search, item);
    }
    W = block_sum_u64(W, s_red);
    probe = block_sum_u64(probe, s_red);
    skipped = block_sum_u64(skipped, s_red);
    hashed = block_sum_u64(hashed, s_red);
    if (threadIdx.x == 0) {
        atomicAdd((unsigned long long *)&counts[4], (unsigned long long)W);
        atomicAdd((unsigned long long *)&counts[5], (unsigned long long)probe);
        atomicAdd((unsigned long long *)&counts[6], (unsigned long long)skipped);
        atomicAdd((unsigned long long *)&counts[8], (unsigned long long)hashed);
    }
}

__global__ void k_hubs(const uint32_t *__restrict__ dplus, uint64_t n, BinParams p,
                       uint32_t *__restrict__ hubs, uint64_t *__restrict__ counts) {
    uint64_t chunk = 0;
    if (p.world > 1) chunk = (p.work_prefix[n] + p.world - 1) / p.world;
    uint32_t local_max = 0;
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t end = (n + 31) & ~31ull;  // keep whole warps in the loop for warp_append
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < end; u += stride) {
        bool take = false;
        if (u < n) {
            uint32_t du = dplus[u];
            local_max = max(local_max, du);
            uint32_t thr = p.force == TC_VARIANT_HASH ? 2u : p.hub_min;
            take = (p.force < 0 || p.force == TC_VARIANT_HASH) && du >= thr &&
                   owner_of(p.work_prefix, chunk, (uint32_t)u, p.world) == p.rank;
        }
        uint32_t mask = __ballot_sync(0xffffffffu, take);
        if (mask) {
            int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
            uint64_t base = 0;
            if (lane == leader)
                base = atomicAdd((unsigned long long *)&counts[3], (unsigned long long)__popc(mask));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (take) hubs[base + __popc(mask & ((1u << lane) - 1u))] = (uint32_t)u;
        }
    }
    local_max = __reduce_max_sync(0xffffffffu, local_max);
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long *)&counts[7], (unsigned long long)local_max);
}

void bin_edges(Ctx &ctx, const Oriented &g, const BinParams &p, Bins &bins) {
    uint64_t cap = g.m_cap;
    bins.cap = cap;
    bins.count = ctx.alloc<uint64_t>(16);
    TC_CUDA(cudaMemsetAsync(bins.count, 0, 16 * sizeof(uint64_t), ctx.stream));
    for (int k = 0; k < 3; k++) bins.edges[k] = ctx.alloc<uint2>(cap);
    bins.hubs = ctx.alloc<uint32_t>(g.n);
    uint32_t tiles = (uint32_t)((cap + kTileItems - 1) / kTileItems);
    if (tiles) {
        k_bin<<<tiles, kTileThreads, 0, ctx.stream>>>(g.off, g.col, g.dplus, g.n, g.m_dev, p,
                                                      bins.edges[0], bins.edges[1], bins.edges[2],
                                                      bins.count);
        TC_LAUNCHED(ctx);
    }
    k_hubs<<<ctx.persistent_grid(4), 256, 0, ctx.stream>>>(g.dplus, g.n, p, bins.hubs, bins.count);
    TC_LAUNCHED(ctx);
}

// per-source work w(u) = sum_{v in N+(u)} (d+u + d+v), then exclusive prefix.
__global__ void k_work(const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
                       const uint32_t *__restrict__ dplus, uint64_t n, uint64_t *__restrict__ work) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t b = off[u], e = off[u + 1], du = e - b, w = du * du;
        for (uint64_t k = b; k < e; k++) w += dplus[col[k]];
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
