// prune.cu -- NEXT-2: leaf pruning before orientation (TC_PRUNE).
//
// The paper's filtering stage drops what cannot be in a triangle: "nodes with
// degree less than two cannot be matched [to] any query vertex, since every node in
// a triangle has a degree of two"; the non-candidate edges are
// filtered out, the graph is "reconstruct[ed] ... updat[ing] node degree ... for a
// few iterations in order to prune out more edges".  One round deletes
// every edge with an endpoint of degree < 2 in the current graph.
//
// B200 formulation: no per-round compaction.  With G_0 the cleaned graph and d_i
// the degrees of G_i, the edges of G_{i+1} are exactly the edges of G_0 whose two
// endpoints have d_i >= 2 (alive sets are nested), so
//     d_{i+1}(v) = [d_i(v) >= 2] * #{w in N_0(v) : d_i(w) >= 2},
// one streaming pass over the ORIGINAL edge list per round (degree gathers are
// L2-resident), and |E(G_{i+1})| falls out of the same pass.  After the last round
// an edge survives iff both final degrees are > 0 (d_k(v) > 0 implies v alive in
// round k-1, and an alive endpoint pair keeps the edge), so one compaction (dirty
// input) or a degree test inside the orientation filter (clean input) finishes.
// rounds = 0 runs until a round deletes nothing (the 2-core), reading one 8-byte
// counter per round back to the host.
#include "block_scan.cuh"
#include "tc_internal.cuh"

namespace tc {

// Warp-aggregated degree increment: lanes with `live` add 1 to cnt[key]; lanes
// sharing a key issue one atomic.
__device__ __forceinline__ void add_degree(bool live, uint32_t key, uint32_t *cnt) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t peers = __match_any_sync(0xffffffffu, live ? key : 0xffffffffu);
    if (live && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&cnt[key], (uint32_t)__popc(peers));
}

// One round on the undirected edge list E (keys (min << b) | max, sorted).
__global__ void k_prune_pairs(const uint64_t *__restrict__ E, const uint64_t *__restrict__ m_dev, int b,
                              const uint32_t *__restrict__ dcur, uint32_t *__restrict__ dnext,
                              uint64_t *__restrict__ live_edges) {
    __shared__ uint64_t s_red[32];
    uint64_t m = *m_dev, mask = (1ull << b) - 1;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t live_n = 0;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < m; i0 += stride) {
        uint64_t i = i0 + threadIdx.x;
        bool live = false;
        uint32_t a = 0, c = 0;
        if (i < m) {
            uint64_t k = E[i];
            a = (uint32_t)(k >> b);
            c = (uint32_t)(k & mask);
            live = dcur[a] >= 2 && dcur[c] >= 2;
        }
        live_n += live;
        add_degree(live, a, dnext);   // runs of one min: one atomic per run
        if (live) atomicAdd(&dnext[c], 1u);
    }
    live_n = block_sum_u64(live_n, s_red);
    if (threadIdx.x == 0 && live_n) atomicAdd((unsigned long long *)live_edges, (unsigned long long)live_n);
}

// One round on a clean symmetric CSR (each edge twice): counts live ARCS.
__global__ void __launch_bounds__(kTileThreads)
    k_prune_csr(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col, uint64_t n,
                uint64_t M, const uint32_t *__restrict__ dcur, uint32_t *__restrict__ dnext,
                uint64_t *__restrict__ live_arcs) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    __shared__ uint64_t s_red[32];
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
    tile_rows(rowptr, n, t0, len, s_row, s_scan);
    uint64_t live_n = 0;
    for (uint32_t i = threadIdx.x; i < kTileItems; i += kTileThreads) {  // whole warps
        bool live = false;
        uint32_t u = 0;
        if (i < len) {
            u = s_row[i];
            live = dcur[u] >= 2 && dcur[col[t0 + i]] >= 2;
        }
        live_n += live;
        add_degree(live, u, dnext);
    }
    live_n = block_sum_u64(live_n, s_red);
    if (threadIdx.x == 0 && live_n) atomicAdd((unsigned long long *)live_arcs, (unsigned long long)live_n);
}

// Compaction of E to the edges whose endpoints both have degree > 0.
__device__ __forceinline__ uint32_t survives(const uint64_t *__restrict__ E, uint64_t i, int b,
                                             const uint32_t *__restrict__ deg) {
    uint64_t k = E[i];
    return deg[k >> b] > 0 && deg[k & ((1ull << b) - 1)] > 0;
}

__global__ void __launch_bounds__(kTileThreads)
    k_survive_count(const uint64_t *__restrict__ E, const uint64_t *__restrict__ m_dev, int b,
                    const uint32_t *__restrict__ deg, uint32_t *__restrict__ counts) {
    __shared__ uint64_t s_red[32];
    uint64_t m = *m_dev, t0 = (uint64_t)blockIdx.x * kTileItems, c = 0;
    for (int k = 0; k < kItemsPerThread; k++) {
        uint64_t i = t0 + (uint64_t)k * kTileThreads + threadIdx.x;
        if (i < m) c += survives(E, i, b, deg);
    }
    c = block_sum_u64(c, s_red);
    if (threadIdx.x == 0) counts[blockIdx.x] = (uint32_t)c;
}

__global__ void __launch_bounds__(kTileThreads)
    k_survive_scatter(const uint64_t *__restrict__ E, const uint64_t *__restrict__ m_dev, int b,
                      const uint32_t *__restrict__ deg, const uint64_t *__restrict__ offs,
                      uint64_t *__restrict__ out) {
    __shared__ uint32_t s_scan[kTileThreads / 32];
    uint64_t m = *m_dev;
    uint64_t base = (uint64_t)blockIdx.x * kTileItems + (uint64_t)threadIdx.x * kItemsPerThread;
    uint32_t f[kItemsPerThread], c = 0;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        f[k] = base + k < m ? survives(E, base + k, b, deg) : 0u;
        c += f[k];
    }
    uint32_t pos = block_exclusive_scan<SumOp>(c, s_scan);
    uint64_t o = offs[blockIdx.x] + pos;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++)
        if (f[k]) out[o++] = E[base + k];
}

// Shared round driver.  `step(dcur, dnext, live)` launches one round; `initial` is
// the live count before round 1 (host value, needed only in fixed-point mode) and
// `live_div` converts the kernel's count to edges.  Returns the final degree buffer.
template <class Step>
static uint32_t *run_rounds(Ctx &ctx, uint64_t n, uint32_t *deg, uint32_t rounds, uint64_t initial,
                            Step step, PruneInfo &info) {
    // fixed-point mode can need many rounds (a path of length L takes L/2): bound by n+1
    const uint64_t max_rounds = rounds ? rounds : n + 1;
    uint64_t *live = ctx.alloc<uint64_t>(max_rounds < 4096 ? max_rounds : 4096);
    uint32_t *dcur = deg, *dnext = ctx.alloc<uint32_t>(n);
    uint64_t prev = initial, r = 0;
    uint64_t *pin = nullptr;
    if (!rounds) TC_CUDA(cudaMallocHost((void **)&pin, sizeof(uint64_t)));
    struct PinFree {
        uint64_t *p;
        ~PinFree() { if (p) cudaFreeHost(p); }
    } pin_free{pin};
    while (r < max_rounds) {
        uint64_t *lc = live + (r % 4096);
        TC_CUDA(cudaMemsetAsync(dnext, 0, n * sizeof(uint32_t), ctx.stream));
        TC_CUDA(cudaMemsetAsync(lc, 0, sizeof(uint64_t), ctx.stream));
        step(dcur, dnext, lc);
        uint32_t *t = dcur;
        dcur = dnext;
        dnext = t;
        r++;
        if (!rounds) {  // one 8-byte read per round: stop when nothing was deleted
            TC_CUDA(cudaMemcpyAsync(pin, lc, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
            TC_CUDA(cudaStreamSynchronize(ctx.stream));
            uint64_t now = *pin;
            if (now == prev) break;
            prev = now;
        }
    }
    info.rounds = r;
    return dcur;
}

void prune_pairs(Ctx &ctx, uint64_t n, int b, uint32_t rounds, uint64_t *&E, uint64_t *&m_dev,
                 uint32_t *&deg, uint64_t m_host_cap, PruneInfo &info) {
    uint64_t m0 = 0;
    if (!rounds) {
        TC_CUDA(cudaMemcpyAsync(&m0, m_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
        TC_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    const uint64_t *Ec = E, *mc = m_dev;
    int grid = ctx.persistent_grid(8);
    deg = run_rounds(ctx, n, deg, rounds, m0,
                     [&](const uint32_t *dcur, uint32_t *dnext, uint64_t *live) {
                         k_prune_pairs<<<grid, 256, 0, ctx.stream>>>(Ec, mc, b, dcur, dnext, live);
                         TC_LAUNCHED(ctx);
                     },
                     info);
    // compact E to the surviving edges
    uint32_t tiles = (uint32_t)((m_host_cap + kTileItems - 1) / kTileItems);
    uint32_t *counts = ctx.alloc<uint32_t>(tiles + 1);
    uint64_t *offs = ctx.alloc<uint64_t>(tiles + 1);
    uint64_t *out = ctx.alloc<uint64_t>(m_host_cap);
    if (tiles) {
        k_survive_count<<<tiles, kTileThreads, 0, ctx.stream>>>(E, m_dev, b, deg, counts);
        TC_LAUNCHED(ctx);
    }
    scan_exclusive(ctx, counts, offs, tiles);
    if (tiles) {
        k_survive_scatter<<<tiles, kTileThreads, 0, ctx.stream>>>(E, m_dev, b, deg, offs, out);
        TC_LAUNCHED(ctx);
    }
    info.m_before = m_dev;
    E = out;
    m_dev = offs + tiles;
}

void prune_csr(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
               uint32_t rounds, uint32_t *&deg, PruneInfo &info) {
    uint32_t tiles = (uint32_t)((M + kTileItems - 1) / kTileItems);
    deg = run_rounds(ctx, n, deg, rounds, M,
                     [&](const uint32_t *dcur, uint32_t *dnext, uint64_t *live) {
                         k_prune_csr<<<tiles, kTileThreads, 0, ctx.stream>>>(rowptr, col, n, M, dcur,
                                                                            dnext, live);
                         TC_LAUNCHED(ctx);
                     },
                     info);
}

}  // namespace tc
