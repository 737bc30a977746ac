// intersect.cu -- a6 + a7: batched sorted-set intersection of N+(u) and N+(v)
// for every kept edge (Alg. 2 Compute_Intersection P:345-352; "the number of
// triangles formed with e is N") and the reduction
// Count = Reduce(IntersectList) fused into each kernel: per-thread
// uint64 partials -> warp shuffle -> shared memory -> ONE atomicAdd per block.
// The IntersectList itself is never materialised.
//
// Variants (chosen per bin, §4.2.2 P:527-542 and the third kernel of P:704-708):
//   SHORT  one thread per edge, two-pointer merge           ("TwoSmall")
//   MERGE  one warp per edge, merge-path split of |A|+|B|   ("TwoLarge" with the
//          balanced path)
//   SEARCH lanes own elements of the shorter list and binary-search the longer
//          one ("scan each node in the smaller list and search the larger list",
//          P:706-707)
//   HASH   one CTA per hub source u: N+(u) staged in a shared-memory open-
//          addressing hash, every w in N+(v), v in N+(u), probed (north_star).
// Per-vertex mode (TC_PER_VERTEX): each match w of (u,v) adds 1 to t(u), t(v),
// t(w).
#include "block_scan.cuh"
#include "tc_internal.cuh"

namespace tc {

constexpr int kIxThreads = 256;

__device__ __forceinline__ void flush_count(uint64_t acc, uint64_t *total) {
    __shared__ uint64_t s_red[32];
    uint64_t t = block_sum_u64(acc, s_red);
    if (threadIdx.x == 0 && t) atomicAdd((unsigned long long *)total, (unsigned long long)t);
}

template <bool PV>
__device__ __forceinline__ void credit_edge(uint64_t *pv, uint32_t u, uint32_t v, uint32_t c) {
    if (PV && c) {
        atomicAdd((unsigned long long *)&pv[u], (unsigned long long)c);
        atomicAdd((unsigned long long *)&pv[v], (unsigned long long)c);
    }
}

// ------------------------------------------------------------------ SHORT
template <bool PV>
__global__ void __launch_bounds__(kIxThreads)
    k_short(const uint2 *__restrict__ edges, const uint64_t *__restrict__ count,
            const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
            uint64_t *__restrict__ total, uint64_t *__restrict__ pv) {
    uint64_t ne = *count;
    uint64_t acc = 0;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint2 uv = edges[e];
        uint64_t i = off[uv.x], ie = off[uv.x + 1], j = off[uv.y], je = off[uv.y + 1];
        uint32_t c = 0;
        if (i < ie && j < je) {
            uint32_t a = col[i], b = col[j];
            while (true) {
                if (a < b) {
                    if (++i == ie) break;
                    a = col[i];
                } else if (a > b) {
                    if (++j == je) break;
                    b = col[j];
                } else {
                    c++;
                    if (PV) atomicAdd((unsigned long long *)&pv[a], 1ull);
                    if (++i == ie || ++j == je) break;
                    a = col[i];
                    b = col[j];
                }
            }
        }
        credit_edge<PV>(pv, uv.x, uv.y, c);
        acc += c;
    }
    flush_count(acc, total);
}

// ------------------------------------------------------------------ MERGE
// Merge path of A (len na) and B (len nb), rule "take A[i] when A[i] <= B[j]".
// Lane l walks diagonals [k0, k1); a match is counted when A[i] is taken and
// B[j] == A[i] (B[j] is then the first element of B >= A[i]), so every common
// element is counted exactly once across lanes.
template <bool PV>
__global__ void __launch_bounds__(kIxThreads)
    k_merge(const uint2 *__restrict__ edges, const uint64_t *__restrict__ count,
            const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
            uint64_t *__restrict__ total, uint64_t *__restrict__ pv) {
    uint64_t ne = *count;
    int lane = threadIdx.x & 31;
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t acc = 0;
    for (uint64_t e = warp; e < ne; e += nwarps) {
        uint2 uv = edges[e];
        const uint32_t *A = col + off[uv.x];
        const uint32_t *B = col + off[uv.y];
        uint32_t na = (uint32_t)(off[uv.x + 1] - off[uv.x]);
        uint32_t nb = (uint32_t)(off[uv.y + 1] - off[uv.y]);
        uint32_t L = na + nb;
        uint32_t k0 = (uint32_t)(((uint64_t)L * lane) >> 5);
        uint32_t k1 = (uint32_t)(((uint64_t)L * (lane + 1)) >> 5);
        // smallest i in [lo, hi] with (i == na) || (k0-i-1 < 0) || A[i] > B[k0-i-1]
        uint32_t lo = k0 > nb ? k0 - nb : 0, hi = k0 < na ? k0 : na;
        while (lo < hi) {
            uint32_t mid = (lo + hi) >> 1;
            if (A[mid] > B[k0 - mid - 1]) hi = mid; else lo = mid + 1;
        }
        uint32_t i = lo, j = k0 - lo, c = 0;
        for (uint32_t k = k0; k < k1; k++) {
            if (j >= nb || (i < na && A[i] <= B[j])) {
                if (j < nb && A[i] == B[j]) {
                    c++;
                    if (PV) atomicAdd((unsigned long long *)&pv[A[i]], 1ull);
                }
                i++;
            } else {
                j++;
            }
        }
        if (PV) {
            uint32_t ce = __reduce_add_sync(0xffffffffu, c);
            if (lane == 0) credit_edge<PV>(pv, uv.x, uv.y, ce);
        }
        acc += c;
    }
    flush_count(acc, total);
}

// ------------------------------------------------------------------ SEARCH
template <bool PV>
__global__ void __launch_bounds__(kIxThreads)
    k_search(const uint2 *__restrict__ edges, const uint64_t *__restrict__ count,
             const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
             uint64_t *__restrict__ total, uint64_t *__restrict__ pv) {
    uint64_t ne = *count;
    int lane = threadIdx.x & 31;
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t acc = 0;
    for (uint64_t e = warp; e < ne; e += nwarps) {
        uint2 uv = edges[e];
        const uint32_t *A = col + off[uv.x];
        const uint32_t *B = col + off[uv.y];
        uint32_t na = (uint32_t)(off[uv.x + 1] - off[uv.x]);
        uint32_t nb = (uint32_t)(off[uv.y + 1] - off[uv.y]);
        if (na > nb) {  // A := the shorter list
            const uint32_t *t = A; A = B; B = t;
            uint32_t tn = na; na = nb; nb = tn;
        }
        uint32_t c = 0;
        for (uint32_t k = lane; k < na; k += 32) {
            uint32_t x = A[k], lo = 0, hi = nb;
            while (lo < hi) {
                uint32_t mid = (lo + hi) >> 1;
                if (B[mid] < x) lo = mid + 1; else hi = mid;
            }
            if (lo < nb && B[lo] == x) {
                c++;
                if (PV) atomicAdd((unsigned long long *)&pv[x], 1ull);
            }
        }
        if (PV) {
            uint32_t ce = __reduce_add_sync(0xffffffffu, c);
            if (lane == 0) credit_edge<PV>(pv, uv.x, uv.y, ce);
        }
        acc += c;
    }
    flush_count(acc, total);
}

// ------------------------------------------------------------------ HASH
constexpr uint32_t kHashSlots = 4096;  // shared-memory table capacity (power of two)
constexpr uint32_t kHashChunk = 2048;  // N+(u) elements per table build (load factor <= 1/2)
constexpr uint32_t kVChunk = 1024;     // neighbour descriptors staged per round

__device__ __forceinline__ uint32_t hash_slot(uint32_t x, int bits) {
    return (x * 0x9E3779B1u) >> (32 - bits);
}

template <bool PV>
__global__ void __launch_bounds__(kIxThreads)
    k_hash(const uint32_t *__restrict__ hubs, const uint64_t *__restrict__ count,
           const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
           uint64_t *__restrict__ total, uint64_t *__restrict__ pv) {
    __shared__ uint32_t s_table[kHashSlots];
    __shared__ uint64_t s_vstart[kVChunk];
    __shared__ uint32_t s_vid[kVChunk];
    __shared__ uint32_t s_vpre[kVChunk + 1];
    __shared__ uint32_t s_scan[kIxThreads / 32];
    __shared__ unsigned long long s_uhits;
    uint64_t nh = count[3];
    uint64_t acc = 0;
    for (uint64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        uint32_t u = hubs[h];
        uint64_t ub = off[u];
        uint32_t du = (uint32_t)(off[u + 1] - ub);
        if (PV && threadIdx.x == 0) s_uhits = 0;
        for (uint32_t c0 = 0; c0 < du; c0 += kHashChunk) {
            uint32_t clen = min(kHashChunk, du - c0);
            int bits = 6;
            while ((1u << bits) < 2 * clen) bits++;
            uint32_t tsize = 1u << bits;
            for (uint32_t s = threadIdx.x; s < tsize; s += blockDim.x) s_table[s] = kEmpty;
            __syncthreads();
            for (uint32_t k = threadIdx.x; k < clen; k += blockDim.x) {
                uint32_t x = col[ub + c0 + k], slot = hash_slot(x, bits);
                while (atomicCAS(&s_table[slot], kEmpty, x) != kEmpty) slot = (slot + 1) & (tsize - 1);
            }
            __syncthreads();
            for (uint32_t v0 = 0; v0 < du; v0 += kVChunk) {
                uint32_t vlen = min(kVChunk, du - v0);
                // stage descriptors of N+(v) for v = N+(u)[v0 .. v0+vlen) and scan lengths
                uint32_t lens[kVChunk / kIxThreads], run = 0;
#pragma unroll
                for (int q = 0; q < (int)(kVChunk / kIxThreads); q++) {
                    uint32_t i = threadIdx.x * (kVChunk / kIxThreads) + q;
                    uint32_t l = 0;
                    if (i < vlen) {
                        uint32_t v = col[ub + v0 + i];
                        uint64_t s = off[v];
                        l = (uint32_t)(off[v + 1] - s);
                        s_vstart[i] = s;
                        s_vid[i] = v;
                    }
                    lens[q] = run;
                    run += l;
                }
                uint32_t items;
                uint32_t pre = block_exclusive_scan<SumOp>(run, s_scan, &items);
#pragma unroll
                for (int q = 0; q < (int)(kVChunk / kIxThreads); q++) {
                    uint32_t i = threadIdx.x * (kVChunk / kIxThreads) + q;
                    if (i < vlen) s_vpre[i] = pre + lens[q];
                }
                if (threadIdx.x == 0) s_vpre[vlen] = items;
                __syncthreads();
                for (uint32_t t = threadIdx.x; t < items; t += blockDim.x) {
                    // list index: largest i with s_vpre[i] <= t
                    uint32_t lo = 0, hi = vlen;
                    while (hi - lo > 1) {
                        uint32_t mid = (lo + hi) >> 1;
                        if (s_vpre[mid] <= t) lo = mid; else hi = mid;
                    }
                    uint32_t w = col[s_vstart[lo] + (t - s_vpre[lo])];
                    uint32_t slot = hash_slot(w, bits);
                    while (true) {
                        uint32_t y = s_table[slot];
                        if (y == w) {
                            acc++;
                            if (PV) {
                                atomicAdd((unsigned long long *)&pv[w], 1ull);
                                atomicAdd((unsigned long long *)&pv[s_vid[lo]], 1ull);
                                atomicAdd(&s_uhits, 1ull);
                            }
                            break;
                        }
                        if (y == kEmpty) break;
                        slot = (slot + 1) & (tsize - 1);
                    }
                }
                __syncthreads();
            }
        }
        if (PV) {
            __syncthreads();
            if (threadIdx.x == 0 && s_uhits) atomicAdd((unsigned long long *)&pv[u], s_uhits);
            __syncthreads();
        }
    }
    flush_count(acc, total);
}

// ------------------------------------------------------------------ launch all
template <bool PV>
static void launch_all(Ctx &ctx, const Oriented &g, const Bins &bins, uint64_t *total,
                       uint64_t *pv) {
    int grid = ctx.persistent_grid(8);
    k_hash<PV><<<ctx.persistent_grid(4), kIxThreads, 0, ctx.stream>>>(bins.hubs, bins.count, g.off,
                                                                       g.col, total, pv);
    TC_LAUNCHED(ctx);
    k_merge<PV><<<grid, kIxThreads, 0, ctx.stream>>>(bins.edges[1], bins.count + 1, g.off, g.col,
                                                     total, pv);
    TC_LAUNCHED(ctx);
    k_search<PV><<<grid, kIxThreads, 0, ctx.stream>>>(bins.edges[2], bins.count + 2, g.off, g.col,
                                                      total, pv);
    TC_LAUNCHED(ctx);
    k_short<PV><<<grid, kIxThreads, 0, ctx.stream>>>(bins.edges[0], bins.count + 0, g.off, g.col,
                                                     total, pv);
    TC_LAUNCHED(ctx);
}

void intersect_all(Ctx &ctx, const Oriented &g, const Bins &bins, uint64_t *total_dev,
                   uint64_t *per_vertex) {
    if (per_vertex) launch_all<true>(ctx, g, bins, total_dev, per_vertex);
    else launch_all<false>(ctx, g, bins, total_dev, nullptr);
}

}  // namespace tc
