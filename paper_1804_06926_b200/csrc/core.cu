// core.cu -- a6 + a7 for the DENSE CORE: word-parallel intersection of adjacency bitmaps.
//
// After the rank relabelling (orient.cu) the highest-ranked vertices -- the highest
// degrees -- are the last ids, and their mutual adjacency is dense (R-MAT / power-law hubs
// form a dense core).  For an oriented edge (u, x), u < x, the triangles it closes are
// w in N+(u) with w > x and w in N+(x) (the forward algorithm, Alg. 2 Compute_Intersection
// P:345-352, "the number of triangles formed with e is N"); if u lies in the core
// [core_lo, n) then so do x and every w.  So with one bitmap per core vertex y -- bit
// (z - core_lo) set iff z in N+(y) -- the count is
//
//     c(u, x) = sum over words k in [w0, w1] of popc(B_u[k] & B_x[k])
//
// over the words covering (x, min(last N+(u), last N+(x))] (B_x has no bit <= x, so the
// AND needs no mask).  That costs w1 - w0 + 1 word operations instead of min(suf, d+x)
// shared-memory probes (intersect.cu HASH); binning (bin.cu) sends an edge here when its
// word count is at most its probe count (core_edge, tc_internal.cuh).  Only the plain
// count uses it (per-vertex / edge / list credits need the individual matches).
//
// Layout: K = core_words * 32 core ids (the top K ranks, K = 16384 or 32768 below / from 2^23
// vertices, at most n rounded up to 128), row r = vertex core_lo + r, words [0, core_words)
// each (K^2 / 8 bytes: 32 MB at K = 16384, L2-resident); only the words a row can ever be
// read at -- from the 16-byte group holding its own vertex's word on -- are written (about
// half).  core_info[r] = (first, last element, d+) of N+(core_lo + r) bounds the word range
// of every core edge.  The paper has no such path (its kernels merge or
// binary-search); this is the B200-first replacement of its "TwoLarge"
// kernel for the densest lists.
#include "tc_internal.cuh"

namespace tc {

#ifndef TC_CORE_MAX
#define TC_CORE_MAX 32768
#endif
#ifndef TC_CORE_SMALL
#define TC_CORE_SMALL 16384
#endif
// core ids K (multiple of 128): TC_CORE_SMALL below 2^23 vertices (the core bitmaps stay
// L2-resident next to the rest of the a6 working set), TC_CORE_MAX from there on (measured:
// s21 16384 vs 32768 equal, s24 32768 -1.4 ms)
constexpr uint32_t kCoreMax = TC_CORE_MAX;
constexpr uint32_t kCoreMaxWords = kCoreMax / 32;
static_assert(kCoreMax % 128 == 0 && TC_CORE_SMALL % 128 == 0 && TC_CORE_SMALL <= kCoreMax,
              "rows are read as 16-byte groups");
constexpr int kCoreBuildWarps = 8;

// One warp per core vertex y: its row is assembled in shared memory (zero, set the bits of
// N+(y) with shared atomics) and stored from y's own word on, 16 bytes per lane.
__global__ void __launch_bounds__(kCoreBuildWarps * 32)
    k_core_build(const uint64_t *__restrict__ off, const uint32_t *__restrict__ col, uint32_t n,
                 uint32_t core_lo, uint32_t words, uint32_t *__restrict__ bm,
                 uint4 *__restrict__ info) {
    __shared__ __align__(16) uint32_t s_row[kCoreBuildWarps][kCoreMaxWords];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t *row = s_row[wib];
    for (uint32_t y = core_lo + blockIdx.x * kCoreBuildWarps + wib; y < n;
         y += gridDim.x * kCoreBuildWarps) {
        const uint32_t w_first = ((y - core_lo) >> 5) & ~3u;   // 16-byte aligned start
        for (uint32_t k = w_first + lane; k < words; k += 32) row[k] = 0u;
        __syncwarp();
        const uint64_t b = off[y], e = off[y + 1];
        if (lane == 0)
            info[y - core_lo] = e > b ? make_uint4(col[b], col[e - 1], (uint32_t)(e - b), 0u)
                                      : make_uint4(~0u, 0u, 0u, 0u);
        for (uint64_t k = b + lane; k < e; k += 32) {
            const uint32_t o = col[k] - core_lo;
            atomicOr(&row[o >> 5], 1u << (o & 31));
        }
        __syncwarp();
        uint4 *dst = reinterpret_cast<uint4 *>(bm + (uint64_t)(y - core_lo) * words);
        const uint4 *src = reinterpret_cast<const uint4 *>(row);
        for (uint32_t q = (w_first >> 2) + lane; q < (words >> 2); q += 32) dst[q] = src[q];
        __syncwarp();
    }
}

// One CTA per core source u (grid-strided; the longest rows, just above core_lo, come first,
// so every CTA starts with one of them): B_u is staged in shared memory once, then groups of
// 8 lanes take the edges (u, x) of its row that binning sent here -- the HASH-bin edges of a
// core source (bin.cu) -- and AND B_u with B_x (from L2) over the words covering the common
// range [max(next, first(x)), min(last(u), last(x))]; an empty range closes no triangle.
#ifndef TC_CORE_GROUP
#define TC_CORE_GROUP 4   // measured s21 ix: 2 2.35, 4 2.29, 8 2.41, 16 2.68 ms
#endif
constexpr int kCoreGroup = TC_CORE_GROUP;   // lanes per core edge
__global__ void __launch_bounds__(256)
    k_core_count(HashParams hp, const uint64_t *__restrict__ m_dev, uint64_t *__restrict__ total,
                 uint64_t *__restrict__ words_out) {
    __shared__ __align__(16) uint32_t s_bu[kCoreMaxWords];
    __shared__ uint64_t s_red[32];
    const uint64_t m = *m_dev;
    const uint32_t gl = threadIdx.x % kCoreGroup, grp = threadIdx.x / kCoreGroup;
    constexpr uint32_t kGroups = 256 / kCoreGroup;
    uint64_t acc = 0, words = 0;
    for (uint32_t u = hp.core_lo + blockIdx.x; u < hp.n; u += gridDim.x) {
        const uint64_t ub = hp.off[u], ue = hp.off[u + 1];
        if (ue - ub < 2) continue;   // block-uniform: a single edge has no suffix
        __syncthreads();             // the previous row's B_u is no longer read
        const uint4 *src = reinterpret_cast<const uint4 *>(hp.core + (uint64_t)(u - hp.core_lo) * hp.core_words);
        uint4 *dst = reinterpret_cast<uint4 *>(s_bu);
        for (uint32_t q = ((u - hp.core_lo) >> 7) + threadIdx.x; q < (hp.core_words >> 2); q += 256)
            dst[q] = __ldg(src + q);
        __syncthreads();
        const uint32_t du = (uint32_t)(ue - ub), last_u = hp.core_info[u - hp.core_lo].y;
        // the next edge's target is loaded one iteration ahead (the chain per edge is then
        // core_info[x] -> B_x words)
        uint64_t e = ub + grp;
        uint32_t x_next = e + 1 < ue ? hp.col[e] : 0u;
        for (; e + 1 < ue; e += kGroups) {
            const uint32_t x = x_next, nxt = hp.col[e + 1];
            x_next = e + kGroups + 1 < ue ? hp.col[e + kGroups] : 0u;
            if (hp.world > 1 && edge_rank(e, hp.world) != hp.rank) continue;
            const uint4 rx = hp.core_info[x - hp.core_lo];   // first, last, d+ of x
            const uint32_t suf = (uint32_t)(ue - e - 1);
            if (edge_bin(hp, du, rx.z, suf) != TC_VARIANT_HASH) continue;
            const uint32_t lo = max(nxt, rx.x), hi = min(last_u, rx.y);
            if (hi < lo) continue;
            const uint32_t w0 = (lo - hp.core_lo) >> 5, w1 = (hi - hp.core_lo) >> 5;
            if (gl == 0) words += w1 - w0 + 1;
            // 16-byte groups from w0 & ~3: row x is written from its 16-byte group holding x's
            // own word on (k_core_build), and its words below w0 cover ids <= x, so they are 0
            const uint4 *bx = reinterpret_cast<const uint4 *>(hp.core + (uint64_t)(x - hp.core_lo) * hp.core_words);
            for (uint32_t q = (w0 >> 2) + gl; q <= (w1 >> 2); q += kCoreGroup) {
                const uint4 a = dst[q], b = __ldg(bx + q);
                acc += __popc(a.x & b.x) + __popc(a.y & b.y) + __popc(a.z & b.z) + __popc(a.w & b.w);
            }
        }
    }
    const uint64_t t = block_sum_u64(acc, s_red);
    const uint64_t wsum = block_sum_u64(words, s_red);
    if (threadIdx.x == 0 && t) atomicAdd((unsigned long long *)total, (unsigned long long)t);
    if (threadIdx.x == 0 && wsum) atomicAdd((unsigned long long *)words_out, (unsigned long long)wsum);
    (void)m;
}

// Core size K and first core rank id: the top K = 16384 ranks below 2^23 vertices, 32768
// from there on (rounded to whole 128-id groups for small n).
static uint32_t core_size(uint32_t n) {
    const uint32_t cap = n < (1u << 23) ? TC_CORE_SMALL : kCoreMax;
    return (uint32_t)std::min<uint64_t>(cap, ((uint64_t)n + 127) / 128 * 128);
}
uint32_t core_first(uint64_t n) {
    const uint32_t K = core_size((uint32_t)n);
    return n > K ? (uint32_t)n - K : 0u;
}

void core_build(Ctx &ctx, const Oriented &g, HashParams &hp) {
    hp.core = nullptr;
    const uint32_t n = (uint32_t)g.n;
    if (n == 0) return;
    const uint32_t K = core_size(n);
    hp.core_lo = core_first(n);
    hp.core_words = K / 32;
    uint32_t *bm = ctx.alloc<uint32_t>((uint64_t)K * hp.core_words);
    uint4 *info = ctx.alloc<uint4>(K);
    const uint32_t rows = n - hp.core_lo;
    const uint32_t grid = std::min<uint32_t>((rows + kCoreBuildWarps - 1) / kCoreBuildWarps,
                                             (uint32_t)ctx.persistent_grid(4));
    k_core_build<<<grid, kCoreBuildWarps * 32, 0, ctx.stream>>>(g.off, g.col, n, hp.core_lo,
                                                                 hp.core_words, bm, info);
    TC_LAUNCHED(ctx);
    hp.core = bm;
    hp.core_info = info;
}

void core_count(Ctx &ctx, const Oriented &g, const HashParams &hp, uint64_t *total_dev,
                uint64_t *words_dev, cudaStream_t stream) {
    if (!hp.core) return;
    const uint32_t rows = (uint32_t)g.n - hp.core_lo;
    const uint32_t grid = std::min<uint32_t>(rows, (uint32_t)ctx.persistent_grid(8));
    k_core_count<<<grid, 256, 0, stream>>>(hp, g.m_dev, total_dev, words_dev);
    TC_LAUNCHED(ctx);
}

}  // namespace tc
