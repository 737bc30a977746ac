// shard.cu -- multi-GPU with a2-a5 SHARDED over the ranks (north_star: "the edge
// range is split by a prefix sum over estimated intersection work, followed by one NCCL
// allreduce"), round 2.  After the sharded cleaning step (tc_clean_shard: rank r holds the
// unique edges whose smaller endpoint is r mod G, and the degrees are all-reduced) nothing is
// repeated on every rank except n-sized passes:
//
//   P1 tc_shard_orient     rank relabelling (n-sized, replicated), the rank's OWN edges
//                          oriented low -> high rank -> pairs, d+ partials
//      [all-reduce d+]
//   P2 tc_shard_partition  off+ = scan(d+) (replicated); source-row ranges R_q holding m/G
//                          pairs each; the rank's pairs grouped by the range of their source
//      [all-to-all pairs]
//   P3 tc_shard_rows       the received pairs (rows [R_r, R_r+1)) sorted (target, then
//                          source: LSD) -> that slice of col+, rows ascending (a3 + a4)
//      [all-gather col+ slices: every rank holds the whole oriented CSR, as the probes of a6
//       read any N+(u)]
//   P4 tc_shard_work       the slice's edges classified (a5: skip / SHORT / SEARCH / dense
//                          core / HASH in-part of owner x / out-part of owner u) -> per-owner
//                          probe entries and probe lengths (partials)
//      [all-reduce entries, lengths]
//   P5 tc_shard_route      owner work w(x) (replicated, the single-GPU owner split's model),
//                          its exclusive prefix, owner x -> rank split_rank(prefix); the
//                          slice's HASH entries grouped by the owner's rank
//      [all-to-all entries]
//   P6 tc_shard_count      in-lists / out-part lists of the rank's owners from the received
//                          entries, owner classes, tasks; the slice's SHORT / SEARCH edges;
//                          the dense core by interleaved 2048-edge blocks (core.cu); a6 + a7
//      [all-reduce the count]
//
// Every edge is classified by exactly one rank (the one whose row range holds its source),
// every HASH owner's table is built on exactly one rank, so the partials sum to tc_count's
// total.  The collectives are the caller's (paper_1804_06926_b200/dist.py: NCCL); the phases
// are synchronous and exchange only through caller-owned device buffers.
#include <algorithm>

#include "block_scan.cuh"
#include "tc_internal.cuh"

namespace tc {

static int sh_id_bits(uint64_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) b++;
    return b;
}

// Destination of id v under bounds b[0..G] (b[0] = 0, b[G] = n): the q with b[q] <= v < b[q+1].
__device__ __forceinline__ int range_of(const uint32_t *b, int G, uint32_t v) {
    int lo = 0, hi = G;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (b[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

// ------------------------------------------------------------------ P1
__global__ void k_shard_orient(const uint64_t *__restrict__ E, uint64_t m, int b,
                               const uint32_t *__restrict__ newid, uint32_t *__restrict__ src,
                               uint32_t *__restrict__ dst, uint32_t *__restrict__ dplus) {
    const uint64_t mask = (1ull << b) - 1;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < m; i0 += stride) {
        const uint64_t i = i0 + threadIdx.x;
        uint32_t s = 0xffffffffu;
        if (i < m) {
            const uint64_t k = E[i];
            const uint32_t a = newid[k >> b], c = newid[k & mask];
            s = min(a, c);
            src[i] = s;
            dst[i] = max(a, c);
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, s);
        if (i < m && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&dplus[s], (uint32_t)__popc(peers));
    }
}

// ------------------------------------------------------------------ P2
// bounds[q] = first x with prefix[x] >= ceil(q * total / G) (q = 0..G; bounds[G] = n).
__global__ void k_split_bounds(const uint64_t *__restrict__ prefix, uint64_t n, int G,
                               uint32_t *__restrict__ bounds) {
    const int q = threadIdx.x;
    if (q > G) return;
    const uint64_t total = prefix[n];
    if (q == 0) {
        bounds[0] = 0;
        return;
    }
    if (q == G) {
        bounds[G] = (uint32_t)n;
        return;
    }
    const uint64_t target = (total * (uint64_t)q + G - 1) / G;
    uint64_t lo = 0, hi = n;   // first x in [0, n] with prefix[x] >= target
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (prefix[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    bounds[q] = (uint32_t)lo;
}

// Pairs grouped by the range of their source: per-block counts per destination, one atomic
// per (block, destination) for the block's run, then the writes.  count pass: cur == nullptr.
constexpr int kMaxWorld = 64;
__global__ void __launch_bounds__(256)
    k_part_pairs(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst, uint64_t m,
                 const uint32_t *__restrict__ bounds, int G, unsigned long long *__restrict__ cnt,
                 unsigned long long *__restrict__ cur, const uint64_t *__restrict__ base,
                 uint64_t *__restrict__ out) {
    __shared__ uint32_t s_b[kMaxWorld + 1];
    __shared__ uint32_t s_c[kMaxWorld];
    __shared__ unsigned long long s_o[kMaxWorld];
    for (int q = threadIdx.x; q <= G; q += blockDim.x) s_b[q] = bounds[q];
    const uint64_t per = (m + gridDim.x - 1) / gridDim.x;
    const uint64_t i0 = (uint64_t)blockIdx.x * per, i1 = min(m, i0 + per);
    for (uint64_t c0 = i0; c0 < i1; c0 += 256 * 8) {
        for (int q = threadIdx.x; q < G; q += blockDim.x) s_c[q] = 0;
        __syncthreads();
        int d[8];
        uint32_t slot[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint64_t i = c0 + (uint64_t)k * 256 + threadIdx.x;
            d[k] = -1;
            if (i < i1) {
                d[k] = range_of(s_b, G, src[i]);
                slot[k] = atomicAdd(&s_c[d[k]], 1u);
            }
        }
        __syncthreads();
        for (int q = threadIdx.x; q < G; q += blockDim.x)
            if (s_c[q]) {
                if (cur) s_o[q] = base[q] + atomicAdd(&cur[q], (unsigned long long)s_c[q]);
                else atomicAdd(&cnt[q], (unsigned long long)s_c[q]);
            }
        __syncthreads();
        if (cur) {
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (d[k] >= 0) {
                    const uint64_t i = c0 + (uint64_t)k * 256 + threadIdx.x;
                    out[s_o[d[k]] + slot[k]] = ((uint64_t)dst[i] << 32) | src[i];
                }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ P3
__global__ void k_unpack_pairs(const uint64_t *__restrict__ p, uint64_t m, uint32_t *__restrict__ s,
                               uint32_t *__restrict__ t) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = p[i];
        s[i] = (uint32_t)v;
        t[i] = (uint32_t)(v >> 32);
    }
}

// ------------------------------------------------------------------ P4 / P5 / P6: the slice
// Edge e = (u -> x) of the global CSR (rows ascending), classified as k_edges does (bin.cu).
enum SliceKind { kSkip = 0, kShort, kSearch, kCoreEdge, kHashIn, kHashOut };
struct SliceParams {
    HashParams hp;       // off, col, dplus, n, short_max, skew_ratio, force (-1)
    bool core = false;   // count mode: HASH edges of core sources go to core.cu
    uint32_t core_lo = 0;
};
__device__ __forceinline__ int slice_kind(const SliceParams &sp, uint32_t u, uint32_t du, uint32_t dv,
                                          uint32_t suf) {
    const int bin = edge_bin(sp.hp, du, dv, suf);
    if (bin < 0) return kSkip;
    if (bin == TC_VARIANT_SHORT) return kShort;
    if (bin == TC_VARIANT_SEARCH) return kSearch;
    if (sp.core && u >= sp.core_lo) return kCoreEdge;
    return suf <= dv && suf <= kSufMax ? kHashIn : kHashOut;
}

// mode 0 (P4): per owner, HASH probe entries (cnt) and probe lengths (len), atomics.
// mode 1 (P5, count pass / write pass): HASH entries to the owner's rank.
// mode 2 (P6): SHORT / SEARCH edges appended to their bins.
template <int kMode>
__global__ void __launch_bounds__(kTileThreads)
    k_slice(SliceParams sp, uint64_t e0, uint64_t e1, uint32_t *__restrict__ cnt,
            unsigned long long *__restrict__ len, const uint64_t *__restrict__ wprefix, int G, int self_rank,
            unsigned long long *__restrict__ dcnt, unsigned long long *__restrict__ dcur,
            const uint64_t *__restrict__ dbase, uint32_t *__restrict__ ent, uint2 *__restrict__ b_short,
            uint2 *__restrict__ b_search, uint64_t *__restrict__ counts) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    __shared__ uint32_t s_c[kMaxWorld];
    __shared__ unsigned long long s_o[kMaxWorld];
    const HashParams &hp = sp.hp;
    const uint64_t t0 = e0 + (uint64_t)blockIdx.x * kTileItems;
    if (t0 >= e1) return;
    const uint32_t len_t = (uint32_t)min((uint64_t)kTileItems, e1 - t0);
    tile_rows(hp.off, hp.n, t0, len_t, s_row, s_scan);
    if (kMode == 1) {
        for (int q = threadIdx.x; q < G; q += blockDim.x) s_c[q] = 0;
        __syncthreads();
    }
    const uint64_t wtot = kMode == 1 ? wprefix[hp.n] : 0;
    int dq[kItemsPerThread];
    uint32_t slot[kItemsPerThread], own[kItemsPerThread], oth[kItemsPerThread], ee[kItemsPerThread];
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        dq[k] = -1;
        const uint32_t i = k * kTileThreads + threadIdx.x;   // striped: coalesced col+ loads
        if (i >= len_t) continue;
        const uint64_t e = t0 + i;
        const uint32_t u = s_row[i], x = hp.col[e];
        const uint64_t ub = hp.off[u], ue = hp.off[u + 1];
        const uint32_t du = (uint32_t)(ue - ub), dv = hp.dplus[x], suf = (uint32_t)(ue - e - 1);
        const int kind = slice_kind(sp, u, du, dv, suf);
        if (kMode == 0) {
            if (kind == kHashIn) {
                atomicAdd(&cnt[x], 1u);
                atomicAdd(&len[x], (unsigned long long)suf);
            } else if (kind == kHashOut) {
                atomicAdd(&cnt[u], 1u);
                atomicAdd(&len[u], (unsigned long long)dv);
            }
        } else if (kMode == 1) {
            if (kind == kHashIn || kind == kHashOut) {
                const uint32_t o = kind == kHashIn ? x : u;
                own[k] = o;
                oth[k] = kind == kHashIn ? u : x;
                ee[k] = (uint32_t)e | (kind == kHashOut ? 0x80000000u : 0u);
                dq[k] = split_rank(wprefix[o], wtot, G);
                slot[k] = atomicAdd(&s_c[dq[k]], 1u);
            } else if (kind == kShort || kind == kSearch) {   // per-edge bins stay on this rank
                own[k] = u | 0x80000000u;
                oth[k] = x;
                ee[k] = (uint32_t)e | (kind == kSearch ? 0x80000000u : 0u);
                dq[k] = self_rank;
                slot[k] = atomicAdd(&s_c[dq[k]], 1u);
            }
        } else {
            if (kind == kShort) {
                const unsigned long long p = atomicAdd((unsigned long long *)&counts[0], 1ull);
                b_short[p] = make_uint2(u, x);
            } else if (kind == kSearch) {
                const unsigned long long p = atomicAdd((unsigned long long *)&counts[2], 1ull);
                b_search[p] = make_uint2(u, x);
            }
        }
    }
    if (kMode == 1) {
        __syncthreads();
        for (int q = threadIdx.x; q < G; q += blockDim.x)
            if (s_c[q]) {
                if (dcur) s_o[q] = dbase[q] + atomicAdd(&dcur[q], (unsigned long long)s_c[q]);
                else atomicAdd(&dcnt[q], (unsigned long long)s_c[q]);
            }
        __syncthreads();
        if (dcur) {
#pragma unroll
            for (int k = 0; k < kItemsPerThread; k++)
                if (dq[k] >= 0) {
                    uint32_t *p = ent + 3 * (s_o[dq[k]] + slot[k]);
                    p[0] = own[k];
                    p[1] = oth[k];
                    p[2] = ee[k];
                }
        }
    }
}

// Rank span last - first + 1 of N+(x) for the rows x in [r0, r1) (0 elsewhere: all-reduced by
// summation), so the owner work needs no remote rows of col+.
__global__ void k_row_spans(const uint64_t *__restrict__ off, const uint32_t *__restrict__ col, uint64_t r0,
                            uint64_t r1, uint32_t *__restrict__ spans) {
    for (uint64_t x = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < r1;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = off[x], b = off[x + 1];
        spans[x] = b > a ? col[b - 1] - col[a] + 1 : 0u;
    }
}

// Owner work w(x) from its HASH entries c and their probe lengths l: the single-GPU owner
// split's model (bin.cu k_owner_work: a fixed cost per entry, class weights, table builds).
#ifndef TC_SHARD_ENTRY_COST
#define TC_SHARD_ENTRY_COST 64
#endif
#ifndef TC_SHARD_HASH_WEIGHT
#define TC_SHARD_HASH_WEIGHT 3
#endif
#ifndef TC_SHARD_WARP_WEIGHT
#define TC_SHARD_WARP_WEIGHT 2
#endif
__global__ void k_shard_owner_work(const uint32_t *__restrict__ cnt, const unsigned long long *__restrict__ len,
                                   const uint32_t *__restrict__ spans, const uint32_t *__restrict__ dplus,
                                   uint64_t n, uint32_t cta_min, uint64_t *__restrict__ work) {
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = cnt[x], du = dplus[x];
        uint64_t w = 0;
        if (c) {
            w = (uint64_t)c * TC_SHARD_ENTRY_COST + len[x];
            if (du < cta_min) {
                w = w * TC_SHARD_WARP_WEIGHT + (uint64_t)((c + kWarpTaskLists - 1) / kWarpTaskLists) * du;
            } else {
                const uint64_t span = spans[x];
                const bool bitmap = span + 32 <= kCtaBitmapBits;
                if (!bitmap) w *= TC_SHARD_HASH_WEIGHT;
                w += (uint64_t)((c + kCtaTaskLists - 1) / kCtaTaskLists) * (du + (bitmap ? span / 32 : 0));
            }
        }
        work[x] = w;
    }
}

// ------------------------------------------------------------------ P6: owner structures
// Received entries grouped by a stable radix sort of key = out-part flag << b | owner (no
// per-owner atomics: a hub owner receives up to 10^6 entries): in-part entries first, by
// owner, then the out-part entries, by owner.
// Classes: 0 HASH in-part, 1 HASH out-part (flag in bit 31 of the CSR index), 2 SHORT edge,
// 3 SEARCH edge (bit 31 of the owner field marks the per-edge bins; owner = u, other = x).
__global__ void k_ent_keys(const uint32_t *__restrict__ ent, uint64_t k, int b, uint32_t *__restrict__ key) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t o = ent[3 * i], cls = (o >> 31) * 2 + (ent[3 * i + 2] >> 31);
        key[i] = (o & 0x7fffffffu) | (cls << b);
    }
}

// Entries per owner (icnt: class 0, ocnt: class 1) from the runs of the sorted keys (two
// atomics per run, each on its own owner's counter).
__global__ void k_ent_runs(const uint32_t *__restrict__ key, uint64_t k, int b, uint32_t *__restrict__ icnt,
                           uint32_t *__restrict__ ocnt) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = key[i], cls = x >> b;
        if (cls >= 2) continue;
        const uint32_t o = x & ((1u << b) - 1u);
        uint32_t *c = cls ? ocnt : icnt;
        if (i + 1 == k || key[i + 1] != x) atomicAdd(&c[o], (uint32_t)(i + 1));
        if (i == 0 || key[i - 1] != x) atomicSub(&c[o], (uint32_t)i);
    }
}

// Entries per class: the sorted keys hold the class in their top bits, so its boundaries are
// found by binary search (a per-run atomic on 4 counters serialised for ms at s24).
__global__ void k_ent_classes(const uint32_t *__restrict__ key, uint64_t k, int b,
                              unsigned long long *__restrict__ tot) {
    __shared__ uint64_t s_at[5];
    const int c = threadIdx.x;
    if (c <= 4) {
        uint64_t lo = 0, hi = k;   // first i with key[i] >= c << b
        const uint64_t want = (uint64_t)c << b;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if ((uint64_t)key[mid] < want) lo = mid + 1;
            else hi = mid;
        }
        s_at[c] = c == 4 ? k : lo;
    }
    __syncthreads();
    if (c < 4) tot[c] = s_at[c + 1] - s_at[c];
}

// Sorted position i (entry perm[i]): i < k_in -> in-list slot i: in_src = u, ulo = the probe
// length off[u + 1] - e - 1 (probe [e + 1, off[u + 1])); else out-part slot i - k_in: orange = N+(x), ovid = x.
// ... and the SHORT / SEARCH edges into their bins (whose counts come from tot).
__global__ void k_ent_place(const uint32_t *__restrict__ ent, const uint32_t *__restrict__ perm, uint64_t k,
                            const unsigned long long *__restrict__ tot, const uint64_t *__restrict__ off,
                            uint32_t *__restrict__ in_src, uint16_t *__restrict__ ulo,
                            uint2 *__restrict__ orange, uint32_t *__restrict__ ovid,
                            uint2 *__restrict__ b_short, uint2 *__restrict__ b_search,
                            uint64_t *__restrict__ counts) {
    const uint64_t k_in = tot[0], k_o = k_in + tot[1], k_s = k_o + tot[2];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        counts[0] = tot[2];
        counts[2] = tot[3];
    }
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = perm[i];
        const uint32_t y = ent[3 * e + 1], ef = ent[3 * e + 2];
        if (i < k_in) {
            in_src[i] = y;
            ulo[i] = (uint16_t)(off[y + 1] - ef - 1);
        } else if (i < k_o) {
            orange[i - k_in] = make_uint2((uint32_t)off[y], (uint32_t)off[y + 1]);
            ovid[i - k_in] = y;
        } else {
            const uint2 uv = make_uint2(ent[3 * e] & 0x7fffffffu, y);
            if (i < k_s) b_short[i - k_o] = uv;
            else b_search[i - k_s] = uv;
        }
    }
}

// Owner lists (k_owners' classes): warp owners (d+ < cta_min), CTA bitmap owners (effective
// span + a spare word fits kCtaBitmapBits), CTA hash owners; pcnt / in_cnt; max d+ -> counts[7].
__global__ void k_shard_owners(const uint32_t *__restrict__ icnt, const uint32_t *__restrict__ ocnt,
                               const uint32_t *__restrict__ dplus, const uint64_t *__restrict__ off,
                               const uint32_t *__restrict__ col, uint64_t n, uint32_t cta_min,
                               uint32_t *__restrict__ pcnt, uint32_t *__restrict__ in_cnt,
                               uint32_t *__restrict__ owners_warp, uint32_t *__restrict__ owners_cta,
                               uint32_t *__restrict__ owners_bitmap, uint64_t *__restrict__ counts) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    const uint64_t end = (n + 31) & ~31ull, stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t local_max = 0;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < end; x += stride) {
        int kind = -1;
        if (x < n) {
            const uint32_t ic = icnt[x], c = ic + ocnt[x], du = dplus[x];
            local_max = max(local_max, du);
            pcnt[x] = c;
            in_cnt[x] = ic;
            if (c)
                kind = du < cta_min ? 0
                       : ((uint64_t)col[off[x + 1] - 1] - col[off[x]] + 1 + 32 <= kCtaBitmapBits ? 2 : 1);
        }
        uint32_t *dst[3] = {owners_warp, owners_cta, owners_bitmap};
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const uint32_t mk = __ballot_sync(0xffffffffu, kind == k);
            uint64_t base = 0;
            if (lane == 0 && mk)
                base = atomicAdd((unsigned long long *)&counts[8 + k], (unsigned long long)__popc(mk));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (kind == k) dst[k][base + __popc(mk & lt)] = (uint32_t)x;
        }
    }
    local_max = __reduce_max_sync(0xffffffffu, local_max);
    if (lane == 0) atomicMax((unsigned long long *)&counts[7], (unsigned long long)local_max);
}

// ------------------------------------------------------------------ host helpers
static SliceParams slice_params(Ctx &ctx, uint64_t n, const uint64_t *off, const uint32_t *col,
                                const uint32_t *dplus, const tc_options &o, bool core) {
    SliceParams sp;
    sp.hp.off = off;
    sp.hp.col = col;
    sp.hp.dplus = dplus;
    sp.hp.n = (uint32_t)n;
    sp.hp.short_max = o.short_max;
    sp.hp.skew_ratio = o.skew_ratio;
    sp.hp.force = -1;
    sp.core = core;
    sp.core_lo = core_first(n);
    (void)ctx;
    return sp;
}

static uint32_t cta_min_of(const tc_options &o) {
    return o.hub_min_dplus < kWarpTableSlots / 4 + 1 ? o.hub_min_dplus : kWarpTableSlots / 4 + 1;
}

static void check_world(int rank, int world) {
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
        throw Error{TC_EINVAL, "need 0 <= rank < world <= 64"};
}

static void check_opts(const tc_options &o) {
    if (o.force_variant != TC_VARIANT_AUTO)
        throw Error{TC_EINVAL, "the sharded pipeline runs the AUTO policy only (force_variant = -1)"};
}

// Per-destination exclusive offsets of G counts (host side, G <= 64).
static void dest_offsets(Ctx &ctx, const unsigned long long *cnt_dev, int G, uint64_t *base_dev,
                         uint64_t *counts_host) {
    std::vector<unsigned long long> c(G);
    TC_CUDA(cudaMemcpyAsync(c.data(), cnt_dev, G * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            ctx.stream));
    TC_CUDA(cudaStreamSynchronize(ctx.stream));
    std::vector<uint64_t> b(G);
    uint64_t run = 0;
    for (int q = 0; q < G; q++) {
        b[q] = run;
        run += c[q];
        counts_host[q] = c[q];
    }
    TC_CUDA(cudaMemcpyAsync(base_dev, b.data(), G * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx.stream));
    TC_CUDA(cudaStreamSynchronize(ctx.stream));
}

}  // namespace tc

using namespace tc;

extern "C" {

tc_status tc_shard_orient(uint64_t n, uint64_t m_local, const uint64_t *edges, const uint32_t *degrees,
                          uint32_t flags, const tc_options *opt, uint32_t *newid, uint32_t *src,
                          uint32_t *dst, uint32_t *dplus) {
    return run_phase(opt, [&](Ctx &ctx, const tc_options &o) {
        if (flags & ~(uint32_t)TC_ID_ORDER) throw Error{TC_EINVAL, "tc_shard_orient: flags: TC_ID_ORDER only"};
        if (n >= (1ull << 30) || m_local >= (1ull << 31)) throw Error{TC_EINVAL, "the sharded pipeline needs n < 2^30, m < 2^31"};
        check_device(edges, ctx.device, "edges");
        check_device(degrees, ctx.device, "degrees");
        check_device(newid, ctx.device, "newid");
        check_device(src, ctx.device, "src");
        check_device(dst, ctx.device, "dst");
        check_device(dplus, ctx.device, "dplus");
        (void)o;
        if (!n) return;
        TC_CUDA(cudaMemsetAsync(dplus, 0, n * sizeof(uint32_t), ctx.stream));
        rank_relabel(ctx, n, degrees, flags & TC_ID_ORDER, newid);
        if (m_local) {
            k_shard_orient<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(edges, m_local, sh_id_bits(n), newid,
                                                                           src, dst, dplus);
            TC_LAUNCHED(ctx);
        }
    });
}

tc_status tc_shard_partition(uint64_t n, uint64_t m_local, const uint32_t *src, const uint32_t *dst,
                             const uint32_t *dplus, const tc_options *opt, int rank, int world,
                             uint64_t *off_plus, uint64_t *pairs_out, uint64_t *send_counts,
                             uint64_t *row_bounds, uint64_t *col_bounds) {
    return run_phase(opt, [&](Ctx &ctx, const tc_options &o) {
        (void)o;
        check_world(rank, world);
        check_device(dplus, ctx.device, "dplus");
        check_device(off_plus, ctx.device, "off_plus");
        check_device(pairs_out, ctx.device, "pairs_out");
        const int G = world;
        scan_exclusive(ctx, dplus, off_plus, n);
        uint32_t *bounds = ctx.alloc<uint32_t>(G + 1);
        k_split_bounds<<<1, 128, 0, ctx.stream>>>(off_plus, n, G, bounds);
        TC_LAUNCHED(ctx);
        std::vector<uint32_t> hb(G + 1);
        TC_CUDA(cudaMemcpyAsync(hb.data(), bounds, (G + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx.stream));
        TC_CUDA(cudaStreamSynchronize(ctx.stream));
        for (int q = 0; q <= G; q++) {
            row_bounds[q] = hb[q];
            TC_CUDA(cudaMemcpyAsync(&col_bounds[q], off_plus + hb[q], sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    ctx.stream));
        }
        unsigned long long *cnt = ctx.alloc<unsigned long long>(2 * G);
        uint64_t *base = ctx.alloc<uint64_t>(G);
        TC_CUDA(cudaMemsetAsync(cnt, 0, 2 * G * sizeof(unsigned long long), ctx.stream));
        const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((m_local + 2047) / 2048,
                                                                                 (uint64_t)ctx.persistent_grid(4)));
        if (m_local) {
            check_device(src, ctx.device, "src");
            check_device(dst, ctx.device, "dst");
            k_part_pairs<<<grid, 256, 0, ctx.stream>>>(src, dst, m_local, bounds, G, cnt, nullptr, nullptr, nullptr);
            TC_LAUNCHED(ctx);
        }
        dest_offsets(ctx, cnt, G, base, send_counts);
        if (m_local) {
            k_part_pairs<<<grid, 256, 0, ctx.stream>>>(src, dst, m_local, bounds, G, nullptr, cnt + G, base,
                                                       pairs_out);
            TC_LAUNCHED(ctx);
        }
    });
}

tc_status tc_shard_rows(uint64_t n, uint64_t m_recv, const uint64_t *pairs, const tc_options *opt,
                        uint64_t col_begin, uint32_t *col_plus) {
    return run_phase(opt, [&](Ctx &ctx, const tc_options &o) {
        (void)o;
        check_device(pairs, ctx.device, "pairs");
        check_device(col_plus, ctx.device, "col_plus");
        if (!m_recv) return;
        const int b = sh_id_bits(n);
        uint32_t *s = ctx.alloc<uint32_t>(m_recv), *t = ctx.alloc<uint32_t>(m_recv);
        k_unpack_pairs<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(pairs, m_recv, s, t);
        TC_LAUNCHED(ctx);
        uint32_t *kA = ctx.alloc<uint32_t>(m_recv), *kB = ctx.alloc<uint32_t>(m_recv);
        uint32_t *vA = ctx.alloc<uint32_t>(m_recv), *vB = ctx.alloc<uint32_t>(m_recv);
        uint32_t *k1, *v1;   // by target (values: sources)
        radix_sort_pairs_from(ctx, t, s, kA, kB, vA, vB, m_recv, nullptr, b, &k1, &v1);
        // then stably by source (values: the targets): rows ascending
        uint32_t *fk = k1 == kA ? kB : kA, *fv = v1 == vA ? vB : vA;
        uint32_t *k2, *v2;
        radix_sort_pairs_from(ctx, v1, k1, fk, s, fv, t, m_recv, nullptr, b, &k2, &v2);
        TC_CUDA(cudaMemcpyAsync(col_plus + col_begin, v2, m_recv * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                ctx.stream));
    });
}

tc_status tc_shard_work(uint64_t n, const uint64_t *off_plus, const uint32_t *col_plus, const uint32_t *dplus,
                        uint32_t flags, const tc_options *opt, uint64_t row_begin, uint64_t row_end,
                        uint64_t e_begin, uint64_t e_end, uint32_t *ent_cnt, uint64_t *ent_len,
                        uint32_t *spans) {
    return run_phase(opt, [&](Ctx &ctx, const tc_options &o) {
        check_opts(o);
        check_device(ent_cnt, ctx.device, "ent_cnt");
        check_device(ent_len, ctx.device, "ent_len");
        check_device(spans, ctx.device, "spans");
        TC_CUDA(cudaMemsetAsync(ent_cnt, 0, n * sizeof(uint32_t), ctx.stream));
        TC_CUDA(cudaMemsetAsync(ent_len, 0, n * sizeof(uint64_t), ctx.stream));
        TC_CUDA(cudaMemsetAsync(spans, 0, n * sizeof(uint32_t), ctx.stream));
        if (row_end > row_begin) {
            k_row_spans<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(off_plus, col_plus, row_begin, row_end, spans);
            TC_LAUNCHED(ctx);
        }
        if (e_end <= e_begin) return;
        const SliceParams sp = slice_params(ctx, n, off_plus, col_plus, dplus, o, !(flags & TC_PER_VERTEX));
        const uint32_t tiles = (uint32_t)((e_end - e_begin + kTileItems - 1) / kTileItems);
        k_slice<0><<<tiles, kTileThreads, 0, ctx.stream>>>(sp, e_begin, e_end, ent_cnt,
                                                            (unsigned long long *)ent_len, nullptr, 1, 0,
                                                            nullptr, nullptr, nullptr, nullptr, nullptr,
                                                            nullptr, nullptr);
        TC_LAUNCHED(ctx);
    });
}

tc_status tc_shard_route(uint64_t n, const uint64_t *off_plus, const uint32_t *col_plus, const uint32_t *dplus,
                         const uint32_t *ent_cnt, const uint64_t *ent_len, const uint32_t *spans, uint32_t flags,
                         const tc_options *opt, int rank, int world, uint64_t e_begin, uint64_t e_end,
                         uint32_t *entries_out, uint64_t *send_counts) {
    return run_phase(opt, [&](Ctx &ctx, const tc_options &o) {
        check_opts(o);
        check_world(rank, world);
        check_device(entries_out, ctx.device, "entries_out");
        const int G = world;
        uint64_t *work = ctx.alloc<uint64_t>(n), *wprefix = ctx.alloc<uint64_t>(n + 1);
        k_shard_owner_work<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(
            ent_cnt, (const unsigned long long *)ent_len, spans, dplus, n, cta_min_of(o), work);
        TC_LAUNCHED(ctx);
        scan_exclusive(ctx, work, wprefix, n);
        unsigned long long *cnt = ctx.alloc<unsigned long long>(2 * G);
        uint64_t *base = ctx.alloc<uint64_t>(G);
        TC_CUDA(cudaMemsetAsync(cnt, 0, 2 * G * sizeof(unsigned long long), ctx.stream));
        const SliceParams sp = slice_params(ctx, n, off_plus, col_plus, dplus, o, !(flags & TC_PER_VERTEX));
        const uint32_t tiles = e_end > e_begin ? (uint32_t)((e_end - e_begin + kTileItems - 1) / kTileItems) : 0;
        if (tiles) {
            k_slice<1><<<tiles, kTileThreads, 0, ctx.stream>>>(sp, e_begin, e_end, nullptr, nullptr, wprefix, G,
                                                                rank, cnt, nullptr, nullptr, nullptr, nullptr,
                                                                nullptr, nullptr);
            TC_LAUNCHED(ctx);
        }
        dest_offsets(ctx, cnt, G, base, send_counts);
        if (tiles) {
            k_slice<1><<<tiles, kTileThreads, 0, ctx.stream>>>(sp, e_begin, e_end, nullptr, nullptr, wprefix, G,
                                                                rank, nullptr, cnt + G, base, entries_out, nullptr,
                                                                nullptr, nullptr);
            TC_LAUNCHED(ctx);
        }
    });
}

tc_status tc_shard_count(uint64_t n, uint64_t m, const uint64_t *off_plus, const uint32_t *col_plus,
                         const uint32_t *dplus, const uint32_t *newid, uint64_t n_entries,
                         const uint32_t *entries, uint32_t flags, const tc_options *opt, int rank,
                         int world, uint64_t e_begin, uint64_t e_end, uint64_t *partial_dev,
                         uint64_t *per_vertex_partial, double *ms_a6) {
    return run_phase(opt, [&](Ctx &ctx, const tc_options &o) {
        if (ms_a6) *ms_a6 = 0.0;
        check_opts(o);
        check_world(rank, world);
        if (flags & ~(uint32_t)TC_PER_VERTEX) throw Error{TC_EINVAL, "tc_shard_count: flags: TC_PER_VERTEX only"};
        const bool pv = flags & TC_PER_VERTEX;
        if (pv && (!per_vertex_partial || !newid)) throw Error{TC_EINVAL, "TC_PER_VERTEX needs newid and per_vertex_partial"};
        if (n >= (1ull << 30) || m >= (1ull << 31)) throw Error{TC_EINVAL, "the sharded pipeline needs n < 2^30, m < 2^31"};
        check_device(partial_dev, ctx.device, "partial_dev");
        check_device(per_vertex_partial, ctx.device, "per_vertex_partial");
        TC_CUDA(cudaMemsetAsync(partial_dev, 0, sizeof(uint64_t), ctx.stream));
        if (!n) return;
        uint64_t *m_dev = ctx.alloc<uint64_t>(1);
        TC_CUDA(cudaMemcpyAsync(m_dev, &m, sizeof(uint64_t), cudaMemcpyHostToDevice, ctx.stream));
        Oriented g;
        g.n = n;
        g.off = const_cast<uint64_t *>(off_plus);
        g.col = const_cast<uint32_t *>(col_plus);
        g.dplus = const_cast<uint32_t *>(dplus);
        g.newid = const_cast<uint32_t *>(newid);
        g.m_dev = m_dev;
        g.m_cap = m;
        // ---- HASH owners of this rank: in-lists and out-part lists from the received entries
        const uint64_t k = n_entries;
        const int b = sh_id_bits(n);
        uint32_t *icnt = ctx.alloc<uint32_t>(n + 1), *ocnt = ctx.alloc<uint32_t>(n + 1);
        TC_CUDA(cudaMemsetAsync(icnt, 0, (n + 1) * sizeof(uint32_t), ctx.stream));
        TC_CUDA(cudaMemsetAsync(ocnt, 0, (n + 1) * sizeof(uint32_t), ctx.stream));
        const int grid = ctx.persistent_grid(8);
        uint32_t *perm = nullptr;
        unsigned long long *tot = ctx.alloc<unsigned long long>(4);
        TC_CUDA(cudaMemsetAsync(tot, 0, 4 * sizeof(unsigned long long), ctx.stream));
        if (k) {
            check_device(entries, ctx.device, "entries");
            uint32_t *key = ctx.alloc<uint32_t>(k);
            k_ent_keys<<<grid, 256, 0, ctx.stream>>>(entries, k, b, key);
            TC_LAUNCHED(ctx);
            uint32_t *kA = ctx.alloc<uint32_t>(k), *kB = ctx.alloc<uint32_t>(k);
            uint32_t *vA = ctx.alloc<uint32_t>(k), *vB = ctx.alloc<uint32_t>(k);
            uint32_t *sk;
            radix_sort_pairs_from(ctx, key, nullptr, kA, kB, vA, vB, k, nullptr, b + 2, &sk, &perm);
            k_ent_runs<<<grid, 256, 0, ctx.stream>>>(sk, k, b, icnt, ocnt);
            TC_LAUNCHED(ctx);
            k_ent_classes<<<1, 32, 0, ctx.stream>>>(sk, k, b, tot);
            TC_LAUNCHED(ctx);
        }
        uint64_t *in_off = ctx.alloc<uint64_t>(n + 1), *ooff = ctx.alloc<uint64_t>(n + 1);
        scan_exclusive(ctx, icnt, in_off, n);
        scan_exclusive(ctx, ocnt, ooff, n);
        Bins bins;
        bins.cap = m;
        bins.count = ctx.alloc<uint64_t>(16);
        TC_CUDA(cudaMemsetAsync(bins.count, 0, 16 * sizeof(uint64_t), ctx.stream));
        bins.pcnt = ctx.alloc<uint32_t>(n + 1);
        bins.owners_warp = ctx.alloc<uint32_t>(n);
        bins.owners_cta = ctx.alloc<uint32_t>(n);
        bins.owners_bitmap = ctx.alloc<uint32_t>(n);
        uint32_t *in_cnt = ctx.alloc<uint32_t>(n + 1);
        k_shard_owners<<<ctx.persistent_grid(4), 256, 0, ctx.stream>>>(icnt, ocnt, dplus, off_plus, col_plus, n,
                                                                       cta_min_of(o), bins.pcnt, in_cnt,
                                                                       bins.owners_warp, bins.owners_cta,
                                                                       bins.owners_bitmap, bins.count);
        TC_LAUNCHED(ctx);
        uint32_t *in_src = ctx.alloc<uint32_t>(k), *ovid = ctx.alloc<uint32_t>(k);
        uint16_t *ulo = ctx.alloc<uint16_t>(k);
        uint2 *orange = ctx.alloc<uint2>(k);
        // per-edge bins of this rank's rows (routed to itself by tc_shard_route)
        const bool want_short = o.short_max > 0, want_search = o.skew_ratio > 0;
        bins.edges[0] = ctx.alloc<uint2>(want_short ? std::max<uint64_t>(k, 1) : 1);
        bins.edges[1] = ctx.alloc<uint2>(1);
        bins.edges[2] = ctx.alloc<uint2>(want_search ? std::max<uint64_t>(k, 1) : 1);
        bins.has[0] = want_short;
        bins.has[1] = false;
        bins.has[2] = want_search;
        if (k) {
            k_ent_place<<<grid, 256, 0, ctx.stream>>>(entries, perm, k, tot, off_plus, in_src, ulo, orange, ovid,
                                                     bins.edges[0], bins.edges[2], bins.count);
            TC_LAUNCHED(ctx);
        }
        g.in_off = in_off;
        g.in_src = in_src;
        HashParams &hp = bins.hp;
        hp.off = off_plus;
        hp.col = col_plus;
        hp.dplus = dplus;
        hp.in_off = in_off;
        hp.in_src = in_src;
        hp.ulo = ulo;
        hp.in_cnt = in_cnt;
        hp.ooff = ooff;
        hp.orange = orange;
        hp.ovid = ovid;
        hp.n = (uint32_t)n;
        hp.short_max = o.short_max;
        hp.skew_ratio = o.skew_ratio;
        hp.force = -1;
        hp.rank = rank;
        hp.world = world;
        // the dense core by interleaved 2048-edge blocks (core.cu, every rank holds the CSR)
        if (!pv) core_build(ctx, g, hp);
        make_tasks(ctx, n, m, bins.owners_warp, bins.count + 8, bins.pcnt, hp, kWarpTaskLists, bins.count + 11,
                   bins.tasks_warp, bins.ntasks_warp);
        make_tasks(ctx, n, m, bins.owners_cta, bins.count + 9, bins.pcnt, hp, kCtaTaskLists, bins.count + 11,
                   bins.tasks_cta, bins.ntasks_cta);
        make_tasks(ctx, n, m, bins.owners_bitmap, bins.count + 10, bins.pcnt, hp, kBitmapTaskLists,
                   bins.count + 11, bins.tasks_bitmap, bins.ntasks_bitmap);
        Credit cr;
        uint64_t *pv_new = nullptr;
        if (pv) {
            pv_new = ctx.alloc<uint64_t>(n);
            TC_CUDA(cudaMemsetAsync(pv_new, 0, n * sizeof(uint64_t), ctx.stream));
            cr.mode = kCmVertex;
            cr.pv = pv_new;
        }
        Timer *tm = ms_a6 ? new Timer(ctx.stream) : nullptr;
        struct Del {
            Timer *t;
            ~Del() { delete t; }
        } del{tm};
        if (tm) tm->begin(kIntersect);
        intersect_all(ctx, g, bins, partial_dev, cr);
        if (tm) tm->end(kIntersect);
        if (pv) per_vertex_to_original(ctx, g, pv_new, per_vertex_partial);
        if (tm) {
            TC_CUDA(cudaStreamSynchronize(ctx.stream));
            *ms_a6 = tm->ms(kIntersect);
        }
    });
}

}  // extern "C"
