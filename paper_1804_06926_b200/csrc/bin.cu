// bin.cu -- a5: work estimation and binning (§4.2.2 P:527-542 "dynamic
// grouping ... divide the edge lists into groups"; third kernel P:704-708).
//
// Oriented edge (u,v) in rank ids (u < v, rows ascending).  A triangle {u,v,w}
// counted on it needs w in N+(u) and w > v, so only suf = |N+(u) after v| elements
// of N+(u) matter (they sit right after the edge in col+).  Edges with suf = 0 or
// d+(v) = 0 are skipped.  AUTO policy (edge_bin): SHORT if max(d+u, d+v) <=
// short_max, SEARCH if skew_ratio and max >= skew_ratio * min, else HASH.
//
// HASH owners.  An edge costs min(suf, d+v) probes.  If suf <= d+(v) (96% of R-MAT
// edges) its owner is v and it probes the suffix of N+(u) after v into a table of
// N+(v): these entries of v are exactly its in-list (the transposed CSR built in
// a3), so no grouping pass is needed -- k_edges writes each edge's probe range to
// its in-list slot (known from the a3 sort).  Otherwise the owner is u and it
// probes N+(v) into a table of N+(u): such out-part entries are compacted in CSR
// order (so grouped by u) by a tile scan.  Owner x's entries = in-list ++ out-part.
//
// Multi-GPU: every rank bins every edge identically; then the HASH work is
// split by OWNER -- owners are cut into `world` contiguous groups by an exclusive prefix of
// their work w(x) (k_owner_work: probe lengths + a fixed cost per entry + the table builds),
// so each owner's table is built on exactly one rank -- and the SHORT / MERGE / SEARCH / core
// edges by interleaved 2048-edge blocks of CSR order (edge_rank; contiguous ranges would hand
// the whole dense core, the last rows, to the last rank).  No communication: every rank
// computes the same prefix.
#include "block_scan.cuh"
#include "tc_internal.cuh"

namespace tc {

template <class Item>
__device__ __forceinline__ void warp_append(bool take, uint64_t *counter, Item *out, Item item) {
    uint32_t mask = __ballot_sync(0xffffffffu, take);
    if (!mask) return;
    int lane = threadIdx.x & 31;
    int leader = __ffs(mask) - 1;
    uint64_t base = 0;
    if (lane == leader) base = atomicAdd((unsigned long long *)counter, (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (take) out[base + __popc(mask & ((1u << lane) - 1u))] = item;
}

// For every CSR edge e = (u -> x) (row u, rows ascending), with p = pidx[e] its slot
// in x's in-list:
//   - x owns the edge (suf = |N+(u) after x| <= d+(x), and suf <= kSufMax): ulo[p] = suf,
//     16 bits (probe range [off[u+1] - suf, off[u+1]), the end re-read by the kernel from
//     u = in_src[p]),
//     an in-part entry of x;
//   - u owns it (suf > d+(x), ~4% of R-MAT edges): bit e of `obits` is set, an
//     out-part entry of u (probe range N+(x); compacted in CSR order by k_ocompact,
//     which re-derives the range from x = col+[e]);
// Not-HASH / skipped / other-rank edges: neither.  One ballot word per warp round
// (32 consecutive edges) and the tile's out-part count (tcount) replace a per-edge
// range array.  SHORT / MERGE / SEARCH edges are appended to their bins.  Also accumulates
// the work statistics.
#ifndef TC_EDGES_MINBLOCKS
#define TC_EDGES_MINBLOCKS 4   // 64 registers: measured s21 bin -0.09 ms, road -0.19 ms
#endif
#ifndef TC_EDGES_BATCH
#define TC_EDGES_BATCH 4
#endif
__global__ void __launch_bounds__(kTileThreads, TC_EDGES_MINBLOCKS)
    k_edges(HashParams hp, const uint64_t *__restrict__ m_dev, uint16_t *__restrict__ ulo,
            uint32_t *__restrict__ obits, uint32_t *__restrict__ tcount,
            uint2 *__restrict__ b_short, uint2 *__restrict__ b_merge, uint2 *__restrict__ b_search,
            uint64_t *__restrict__ counts, const uint2 *__restrict__ tb) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    __shared__ uint64_t s_red[kTileThreads / 32];
    // SHORT edges (AUTO sends many) are staged per tile and appended with ONE global
    // atomic per block: per-warp appends all hit one counter (~1 M atomics per step at s21)
    __shared__ uint2 s_short[kTileItems];
    __shared__ uint32_t s_nshort;
    __shared__ uint64_t s_short_base;
    if (threadIdx.x == 0) s_nshort = 0;
    uint64_t m = *m_dev;
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    if (t0 >= m) {
        if (threadIdx.x == 0) tcount[blockIdx.x] = 0;
        return;
    }
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, m - t0);
    tile_rows_tb(hp.off, hp.n, blockIdx.x, t0, len, tb, s_row, s_scan);
    uint64_t W = 0, probe = 0, skipped = 0, hashed = 0, outs = 0, cedges = 0, cprobe = 0;
    // striped: each warp handles 32 consecutive edges per round (warp-aggregated
    // appends); the loads of kBatch rounds are issued before any is used
    constexpr int kRounds = kTileItems / kTileThreads, kBatch = TC_EDGES_BATCH;
#pragma unroll 1
    for (int r0 = 0; r0 < kRounds; r0 += kBatch) {
        uint32_t us[kBatch], xs[kBatch], ps[kBatch], dvs[kBatch];
        uint64_t ubs[kBatch], ues[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; j++) {
            uint32_t i = (r0 + j) * kTileThreads + threadIdx.x;
            bool ok = i < len;
            us[j] = ok ? s_row[i] : 0u;
            xs[j] = ok ? hp.col[t0 + i] : 0u;
            ps[j] = ok ? hp.pidx[t0 + i] : 0u;
        }
#pragma unroll
        for (int j = 0; j < kBatch; j++) {
            dvs[j] = hp.dplus[xs[j]];
            ubs[j] = hp.off[us[j]];
            ues[j] = hp.off[us[j] + 1];
        }
#pragma unroll
        for (int j = 0; j < kBatch; j++) {
            uint32_t i = (r0 + j) * kTileThreads + threadIdx.x;
            int bin = -1;
            bool outp = false;
            uint2 item = make_uint2(0, 0);
            if (i < len) {
                uint64_t e = t0 + i;
                uint32_t u = us[j], x = xs[j], dv = dvs[j];
                uint64_t ue = ues[j];
                uint32_t du = (uint32_t)(ue - ubs[j]), suf = (uint32_t)(ue - e - 1);
                bin = edge_bin(hp, du, dv, suf);
                // a HASH edge of a core source is counted by the dense-core path (core.cu)
                if (bin == TC_VARIANT_HASH && hp.core && u >= hp.core_lo) bin = kBinCore;
                // world > 1: HASH edges are binned on every rank (split later by owner, whose
                // statistics k_owners counts); the other bins keep this rank's edge range
                const bool mine = hp.world <= 1 || bin == TC_VARIANT_HASH || edge_rank(e, hp.world) == hp.rank;
                if (!mine) bin = -1;
                if (mine && (hp.world <= 1 || bin != TC_VARIANT_HASH)) {
                    W += du + dv;
                    probe += min(suf, dv);
                    skipped += bin < 0;
                    if (bin == kBinCore) {
                        cedges++;
                        cprobe += min(suf, dv);
                    }
                }
                item = make_uint2(u, x);
                uint32_t ri = 0;
                if (bin == TC_VARIANT_HASH) {
                    hashed += hp.world <= 1;
                    if (suf <= dv && suf <= kSufMax) ri = suf;
                    else outp = true;
                }
                ulo[ps[j]] = (uint16_t)ri;
            }
            const uint32_t ob = __ballot_sync(0xffffffffu, outp);
            if ((threadIdx.x & 31) == 0) {
                obits[(t0 + (uint64_t)(r0 + j) * kTileThreads + (threadIdx.x & ~31u)) >> 5] = ob;
                outs += __popc(ob);
            }
            {   // stage SHORT in shared memory (warp-aggregated shared atomic)
                const bool take = bin == TC_VARIANT_SHORT;
                const uint32_t mask = __ballot_sync(0xffffffffu, take);
                if (mask) {
                    const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
                    uint32_t b0 = 0;
                    if (lane == leader) b0 = atomicAdd(&s_nshort, (uint32_t)__popc(mask));
                    b0 = __shfl_sync(0xffffffffu, b0, leader);
                    if (take) s_short[b0 + __popc(mask & ((1u << lane) - 1u))] = item;
                }
            }
            warp_append(bin == TC_VARIANT_MERGE, &counts[1], b_merge, item);
            warp_append(bin == TC_VARIANT_SEARCH, &counts[2], b_search, item);
        }
    }
    __syncthreads();
    const uint32_t ns = s_nshort;
    if (threadIdx.x == 0 && ns)
        s_short_base = atomicAdd((unsigned long long *)&counts[0], (unsigned long long)ns);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < ns; i += kTileThreads) b_short[s_short_base + i] = s_short[i];
    W = block_sum_u64(W, s_red);
    probe = block_sum_u64(probe, s_red);
    skipped = block_sum_u64(skipped, s_red);
    hashed = block_sum_u64(hashed, s_red);
    outs = block_sum_u64(outs, s_red);
    cedges = block_sum_u64(cedges, s_red);
    cprobe = block_sum_u64(cprobe, s_red);
    if (threadIdx.x == 0) {
        tcount[blockIdx.x] = (uint32_t)outs;
        if (cedges) {
            atomicAdd((unsigned long long *)&counts[13], (unsigned long long)cedges);
            atomicAdd((unsigned long long *)&counts[15], (unsigned long long)cprobe);
        }
        atomicAdd((unsigned long long *)&counts[3], (unsigned long long)hashed);
        atomicAdd((unsigned long long *)&counts[4], (unsigned long long)W);
        atomicAdd((unsigned long long *)&counts[5], (unsigned long long)probe);
        atomicAdd((unsigned long long *)&counts[6], (unsigned long long)skipped);
    }
}

// Compaction of the out-part entries (CSR order => grouped by the owning source): one
// 64-thread block per tile, one thread per ballot word.  Entry = probe range N+(x) of
// the edge's target x and its vid (x, or the edge index for edge support).  Also the
// in-tile exclusive prefix of each word (wpre) for k_ooff.
constexpr int kTileWords = kTileItems / 32;
__global__ void __launch_bounds__(kTileWords)
    k_ocompact(const uint32_t *__restrict__ obits, const uint32_t *__restrict__ col,
               const uint64_t *__restrict__ off, const uint32_t *__restrict__ dplus,
               const uint64_t *__restrict__ m_dev, const uint64_t *__restrict__ toff,
               uint2 *__restrict__ orange, uint32_t *__restrict__ ovid, uint16_t *__restrict__ wpre,
               bool edge_ids) {
    __shared__ uint32_t s_w[kTileWords / 32];
    const uint64_t m = *m_dev, t0 = (uint64_t)blockIdx.x * kTileItems;
    if (t0 >= m) return;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t gw = (t0 >> 5) + threadIdx.x;
    const uint64_t e0 = t0 + 32ull * threadIdx.x;
    uint32_t bits = e0 < m ? obits[gw] : 0u;
    const uint32_t c = __popc(bits);
    const uint32_t inc = warp_inclusive_scan<SumOp>(c);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint32_t excl = inc - c;
    for (uint32_t w = 0; w < warp; w++) excl += s_w[w];
    if (e0 < m) wpre[gw] = (uint16_t)excl;
    uint64_t base = toff[blockIdx.x] + excl;
    while (bits) {
        const uint32_t b = __ffs(bits) - 1;
        bits &= bits - 1;
        const uint64_t e = e0 + b;
        const uint32_t x = col[e];
        const uint64_t xb = off[x];
        orange[base] = make_uint2((uint32_t)xb, (uint32_t)(xb + dplus[x]));
        ovid[base] = edge_ids ? (uint32_t)e : x;
        base++;
    }
}

// Out-part entries before CSR position s = tile prefix + in-tile word prefix + bits below.
struct OutPrefix {
    const uint32_t *obits;
    const uint16_t *wpre;
    const uint64_t *toff;
    uint64_t m, total;
    __device__ __forceinline__ uint64_t at(uint64_t s) const {
        return s < m ? toff[s / kTileItems] + wpre[s >> 5] + __popc(obits[s >> 5] & ((1u << (s & 31)) - 1u))
                     : total;
    }
};

// Owner lists and max d+.  pcnt[x] = probe entries of owner x = its in-degree (empty
// entries included; 0 if none of them is x's) + its compacted out-part entries; warp owners (d+ < cta_min), CTA
// bitmap owners (rank span n-1-x plus a spare zero word fits kCtaBitmapBits) and CTA
// hash owners (the rest).
// Also writes ooff[u] (each owner's first out-part entry; ooff[n] = the total), which the
// owner counts here need anyway: no separate pass over the vertices.
template <bool shard>
__global__ void k_owners(const uint32_t *__restrict__ dplus, const uint32_t *__restrict__ col,
                         const uint64_t *__restrict__ in_off, const uint64_t *__restrict__ pre_cnt,
                         const uint64_t *__restrict__ pre_len,
                         const uint2 *__restrict__ orange, const uint64_t *__restrict__ owner_prefix,
                         int rank, int world,
                         const uint16_t *__restrict__ ulo, uint32_t *__restrict__ in_cnt,
                         uint64_t *__restrict__ ooff, const uint64_t *__restrict__ off,
                         const uint64_t *__restrict__ m_dev, const uint32_t *__restrict__ obits,
                         const uint16_t *__restrict__ wpre, const uint64_t *__restrict__ toff,
                         const uint64_t *__restrict__ ototal,
                         uint64_t n, uint32_t cta_min,
                         uint32_t *__restrict__ pcnt, uint32_t *__restrict__ owners_warp,
                         uint32_t *__restrict__ owners_cta, uint32_t *__restrict__ owners_bitmap,
                         uint64_t *__restrict__ counts) {
    uint32_t local_max = 0;
    const OutPrefix op{obits, wpre, toff, *m_dev, *ototal};
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t end = (n + 31) & ~31ull;  // whole warps stay in the loop (warp-aggregated appends)
    if (blockIdx.x == 0 && threadIdx.x == 0) ooff[n] = op.at(off[n]);
    int lane = threadIdx.x & 31;
    uint32_t lt = (1u << lane) - 1u;
    uint64_t s_hashed = 0, s_probe = 0, s_W = 0;   // shard statistics (this rank's owners)
    // world 1: k_edges counted the HASH edges (counts[3]); none -> every owner is empty (the
    // in-list scans below would read every ulo entry for nothing: road mesh 0.23 ms)
    const bool any_hash = shard || counts[3] != 0;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < end; u += stride) {
        int kind = -1;
        if (u < n) {
            uint32_t du = dplus[u];
            local_max = max(local_max, du);
            uint32_t c = 0, hin = 0;
            (void)hin;
            if (shard) {   // k_owner_work wrote in_cnt, pcnt and the owner work prefix
                c = pcnt[u];
                if (c && split_rank(owner_prefix[u], owner_prefix[n], world) != rank) c = 0;
                if (c) {   // this rank's owner: its HASH statistics (W: out-part entries only)
                    const uint64_t ib = in_off[u], ie = in_off[u + 1];
                    s_hashed += pre_cnt[ie] - pre_cnt[ib];
                    s_probe += pre_len[ie] - pre_len[ib];
                    for (uint64_t k = ooff[u], ke = ooff[u + 1]; k < ke; k++) {
                        const uint2 r = orange[k];
                        s_hashed++;
                        s_probe += r.y - r.x;
                        s_W += du + (r.y - r.x);
                    }
                }
            } else if (!any_hash) {   // no HASH edge at all (road-like graphs): nothing to own
                ooff[u] = 0;
                in_cnt[u] = 0;
                pcnt[u] = 0;
            } else {
                const uint64_t o0 = op.at(off[u]);
                ooff[u] = o0;
                if (du) {
                    // does some in-entry of u carry HASH work?  (first hit exits)
                    uint64_t ib = in_off[u], ie = in_off[u + 1];
                    for (uint64_t p = ib; p < ie; p++)
                        if (ulo[p]) {
                            hin = (uint32_t)(ie - ib);
                            break;
                        }
                    c = hin + (uint32_t)(op.at(off[u + 1]) - o0);
                }
                in_cnt[u] = hin;
                pcnt[u] = c;
            }
            // bitmap owners: N+(u) spans [first, last] element (rows ascending) + a spare word
#if TC_BITMAP_EFFSPAN
            if (c)
                kind = du < cta_min ? 0
                       : ((uint64_t)col[off[u + 1] - 1] - col[off[u]] + 1 + 32 <= kCtaBitmapBits ? 2 : 1);
#else
            if (c) kind = du < cta_min ? 0 : (n - 1 - u + 32 <= kCtaBitmapBits ? 2 : 1);
#endif
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
    if (shard) {
        s_hashed = warp_sum_u64(s_hashed);
        s_probe = warp_sum_u64(s_probe);
        s_W = warp_sum_u64(s_W);
        if (lane == 0 && s_hashed) {
            atomicAdd((unsigned long long *)&counts[3], (unsigned long long)s_hashed);
            atomicAdd((unsigned long long *)&counts[4], (unsigned long long)s_W);
            atomicAdd((unsigned long long *)&counts[5], (unsigned long long)s_probe);
        }
    }
}

// world > 1: per in-list entry p (owner = its in-list's vertex), 1 and its probe length if it is
// HASH work (ulo[p] != 0), else 0 / 0 -- prefix-scanned so every owner's sums are two
// lookups (a thread per owner would walk a hub's 10^5-entry in-list alone).
__global__ void k_entry_vals(const uint64_t *__restrict__ off, const uint32_t *__restrict__ in_src,
                             const uint16_t *__restrict__ ulo, const uint64_t *__restrict__ m_dev,
                             uint32_t *__restrict__ cnt, uint32_t *__restrict__ len) {
    const uint64_t m = *m_dev;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t suf = ulo[p];   // the probe length itself
        cnt[p] = suf ? 1u : 0u;
        len[p] = suf;
    }
}

// world > 1, before k_owners: for every owner x, in_cnt / pcnt as k_owners computes them, the
// first out-part entry ooff[x], and its work w(x) = sum over its probe entries of
// (kEntryCost + probe length) + the table builds per CTA task (d+(x), plus the bitmap words
// for a bitmap owner).
#ifndef TC_SHARD_ENTRY_COST
#define TC_SHARD_ENTRY_COST 64   // fixed cost of a probe entry (descriptor, partial slots), in probes
#endif
#ifndef TC_SHARD_HASH_WEIGHT
#define TC_SHARD_HASH_WEIGHT 3   // bucket-hash owner probes relative to bitmap probes
#endif
#ifndef TC_SHARD_WARP_WEIGHT
#define TC_SHARD_WARP_WEIGHT 2   // warp-table owner probes relative to bitmap probes (measured: s21 w8 max/mean 1.50 -> 1.31)
#endif
__global__ void k_owner_work(const uint32_t *__restrict__ dplus, const uint32_t *__restrict__ col,
                             const uint64_t *__restrict__ off, const uint64_t *__restrict__ in_off,
                             const uint64_t *__restrict__ pre_cnt, const uint64_t *__restrict__ pre_len,
                             const uint64_t *__restrict__ m_dev, const uint32_t *__restrict__ obits,
                             const uint16_t *__restrict__ wpre, const uint64_t *__restrict__ toff,
                             const uint64_t *__restrict__ ototal, const uint2 *__restrict__ orange,
                             uint64_t n, uint32_t cta_min, uint32_t *__restrict__ in_cnt,
                             uint32_t *__restrict__ pcnt, uint64_t *__restrict__ ooff,
                             uint64_t *__restrict__ work) {
    const OutPrefix op{obits, wpre, toff, *m_dev, *ototal};
    if (blockIdx.x == 0 && threadIdx.x == 0) ooff[n] = op.at(off[n]);
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t du = dplus[u];
        const uint64_t o0 = op.at(off[u]), o1 = op.at(off[u + 1]);
        ooff[u] = o0;
        uint64_t w = 0;
        uint32_t c = 0, ic = 0;
        if (du) {
            const uint64_t ib = in_off[u], ie = in_off[u + 1];
            const uint64_t entries = pre_cnt[ie] - pre_cnt[ib];
            w = entries * TC_SHARD_ENTRY_COST + (pre_len[ie] - pre_len[ib]);
            for (uint64_t k = o0; k < o1; k++) {   // out-part: at most d+(u) entries
                const uint2 r = orange[k];
                w += TC_SHARD_ENTRY_COST + (r.y - r.x);
            }
            ic = entries ? (uint32_t)(ie - ib) : 0u;
            c = ic + (uint32_t)(o1 - o0);
            if (c && du < cta_min) {          // warp owner: a warp table per 64 entries
                w = w * TC_SHARD_WARP_WEIGHT + (uint64_t)((c + kWarpTaskLists - 1) / kWarpTaskLists) * du;
            } else if (c) {                   // CTA owner: bitmap (zeroed span) or hash table
                const uint64_t span = (uint64_t)col[off[u + 1] - 1] - col[off[u]] + 1;
                const bool bitmap = span + 32 <= kCtaBitmapBits;
                if (!bitmap) w *= TC_SHARD_HASH_WEIGHT;   // bucket-hash probes cost more
                w += (uint64_t)((c + kCtaTaskLists - 1) / kCtaTaskLists) * (du + (bitmap ? span / 32 : 0));
            }
        }
        in_cnt[u] = ic;
        pcnt[u] = c;
        work[u] = w;
    }
}

// Tasks: owner i of `owners` (i < *ocount) gets ceil(pcnt / L) tasks.
// Also accumulates the table-build loads sum over tasks of d+(owner) into *tloads.
__global__ void k_task_count(const uint32_t *__restrict__ owners, const uint64_t *__restrict__ ocount,
                             const uint32_t *__restrict__ pcnt, const uint32_t *__restrict__ dplus,
                             uint64_t n, uint32_t L, uint32_t *__restrict__ tcnt,
                             uint64_t *__restrict__ tloads) {
    uint64_t no = *ocount, loads = 0;
    (void)n;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < no;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x = owners[i];
        uint32_t t = (pcnt[x] + L - 1) / L;
        loads += (uint64_t)t * dplus[x];
        tcnt[i] = t;
    }
    loads = warp_sum_u64(loads);
    if ((threadIdx.x & 31) == 0 && loads) atomicAdd((unsigned long long *)tloads, (unsigned long long)loads);
}

// Task records: task k of owner x = {x, first entry k*L, d+(x), in_cnt(x)} and {off+[x],
// in_off[x], ooff[x], out-part entries of x} (all offsets < 2^32: m < 2^32), so a6 reads
// its task header with two 16-byte loads instead of a task -> owner -> offsets chain.
__global__ void k_task_expand(const uint32_t *__restrict__ owners, const uint64_t *__restrict__ ocount,
                              const uint32_t *__restrict__ tcnt, const uint64_t *__restrict__ toff,
                              uint32_t L, const uint64_t *__restrict__ off,
                              const uint64_t *__restrict__ in_off, const uint32_t *__restrict__ in_cnt,
                              const uint64_t *__restrict__ ooff, uint4 *__restrict__ tasks) {
    uint64_t no = *ocount;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < no;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = owners[i], c = tcnt[i];
        const uint64_t o = toff[i], xb = off[x], ob = ooff[x];
        const uint4 r1 = make_uint4((uint32_t)xb, (uint32_t)in_off[x], (uint32_t)ob,
                                    (uint32_t)(ooff[x + 1] - ob));
        const uint32_t dx = (uint32_t)(off[x + 1] - xb), ic = in_cnt[x];
        for (uint32_t k = 0; k < c; k++) {
            tasks[2 * (o + k)] = make_uint4(x, k * L, dx, ic);
            tasks[2 * (o + k) + 1] = r1;
        }
    }
}

void make_tasks(Ctx &ctx, uint64_t n, uint64_t cap, const uint32_t *owners,
                       const uint64_t *ocount, const uint32_t *pcnt, const HashParams &hp,
                       uint32_t L, uint64_t *tloads, uint4 *&tasks, uint64_t *&ntasks) {
    uint32_t *tcnt = ctx.alloc<uint32_t>(n);
    uint64_t *toff = ctx.alloc<uint64_t>(n + 1);
    int grid = ctx.persistent_grid(4);
    k_task_count<<<grid, 256, 0, ctx.stream>>>(owners, ocount, pcnt, hp.dplus, n, L, tcnt, tloads);
    TC_LAUNCHED(ctx);
    // the owner list is usually far shorter than n (road mesh: empty): scan only its length
    scan_exclusive_dc(ctx, tcnt, toff, n, ocount, toff + n);
    tasks = ctx.alloc<uint4>(2 * ((2 * cap) / L + n + 1));
    k_task_expand<<<grid, 256, 0, ctx.stream>>>(owners, ocount, tcnt, toff, L, hp.off, hp.in_off,
                                                hp.in_cnt, hp.ooff, tasks);
    TC_LAUNCHED(ctx);
    ntasks = toff + n;
}

void bin_edges(Ctx &ctx, const Oriented &g, const BinParams &p, Bins &bins) {
    uint64_t cap = g.m_cap, n = g.n;
    bins.cap = cap;
    bins.count = ctx.alloc<uint64_t>(16);
    TC_CUDA(cudaMemsetAsync(bins.count, 0, 16 * sizeof(uint64_t), ctx.stream));
    HashParams &hp = bins.hp;
    hp.off = g.off;
    hp.col = g.col;
    hp.dplus = g.dplus;
    hp.in_off = g.in_off;
    hp.in_src = g.in_src;
    hp.pidx = g.pidx;
    hp.n = (uint32_t)n;
    hp.short_max = p.short_max;
    hp.skew_ratio = p.skew_ratio;
    hp.force = p.force;
    hp.rank = p.rank;
    hp.world = p.world;
    uint32_t tiles = (uint32_t)((cap + kTileItems - 1) / kTileItems);
    // dense core (core.cu): plain counts under the AUTO policy only
    if (p.core && p.force < 0) core_build(ctx, g, hp);

    // edge bins for the merge / search / two-pointer variants (filled by k_edges)
    // only the bins that can receive edges get capacity (at s26 each is 8.6 GB): AUTO
    // routes to SHORT (short_max > 0), SEARCH (skew_ratio > 0) or HASH; MERGE only if forced
    const bool want[3] = {p.force == TC_VARIANT_SHORT || (p.force < 0 && p.short_max > 0),
                          p.force == TC_VARIANT_MERGE,
                          p.force == TC_VARIANT_SEARCH || (p.force < 0 && p.skew_ratio > 0)};
    for (int k = 0; k < 3; k++) {
        bins.edges[k] = ctx.alloc<uint2>(want[k] ? cap : 1);
        bins.has[k] = want[k];
    }

    // HASH: in-part ranges (in-list order), out-part entries (compacted, CSR order),
    // statistics, owners, tasks
    uint16_t *ulo = ctx.alloc<uint16_t>(cap);
    uint32_t *obits = ctx.alloc<uint32_t>((uint64_t)tiles * kTileWords + 1);
    uint16_t *wpre = ctx.alloc<uint16_t>((uint64_t)tiles * kTileWords + 1);
    uint2 *orange = ctx.alloc<uint2>(cap);
    uint32_t *ovid = ctx.alloc<uint32_t>(cap);
    uint32_t *tcount = ctx.alloc<uint32_t>(tiles + 1);
    uint64_t *toff = ctx.alloc<uint64_t>(tiles + 1), *ooff = ctx.alloc<uint64_t>(n + 1);
    uint32_t *in_cnt = ctx.alloc<uint32_t>(n + 1);
    if (tiles) {
        uint2 *tb = nullptr;
        if (TC_TILE_BOUNDS) {
            tb = ctx.alloc<uint2>(tiles + 1);
            tile_bounds(ctx, g.off, n, cap, g.m_dev, tb);
        }
        k_edges<<<tiles, kTileThreads, 0, ctx.stream>>>(hp, g.m_dev, ulo, obits, tcount,
                                                        bins.edges[0], bins.edges[1], bins.edges[2],
                                                        bins.count, tb);
        TC_LAUNCHED(ctx);
    }
    scan_exclusive(ctx, tcount, toff, tiles);
    if (tiles) {
        k_ocompact<<<tiles, kTileWords, 0, ctx.stream>>>(obits, g.col, g.off, g.dplus, g.m_dev, toff,
                                                         orange, ovid, wpre, p.edge_ids);
        TC_LAUNCHED(ctx);
    }
    hp.ulo = ulo;
    hp.in_cnt = in_cnt;
    hp.orange = orange;
    hp.ovid = ovid;
    hp.ooff = ooff;
    bins.pcnt = ctx.alloc<uint32_t>(n + 1);
    bins.owners_warp = ctx.alloc<uint32_t>(n);
    bins.owners_cta = ctx.alloc<uint32_t>(n);
    bins.owners_bitmap = ctx.alloc<uint32_t>(n);
    uint32_t cta_min = p.hub_min < kWarpTableSlots / 4 + 1 ? p.hub_min : kWarpTableSlots / 4 + 1;
    // (core owners keep the now-empty entries of their core edges in their in-lists:
    // compacting them in place, one CTA per core owner, measured +0.43 ms in binning for
    // -0.13 ms in a6 at s21)
    if (p.world > 1) {   // owner split: work per owner, its exclusive prefix, then this rank's owners
        uint32_t *ecnt = ctx.alloc<uint32_t>(cap), *elen = ctx.alloc<uint32_t>(cap);
        uint64_t *pre_cnt = ctx.alloc<uint64_t>(cap + 1), *pre_len = ctx.alloc<uint64_t>(cap + 1);
        k_entry_vals<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(g.off, g.in_src, ulo, g.m_dev,
                                                                     ecnt, elen);
        TC_LAUNCHED(ctx);
        scan_exclusive_dc(ctx, ecnt, pre_cnt, cap, g.m_dev, pre_cnt + cap);
        scan_exclusive_dc(ctx, elen, pre_len, cap, g.m_dev, pre_len + cap);
        uint64_t *work = ctx.alloc<uint64_t>(n), *wprefix = ctx.alloc<uint64_t>(n + 1);
        k_owner_work<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(
            g.dplus, g.col, g.off, g.in_off, pre_cnt, pre_len, g.m_dev, obits, wpre, toff,
            toff + tiles, orange, n, cta_min, in_cnt, bins.pcnt, ooff, work);
        TC_LAUNCHED(ctx);
        scan_exclusive(ctx, work, wprefix, n);
        k_owners<true><<<ctx.persistent_grid(4), 256, 0, ctx.stream>>>(
            g.dplus, g.col, g.in_off, pre_cnt, pre_len, orange, wprefix, p.rank, p.world, ulo, in_cnt, ooff,
            g.off, g.m_dev, obits, wpre, toff, toff + tiles, n, cta_min, bins.pcnt, bins.owners_warp,
            bins.owners_cta, bins.owners_bitmap, bins.count);
    } else {
        k_owners<false><<<ctx.persistent_grid(4), 256, 0, ctx.stream>>>(
            g.dplus, g.col, g.in_off, nullptr, nullptr, orange, nullptr, 0, 1, ulo, in_cnt, ooff, g.off,
            g.m_dev, obits, wpre, toff, toff + tiles, n, cta_min, bins.pcnt, bins.owners_warp,
            bins.owners_cta, bins.owners_bitmap, bins.count);
    }
    TC_LAUNCHED(ctx);
    make_tasks(ctx, n, cap, bins.owners_warp, bins.count + 8, bins.pcnt, hp, kWarpTaskLists,
               bins.count + 11, bins.tasks_warp, bins.ntasks_warp);
    make_tasks(ctx, n, cap, bins.owners_cta, bins.count + 9, bins.pcnt, hp, kCtaTaskLists,
               bins.count + 11, bins.tasks_cta, bins.ntasks_cta);
    make_tasks(ctx, n, cap, bins.owners_bitmap, bins.count + 10, bins.pcnt, hp, kBitmapTaskLists,
               bins.count + 11, bins.tasks_bitmap, bins.ntasks_bitmap);
}

}  // namespace tc
