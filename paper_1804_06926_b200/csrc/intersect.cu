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
//   HASH   per edge (u,v), u < v in rank ids, the shorter of (N+(u) after v) and
//          N+(v) is probed into a shared-memory table (bucket hash, or a bitmap
//          over the rank range for hubs) of the other endpoint's N+ ("owner");
//          one warp per small owner task, one CTA per hub task (north_star hub
//          kernel).  Cost: min(|N+(u) > v|, d+v) probes per edge instead of
//          d+u + d+v merge steps.
// Credit modes (template parameter CM, Credit in tc_internal.cuh): every match w of
// an oriented edge (u,v) is the triangle {u,v,w}, and besides the count it can
//   kCmVertex  add 1 to t(u), t(v), t(w)  (TC_PER_VERTEX);
//   kCmEdge    add 1 to the support of its three edges (u,v), (u,w), (v,w), each an
//              entry of col+ (NEXT-3 edge support, the k-truss input);
//   kCmList    write the triangle as three ascending input ids (NEXT-3 enumeration,
//              "the listings of all the triangles for free");
//   kCmTop     add 1 to its TOP edge only, the edge between its two highest-ranked
//              vertices: C = A o (L U) at A's nonzeros (NEXT-4, Alg. 3),
//              since (L U)_ij counts the common neighbours k ranked below i and j.
// In the HASH kernels the owner-side credit (t(w), or the support of (owner, w)) is
// counted in shared memory per owner element and flushed once per task.
#include "block_scan.cuh"
#include "tc_internal.cuh"

namespace tc {

constexpr int kIxThreads = 256;

__device__ __forceinline__ void flush_count(uint64_t acc, uint64_t *total) {
    __shared__ uint64_t s_red[32];
    uint64_t t = block_sum_u64(acc, s_red);
    if (threadIdx.x == 0 && t) atomicAdd((unsigned long long *)total, (unsigned long long)t);
}

template <int CM>
__device__ __forceinline__ void credit_edge(const Credit &cr, uint32_t u, uint32_t v, uint32_t c) {
    if (CM == kCmVertex && c) {
        atomicAdd((unsigned long long *)&cr.pv[u], (unsigned long long)c);
        atomicAdd((unsigned long long *)&cr.pv[v], (unsigned long long)c);
    }
}

// Index of w in the ascending list a[0, len) (w must be present): edge-support credit.
__device__ __forceinline__ uint32_t list_pos(const uint32_t *__restrict__ a, uint32_t len, uint32_t w) {
    uint32_t lo = 0, hi = len;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < w) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// CSR index of oriented edge (u, v) (v in N+(u)).
__device__ __forceinline__ uint64_t edge_index(const uint64_t *__restrict__ off,
                                               const uint32_t *__restrict__ col, uint32_t u, uint32_t v) {
    uint64_t b = off[u];
    return b + list_pos(col + b, (uint32_t)(off[u + 1] - b), v);
}

// kCmList: triangle {a, b, c} (rank ids) -> slot s as ascending input ids (if s < cap).
__device__ __forceinline__ void put_triangle(const Credit &cr, uint64_t s, uint32_t a, uint32_t b,
                                             uint32_t c) {
    if (s >= cr.cap) return;
    uint32_t x = cr.order[a], y = cr.order[b], z = cr.order[c];
    uint32_t lo = min(x, min(y, z)), hi = max(x, max(y, z));
    uint32_t* t = cr.tri + 3 * s;
    t[0] = lo;
    t[1] = x ^ y ^ z ^ lo ^ hi;
    t[2] = hi;
}

// ------------------------------------------------------------------ SHORT
// Two-pointer merge of col+[i, ie) and col+[j, je); hit(i, j, w) per common w.
template <class Hit>
__device__ __forceinline__ uint32_t merge_short(const uint32_t *__restrict__ col, uint64_t i, uint64_t ie,
                                                uint64_t j, uint64_t je, Hit hit) {
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
                hit(i, j, a);
                if (++i == ie || ++j == je) break;
                a = col[i];
                b = col[j];
            }
        }
    }
    return c;
}

template <int CM>
__global__ void __launch_bounds__(kIxThreads)
    k_short(const uint2 *__restrict__ edges, const uint64_t *__restrict__ count,
            const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
            uint64_t *__restrict__ total, Credit cr) {
    uint64_t ne = *count;
    uint64_t acc = 0;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint2 uv = edges[e];
        uint64_t i = off[uv.x], ie = off[uv.x + 1], j = off[uv.y], je = off[uv.y + 1];
        uint32_t c = merge_short(col, i, ie, j, je, [&](uint64_t pi, uint64_t pj, uint32_t w) {
            if (CM == kCmVertex) atomicAdd((unsigned long long *)&cr.pv[w], 1ull);
            if (CM == kCmEdge) {
                atomicAdd(&cr.sup[pi], 1u);
                atomicAdd(&cr.sup[pj], 1u);
            }
            if (CM == kCmTop) atomicAdd(&cr.sup[pj], 1u);   // (v, w): u < v < w
        });
        credit_edge<CM>(cr, uv.x, uv.y, c);
        if (CM == kCmEdge && c) atomicAdd(&cr.sup[edge_index(off, col, uv.x, uv.y)], c);
        if (CM == kCmList && c) {  // reserve c slots, then merge again to write them
            uint64_t s = atomicAdd((unsigned long long *)cr.cursor, (unsigned long long)c);
            merge_short(col, i, ie, j, je,
                        [&](uint64_t, uint64_t, uint32_t w) { put_triangle(cr, s++, uv.x, uv.y, w); });
        }
        acc += c;
    }
    flush_count(acc, total);
}

// ------------------------------------------------------------------ MERGE
// Merge path of A (len na) and B (len nb), rule "take A[i] when A[i] <= B[j]".
// Lane l walks diagonals [k0, k1); a match is counted when A[i] is taken and
// B[j] == A[i] (B[j] is then the first element of B >= A[i]), so every common
// element is counted exactly once across lanes.
template <int CM>
__global__ void __launch_bounds__(kIxThreads)
    k_merge(const uint2 *__restrict__ edges, const uint64_t *__restrict__ count,
            const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
            uint64_t *__restrict__ total, Credit cr) {
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
        auto walk = [&](auto hit) {
            uint32_t i = lo, j = k0 - lo, c = 0;
            for (uint32_t k = k0; k < k1; k++) {
                if (j >= nb || (i < na && A[i] <= B[j])) {
                    if (j < nb && A[i] == B[j]) {
                        c++;
                        hit(i, j, A[i]);
                    }
                    i++;
                } else {
                    j++;
                }
            }
            return c;
        };
        const uint64_t ab = off[uv.x], bb = off[uv.y];
        uint32_t c = walk([&](uint32_t i, uint32_t j, uint32_t w) {
            if (CM == kCmVertex) atomicAdd((unsigned long long *)&cr.pv[w], 1ull);
            if (CM == kCmEdge) {
                atomicAdd(&cr.sup[ab + i], 1u);
                atomicAdd(&cr.sup[bb + j], 1u);
            }
            if (CM == kCmTop) atomicAdd(&cr.sup[bb + j], 1u);   // B = N+(v)
        });
        if (CM == kCmVertex || CM == kCmEdge) {
            uint32_t ce = __reduce_add_sync(0xffffffffu, c);
            if (lane == 0) credit_edge<CM>(cr, uv.x, uv.y, ce);
            if (CM == kCmEdge && lane == 0 && ce) atomicAdd(&cr.sup[edge_index(off, col, uv.x, uv.y)], ce);
        }
        if (CM == kCmList && c) {
            uint64_t s = atomicAdd((unsigned long long *)cr.cursor, (unsigned long long)c);
            walk([&](uint32_t, uint32_t, uint32_t w) { put_triangle(cr, s++, uv.x, uv.y, w); });
        }
        acc += c;
    }
    flush_count(acc, total);
}

// ------------------------------------------------------------------ SEARCH
template <int CM>
__global__ void __launch_bounds__(kIxThreads)
    k_search(const uint2 *__restrict__ edges, const uint64_t *__restrict__ count,
             const uint64_t *__restrict__ off, const uint32_t *__restrict__ col,
             uint64_t *__restrict__ total, Credit cr) {
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
        const bool swapped = na > nb;   // then A = N+(v)
        if (na > nb) {  // A := the shorter list
            const uint32_t *t = A; A = B; B = t;
            uint32_t tn = na; na = nb; nb = tn;
        }
        auto scan = [&](auto hit) {
            uint32_t c = 0;
            for (uint32_t k = lane; k < na; k += 32) {
                uint32_t x = A[k], lo = 0, hi = nb;
                while (lo < hi) {
                    uint32_t mid = (lo + hi) >> 1;
                    if (B[mid] < x) lo = mid + 1; else hi = mid;
                }
                if (lo < nb && B[lo] == x) {
                    c++;
                    hit(k, lo, x);
                }
            }
            return c;
        };
        uint32_t c = scan([&](uint32_t k, uint32_t l, uint32_t w) {
            if (CM == kCmVertex) atomicAdd((unsigned long long *)&cr.pv[w], 1ull);
            if (CM == kCmEdge) {
                atomicAdd(&cr.sup[A - col + k], 1u);
                atomicAdd(&cr.sup[B - col + l], 1u);
            }
            if (CM == kCmTop) atomicAdd(&cr.sup[swapped ? A - col + k : B - col + l], 1u);
        });
        if (CM == kCmVertex || CM == kCmEdge) {
            uint32_t ce = __reduce_add_sync(0xffffffffu, c);
            if (lane == 0) credit_edge<CM>(cr, uv.x, uv.y, ce);
            if (CM == kCmEdge && lane == 0 && ce) atomicAdd(&cr.sup[edge_index(off, col, uv.x, uv.y)], ce);
        }
        if (CM == kCmList && c) {
            uint64_t s = atomicAdd((unsigned long long *)cr.cursor, (unsigned long long)c);
            scan([&](uint32_t, uint32_t, uint32_t w) { put_triangle(cr, s++, uv.x, uv.y, w); });
        }
        acc += c;
    }
    flush_count(acc, total);
}

// ------------------------------------------------------------------ HASH
// Owner x's list N+(x) (the longer one of each of its edges) lives in a
// shared-memory hash table (load factor <= 1/2, multiplicative hash, buckets of
// 4 slots read with one 16-byte shared load, linear probing over buckets).
// For each probe vertex y of x every element w of N+(y) is looked up; a hit is
// the triangle {x, y, w}.
// A task = (owner, up to L probe lists).  The task's list descriptors go to
// shared memory (exclusive prefix of lengths, start - prefix, id), the items of
// all its lists are flattened, and each warp takes an equal contiguous item
// range.  In each 32-item window lane t finds its list from a bitmap of the list
// starts inside the window (reduce-or + popc): no per-item search.
constexpr uint32_t kHashSlots = 4096;  // CTA table capacity (power of two), 16 KB
constexpr uint32_t kHashChunk = 1024;  // owner elements per table build (load factor <= 1/4)
#ifndef TC_BITMAP_REUSE
#define TC_BITMAP_REUSE 1
#endif
#ifndef TC_HASH_UNROLL
#define TC_HASH_UNROLL 1
#endif
#ifndef TC_HASH_WARP_MINBLOCKS
#define TC_HASH_WARP_MINBLOCKS 1
#endif
#ifndef TC_HASH_CTA_MINBLOCKS
#define TC_HASH_CTA_MINBLOCKS 8
#endif
#ifndef TC_HASH_PREFETCH
#define TC_HASH_PREFETCH 0
#endif
#ifndef TC_HASH_RR
#define TC_HASH_RR 0   // measured: round-robin windows s21 a6 2.50 vs contiguous shares 2.26 ms
#endif
constexpr int kUnroll = TC_HASH_UNROLL;  // independent 32-slot windows per probe step
constexpr uint32_t kCtaStride = TC_HASH_RR ? 32u * (kIxThreads / 32) : 32u;   // window stride of a CTA task's warps
constexpr int kHashWarps = kIxThreads / 32;

// Explicit shared-memory accesses on 32-bit shared addresses (keeps the hot
// loop free of generic-address conversions).
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t hash_slot(uint32_t x, int bits) {
    return (x * 0x9E3779B1u) >> (32 - bits);
}

// Table of 2^bits slots (>= 4 * len: load factor <= 1/4) = 2^(bits-2) buckets of 4.
__device__ __forceinline__ int table_bits(uint32_t len) {
    int bits = 5;
    while ((1u << bits) < 4 * len) bits++;
    return bits;
}

// Build: `nthreads` cooperating threads (index `tid`) insert keys[0..len).  A key
// goes to the first free slot of its home bucket or of the following buckets;
// within a bucket slots fill in order, so a bucket with an EMPTY slot ends every
// probe sequence that reaches it.
__device__ __forceinline__ void table_insert(uint32_t *tab, int bits, const uint32_t *__restrict__ keys,
                                             uint32_t len, uint32_t tid, uint32_t nthreads) {
    uint32_t bmask = (1u << (bits - 2)) - 1u;
    for (uint32_t k = tid; k < len; k += nthreads) {
        uint32_t x = keys[k], b = hash_slot(x, bits - 2);
        while (true) {
            uint32_t *slot = tab + 4 * b;
            if (atomicCAS(slot + 0, kEmpty, x) == kEmpty) break;
            if (atomicCAS(slot + 1, kEmpty, x) == kEmpty) break;
            if (atomicCAS(slot + 2, kEmpty, x) == kEmpty) break;
            if (atomicCAS(slot + 3, kEmpty, x) == kEmpty) break;
            b = (b + 1) & bmask;
        }
    }
}

// Rare slow path: w's home bucket was full and did not hold it.
__device__ __noinline__ uint32_t table_contains_slow(uint32_t tab, uint32_t bmask, uint32_t b,
                                                     uint32_t w) {
    while (true) {
        b = (b + 1) & bmask;
        uint4 q = lds128(tab + 16 * b);
        if (q.x == w || q.y == w || q.z == w || q.w == w) return 1u;
        if (q.w == kEmpty) return 0u;
    }
}

// Slot index of w, which is known to be in the table (per-vertex credits).
__device__ __forceinline__ uint32_t table_find(uint32_t tab, int bits, uint32_t w) {
    uint32_t bmask = (1u << (bits - 2)) - 1u, b = hash_slot(w, bits - 2);
    while (true) {
        uint4 q = lds128(tab + 16 * b);
        if (q.x == w) return 4 * b;
        if (q.y == w) return 4 * b + 1;
        if (q.z == w) return 4 * b + 2;
        if (q.w == w) return 4 * b + 3;
        b = (b + 1) & bmask;
    }
}

// 1 if w is in the table at shared address `tab`.
__device__ __forceinline__ uint32_t table_contains(uint32_t tab, int bits, uint32_t w) {
    uint32_t b = hash_slot(w, bits - 2);
    uint4 q = lds128(tab + 16 * b);
    bool hit = q.x == w || q.y == w || q.z == w || q.w == w;
    if (hit || q.w == kEmpty) return hit;  // slots fill in order: a free last slot ends the search
    return table_contains_slow(tab, (1u << (bits - 2)) - 1u, b, w);
}

// Probe-list loads: read-only path, L1-allocating (48 % L1 hits at s21; the
// L1::no_allocate hint measured slower).
__device__ __forceinline__ uint4 ld_probe(const uint4 *p) { return __ldg(p); }

// Keep a shared-memory base address in a register (stops the compiler from
// re-deriving it from SR_CgaCtaId at every use).
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}

// Membership tests used by probe_quads.
// Membership tests used by probe_quads: key(e, valid) maps a loaded element (or a
// masked slot outside the probe range) to a probe key; test(key) answers 0/1.
struct HashProbe {  // bucket hash of the owner's N+ (any id range)
    uint32_t tab, absent;  // absent = the owner itself: never in its own N+
    int bits;
    // per-vertex / edge mode: hit counters per table slot (cnt != nullptr), else global atomics
    uint32_t *cnt = nullptr;
    const uint32_t *xl = nullptr;  // edge mode without counters: the owner's N+ (col+ at xb)
    uint32_t xlen = 0;
    uint64_t xb = 0;
    // bit c set iff element c of the slot is in the list (rel + c < len, mod 2^32)
    // and in the table
    template <int N>
    __device__ __forceinline__ uint32_t hit_mask(const uint32_t (&e)[N], uint32_t rel,
                                                 uint32_t len) const {
        uint32_t h = 0;
#pragma unroll
        for (int c = 0; c < N; c++)
            h |= table_contains(tab, bits, rel + c < len ? e[c] : absent) << c;
        return h;
    }
    // owner-side credit of a hit w: t(w) (vertex mode) or sup(owner, w) (edge mode)
    template <int CM>
    __device__ __forceinline__ void credit(uint32_t w, const Credit &cr) const {
        if (!cnt) {
            if (CM == kCmVertex) atomicAdd((unsigned long long *)&cr.pv[w], 1ull);
            if (CM == kCmEdge || CM == kCmTop) atomicAdd(&cr.sup[xb + list_pos(xl, xlen, w)], 1u);
            return;
        }
        atomicAdd(&cnt[table_find(tab, bits, w)], 1u);
    }
};
struct BitProbe {   // bitmap over the rank-id range [base, base + span) of the owner's N+
    // Any element e of col+ maps to bit min(e - base, zero) (mod 2^32): ids below base
    // wrap high and land on `zero`, a bit of the spare all-zero word after the bitmap,
    // so no load leaves the bitmap; elements outside the slot's list range are then
    // removed by a per-slot mask instead of a per-element select.
    uint32_t bm, base, zero;
    // per-vertex mode: hits of w are counted in shared memory at w's rank among the
    // owner's set bits (wpre = per-word prefix popcounts) when cnt != nullptr
    uint32_t *cnt = nullptr;
    const uint16_t *wpre = nullptr;
    const uint32_t *xl = nullptr;  // edge mode without counters: the owner's N+ (col+ at xb)
    uint32_t xlen = 0;
    uint64_t xb = 0;
    template <int N>
    __device__ __forceinline__ uint32_t hit_mask(const uint32_t (&e)[N], uint32_t rel,
                                                 uint32_t len) const {
        static_assert(N <= 32, "slot hit vector is one word");
        uint32_t hv = 0;
#if TC_BITMAP_REUSE
        // A slot's elements are consecutive entries of a sorted row, so neighbours often
        // share a bitmap word: load a word only when its index changes (the other lanes
        // sit the load out, so the shared-memory wavefronts of each probe drop).
        uint32_t wi_prev = 0xffffffffu, w = 0;
#endif
#pragma unroll
        for (int c = 0; c < N; c++) {
            uint32_t o = min(e[c] - base, zero);
#if TC_BITMAP_REUSE
            const uint32_t wi = o >> 5;
            if (wi != wi_prev) w = lds32(bm + 4 * wi);
            wi_prev = wi;
#else
            uint32_t w = lds32(bm + 4 * (o >> 5));
#endif
            // rotate bit (o & 31) of w to position c, collect it in hv
            hv |= __funnelshift_r(w, w, o - c) & (1u << c);
        }
        // valid elements: c in [a, b).  rel < len: the slot starts inside the list,
        // a = 0, b = min(N, hi - e0); else it starts before lo (a = min(N, lo - e0),
        // b = min(N, hi - e0)) or at/after hi (a = N: none); len == 0 (masked lane): none
        uint32_t a = rel < len ? 0u : min((uint32_t)N, 0u - rel);
        uint32_t b = min((uint32_t)N, len - rel);
        uint32_t m = len ? ((1u << b) - 1u) & ~((1u << a) - 1u) : 0u;
        return hv & m;
    }
    template <int CM>
    __device__ __forceinline__ void credit(uint32_t w, const Credit &cr) const {
        if (!cnt) {
            if (CM == kCmVertex) atomicAdd((unsigned long long *)&cr.pv[w], 1ull);
            if (CM == kCmEdge || CM == kCmTop) atomicAdd(&cr.sup[xb + list_pos(xl, xlen, w)], 1u);
            return;
        }
        uint32_t o = w - base, word = lds32(bm + 4 * (o >> 5));
        uint32_t idx = wpre[o >> 5] + __popc(word & ((1u << (o & 31)) - 1u));
        atomicAdd(&cnt[idx], 1u);
    }
};

// Probe-list descriptors in shared memory, in QUAD space: list i covers the
// aligned 16-byte quads [qlo_i, qhi_i) of col+ that overlap its element range
// [lo_i, hi_i).  s_pre[i] = exclusive prefix of quad counts (s_pre[nl] = total),
// pk[i] = {qlo_i - s_pre[i] (mod 2^32), lo_i, hi_i, vid_i}: one 16-byte shared load per
// window (measured ~1.5 % faster than separate qb / rng / vid arrays).  All offsets fit
// in 32 bits (the host routes graphs with >= 2^32 oriented edges away).
struct QuadDesc {
    uint32_t *pre;
    uint4 *pk;
};

// Probe slots are aligned groups of kSlot elements of col+ (kSlot / 4 128-bit loads).
#ifndef TC_SLOT_SHIFT
#define TC_SLOT_SHIFT 3
#endif
constexpr int kSlotShift = TC_SLOT_SHIFT;
constexpr int kSlot = 1 << kSlotShift;

__device__ __forceinline__ void put_desc(const QuadDesc &d, uint32_t i, uint32_t lo, uint32_t hi,
                                         uint32_t pre, uint32_t y, bool pv) {
    d.pre[i] = pre;
    d.pk[i] = make_uint4((lo >> kSlotShift) - pre, lo, hi, pv ? y : 0u);
}

__device__ __forceinline__ uint32_t quad_count(uint32_t lo, uint32_t hi) {
    return ((hi + kSlot - 1) >> kSlotShift) - (lo >> kSlotShift);
}

// The calling warp probes quads [ib, ie) of the flattened quad space: one aligned
// uint4 load and four probes per lane per window.  In each 32-quad window lane t
// finds its list from a bitmap of the list starts inside the window (reduce-or +
// popc): no per-item search.  Returns the number of hits.
// kCmList: the hits are staged per warp in shared memory as (list vertex, w) input-id
// pairs (kStage of them; the owner is common to the task) and written out as one
// contiguous run of ascending triples per flush, with ONE global slot reservation.
constexpr uint32_t kStage = 256;   // >= the hits of one window (32 lanes x kSlot)

__device__ __forceinline__ void flush_stage(const uint2 *stage, uint32_t staged, uint32_t b,
                                            const Credit &cr) {
    const uint32_t lane = threadIdx.x & 31;
    __syncwarp();
    uint64_t base = 0;
    if (lane == 0) base = atomicAdd((unsigned long long *)cr.cursor, (unsigned long long)staged);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (uint32_t i = lane; i < staged; i += 32) {
        if (base + i >= cr.cap) break;
        const uint2 aw = stage[i];
        const uint32_t lo3 = min(aw.x, min(b, aw.y)), hi3 = max(aw.x, max(b, aw.y));
        uint32_t *t = cr.tri + 3 * (base + i);
        t[0] = lo3;
        t[1] = aw.x ^ b ^ aw.y ^ lo3 ^ hi3;
        t[2] = hi3;
    }
    __syncwarp();
}

template <int CM, class Probe>
__device__ __forceinline__ uint64_t probe_quads(const Probe &contains,
                                                const QuadDesc &d, uint32_t nl, uint32_t ib,
                                                uint32_t ie,
                                                const uint32_t *__restrict__ col,
                                                uint32_t owner, const Credit &cr,
                                                uint2 *stage = nullptr,
                                                uint32_t stride = 32 * kUnroll) {
    uint32_t staged = 0, ord_owner = 0;
    if (CM == kCmList) ord_owner = cr.order[owner];
    const int lane = threadIdx.x & 31;
    uint32_t hits = 0;
    if (ib >= ie) return 0;   // warp-uniform: nothing staged
    uint32_t lo = 0, hi = nl;  // i0 = the list containing quad ib
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (d.pre[mid] <= ib) lo = mid; else hi = mid;
    }
    uint32_t i0 = lo;
    const uint32_t le_mask = (2u << lane) - 1u;
    const uint4 *col4 = reinterpret_cast<const uint4 *>(col);
    for (uint32_t wb = ib; wb < ie; wb += stride) {
        if (stride > 32 * kUnroll && wb != ib) {   // strided windows: the list holding quad wb,
            uint32_t lo2 = i0, hi2 = nl;          // searched from the previous window's last
            while (hi2 - lo2 > 1) {
                const uint32_t mid = (lo2 + hi2) >> 1;
                if (d.pre[mid] <= wb) lo2 = mid; else hi2 = mid;
            }
            i0 = lo2;
        }
        uint4 q[kUnroll][kSlot / 4];
        uint2 r[kUnroll];
        uint32_t e0[kUnroll], ly[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; k++) {
            uint32_t wk = wb + 32 * k;
            uint32_t j = i0 + 1 + lane;           // candidate list starts after list i0
            uint32_t s = (j < nl ? d.pre[j] : 0xffffffffu) - wk;
            uint32_t starts = __reduce_or_sync(0xffffffffu, s < 32 ? (1u << s) : 0u);
            uint32_t li = i0 + __popc(starts & le_mask);
            const uint32_t t = wk + lane;
            const bool live = t < ie;
            // lanes past ie load slot 0 of col+ (always allocated, >= 256 bytes) and are
            // masked by an empty range
            const uint4 dd = d.pk[li];
            uint32_t qi = live ? dd.x + t : 0u;
            r[k] = make_uint2(dd.y, dd.z);
            ly[k] = dd.w;
            if (!live) r[k].y = r[k].x;
            e0[k] = qi << kSlotShift;
#pragma unroll
            for (int v = 0; v < kSlot / 4; v++) q[k][v] = ld_probe(col4 + (uint64_t)qi * (kSlot / 4) + v);
            i0 = __shfl_sync(0xffffffffu, li, 31);  // list holding slot wk + 31
#if TC_HASH_PREFETCH
            {   // this lane's slot of the NEXT window, found the same way, prefetched into L1 so
                // its loads hit while this window is probed (no registers held across)
                const uint32_t wn = wk + 32 * kUnroll, jn = i0 + 1 + lane;
                const uint32_t sn = (jn < nl ? d.pre[jn] : 0xffffffffu) - wn;
                const uint32_t stn = __reduce_or_sync(0xffffffffu, sn < 32 ? (1u << sn) : 0u);
                const uint32_t tn = wn + lane;
                if (tn < ie) {
                    const uint32_t qn = d.pk[i0 + __popc(stn & le_mask)].x + tn;
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(col4 + (uint64_t)qn * (kSlot / 4)));
                }
            }
#endif
        }
#pragma unroll
        for (int k = 0; k < kUnroll; k++) {
            const uint32_t rel = e0[k] - r[k].x, len = r[k].y - r[k].x;  // mod 2^32
            uint32_t e[kSlot];
#pragma unroll
            for (int v = 0; v < kSlot / 4; v++) {
                e[4 * v + 0] = q[k][v].x;
                e[4 * v + 1] = q[k][v].y;
                e[4 * v + 2] = q[k][v].z;
                e[4 * v + 3] = q[k][v].w;
            }
            const uint32_t hm = contains.hit_mask(e, rel, len);
            hits += __popc(hm);
            if (CM == kCmVertex && hm) {
#pragma unroll
                for (int c = 0; c < kSlot; c++)
                    if ((hm >> c) & 1u) contains.template credit<CM>(e[c], cr);
                atomicAdd((unsigned long long *)&cr.pv[ly[k]], (unsigned long long)__popc(hm));
            }
            if (CM == kCmEdge && hm) {   // (list vertex, w) at its col+ slot; base edge ly
#pragma unroll
                for (int c = 0; c < kSlot; c++)
                    if ((hm >> c) & 1u) {
                        contains.template credit<CM>(e[c], cr);
                        atomicAdd(&cr.sup[e0[k] + c], 1u);
                    }
                atomicAdd(&cr.sup[ly[k]], (uint32_t)__popc(hm));
            }
            if (CM == kCmTop && hm) {
                // in-part entry (ly = 0): list N+(u) after owner x, triangle u < x < w, top
                // edge (x, w) = the owner's element; out-part entry (ly = 1): owner u, list
                // N+(x), top edge (x, w) = the probed slot
#pragma unroll
                for (int c = 0; c < kSlot; c++)
                    if ((hm >> c) & 1u) {
                        if (ly[k]) atomicAdd(&cr.sup[e0[k] + c], 1u);
                        else contains.template credit<CM>(e[c], cr);
                    }
            }
            if (CM == kCmList) {         // stage as ascending input ids, flush when full
                const uint32_t nh = __popc(hm);
                const uint32_t incl = warp_inclusive_scan<SumOp>(nh);
                const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
                if (staged + tot > kStage) {
                    flush_stage(stage, staged, ord_owner, cr);
                    staged = 0;
                }
                if (hm) {
                    uint32_t pos = staged + incl - nh;
                    const uint32_t a = cr.order[ly[k]];
#pragma unroll
                    for (int c = 0; c < kSlot; c++)
                        if ((hm >> c) & 1u) stage[pos++] = make_uint2(a, cr.order[e[c]]);
                }
                staged += tot;
            }
        }
    }
    if (CM == kCmList && staged) flush_stage(stage, staged, ord_owner, cr);
    return hits;
}

// Probe entry j of HASH owner x (bin.cu header): j < indeg -> the j-th in-edge
// (u -> x) of x's in-list, range = N+(u) after x (empty if x does not own it), y = u;
// else the (j - indeg)-th compacted out-part entry of x: range = N+(v), y = v.
// Edge mode: y = the CSR index of the entry's own edge instead (in-part: lo - 1;
// out-part: ovid holds edge indices, bin_edges' edge_ids).
template <int CM>
__device__ __forceinline__ void hash_desc(const HashParams &hp, uint64_t inb, uint32_t indeg,
                                          uint64_t ob, uint32_t ocnt, uint32_t j, uint32_t &lo,
                                          uint32_t &hi, uint32_t &y) {
    lo = hi = y = 0;
    if (j < indeg) {
        const uint32_t suf = hp.ulo[inb + j];   // probe length (0: not this owner's entry)
        uint32_t u = hp.in_src[inb + j];
        if (suf) {
            hi = (uint32_t)hp.off[u + 1];
            lo = hi - suf;
        }
        y = CM == kCmEdge ? lo - 1 : (CM == kCmTop ? 0u : u);
    } else if (j - indeg < ocnt) {
        uint2 r = hp.orange[ob + (j - indeg)];
        y = CM == kCmTop ? 1u : hp.ovid[ob + (j - indeg)];
        lo = r.x;
        hi = r.y;
    }
}

// Warp tasks: owners with d+(x) <= kWarpTableSlots/4 (table in the warp's smem slice).
template <int CM>
__global__ void __launch_bounds__(kIxThreads, TC_HASH_WARP_MINBLOCKS)
    k_hash_warp(const uint4 *__restrict__ tasks, const uint64_t *__restrict__ ntasks, HashParams hp,
                uint64_t *__restrict__ total, Credit cr) {
    constexpr uint32_t L = kWarpTaskLists;
    constexpr bool PV = CM != kCmNone;                        // descriptors carry vid
    constexpr bool kCnt = CM == kCmVertex || CM == kCmEdge || CM == kCmTop;  // owner-side hits
    __shared__ __align__(16) uint32_t s_tab[kHashWarps][kWarpTableSlots];
    __shared__ uint4 s_pk[kHashWarps][L];
    __shared__ uint32_t s_pre[kHashWarps][L + 1];
    __shared__ uint32_t s_cnt[kCnt ? kHashWarps : 1][kCnt ? kWarpTableSlots : 1];  // owner hits per slot
    __shared__ uint2 s_stage[CM == kCmList ? kHashWarps : 1][CM == kCmList ? kStage : 1];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const QuadDesc d{s_pre[wib], s_pk[wib]};
    uint64_t nt = *ntasks;
    uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t *tab = s_tab[wib];
    const uint32_t *col = hp.col;
    uint64_t acc = 0;
    for (uint64_t i = gw; i < nt; i += nw) {
        const uint4 t0 = tasks[2 * i], t1 = tasks[2 * i + 1];   // bin.cu k_task_expand
        const uint32_t x = t0.x, j0 = t0.y, dx = t0.z, indeg = t0.w, ocnt = t1.w;
        const uint64_t xb = t1.x, inb = t1.y, ob = t1.z;
        // descriptors of entries j0 + lane, j0 + 32 + lane; non-empty ones compacted in
        // order (the list-start bitmap of probe_quads needs distinct starts)
        uint32_t run = 0, nl = 0;
#pragma unroll
        for (uint32_t h = 0; h < L; h += 32) {
            uint32_t lo = 0, hi = 0, y = 0;
            hash_desc<CM>(hp, inb, indeg, ob, ocnt, j0 + h + lane, lo, hi, y);
            uint32_t nq = quad_count(lo, hi);
            uint32_t inc = warp_inclusive_scan<SumOp>(nq);
            uint32_t keep = __ballot_sync(0xffffffffu, nq != 0);
            if (nq) put_desc(d, nl + __popc(keep & ((1u << lane) - 1u)), lo, hi, run + inc - nq, y, PV);
            run += __shfl_sync(0xffffffffu, inc, 31);
            nl += __popc(keep);
        }
        if (lane == 0) d.pre[nl] = run;
        int bits = table_bits(dx);
        for (uint32_t s = lane; s < (1u << bits); s += 32) {
            tab[s] = kEmpty;
            if (kCnt) s_cnt[wib][s] = 0u;
        }
        __syncwarp();
        table_insert(tab, bits, col + xb, dx, lane, 32);
        __syncwarp();
        HashProbe hpb{opaque(smem_addr(tab)), x, bits};
        if (kCnt) hpb.cnt = s_cnt[wib];
        uint64_t h = probe_quads<CM>(hpb, d, nl, 0, run, col, x, cr, s_stage[CM == kCmList ? wib : 0]);
        if (kCnt) {
            __syncwarp();
            for (uint32_t s = lane; s < (1u << bits); s += 32) {
                uint32_t c = s_cnt[wib][s];
                if (!c) continue;
                if (CM == kCmVertex) atomicAdd((unsigned long long *)&cr.pv[tab[s]], (unsigned long long)c);
                if (CM == kCmEdge || CM == kCmTop) atomicAdd(&cr.sup[xb + list_pos(col + xb, dx, tab[s])], c);
            }
        }
        if (CM == kCmVertex) {
            uint64_t hw = warp_sum_u64(h);
            if (lane == 0 && hw) atomicAdd((unsigned long long *)&cr.pv[x], (unsigned long long)hw);
        }
        acc += h;
        __syncwarp();
    }
    flush_count(acc, total);
}

// CTA tasks: large owners ("hubs"); the task's items are split evenly over the warps.
// kBitmap: the owner's N+ (rank ids in (x, n)) is a bitmap over [x+1, n) -- one
// 32-bit shared load per probe; otherwise the bucket hash (chunked if d+ > 2048).
constexpr uint32_t kSmemWords = kHashSlots;            // 16 KB of table / bitmap per CTA
static_assert(kCtaTaskLists * kBitmapBatches == kBitmapTaskLists, "bitmap task size (bin.cu)");
constexpr uint32_t kPvCounters = 4096;                 // per-vertex: smem hit counters (16 KB)
static_assert(kCtaBitmapBits == kSmemWords * 32, "bitmap owners are classified in bin.cu");
template <int CM, bool kBitmap>
__global__ void __launch_bounds__(kIxThreads, CM != kCmNone ? 4 : TC_HASH_CTA_MINBLOCKS)
    k_hash_cta(const uint4 *__restrict__ tasks, const uint64_t *__restrict__ ntasks, HashParams hp,
               uint64_t *__restrict__ total, Credit cr) {
    constexpr uint32_t L = kCtaTaskLists;
    constexpr bool PV = CM != kCmNone;   // descriptors carry vid
    static_assert(L == kIxThreads, "one descriptor per thread");
    __shared__ __align__(16) uint32_t s_tab[kSmemWords];
    __shared__ uint4 s_pk[L];
    __shared__ uint32_t s_pre[L + 1];
    __shared__ uint64_t s_scan[kHashWarps];
    // per-vertex bitmap owners: hit counters per element of N+(x) (owners with
    // d+ <= kPvCounters; others credit w with global atomics) + word prefix popcounts
    constexpr bool kCnt = CM == kCmVertex || CM == kCmEdge || CM == kCmTop;  // per set bit / slot
    static_assert(kPvCounters == kHashSlots, "hash owners count hits per table slot");
    __shared__ uint32_t s_cnt[kCnt ? kPvCounters : 1];
    __shared__ uint16_t s_wpre[kCnt && kBitmap ? kSmemWords + 1 : 1];
    __shared__ uint2 s_stage[CM == kCmList ? kHashWarps : 1][CM == kCmList ? kStage : 1];
    uint2 *stage = s_stage[CM == kCmList ? (threadIdx.x >> 5) : 0];
    const int wib = threadIdx.x >> 5;
    const QuadDesc d{s_pre, s_pk};
    const uint32_t tab = opaque(smem_addr(s_tab));
    const uint32_t *col = hp.col;
    const uint32_t n = hp.n;
    uint64_t nt = *ntasks;
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x; i < nt; i += gridDim.x) {
        const uint4 t0 = tasks[2 * i], t1 = tasks[2 * i + 1];   // bin.cu k_task_expand
        const uint32_t x = t0.x, j_task = t0.y, dx = t0.z, indeg = t0.w, ocnt = t1.w;
        const uint64_t xb = t1.x, inb = t1.y, ob = t1.z;
        uint64_t h = 0;
        // descriptors of the probe entries j0 + threadIdx.x (one per thread), compacted, and
        // this warp's equal share [ib, ie) of their quads
        uint32_t nl = 0, ib = 0, ie = 0;
        auto batch = [&](uint32_t j0) {
            uint32_t lo, hi, y;
            hash_desc<CM>(hp, inb, indeg, ob, ocnt, j0 + threadIdx.x, lo, hi, y);
            uint32_t nq = quad_count(lo, hi);
            // one 64-bit scan: high word = compacted index of non-empty entries, low = quads
            uint64_t tot;
            uint64_t pre = block_exclusive_scan<SumOp64>(((uint64_t)(nq != 0) << 32) | nq, s_scan, &tot);
            const uint32_t items = (uint32_t)tot;
            nl = (uint32_t)(tot >> 32);
            if (nq) put_desc(d, (uint32_t)(pre >> 32), lo, hi, (uint32_t)pre, y, PV);
            if (threadIdx.x == 0) d.pre[nl] = items;
#if TC_HASH_RR
            // windows of 32 slots dealt round-robin to the warps (full windows even for small
            // tasks; contiguous per-warp shares left most lanes of a small task's windows idle)
            ib = 32u * wib;
            ie = items;
#else
            ib = (uint32_t)(((uint64_t)items * wib) / kHashWarps);
            ie = (uint32_t)(((uint64_t)items * (wib + 1)) / kHashWarps);
#endif
            __syncthreads();   // every descriptor is written before any warp probes
        };
        if (kBitmap) {
            // N+(x) lies in [lo_x, hi_x] (its first and last element, rows ascending): bits
            // [0, span) for ids lo_x .. hi_x, then one spare zero word; every other id maps to it
#if TC_BITMAP_EFFSPAN
            const uint32_t base = col[xb], span = col[xb + dx - 1] - base + 1, words = span / 32 + 1;
#else
            const uint32_t base = x + 1, span = n - 1 - x, words = span / 32 + 1;
#endif
            for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) s_tab[w] = 0u;
            __syncthreads();
            for (uint32_t k = threadIdx.x; k < dx; k += blockDim.x) {
                uint32_t o = col[xb + k] - base;
                atomicOr(&s_tab[o >> 5], 1u << (o & 31));
            }
            // (the first batch's block scan below orders these writes before any probe)
            BitProbe bp{tab, base, (words - 1) * 32 + 31};
            bp.xl = col + xb;
            bp.xlen = dx;
            bp.xb = xb;
            const bool use_cnt = kCnt && kBitmap && dx <= kPvCounters;
            if (use_cnt) {
                __syncthreads();   // the bitmap is complete before its words are counted
                // exclusive prefix popcount per bitmap word (blocked: thread t owns a run)
                const uint32_t per = (words + kIxThreads - 1) / kIxThreads;
                const uint32_t w0 = min(words, threadIdx.x * per), w1 = min(words, w0 + per);
                uint32_t c = 0;
                for (uint32_t w = w0; w < w1; w++) c += __popc(s_tab[w]);
                uint32_t run = (uint32_t)block_exclusive_scan<SumOp64>((uint64_t)c, s_scan);
                for (uint32_t w = w0; w < w1; w++) {
                    s_wpre[w] = (uint16_t)run;
                    run += __popc(s_tab[w]);
                }
                for (uint32_t k = threadIdx.x; k < dx; k += blockDim.x) s_cnt[k] = 0u;
                __syncthreads();
                bp.cnt = s_cnt;
                bp.wpre = s_wpre;
            }
            // one bitmap serves up to kBitmapBatches batches of kCtaTaskLists probe entries
            const uint32_t npe = indeg + ocnt;
            for (uint32_t bt = 0; bt < kBitmapBatches; bt++) {
                const uint32_t j0 = j_task + bt * L;
                if (j0 >= npe) break;   // block-uniform
                batch(j0);
                h += probe_quads<CM>(bp, d, nl, ib, ie, col, x, cr, stage, kCtaStride);
                __syncthreads();   // descriptors are rewritten by the next batch
            }
            if (use_cnt) {   // the k-th set bit is the k-th element of the sorted N+(x)
                for (uint32_t k = threadIdx.x; k < dx; k += blockDim.x) {
                    uint32_t c = s_cnt[k];
                    if (!c) continue;
                    if (CM == kCmVertex) atomicAdd((unsigned long long *)&cr.pv[col[xb + k]], (unsigned long long)c);
                    if (CM == kCmEdge || CM == kCmTop) atomicAdd(&cr.sup[xb + k], c);
                }
                __syncthreads();
            }
        } else {
            batch(j_task);
            for (uint32_t c0 = 0; c0 < dx; c0 += kHashChunk) {
                uint32_t clen = min(kHashChunk, dx - c0);
                int bits = table_bits(clen);
                for (uint32_t s = threadIdx.x; s < (1u << bits); s += blockDim.x) {
                    s_tab[s] = kEmpty;
                    if (kCnt) s_cnt[s] = 0u;
                }
                __syncthreads();
                table_insert(s_tab, bits, col + xb + c0, clen, threadIdx.x, blockDim.x);
                __syncthreads();
                HashProbe hpb{tab, x, bits};
                if (kCnt) hpb.cnt = s_cnt;
                h += probe_quads<CM>(hpb, d, nl, ib, ie, col, x, cr, stage, kCtaStride);
                __syncthreads();
                if (kCnt) {
                    for (uint32_t s = threadIdx.x; s < (1u << bits); s += blockDim.x) {
                        uint32_t c = s_cnt[s];
                        if (!c) continue;
                        if (CM == kCmVertex)
                            atomicAdd((unsigned long long *)&cr.pv[s_tab[s]], (unsigned long long)c);
                        if (CM == kCmEdge || CM == kCmTop)   // chunk col+[xb + c0, + clen), ascending
                            atomicAdd(&cr.sup[xb + c0 + list_pos(col + xb + c0, clen, s_tab[s])], c);
                    }
                    __syncthreads();
                }
            }
        }
        if (CM == kCmVertex) {
            uint64_t hw = warp_sum_u64(h);
            if ((threadIdx.x & 31) == 0 && hw)
                atomicAdd((unsigned long long *)&cr.pv[x], (unsigned long long)hw);
        }
        acc += h;
    }
    flush_count(acc, total);
}

template <int CM>
static void launch_all(Ctx &ctx, const Oriented &g, const Bins &bins, uint64_t *total,
                       const Credit &cr) {
    int grid = ctx.persistent_grid(8);
    // The bitmap hub kernel (most of the work) goes first on the call's stream; the
    // independent warp-owner / SHORT / MERGE / SEARCH kernels run on a side stream and
    // fill the SMs the hub kernel's tail leaves idle (all add into the same total).
    SideStream side(ctx);   // the side work depends only on binning; joined on every path
    cudaStream_t s2 = side.s;
#ifndef TC_HASH_CTA_GRID
#define TC_HASH_CTA_GRID 8   // CTAs per SM of the persistent bitmap-owner kernel
#endif
    k_hash_cta<CM, true><<<ctx.persistent_grid(TC_HASH_CTA_GRID), kIxThreads, 0, ctx.stream>>>(
        bins.tasks_bitmap, bins.ntasks_bitmap, bins.hp, total, cr);
    TC_LAUNCHED(ctx);
    k_hash_cta<CM, false><<<ctx.persistent_grid(8), kIxThreads, 0, ctx.stream>>>(
        bins.tasks_cta, bins.ntasks_cta, bins.hp, total, cr);
    TC_LAUNCHED(ctx);
    k_hash_warp<CM><<<grid, kIxThreads, 0, s2>>>(bins.tasks_warp, bins.ntasks_warp, bins.hp, total, cr);
    TC_LAUNCHED(ctx);
    // bins the policy cannot fill (bin.cu gives them no capacity) are not launched
    if (bins.has[1]) {
        k_merge<CM><<<grid, kIxThreads, 0, s2>>>(bins.edges[1], bins.count + 1, g.off, g.col, total, cr);
        TC_LAUNCHED(ctx);
    }
    if (bins.has[2]) {
        k_search<CM><<<grid, kIxThreads, 0, s2>>>(bins.edges[2], bins.count + 2, g.off, g.col, total, cr);
        TC_LAUNCHED(ctx);
    }
    if (bins.has[0]) {
        k_short<CM><<<grid, kIxThreads, 0, s2>>>(bins.edges[0], bins.count + 0, g.off, g.col, total, cr);
        TC_LAUNCHED(ctx);
    }
    if (CM == kCmNone)   // dense-core edges (core.cu); their word count -> stats
        core_count(ctx, g, bins.hp, total, bins.count + 14, s2);
    side.join();
}

void intersect_all(Ctx &ctx, const Oriented &g, const Bins &bins, uint64_t *total_dev,
                   const Credit &cr) {
    switch (cr.mode) {
        case kCmVertex: launch_all<kCmVertex>(ctx, g, bins, total_dev, cr); break;
        case kCmEdge: launch_all<kCmEdge>(ctx, g, bins, total_dev, cr); break;
        case kCmList: launch_all<kCmList>(ctx, g, bins, total_dev, cr); break;
        case kCmTop: launch_all<kCmTop>(ctx, g, bins, total_dev, cr); break;
        default: launch_all<kCmNone>(ctx, g, bins, total_dev, cr); break;
    }
}

}  // namespace tc
