// radix.cu -- hand-written stable LSD radix sort (8-bit digits), onesweep style:
//   1. one histogram kernel reads the keys once and counts the digits of EVERY
//      pass (shared-memory histograms, one global atomic per digit per block);
//   2. per pass ONE kernel (the pass's digit offsets are the exclusive prefix of its histogram,
//      scanned by every tile together with its own digit counts): each CTA takes the next tile (atomic ticket, so a
//      tile only ever waits on tiles that already started), ranks its keys
//      stably inside the tile (ballot-built digit peer masks per warp round), publishes its
//      per-digit counts, and obtains the exclusive prefix of earlier tiles by
//      DECOUPLED LOOK-BACK over their published (aggregate | inclusive) words.
//      The tile is then reordered by digit in shared memory and written out as
//      coalesced runs (global position = digit offset + look-back prefix + rank).
// Keys are read once and written once per pass.
#include "tc_internal.cuh"

namespace tc {

// Tile geometry, re-swept after the 4-op ballot form (s21 / road / s24 total ms): 512x8, 2 CTAs/SM
// 6.96 / 3.52 / 78.98; 384x8, 3/SM 6.85 / 3.53 / 78.44; 256x16, 4/SM 6.93 / 3.48 / 77.87;
// 512x6, 3/SM 7.02 / 3.59 / 80.18.
#ifndef TC_RS_THREADS
#define TC_RS_THREADS 384
#endif
#ifndef TC_RS_ROUNDS
#define TC_RS_ROUNDS 8
#endif
#ifndef TC_RS_LB
#define TC_RS_LB 8   // look-back batch: predecessor status words loaded together
#endif
#ifndef TC_RS_MINBLOCKS
#define TC_RS_MINBLOCKS 3
#endif
constexpr int kRsThreads = TC_RS_THREADS;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsRounds = TC_RS_ROUNDS;                // 32-item rounds per warp
constexpr int kRsWarpItems = 32 * kRsRounds;           // 256
constexpr int kRsTile = kRsWarps * kRsWarpItems;       // 4096 items per tile
constexpr int kDigits = 256;
constexpr int kMaxPasses = 8;

// Look-back status words: 2 flag bits (aggregate / inclusive prefix published) over the
// count.  32-bit words (half the look-back traffic) whenever every prefix fits in 30 bits.
template <class S>
struct Status {
    static constexpr int kBits = 8 * sizeof(S);
    static constexpr S kFlagAgg = (S)1 << (kBits - 2);
    static constexpr S kFlagPre = (S)2 << (kBits - 2);
    static constexpr S kCountMask = ((S)1 << (kBits - 2)) - 1;
};

__device__ __forceinline__ uint64_t valid_count(uint64_t cap, const uint64_t *count_dev) {
    if (!count_dev) return cap;
    uint64_t c = *count_dev;
    return c < cap ? c : cap;
}

// Status words carry their own payload (flag | count in one 64-bit word), so
// relaxed gpu-scope single-copy-atomic accesses suffice: no acquire/release
// (which would invalidate L1 on every spin iteration).
__device__ __forceinline__ void st_relaxed(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// All-pass digit histogram: hist[pass * 256 + digit].
template <class K>
__global__ void __launch_bounds__(kRsThreads)
    k_rs_hist(const K *__restrict__ keys, uint64_t cap, const uint64_t *__restrict__ count_dev,
              int passes, int db, uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[kMaxPasses][kDigits];
    const uint32_t dmask = (1u << db) - 1u;
    uint64_t n = valid_count(cap, count_dev);
    for (int i = threadIdx.x; i < kMaxPasses * kDigits; i += kRsThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * kRsThreads + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * kRsThreads) {
        K k = keys[i];
        for (int p = 0; p < passes; p++) atomicAdd(&h[p][(uint32_t)(k >> (db * p)) & dmask], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kDigits; i += kRsThreads) {
        uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// Lanes of `active` holding the same DB-bit digit d as this lane: DB ballots, measured
// a little faster than __match_any_sync on sm_100a.
// Per bit: one predicate test, the ballot, one select and one 3-input LOP
// (peers &= ballot ^ (bit ? 0 : ~0)): 4 SASS instructions (the C++ form compiled to 6-7).
template <int DB>
__device__ __forceinline__ uint32_t digit_peers(uint32_t active, uint32_t d) {
    uint32_t peers = active;
#pragma unroll
    for (int b = 0; b < DB; b++) {
        asm("{\n\t.reg .pred p;\n\t.reg .b32 m, x;\n\t"
            "and.b32 x, %1, %3;\n\t"
            "setp.ne.u32 p, x, 0;\n\t"
            "vote.sync.ballot.b32 m, p, %2;\n\t"
            "selp.b32 x, 0, -1, p;\n\t"
            "xor.b32 m, m, x;\n\t"
            "and.b32 %0, %0, m;\n\t}"
            : "+r"(peers) : "r"(d), "r"(active), "r"(1u << b));
    }
    return peers;
}

template <class K, bool kVals>
struct RsSmem {
    K keys[kRsTile];
    uint32_t vals[kVals ? kRsTile : 1];
    uint32_t wc[kRsWarps][kDigits];   // per-warp digit counters -> per-warp exclusive offsets
    uint32_t dstart[kDigits];         // tile-local digit start
    uint64_t gbase[kDigits];          // global start of this tile's run of each digit
    uint64_t scan[kRsWarps];
    uint32_t tile;
};

template <class K, bool kVals, class SW, int DB>
__global__ void __launch_bounds__(kRsThreads, TC_RS_MINBLOCKS)
    k_rs_pass(const K *__restrict__ keys, const uint32_t *__restrict__ vals, K *__restrict__ keys_out,
              uint32_t *__restrict__ vals_out, uint64_t cap, const uint64_t *__restrict__ count_dev,
              int shift, const uint32_t *__restrict__ hist_p, uint32_t *__restrict__ ticket,
              SW *__restrict__ status, const uint32_t *__restrict__ gather,
              uint32_t *__restrict__ gather_out, uint32_t *__restrict__ inverse) {
    constexpr SW kFlagAgg = Status<SW>::kFlagAgg, kFlagPre = Status<SW>::kFlagPre;
    constexpr SW kCountMask = Status<SW>::kCountMask;
    constexpr uint32_t kD = 1u << DB, kDMask = kD - 1u;   // digits of this pass
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RsSmem<K, kVals> &S = *reinterpret_cast<RsSmem<K, kVals> *>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n = valid_count(cap, count_dev);
    if (threadIdx.x == 0) S.tile = atomicAdd(ticket, 1u);
    for (int i = threadIdx.x; i < kRsWarps * kDigits; i += kRsThreads) (&S.wc[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = S.tile;
    const uint64_t tile_base = (uint64_t)tile * kRsTile;
    if (tile_base >= n) return;  // empty tail tiles: nobody waits on them
    const uint32_t tile_n = (uint32_t)min((uint64_t)kRsTile, n - tile_base);

    // ---- load (warp-blocked, coalesced rounds) and rank stably inside the tile
    const uint32_t wlocal = (uint32_t)warp * kRsWarpItems;
    const K *kp = keys + tile_base + wlocal + lane;
    // vals == nullptr: the values are the input positions (identity permutation)
    const uint32_t *vp = kVals && vals ? vals + tile_base + wlocal + lane : nullptr;
    const uint32_t vid0 = (uint32_t)(tile_base + wlocal + lane);
    K key[kRsRounds];
    uint32_t val[kRsRounds], rank[kRsRounds];
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t *wc = S.wc[warp];
    if (tile_n == kRsTile) {  // full tile: no bounds checks, straight-line ranking
#pragma unroll
        for (int j = 0; j < kRsRounds; j++) {
            key[j] = kp[32 * j];
            if (kVals) val[j] = vp ? vp[32 * j] : vid0 + 32 * j;
        }
#pragma unroll
        for (int j = 0; j < kRsRounds; j++) {
            uint32_t d = (uint32_t)(key[j] >> shift) & kDMask;
            uint32_t peers = digit_peers<DB>(0xffffffffu, d);
            uint32_t old = wc[d];
            __syncwarp();
            if ((peers & lt) == 0) wc[d] = old + __popc(peers);
            __syncwarp();
            rank[j] = old + __popc(peers & lt);
        }
    } else {
#pragma unroll
        for (int j = 0; j < kRsRounds; j++) {
            bool ok = wlocal + 32 * j + lane < tile_n;
            key[j] = ok ? kp[32 * j] : (K)0;
            if (kVals) val[j] = ok ? (vp ? vp[32 * j] : vid0 + 32 * j) : 0u;
        }
#pragma unroll
        for (int j = 0; j < kRsRounds; j++) {
            bool ok = wlocal + 32 * j + lane < tile_n;
            uint32_t d = (uint32_t)(key[j] >> shift) & kDMask;
            uint32_t active = __ballot_sync(0xffffffffu, ok);
            uint32_t old = 0, peers = 0;
            if (ok) {
                peers = digit_peers<DB>(active, d);
                old = wc[d];
            }
            __syncwarp();
            if (ok && (peers & lt) == 0) wc[d] = old + __popc(peers);
            __syncwarp();
            rank[j] = old + __popc(peers & lt);
        }
    }
    __syncthreads();

    // ---- per digit (threads 0..255): warp-exclusive offsets, tile count, publish the
    // aggregate, look back
    static_assert(kRsThreads >= kDigits, "one thread per digit");
    const uint32_t d = threadIdx.x;
    const bool is_digit = d < kD;
    uint32_t cnt = 0, hd = 0;
    SW *my = status + (uint64_t)tile * kD + d;
    if (is_digit) {
#pragma unroll
        for (int w = 0; w < kRsWarps; w++) {
            uint32_t c = S.wc[w][d];
            S.wc[w][d] = cnt;
            cnt += c;
        }
        st_relaxed(my, (SW)((tile == 0 ? kFlagPre : kFlagAgg) | (SW)cnt));
        hd = hist_p[d];   // this pass's global count of digit d
    }
    // one 64-bit scan gives both the tile-local digit starts (low word) and the pass's global
    // digit offsets (high word: exclusive prefix of the histogram; no separate offsets kernel)
    const uint64_t both = block_exclusive_scan<SumOp64>(((uint64_t)hd << 32) | cnt, S.scan);
    const uint32_t dstart = (uint32_t)both;
    if (is_digit) S.dstart[d] = dstart;
    __syncthreads();
    // ---- reorder by digit in shared memory (needs only tile-local offsets) overlapped
    // with the decoupled look-back: the warps holding no digit reorder first, the digit
    // warps look back first and reorder after, so the look-back latency hides behind the
    // other warps' shared-memory traffic
    auto reorder = [&]() {
#pragma unroll
        for (int j = 0; j < kRsRounds; j++) {
            uint32_t local = wlocal + 32 * j + lane;
            if (local < tile_n) {
                uint32_t dg = (uint32_t)(key[j] >> shift) & kDMask;
                uint32_t pos = S.dstart[dg] + S.wc[warp][dg] + rank[j];
                S.keys[pos] = key[j];
                if (kVals) S.vals[pos] = val[j];
            }
        }
    };
    if (!is_digit) reorder();
    if (is_digit) {
        uint64_t excl = 0;
        if (tile > 0) {
            // look back in batches of kLb predecessors (loads in flight together); a
            // missing tile index (< 0) reads as an inclusive prefix of 0
            constexpr int kLb = TC_RS_LB;
            for (int64_t t = (int64_t)tile - 1;; t -= kLb) {
                SW sw[kLb];
#pragma unroll
                for (int k = 0; k < kLb; k++)
                    sw[k] = t - k >= 0 ? ld_relaxed(status + (uint64_t)(t - k) * kD + d) : kFlagPre;
                bool done = false;
#pragma unroll
                for (int k = 0; k < kLb; k++) {
                    if (done) break;
                    while ((sw[k] & ~kCountMask) == 0)
                        sw[k] = ld_relaxed(status + (uint64_t)(t - k) * kD + d);
                    excl += sw[k] & kCountMask;
                    done = (sw[k] & kFlagPre) != 0;
                }
                if (done) break;
            }
            st_relaxed(my, (SW)(kFlagPre | (SW)(excl + cnt)));
        }
        S.gbase[d] = (both >> 32) + excl;
        reorder();
    }
    __syncthreads();
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < tile_n; i += kRsThreads) {
        K k = S.keys[i];
        uint32_t dg = (uint32_t)(k >> shift) & kDMask;
        uint64_t g = S.gbase[dg] + (i - S.dstart[dg]);
        keys_out[g] = k;
        if (kVals) {
            const uint32_t v = S.vals[i];
            vals_out[g] = v;
            if (gather) gather_out[g] = gather[v];   // fused gather (last pass only)
            if (inverse) inverse[v] = (uint32_t)g;   // fused inverse permutation (last pass)
        }
    }
}

// Passes read (kin0, vin0) first, then ping-pong between (A) and (B); the inputs
// are never written.  Returns the buffers holding the sorted result.
template <class K, bool kVals>
static void radix_impl(Ctx &ctx, const K *kin0, const uint32_t *vin0, K *kA, K *kB, uint32_t *vA,
                       uint32_t *vB, uint64_t capacity, const uint64_t *count_dev, int bits,
                       K **kres, uint32_t **vres, const uint32_t *gather = nullptr,
                       uint32_t *gather_out = nullptr, const uint32_t *hist_in = nullptr,
                       uint32_t *inverse = nullptr) {
    *kres = const_cast<K *>(kin0);
    *vres = const_cast<uint32_t *>(vin0);
    if (capacity == 0 || bits <= 0) return;
    const int db = radix_digit_bits(bits);   // 7-bit digits when they need no extra pass
    const int passes = (bits + db - 1) / db;
    const uint32_t tiles = (uint32_t)((capacity + kRsTile - 1) / kRsTile);
    const uint32_t *hist = hist_in;   // digit histograms counted by the producer, or here
    uint32_t *tickets = ctx.alloc<uint32_t>(passes);
    // 32-bit status words when every digit prefix (<= capacity) fits in 30 bits
    const bool narrow = capacity < (1ull << 30);
    const size_t sw = narrow ? sizeof(uint32_t) : sizeof(uint64_t);
    void *status = ctx.alloc<uint64_t>(((uint64_t)tiles * kDigits * sw + 7) / 8);  // reused per pass
    TC_CUDA(cudaMemsetAsync(tickets, 0, passes * sizeof(uint32_t), ctx.stream));
    if (!hist) {
        uint32_t *h = ctx.alloc<uint32_t>((uint64_t)passes * kDigits);
        TC_CUDA(cudaMemsetAsync(h, 0, (size_t)passes * kDigits * sizeof(uint32_t), ctx.stream));
        k_rs_hist<K><<<ctx.persistent_grid(4), kRsThreads, 0, ctx.stream>>>(kin0, capacity, count_dev,
                                                                            passes, db, h);
        TC_LAUNCHED(ctx);
        hist = h;
    }
    const size_t smem = sizeof(RsSmem<K, kVals>);
    auto set_smem = [&](auto kern) {
        TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    };
    set_smem(k_rs_pass<K, kVals, uint32_t, 7>);
    set_smem(k_rs_pass<K, kVals, uint32_t, 8>);
    set_smem(k_rs_pass<K, kVals, uint64_t, 7>);
    set_smem(k_rs_pass<K, kVals, uint64_t, 8>);
    const K *kin = kin0;
    const uint32_t *vin = vin0;
    for (int p = 0; p < passes; p++) {
        K *kout = (p & 1) ? kB : kA;
        uint32_t *vout = (p & 1) ? vB : vA;
        TC_CUDA(cudaMemsetAsync(status, 0, (size_t)tiles * kDigits * sw, ctx.stream));
        const uint32_t *ga = p == passes - 1 ? gather : nullptr;
        uint32_t *inv = p == passes - 1 ? inverse : nullptr;
        const uint32_t *dop = hist + (uint64_t)p * kDigits;
#define TC_RS_LAUNCH(SWT, DBV)                                                                  \
    k_rs_pass<K, kVals, SWT, DBV><<<tiles, kRsThreads, smem, ctx.stream>>>(                     \
        kin, vin, kout, vout, capacity, count_dev, db * p, dop, tickets + p, (SWT *)status, ga, \
        gather_out, inv)
        if (narrow) {
            if (db == 7) TC_RS_LAUNCH(uint32_t, 7);
            else TC_RS_LAUNCH(uint32_t, 8);
        } else {
            if (db == 7) TC_RS_LAUNCH(uint64_t, 7);
            else TC_RS_LAUNCH(uint64_t, 8);
        }
#undef TC_RS_LAUNCH
        TC_LAUNCHED(ctx);
        kin = kout;
        vin = vout;
    }
    *kres = const_cast<K *>(kin);
    *vres = const_cast<uint32_t *>(vin);
}

bool radix_sort(Ctx &ctx, uint64_t *keys, uint64_t *keys_alt, uint64_t capacity,
                const uint64_t *count_dev, int bits, const uint32_t *hist_in) {
    // (keys -> alt -> keys ...): first pass reads `keys`, then alt/keys alternate
    uint64_t *kr;
    uint32_t *vr;
    radix_impl<uint64_t, false>(ctx, keys, nullptr, keys_alt, keys, nullptr, nullptr, capacity,
                                count_dev, bits, &kr, &vr, nullptr, nullptr, hist_in);
    return kr == keys_alt;
}

bool radix_sort_pairs(Ctx &ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                      uint32_t *vals_alt, uint64_t capacity, const uint64_t *count_dev, int bits,
                      const uint32_t *hist_in) {
    uint32_t *kr, *vr;
    radix_impl<uint32_t, true>(ctx, keys, vals, keys_alt, keys, vals_alt, vals, capacity, count_dev,
                               bits, &kr, &vr, nullptr, nullptr, hist_in);
    return kr == keys_alt;
}

void radix_sort_pairs_from(Ctx &ctx, const uint32_t *keys_in, const uint32_t *vals_in,
                           uint32_t *kA, uint32_t *kB, uint32_t *vA, uint32_t *vB,
                           uint64_t capacity, const uint64_t *count_dev, int bits,
                           uint32_t **keys_out, uint32_t **vals_out, const uint32_t *gather,
                           uint32_t *gather_out, const uint32_t *hist_in, uint32_t *inverse) {
    radix_impl<uint32_t, true>(ctx, keys_in, vals_in, kA, kB, vA, vB, capacity, count_dev, bits,
                               keys_out, vals_out, gather, gather_out, hist_in, inverse);
}

}  // namespace tc
