// tc_internal.cuh -- shared device helpers and host-side declarations of the
// B200 triangle-counting pipeline.  Product code only: nothing here is shared
// with oracle/ (which is independent test infrastructure).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/tc.h"
#include "block_scan.cuh"

namespace tc {

constexpr uint32_t kEmpty = 0xffffffffu;

// ------------------------------------------------------------------ errors
struct Error {
    tc_status status;
    std::string msg;
};

void set_error(const std::string &msg);

#define TC_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            throw ::tc::Error{e_ == cudaErrorMemoryAllocation ? TC_ENOMEM : TC_ECUDA, \
                              std::string(#call) + ": " + cudaGetErrorString(e_)};    \
    } while (0)

#define TC_LAUNCHED(ctx)                                                                   \
    do {                                                                                   \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess)                                                             \
            throw ::tc::Error{TC_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)}; \
        (ctx).launches++;                                                                  \
    } while (0)

// ------------------------------------------------------------------ context
// Stream-ordered workspace (include/tc.h OWNERSHIP): every block comes from the caller's
// hook (tc_options.alloc / free) or, without one, from the library's own per-device pool
// (cudaMallocFromPoolAsync), on the call's stream, and is freed stream-ordered when the
// context is destroyed (or earlier with free_now).
uint64_t &thread_launches();   // kernels launched by this thread's calls (tc_launches_issued)

struct Ctx {
    cudaStream_t stream = nullptr;
    int device = 0;
    int num_sms = 148;
    uint64_t launches = 0;
    tc_alloc_fn hook_alloc = nullptr;
    tc_free_fn hook_free = nullptr;
    void *hook_ctx = nullptr;
    cudaMemPool_t pool = nullptr;    // library pool (no hook)
    bool graph_alloc = false;        // under CUDA graph capture: graph memory nodes
    uint64_t bytes_live = 0, bytes_peak = 0, n_allocs = 0;
    std::vector<std::pair<void *, size_t>> allocs;

    template <class T>
    T *alloc(uint64_t count) {
        void *p = nullptr;
        size_t bytes = (size_t)(count ? count : 1) * sizeof(T);
        bytes = (bytes + 255) & ~(size_t)255;   // whole 256-byte granules: aligned slot loads
        if (hook_alloc) {
            p = hook_alloc(hook_ctx, bytes, (void *)stream);
            if (!p)
                throw Error{TC_ENOMEM, "tc_options.alloc(" + std::to_string(bytes) + " B) returned NULL"};
        } else if (graph_alloc) {
            cudaError_t e = cudaMallocAsync(&p, bytes, stream);
            if (e != cudaSuccess) {
                cudaGetLastError();
                throw Error{TC_ECUDA, std::string("cudaMallocAsync under capture: ") + cudaGetErrorString(e)};
            }
        } else {
            cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, stream);
            if (e != cudaSuccess) {
                cudaGetLastError();
                throw Error{TC_ENOMEM, "cudaMallocFromPoolAsync(" + std::to_string(bytes) +
                                           " B) failed: " + cudaGetErrorString(e)};
            }
        }
        allocs.push_back({p, bytes});
        n_allocs++;
        bytes_live += bytes;
        if (bytes_live > bytes_peak) bytes_peak = bytes_live;
        return (T *)p;
    }
    void give_back(void *p, size_t bytes) {
        if (hook_free) hook_free(hook_ctx, p, (void *)stream);
        else cudaFreeAsync(p, stream);
        bytes_live -= bytes;
    }
    void release() {
        for (auto &a : allocs) give_back(a.first, a.second);
        allocs.clear();
    }
    // Stream-ordered early free (the pool reuses it for later allocations of this call).
    void free_now(void *p) {
        for (size_t i = 0; i < allocs.size(); i++)
            if (allocs[i].first == p) {
                give_back(p, allocs[i].second);
                allocs[i] = allocs.back();
                allocs.pop_back();
                return;
            }
    }
    ~Ctx() {
        release();
        thread_launches() += launches;
    }
    // Grid for a persistent (grid-stride) kernel: `per_sm` resident CTAs per SM.
    int persistent_grid(int per_sm) const { return num_sms * per_sm; }

    // A second (non-blocking) stream for independent kernels, cached per thread and
    // device, with fork / join events: work on it starts after everything enqueued on
    // `stream` so far, and `stream` waits for it at join().
    cudaStream_t side() {
        static thread_local cudaStream_t s[64] = {};
        static thread_local cudaEvent_t e[64][2] = {};
        int d = device >= 0 && device < 64 ? device : 0;
        if (!s[d]) {
            if (cudaStreamCreateWithFlags(&s[d], cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&e[d][0], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&e[d][1], cudaEventDisableTiming) != cudaSuccess)
                throw Error{TC_ECUDA, "side stream / event creation failed"};
        }
        ev_fork = e[d][0];
        ev_join = e[d][1];
        return s[d];
    }
    void fork(cudaStream_t s2) {
        if (cudaEventRecord(ev_fork, stream) != cudaSuccess || cudaStreamWaitEvent(s2, ev_fork, 0) != cudaSuccess)
            throw Error{TC_ECUDA, "fork failed"};
    }
    void join(cudaStream_t s2) {
        if (cudaEventRecord(ev_join, s2) != cudaSuccess || cudaStreamWaitEvent(stream, ev_join, 0) != cudaSuccess)
            throw Error{TC_ECUDA, "join failed"};
    }
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

// Fork work onto the side stream for the lifetime of this object; the destructor joins
// it back into the call's stream on EVERY path (also when a launch throws), so the
// workspace is never freed while side-stream kernels may still read it.
struct SideStream {
    Ctx &ctx;
    cudaStream_t s;
    bool joined = false;
    explicit SideStream(Ctx &c) : ctx(c), s(c.side()) {
        if (s != ctx.stream) ctx.fork(s);
    }
    void join() {
        if (!joined && s != ctx.stream) ctx.join(s);
        joined = true;
    }
    ~SideStream() {
        if (!joined && s != ctx.stream) {   // error path: never throw from a destructor
            cudaEventRecord(ctx.ev_join, s);
            cudaStreamWaitEvent(ctx.stream, ctx.ev_join, 0);
        }
    }
};

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum of a per-thread uint64; result valid in thread 0.  `scratch`
// must hold blockDim.x/32 entries.
__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v, uint64_t *scratch) {
    v = warp_sum_u64(v);
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    uint64_t total = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) total += scratch[w];
    __syncthreads();
    return total;
}

// ------------------------------------------------------------------ tiles
// A "tile" is a contiguous range of kTileItems arcs (or oriented edges) handled
// by one CTA of kTileThreads threads, each owning kItemsPerThread consecutive
// items (blocked arrangement, so block scans preserve index order).
constexpr int kTileThreads = 256;
constexpr int kItemsPerThread = 8;
constexpr int kTileItems = kTileThreads * kItemsPerThread;

// Fill s_row[0..len) with the CSR row of items tile_start .. tile_start+len-1
// (load-balanced row search: rows whose start falls inside the tile mark their
// first item, then an inclusive max-scan propagates row ids).  Must be called
// by all threads of the block.  s_scan: kTileThreads/32 uint32 scratch.
// First i in [0, len] with a[i] >= x (a non-decreasing), found by one warp with a
// 33-ary search (each round 32 lanes probe 32 split points: ~log33(len) dependent
// L2 round trips instead of log2(len)).  Every lane returns the answer.
__device__ __forceinline__ uint64_t warp_lower_bound(const uint64_t *__restrict__ a, uint64_t len,
                                                     uint64_t x) {
    const uint32_t lane = threadIdx.x & 31;
    uint64_t lo = 0, hi = len;  // answer in [lo, hi]; a[lo-1] < x, a[hi] >= x (or hi = len)
    while (hi - lo > 32) {
        uint64_t idx = lo + (hi - lo) * (lane + 1) / 33;   // strictly inside [lo, hi)
        uint32_t ge = __ballot_sync(0xffffffffu, a[idx] >= x);
        int f = __ffs(ge) - 1;                               // first probe with a >= x
        uint64_t below = __shfl_sync(0xffffffffu, idx, f > 0 ? f - 1 : 0);
        uint64_t at = __shfl_sync(0xffffffffu, idx, f >= 0 ? f : 31);
        if (f < 0) lo = at + 1;
        else {
            hi = at;
            if (f > 0) lo = below + 1;
        }
    }
    uint64_t i = lo + lane;
    uint32_t ge = __ballot_sync(0xffffffffu, i < hi && a[i] >= x);
    return ge ? lo + (uint64_t)(__ffs(ge) - 1) : hi;
}

__device__ __forceinline__ void tile_rows(const uint64_t *__restrict__ rowptr, uint64_t n, uint64_t tile_start,
                          uint32_t len, uint32_t *s_row, uint32_t *s_scan) {
    __shared__ uint64_t s_bounds[2];
    for (int i = threadIdx.x; i < kTileItems; i += blockDim.x) s_row[i] = 0;
    // warp 0: first row starting after tile_start (its predecessor holds item
    // tile_start); warp 1: first row starting at or after the tile's last item
    if (threadIdx.x < 64) {
        uint64_t b = warp_lower_bound(rowptr, n + 1, threadIdx.x < 32 ? tile_start + 1 : tile_start + len);
        if ((threadIdx.x & 31) == 0) s_bounds[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    uint64_t ulo = s_bounds[0], uhi = s_bounds[1];
    // row of item tile_start = last u with rowptr[u] <= tile_start = ulo - 1 (ulo >= 1)
    if (threadIdx.x == 0) atomicMax(&s_row[0], (uint32_t)(ulo - 1));
    for (uint64_t u = ulo + threadIdx.x; u < uhi; u += blockDim.x)
        atomicMax(&s_row[rowptr[u] - tile_start], (uint32_t)u);
    __syncthreads();
    // inclusive max-scan over the tile (blocked: thread t owns items [8t, 8t+8))
    uint32_t v[kItemsPerThread];
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        run = max(run, s_row[threadIdx.x * kItemsPerThread + k]);
        v[k] = run;
    }
    uint32_t prefix = block_exclusive_scan<MaxOp>(run, s_scan);
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++)
        s_row[threadIdx.x * kItemsPerThread + k] = max(v[k], prefix);
    __syncthreads();
}

// Same, with the row bounds of the tile precomputed by tile_bounds (round 2): the two warp
// searches above are a chain of dependent L2 round trips per tile, which a persistent loop
// pays once per tile in series.  b = (first row starting after tile_start, first row starting
// at or after the tile's last item).
__device__ __forceinline__ void tile_rows_b(const uint64_t *__restrict__ rowptr, uint64_t tile_start,
                                            uint32_t len, uint2 b, uint32_t *s_row, uint32_t *s_scan) {
    for (int i = threadIdx.x; i < kTileItems; i += blockDim.x) s_row[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&s_row[0], b.x - 1u);
    for (uint64_t u = b.x + threadIdx.x; u < b.y; u += blockDim.x)
        atomicMax(&s_row[rowptr[u] - tile_start], (uint32_t)u);
    __syncthreads();
    uint32_t v[kItemsPerThread];
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++) {
        run = max(run, s_row[threadIdx.x * kItemsPerThread + k]);
        v[k] = run;
    }
    uint32_t prefix = block_exclusive_scan<MaxOp>(run, s_scan);
#pragma unroll
    for (int k = 0; k < kItemsPerThread; k++)
        s_row[threadIdx.x * kItemsPerThread + k] = max(v[k], prefix);
    __syncthreads();
}
#ifndef TC_TILE_BOUNDS
#define TC_TILE_BOUNDS 0   // k_edges / k_clean_keys on precomputed row bounds: measured no change (s21 6.57 vs 6.57 ms)
#endif
// tile_rows with the bounds precomputed when tb != nullptr (TC_TILE_BOUNDS), else searched.
__device__ __forceinline__ void tile_rows_tb(const uint64_t *__restrict__ rowptr, uint64_t n, uint64_t tile,
                                             uint64_t tile_start, uint32_t len, const uint2 *__restrict__ tb,
                                             uint32_t *s_row, uint32_t *s_scan) {
    if (tb) tile_rows_b(rowptr, tile_start, len, tb[tile], s_row, s_scan);
    else tile_rows(rowptr, n, tile_start, len, s_row, s_scan);
}
// bounds[t] for the tiles of `items` (host count, or *items_dev when given) CSR items.
void tile_bounds(Ctx &ctx, const uint64_t *rowptr, uint64_t n, uint64_t items, const uint64_t *items_dev,
                 uint2 *bounds);

// Digit width of an LSD radix sort over `bits` key bits: 7 when 7-bit digits need no
// more passes than 8-bit ones (fewer ballots per rank, half the look-back digits), else 8.
inline int radix_digit_bits(int bits) { return (bits + 6) / 7 == (bits + 7) / 8 ? 7 : 8; }

// ------------------------------------------------------------------ fused digit histograms
// Producers of radix-sort keys count the 8-bit digits of every pass on the fly:
// shared-memory counters (RsHist) flushed with one global atomic per non-zero digit.
constexpr int kHistDigits = 256;
template <int P>
struct RsHist {
    uint32_t h[P][kHistDigits];
    __device__ __forceinline__ void clear() {
        for (int i = threadIdx.x; i < P * kHistDigits; i += blockDim.x) (&h[0][0])[i] = 0;
    }
    template <class K>
    __device__ __forceinline__ void add(K key, int passes, int db) {
        const uint32_t mask = (1u << db) - 1u;
#pragma unroll
        for (int p = 0; p < P; p++)
            if (p < passes) atomicAdd(&h[p][(uint32_t)(key >> (db * p)) & mask], 1u);
    }
    __device__ __forceinline__ void flush(uint32_t *g, int passes) {
        for (int i = threadIdx.x; i < passes * kHistDigits; i += blockDim.x) {
            uint32_t v = (&h[0][0])[i];
            if (v) atomicAdd(&g[i], v);
        }
    }
};

// ------------------------------------------------------------------ host primitives
// Exclusive scan: out[i] = sum_{j<i} in[j] for i in [0, count], out[count] = total.
void scan_exclusive(Ctx &ctx, const uint32_t *in, uint64_t *out, uint64_t count);
void scan_exclusive(Ctx &ctx, const uint64_t *in, uint64_t *out, uint64_t count);
// Same over the first *count_dev (<= cap) items only; the total also goes to *total_out.
void scan_exclusive_dc(Ctx &ctx, const uint32_t *in, uint64_t *out, uint64_t cap,
                       const uint64_t *count_dev, uint64_t *total_out);

// Stable LSD radix sort on bits [0, bits) of the keys.  `count_dev`, if non-null,
// is a device counter that caps the number of valid items (<= capacity).
// Returns true if the sorted result ended in the *_alt buffers.
// hist_in (optional): the digit histograms of the keys, hist_in[pass * 256 + digit] for
// the (bits + 7) / 8 passes, counted by the kernel that produced the keys (skips the
// histogram pass).
bool radix_sort(Ctx &ctx, uint64_t *keys, uint64_t *keys_alt, uint64_t capacity,
                const uint64_t *count_dev, int bits, const uint32_t *hist_in = nullptr);
bool radix_sort_pairs(Ctx &ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                      uint32_t *vals_alt, uint64_t capacity, const uint64_t *count_dev, int bits,
                      const uint32_t *hist_in = nullptr);
// Same, reading (keys_in, vals_in) without modifying them; passes ping-pong between
// A and B; *keys_out / *vals_out receive the buffers holding the result.
// vals_in == nullptr: the values are the input positions 0, 1, 2, ...  With `gather`, the
// last pass also writes gather_out[i] = gather[value of sorted item i] (fused gather); with
// `inverse`, inverse[value of sorted item i] = i (fused inverse permutation).
void radix_sort_pairs_from(Ctx &ctx, const uint32_t *keys_in, const uint32_t *vals_in,
                           uint32_t *kA, uint32_t *kB, uint32_t *vA, uint32_t *vB,
                           uint64_t capacity, const uint64_t *count_dev, int bits,
                           uint32_t **keys_out, uint32_t **vals_out,
                           const uint32_t *gather = nullptr, uint32_t *gather_out = nullptr,
                           const uint32_t *hist_in = nullptr, uint32_t *inverse = nullptr);

// ------------------------------------------------------------------ pipeline stages
// Oriented CSR in RANK-RELABELLED ids: vertex v of the input is newid[v] here,
// order[i] is the input vertex of new id i, and newid[u] < newid[v] <=> rank(u) < rank(v).
struct Oriented {
    uint64_t n = 0;
    uint64_t *off = nullptr;     // off+[n+1]   (indexed by new id)
    uint32_t *col = nullptr;     // col+[m]     (new ids; every row ascending)
    uint32_t *dplus = nullptr;   // d+[n]       (indexed by new id)
    uint64_t *in_off = nullptr;  // transposed CSR: in-lists N-(x) (edge-list order)
    uint32_t *in_src = nullptr;
    uint32_t *pidx = nullptr;    // CSR edge e -> its slot in the transposed CSR
    uint32_t *order = nullptr;   // new id -> input id
    uint32_t *newid = nullptr;   // input id -> new id
    uint64_t *m_dev = nullptr;   // device scalar m
    uint64_t *stage_work = nullptr;  // device scalar sum_v d-(v) d+(v) (stats)
    uint32_t *claim_err = nullptr;   // clean input: set if more arcs passed the rank filter
                                     // than a simple symmetric graph allows (false TC_CLEAN)
    uint64_t m_cap = 0;          // capacity bound for m (host-known)
};

// NVTX ranges per phase (header-only NVTX v3: free unless a profiler is attached), so
// Nsight Systems timelines show clean / orient / prune / bin / intersect by name.
inline const char *phase_name(int p) {
    static const char *names[] = {"tc.clean (a1)", "tc.orient (a2-a4)", "tc.sort",
                                  "tc.bin (a5)", "tc.intersect (a6-a7)", "tc.prune (NEXT-2)"};
    return p >= 0 && p < 6 ? names[p] : "tc.phase";
}
// Phase timer: CUDA events on the call's stream, read after the final sync.
enum Phase { kClean = 0, kOrient, kSort, kBin, kIntersect, kPrune, kNumPhases };
struct Timer {
    cudaEvent_t ev[kNumPhases][2] = {};
    bool used[kNumPhases] = {};
    cudaStream_t stream = nullptr;
    explicit Timer(cudaStream_t s) : stream(s) {
        for (auto &p : ev) {
            cudaEventCreate(&p[0]);
            cudaEventCreate(&p[1]);
        }
    }
    ~Timer() {
        for (auto &p : ev) {
            cudaEventDestroy(p[0]);
            cudaEventDestroy(p[1]);
        }
    }
    void begin(Phase p) { cudaEventRecord(ev[p][0], stream); used[p] = true; }
    void end(Phase p) { cudaEventRecord(ev[p][1], stream); }
    double ms(Phase p) const {
        float t = 0.f;
        if (!used[p] || cudaEventElapsedTime(&t, ev[p][0], ev[p][1]) != cudaSuccess) return 0.0;
        return (double)t;
    }
};

// Phase boundary: NVTX range always, CUDA events when stats were requested (tm != null).
inline void phase_begin(Timer *tm, Phase p) {
    nvtxRangePushA(phase_name(p));
    if (tm) tm->begin(p);
}
inline void phase_end(Timer *tm, Phase p) {
    if (tm) tm->end(p);
    nvtxRangePop();
}

// NEXT-2 leaf pruning (prune.cu).  enabled: TC_PRUNE given; rounds: 0 = to the
// fixed point (2-core).  Filled in: rounds executed, the edge count before pruning.
struct PruneInfo {
    bool enabled = false;
    uint32_t rounds_wanted = 0;
    uint64_t rounds = 0;
    const uint64_t *m_before = nullptr;  // device scalar (dirty path)
    uint64_t m_before_host = 0;          // clean path: arcs / 2
};
// Dirty path: E (unique (min << b | max) keys, any order, *m_dev of them), deg = degrees of E.
// On return E / m_dev / deg describe the pruned graph (E compacted).
void prune_pairs(Ctx &ctx, uint64_t n, int b, uint32_t rounds, uint64_t *&E, uint64_t *&m_dev,
                 uint32_t *&deg, uint64_t m_host_cap, PruneInfo &info);
// Clean path: deg = row lengths on entry; on return the pruned degrees (0 = deleted
// vertex); an arc survives iff both endpoint degrees are > 0.
void prune_csr(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
               uint32_t rounds, uint32_t *&deg, PruneInfo &info);

// a1 (dirty input) + a2 + a3 + a4: raw CSR -> oriented relabelled CSR, rows ascending.
// method: tc_options.clean_method (0 = hashed sort order, 1 = full (min, max) order).
void orient_dirty(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
                  Oriented &out, Timer *tm,
                  PruneInfo &prune, bool id_order, uint32_t method);
// a2 + a3 + a4 from unique undirected edges E (keys (min << b) | max, b = id bits of n, any
// order; m_dev of them, at most M) and their graph's degrees deg (both kept by the caller).
void orient_edges(Ctx &ctx, uint64_t n, uint64_t M, uint64_t *E, uint64_t *m_dev, uint32_t *deg,
                  Oriented &out, Timer *tm, PruneInfo &prune, bool id_order,
                  void *free0 = nullptr, void *free1 = nullptr);
// tc_clean_shard: a1 on the arcs of this rank's edges (min endpoint mod world == rank): the
// unique edges (any order) into edges[0, *m_dev_out) and their degrees added into deg.
void clean_shard(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
                 int rank, int world, uint64_t *edges, uint32_t *deg, uint64_t *m_dev_out,
                 uint32_t method);
// a2 + a3 + a4 for clean symmetric input.
void orient_clean(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr, const uint32_t *col,
                  Oriented &out, Timer *tm,
                  PruneInfo &prune, bool id_order);
// The oriented CSR in INPUT ids with ascending rows (tc_orient output).
// With pay_in (m entries in CSR order, e.g. edge supports) also pay_out[k] = the
// payload of the edge written to col_out[k].
void to_original(Ctx &ctx, const Oriented &g, uint64_t *off_out, uint32_t *col_out,
                 const uint32_t *pay_in = nullptr, uint32_t *pay_out = nullptr);
// pv_out[v] = pv_new[newid[v]].
void per_vertex_to_original(Ctx &ctx, const Oriented &g, const uint64_t *pv_new, uint64_t *pv_out);

// NEXT-1: local clustering coefficients (input ids, nullable) from t (rank ids);
// out2 (device) = {sum_v C(d(v),2), bits of sum_v c(v)}.
void clustering(Ctx &ctx, const Oriented &g, const uint64_t *t_new, double *cc, uint64_t *out2);

// HASH-variant context passed by value to the binning and intersection kernels.
struct HashParams {
    const uint64_t *off = nullptr;     // oriented CSR (rank ids, rows ascending)
    const uint32_t *col = nullptr;
    const uint32_t *dplus = nullptr;
    const uint64_t *in_off = nullptr;  // transposed CSR: in-lists
    const uint32_t *in_src = nullptr;
    const uint32_t *pidx = nullptr;    // CSR edge e -> its in-list slot
    const uint32_t *in_cnt = nullptr;  // x: entries of its in-list its tasks take (0 = none: no
                                       // in-part entry of x is this rank's HASH work)
    const uint16_t *ulo = nullptr;     // in-edge p = (u,x) at CSR position e: its probe length
                                       // suf = off[u+1] - e - 1 (range [off[u+1] - suf, off[u+1])
                                       // of col+), 0 if not this rank's in-part HASH work.
                                       // 16 bits (round 2): the in-slot-indexed scatter of a5
                                       // touches half the bytes; in-part needs suf <= kSufMax
    const uint64_t *ooff = nullptr;    // compacted out-part entries of each owner:
    const uint2 *orange = nullptr;     //   probe ranges [lo, hi) of col+
    const uint32_t *ovid = nullptr;    //   the edge's target (per-vertex credit), or its CSR
                                       //   index when binned with edge_ids (edge support)
    uint32_t n = 0, short_max = 0, skew_ratio = 0;
    int force = -1, rank = 0, world = 1;
    // dense core (core.cu): rank ids [core_lo, n) have adjacency bitmaps of core_words words
    // each; nullptr = no core path (per-vertex / edge / list modes, forced variants)
    const uint32_t *core = nullptr;
    const uint4 *core_info = nullptr;    // (first, last element, d+) of N+(y), y in the core
    uint32_t core_lo = 0, core_words = 0;
};

constexpr int kBinCore = 4;   // internal bin of k_edges: dense-core edge (core.cu)


// Multi-GPU split of the per-edge bins (SHORT / MERGE / SEARCH / dense core): interleaved
// blocks of 2048 CSR edges.
__device__ __forceinline__ int edge_rank(uint64_t e, int world) {
    return world <= 1 ? 0 : (int)((e >> 11) % (uint64_t)world);
}
// Multi-GPU split (world > 1): the rank of a unit whose exclusive work prefix is
// `pre`, out of `total`: floor(pre / ceil(total / world)), clamped.  Deterministic on every
// rank, no communication.
__device__ __forceinline__ int split_rank(uint64_t pre, uint64_t total, int world) {
    if (world <= 1) return 0;
    const uint64_t chunk = (total + world - 1) / world;
    const uint64_t r = chunk ? pre / chunk : 0;
    return r >= (uint64_t)world ? world - 1 : (int)r;
}
// Variant of oriented edge (u,v): -1 = cannot close a triangle (suf = |N+(u) after
// v| = 0, or d+(v) = 0); else the forced variant, or the AUTO policy.
// An in-part HASH entry stores its probe length in 16 bits; a longer suffix (possible only when
// d+ is unbounded, TC_ID_ORDER, or m >= 2^31) makes the edge an out-part entry of u instead.
constexpr uint32_t kSufMax = 0xffffu;
__device__ __forceinline__ int edge_bin(const HashParams &hp, uint32_t du, uint32_t dv, uint32_t suf) {
    if (suf == 0 || dv == 0) return -1;
    if (hp.force >= 0) return hp.force;
    uint32_t a = du < dv ? du : dv, b = du < dv ? dv : du;
    if (b <= hp.short_max) return TC_VARIANT_SHORT;
    if (hp.skew_ratio && (uint64_t)b >= (uint64_t)hp.skew_ratio * a) return TC_VARIANT_SEARCH;
    return TC_VARIANT_HASH;
}

// Edge bins (a5).  SHORT / MERGE / SEARCH hold (u, v) pairs.  HASH edges are
// handled per owner (bin.cu header): owner x's probe entries are its in-list
// followed, if it owns out-part edges, by its own row.
struct Bins {
    uint2 *edges[3] = {nullptr, nullptr, nullptr};  // SHORT, MERGE, SEARCH: (u, v) pairs
    bool has[3] = {false, false, false};            // the policy can route edges there
    uint64_t *count = nullptr;  // device: [0..3] SHORT/MERGE/SEARCH/HASH edges, [4] W,
                                // [5] sum min(|N+(u) after v|, d+(v)), [6] skipped, [7] max d+,
                                // [8] warp owners, [9] CTA hash owners, [10] CTA bitmap owners,
                                // [11] table-build loads (sum over tasks of d+(owner))
    uint32_t *pcnt = nullptr;   // per owner: probe entries
    uint32_t *owners_warp = nullptr;   // owners with d+ < hub_min: tables of one warp
    uint32_t *owners_cta = nullptr;    // larger owners ("hubs"): tables of one CTA
    uint32_t *owners_bitmap = nullptr; // hubs whose rank span (x, n) fits a smem bitmap
    // Tasks = (owner, k): the k-th block of kWarpTaskLists / kCtaTaskLists probe
    // entries of an owner, so no warp / CTA is stuck with a hub's whole group.
    uint4 *tasks_warp = nullptr, *tasks_cta = nullptr, *tasks_bitmap = nullptr;   // 2 per task
    uint64_t *ntasks_warp = nullptr, *ntasks_cta = nullptr, *ntasks_bitmap = nullptr;  // device
    HashParams hp;
    uint64_t cap = 0;
};

constexpr uint32_t kWarpTableSlots = 512;   // per-warp hash table (owner d+ <= 128, load <= 1/4)
constexpr uint32_t kWarpTaskLists = 64;     // probe entries per warp task
constexpr uint32_t kCtaTaskLists = 256;     // probe entries per CTA task (one descriptor batch)
#ifndef TC_BITMAP_EFFSPAN
#define TC_BITMAP_EFFSPAN 1   // bitmap over [min, max] of N+(x) (1) or over (x, n) (0)
#endif
#ifndef TC_BITMAP_BATCHES
#define TC_BITMAP_BATCHES 1
#endif
constexpr uint32_t kBitmapBatches = TC_BITMAP_BATCHES;   // bitmap tasks: batches per bitmap build
constexpr uint32_t kBitmapTaskLists = kCtaTaskLists * kBitmapBatches;
constexpr uint32_t kCtaBitmapBits = 4096 * 32;  // rank span of a CTA bitmap (16 KB)

struct BinParams {
    uint32_t short_max, skew_ratio, hub_min;
    int force;
    int rank, world;
    bool edge_ids = false;        // out-part entries record their edge's CSR index (kCmEdge)
    bool core = false;            // route dense-core edges to the core path (count mode, AUTO)
};

void bin_edges(Ctx &ctx, const Oriented &g, const BinParams &p, Bins &bins);

// Dense core (core.cu): builds the adjacency bitmaps of the top-ranked vertices into
// hp.core / core_lo / core_words (count mode only; a no-op when the graph is empty).
void core_build(Ctx &ctx, const Oriented &g, HashParams &hp);
// First rank id of the dense core (the same rule as core_build).
uint32_t core_first(uint64_t n);
// a6 + a7 for the core edges (plain count): popc of bitmap ANDs, added into total_dev.
void core_count(Ctx &ctx, const Oriented &g, const HashParams &hp, uint64_t *total_dev,
                uint64_t *words_dev, cudaStream_t stream);

// What each triangle found in a6 credits besides the total (intersect.cu header).
enum CreditMode { kCmNone = 0, kCmVertex = 1, kCmEdge = 2, kCmList = 3, kCmTop = 4 };
struct Credit {
    int mode = kCmNone;
    uint64_t *pv = nullptr;           // kCmVertex: t(v), rank ids, n entries
    uint32_t *sup = nullptr;          // kCmEdge / kCmTop: per entry of col+ (m entries)
    uint32_t *tri = nullptr;          // kCmList: cap triples of ascending input ids
    uint64_t *cursor = nullptr;       // kCmList: triples found so far (device counter)
    uint64_t cap = 0;
    const uint32_t *order = nullptr;  // kCmList: rank id -> input id
};

// a6 + a7: all intersection kernels; adds into total_dev and credits per `cr`.
void intersect_all(Ctx &ctx, const Oriented &g, const Bins &bins, uint64_t *total_dev,
                   const Credit &cr);

// tiny.cu: the whole count in one CTA for n <= kTinyMaxN (total, per-vertex t(v) in input
// ids if pv_dev, and the undirected edge count m into m_dev).
constexpr uint64_t kTinyMaxN = 1024;
void tiny_count(Ctx &ctx, uint64_t n, const uint64_t *rowptr, const uint32_t *col,
                uint64_t *total_dev, uint64_t *pv_dev, uint64_t *m_dev);

// lowdeg.cu: the bounded-degree path (every vertex has <= L <= kLowDegMax incidences).
// lowdeg_prepare enqueues the eligibility passes (they set *flag_dev when some vertex has
// more); lowdeg_count finishes a1-a2 and counts -- its kernels do nothing when the flag is
// set, and the host, reading the flag with the count, re-runs the call on the pipeline --
// (total, per-vertex t(v) in input ids, and into out_dev[6]: W, probe work, max d+,
// Sum d- d+, skipped edges (these with stats), Sum d+).
constexpr uint32_t kLowDegMax = 32;
struct LowDeg {
    uint64_t n = 0;
    const uint64_t *rowptr = nullptr, *aoff = nullptr;
    const uint32_t *col = nullptr, *adj = nullptr;
    uint32_t *inc = nullptr;
    uint64_t *pk = nullptr;           // d(v) << 40 | offset of v's row in adj
    uint8_t *slot8 = nullptr;         // dirty input: each arc's slot in its target's row
    const uint32_t *flag = nullptr;   // device: set when some vertex has more than L incidences
    uint64_t *m2 = nullptr;     // device: Sum d(v) (dirty input)
    uint64_t m2_host = 0;       // clean input: M
    uint64_t adj_cap = 0;             // entries of adj
};
void lowdeg_prepare(Ctx &ctx, LowDeg &ld, uint64_t n, uint64_t M, const uint64_t *rowptr,
                    const uint32_t *col, bool clean, bool sorted, uint32_t L, uint32_t *flag_dev);
void lowdeg_count(Ctx &ctx, LowDeg &ld, uint64_t M, Timer *tm, uint64_t *total_dev, uint64_t *pv_dev,
                  uint64_t *out_dev, bool stats);

// Multi-GPU phases (shard.cu): tc_api.cu's option / workspace / error wrapper.
tc_status run_phase(const tc_options *opt, const std::function<void(Ctx &, const tc_options &)> &fn);
void check_device(const void *p, int dev, const char *what);   // TC_EINVAL unless on `dev`
// rank relabelling (a2): newid_out[v] = rank position of v (orient.cu)
void rank_relabel(Ctx &ctx, uint64_t n, const uint32_t *deg, bool id_order, uint32_t *newid_out);
// Tasks of an owner list (bin.cu): ceil(pcnt / L) per owner, their records, *ntasks.
void make_tasks(Ctx &ctx, uint64_t n, uint64_t cap, const uint32_t *owners, const uint64_t *ocount,
                const uint32_t *pcnt, const HashParams &hp, uint32_t L, uint64_t *tloads,
                uint4 *&tasks, uint64_t *&ntasks);

// Validation (TC_VALIDATE); returns a TC_EGRAPH message or "".
std::string validate_graph(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr,
                           const uint32_t *col, bool clean, bool sorted);

}  // namespace tc
