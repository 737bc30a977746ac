// validate.cu -- TC_VALIDATE: device checks of the input CSR (SPEC S:37-40 / S:66
// invariants: offsets, id range).  Under TC_CLEAN also the clean-graph promise of
// tc.h: no self-loops, no duplicate arcs, every arc has its reverse.  With TC_SORTED
// rows must be strictly increasing (which excludes duplicates) and symmetry is a binary
// search in the reverse row; without it the arcs' (u << b | v) keys are radix-sorted and
// duplicates / missing reverses are found in the sorted key array.
#include "tc_internal.cuh"

namespace tc {

enum : uint32_t {
    kBadFirst = 1, kBadLast = 2, kNonMonotone = 4, kIdRange = 8, kSelfLoop = 16,
    kUnsorted = 32, kAsymmetric = 64, kDuplicate = 128
};

__global__ void k_val_offsets(const uint64_t *__restrict__ rowptr, uint64_t n, uint64_t M,
                              uint32_t *__restrict__ err) {
    uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid == 0) {
        if (rowptr[0] != 0) atomicOr(err, kBadFirst);
        if (rowptr[n] != M) atomicOr(err, kBadLast);
    }
    for (uint64_t u = tid; u < n; u += (uint64_t)gridDim.x * blockDim.x)
        if (rowptr[u] > rowptr[u + 1]) atomicOr(err, kNonMonotone);
}

__global__ void __launch_bounds__(kTileThreads)
    k_val_arcs(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col, uint64_t n,
               uint64_t M, bool clean, bool sorted, uint32_t *__restrict__ err) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
    tile_rows(rowptr, n, t0, len, s_row, s_scan);
    uint32_t e = 0;
    for (uint32_t i = threadIdx.x; i < len; i += kTileThreads) {
        uint64_t k = t0 + i;
        uint32_t u = s_row[i], v = col[k];
        if (v >= n) { e |= kIdRange; continue; }
        if (!clean) continue;
        if (u == v) e |= kSelfLoop;
        if (!sorted) continue;
        if (k > rowptr[u] && col[k - 1] >= v) e |= kUnsorted;
        // symmetry: u must appear in row v (binary search, rows sorted)
        uint64_t lo = rowptr[v], hi = rowptr[v + 1];
        while (lo < hi) {
            uint64_t mid = (lo + hi) >> 1;
            if (col[mid] < u) lo = mid + 1; else hi = mid;
        }
        if (lo >= rowptr[v + 1] || col[lo] != u) e |= kAsymmetric;
    }
    if (e) atomicOr(err, e);
}

// TC_CLEAN without TC_SORTED: directed keys (u << b) | v of every arc.
__global__ void __launch_bounds__(kTileThreads)
    k_val_keys(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col, uint64_t n,
               uint64_t M, int b, uint64_t *__restrict__ keys) {
    __shared__ uint32_t s_row[kTileItems];
    __shared__ uint32_t s_scan[kTileThreads / 32];
    uint64_t t0 = (uint64_t)blockIdx.x * kTileItems;
    uint32_t len = (uint32_t)min((uint64_t)kTileItems, M - t0);
    tile_rows(rowptr, n, t0, len, s_row, s_scan);
    for (uint32_t i = threadIdx.x; i < len; i += kTileThreads)
        keys[t0 + i] = ((uint64_t)s_row[i] << b) | col[t0 + i];
}

// Sorted directed keys: a key equal to its predecessor is a duplicate arc; a key whose
// reverse (v << b | u) is absent (binary search) is an arc without its reverse.
__global__ void k_val_sorted_keys(const uint64_t *__restrict__ keys, uint64_t M, int b,
                                  uint32_t *__restrict__ err) {
    const uint64_t mask = (1ull << b) - 1;
    uint32_t e = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        if (i > 0 && keys[i - 1] == k) e |= kDuplicate;
        const uint64_t r = ((k & mask) << b) | (k >> b);
        uint64_t lo = 0, hi = M;
        while (lo < hi) {
            uint64_t mid = (lo + hi) >> 1;
            if (keys[mid] < r) lo = mid + 1; else hi = mid;
        }
        if (lo >= M || keys[lo] != r) e |= kAsymmetric;
    }
    if (e) atomicOr(err, e);
}

std::string validate_graph(Ctx &ctx, uint64_t n, uint64_t M, const uint64_t *rowptr,
                           const uint32_t *col, bool clean, bool sorted) {
    uint32_t *err = ctx.alloc<uint32_t>(1);
    TC_CUDA(cudaMemsetAsync(err, 0, sizeof(uint32_t), ctx.stream));
    k_val_offsets<<<ctx.persistent_grid(4), 256, 0, ctx.stream>>>(rowptr, n, M, err);
    TC_LAUNCHED(ctx);
    uint32_t h = 0;
    TC_CUDA(cudaMemcpyAsync(&h, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx.stream));
    TC_CUDA(cudaStreamSynchronize(ctx.stream));
    if (h == 0 && M > 0) {
        uint64_t tiles = (M + kTileItems - 1) / kTileItems;
        k_val_arcs<<<(unsigned)tiles, kTileThreads, 0, ctx.stream>>>(rowptr, col, n, M, clean,
                                                                      sorted, err);
        TC_LAUNCHED(ctx);
        if (clean && !sorted) {   // symmetry and uniqueness over the sorted directed keys
            int b = 1;
            while (b < 32 && (1ull << b) < n) b++;
            uint64_t *keys = ctx.alloc<uint64_t>(M), *alt = ctx.alloc<uint64_t>(M);
            k_val_keys<<<(unsigned)tiles, kTileThreads, 0, ctx.stream>>>(rowptr, col, n, M, b, keys);
            TC_LAUNCHED(ctx);
            uint64_t *sk = radix_sort(ctx, keys, alt, M, nullptr, 2 * b) ? alt : keys;
            k_val_sorted_keys<<<ctx.persistent_grid(8), 256, 0, ctx.stream>>>(sk, M, b, err);
            TC_LAUNCHED(ctx);
        }
        TC_CUDA(cudaMemcpyAsync(&h, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx.stream));
        TC_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    std::string msg;
    if (h & kBadFirst) msg += "row_offsets[0] != 0; ";
    if (h & kBadLast) msg += "row_offsets[n] != m; ";
    if (h & kNonMonotone) msg += "row_offsets not non-decreasing; ";
    if (h & kIdRange) msg += "column index >= n; ";
    if (h & kSelfLoop) msg += "self-loop under TC_CLEAN; ";
    if (h & kUnsorted) msg += "row not strictly increasing under TC_SORTED; ";
    if (h & kAsymmetric) msg += "arc without its reverse under TC_CLEAN; ";
    if (h & kDuplicate) msg += "duplicate arc under TC_CLEAN; ";
    return msg;
}

}  // namespace tc
