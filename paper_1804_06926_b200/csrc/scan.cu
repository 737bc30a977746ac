// scan.cu -- device-wide exclusive scan (reduce-then-scan) and the block-level
// scan / tile row-search helpers every tile kernel uses.
#include <algorithm>

#include "tc_internal.cuh"
#include "block_scan.cuh"

namespace tc {

// ------------------------------------------------------------------ global scan
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const T *__restrict__ in,
                                                              uint64_t count,
                                                              uint64_t *__restrict__ partial) {
    __shared__ uint64_t s_scratch[kScanThreads / 32];
    uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    uint64_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
        if (i < count) sum += (uint64_t)in[i];
    }
    sum = block_sum_u64(sum, s_scratch);
    if (threadIdx.x == 0) partial[blockIdx.x] = sum;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const T *__restrict__ in,
                                                             uint64_t count,
                                                             const uint64_t *__restrict__ offsets,
                                                             uint64_t *__restrict__ out) {
    __shared__ uint64_t s_scan[kScanThreads / 32];
    uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint64_t v[kScanItems];
    uint64_t run = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        uint64_t i = base + k;
        uint64_t x = i < count ? (uint64_t)in[i] : 0;
        v[k] = run;
        run += x;
    }
    uint64_t prefix = block_exclusive_scan<SumOp64>(run, s_scan) + offsets[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        uint64_t i = base + k;
        if (i <= count) out[i] = v[k] + prefix;   // out[count] = total
    }
}

template <class T>
static void scan_impl(Ctx &ctx, const T *in, uint64_t *out, uint64_t count) {
    // tiles cover [0, count] inclusive so the total lands in out[count]
    uint64_t items = count + 1;
    uint64_t tiles = (items + kScanTile - 1) / kScanTile;
    uint64_t *partial = ctx.alloc<uint64_t>(tiles);
    uint64_t *offsets = ctx.alloc<uint64_t>(tiles + 1);
    k_scan_reduce<T><<<(unsigned)tiles, kScanThreads, 0, ctx.stream>>>(in, count, partial);
    TC_LAUNCHED(ctx);
    if (tiles == 1) {
        TC_CUDA(cudaMemsetAsync(offsets, 0, sizeof(uint64_t), ctx.stream));
    } else {
        scan_impl<uint64_t>(ctx, partial, offsets, tiles);
    }
    k_scan_apply<T><<<(unsigned)tiles, kScanThreads, 0, ctx.stream>>>(in, count, offsets, out);
    TC_LAUNCHED(ctx);
}

// Device-count variant: only the first *count_dev (<= cap) items are scanned; blocks past
// them exit at once (no n-sized traffic when few items are live), and the total is also
// written to *total_out.
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce_dc(const uint32_t *__restrict__ in,
                                                                 const uint64_t *__restrict__ count_dev,
                                                                 uint64_t *__restrict__ partial) {
    __shared__ uint64_t s_scratch[kScanThreads / 32];
    const uint64_t count = *count_dev;
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    if (base >= count) {
        if (threadIdx.x == 0) partial[blockIdx.x] = 0;
        return;
    }
    uint64_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
        if (i < count) sum += (uint64_t)in[i];
    }
    sum = block_sum_u64(sum, s_scratch);
    if (threadIdx.x == 0) partial[blockIdx.x] = sum;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply_dc(const uint32_t *__restrict__ in,
                                                                const uint64_t *__restrict__ count_dev,
                                                                const uint64_t *__restrict__ offsets,
                                                                uint64_t *__restrict__ out,
                                                                uint64_t *__restrict__ total_out) {
    __shared__ uint64_t s_scan[kScanThreads / 32];
    const uint64_t count = *count_dev;
    if ((uint64_t)blockIdx.x * kScanTile > count) return;   // block-uniform
    uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint64_t v[kScanItems];
    uint64_t run = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        uint64_t i = base + k;
        uint64_t x = i < count ? (uint64_t)in[i] : 0;
        v[k] = run;
        run += x;
    }
    uint64_t prefix = block_exclusive_scan<SumOp64>(run, s_scan) + offsets[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        uint64_t i = base + k;
        if (i <= count) out[i] = v[k] + prefix;
        if (i == count) *total_out = v[k] + prefix;
    }
}

void scan_exclusive_dc(Ctx &ctx, const uint32_t *in, uint64_t *out, uint64_t cap,
                       const uint64_t *count_dev, uint64_t *total_out) {
    uint64_t tiles = (cap + 1 + kScanTile - 1) / kScanTile;
    uint64_t *partial = ctx.alloc<uint64_t>(tiles);
    uint64_t *offsets = ctx.alloc<uint64_t>(tiles + 1);
    k_scan_reduce_dc<<<(unsigned)tiles, kScanThreads, 0, ctx.stream>>>(in, count_dev, partial);
    TC_LAUNCHED(ctx);
    if (tiles == 1) {
        TC_CUDA(cudaMemsetAsync(offsets, 0, sizeof(uint64_t), ctx.stream));
    } else {
        scan_impl<uint64_t>(ctx, partial, offsets, tiles);
    }
    k_scan_apply_dc<<<(unsigned)tiles, kScanThreads, 0, ctx.stream>>>(in, count_dev, offsets, out,
                                                                       total_out);
    TC_LAUNCHED(ctx);
}

void scan_exclusive(Ctx &ctx, const uint32_t *in, uint64_t *out, uint64_t count) {
    scan_impl<uint32_t>(ctx, in, out, count);
}
void scan_exclusive(Ctx &ctx, const uint64_t *in, uint64_t *out, uint64_t count) {
    scan_impl<uint64_t>(ctx, in, out, count);
}

// ------------------------------------------------------------------ tile row bounds
__device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t *__restrict__ a, uint64_t len, uint64_t x) {
    uint64_t lo = 0, hi = len;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__global__ void k_tile_bounds(const uint64_t *__restrict__ rowptr, uint64_t n, uint64_t items,
                              const uint64_t *__restrict__ items_dev, uint2 *__restrict__ bounds) {
    const uint64_t m = items_dev ? min(*items_dev, items) : items;
    const uint64_t tiles = (m + kTileItems - 1) / kTileItems;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tiles;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t0 = t * kTileItems, len = min((uint64_t)kTileItems, m - t0);
        bounds[t] = make_uint2((uint32_t)lower_bound_u64(rowptr, n + 1, t0 + 1),
                               (uint32_t)lower_bound_u64(rowptr, n + 1, t0 + len));
    }
}

void tile_bounds(Ctx &ctx, const uint64_t *rowptr, uint64_t n, uint64_t items, const uint64_t *items_dev,
                 uint2 *bounds) {
    const uint64_t tiles = (items + kTileItems - 1) / kTileItems;
    if (!tiles) return;
    const uint32_t grid = (uint32_t)std::min<uint64_t>((tiles + 255) / 256, (uint64_t)ctx.persistent_grid(8));
    k_tile_bounds<<<grid, 256, 0, ctx.stream>>>(rowptr, n, items, items_dev, bounds);
    TC_LAUNCHED(ctx);
}

}  // namespace tc
