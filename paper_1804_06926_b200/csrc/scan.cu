// scan.cu -- device-wide exclusive scan (single pass, decoupled look-back) and the block-level
// scan / tile row-search helpers every tile kernel uses.
#include <algorithm>

#include "tc_internal.cuh"
#include "block_scan.cuh"

namespace tc {

// ------------------------------------------------------------------ global scan
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// Single pass (round 2): tiles take a ticket, publish their aggregate, and get the exclusive
// prefix of earlier tiles by decoupled look-back (one warp, 32 predecessors per step): one
// launch and one read of the input instead of reduce + (recursive scan) + apply.  With
// count_dev only the first *count_dev (<= cap) items are scanned; out[count] = the total,
// also written to *total_out when given.
constexpr uint64_t kScAgg = 1ull << 62, kScPre = 2ull << 62, kScMask = (1ull << 62) - 1;
template <class T>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_1p(const T *__restrict__ in, uint64_t cap, const uint64_t *__restrict__ count_dev,
              uint64_t *__restrict__ out, uint64_t *__restrict__ total_out, uint32_t *__restrict__ ticket,
              uint64_t *__restrict__ status) {
    __shared__ uint64_t s_scan[kScanThreads / 32];
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_excl;
    const uint64_t count = count_dev ? min(*count_dev, cap) : cap;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if ((uint64_t)tile * kScanTile > count) return;   // tiles cover [0, count]; nobody waits here
    const uint64_t base = (uint64_t)tile * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint64_t v[kScanItems];
    uint64_t run = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        const uint64_t i = base + k;
        const uint64_t x = i < count ? (uint64_t)in[i] : 0;
        v[k] = run;
        run += x;
    }
    uint64_t total;
    const uint64_t pre = block_exclusive_scan<SumOp64>(run, s_scan, &total);
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        uint64_t excl = 0;
        if (lane == 0)
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(status + tile),
                         "l"((tile == 0 ? kScPre : kScAgg) | total) : "memory");
        if (tile > 0) {
            for (int64_t t = (int64_t)tile - 1;; t -= 32) {
                const int64_t idx = t - (int64_t)lane;
                uint64_t sw = kScPre;
                if (idx >= 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(sw) : "l"(status + idx) : "memory");
                while (__any_sync(0xffffffffu, (sw & ~kScMask) == 0))
                    if ((sw & ~kScMask) == 0)
                        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(sw) : "l"(status + idx) : "memory");
                const uint32_t pm = __ballot_sync(0xffffffffu, (sw & kScPre) != 0);
                const int first = pm ? __ffs(pm) - 1 : 32;
                excl += warp_sum_u64((int)lane <= first ? (sw & kScMask) : 0ull);
                if (pm) break;
            }
            if (lane == 0)
                asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(status + tile),
                             "l"(kScPre | (excl + total)) : "memory");
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    const uint64_t prefix = pre + s_excl;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        const uint64_t i = base + k;
        if (i <= count) out[i] = v[k] + prefix;
        if (i == count && total_out) *total_out = v[k] + prefix;
    }
}

template <class T>
static void scan_1p(Ctx &ctx, const T *in, uint64_t *out, uint64_t cap, const uint64_t *count_dev,
                    uint64_t *total_out) {
    const uint64_t tiles = (cap + 1 + kScanTile - 1) / kScanTile;
    uint64_t *st = ctx.alloc<uint64_t>(tiles + 1);   // status words, then the ticket
    TC_CUDA(cudaMemsetAsync(st, 0, (tiles + 1) * sizeof(uint64_t), ctx.stream));
    k_scan_1p<T><<<(unsigned)tiles, kScanThreads, 0, ctx.stream>>>(in, cap, count_dev, out, total_out,
                                                                   (uint32_t *)(st + tiles), st);
    TC_LAUNCHED(ctx);
}

void scan_exclusive_dc(Ctx &ctx, const uint32_t *in, uint64_t *out, uint64_t cap,
                       const uint64_t *count_dev, uint64_t *total_out) {
    scan_1p<uint32_t>(ctx, in, out, cap, count_dev, total_out);
}

void scan_exclusive(Ctx &ctx, const uint32_t *in, uint64_t *out, uint64_t count) {
    scan_1p<uint32_t>(ctx, in, out, count, nullptr, nullptr);
}
void scan_exclusive(Ctx &ctx, const uint64_t *in, uint64_t *out, uint64_t count) {
    scan_1p<uint64_t>(ctx, in, out, count, nullptr, nullptr);
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
