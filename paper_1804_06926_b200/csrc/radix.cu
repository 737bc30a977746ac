// radix.cu -- hand-written stable LSD radix sort (8-bit digits) for 64-bit keys
// and for 32-bit key / 32-bit value pairs.  Per pass: a per-tile digit
// histogram, a device-wide exclusive scan of the digit-major histogram, and a
// stable scatter that ranks equal digits inside each warp with __match_any_sync.
#include "tc_internal.cuh"

namespace tc {

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixRounds = 16;                         // 32-item rounds per warp
constexpr int kRadixWarpItems = 32 * kRadixRounds;       // 512
constexpr int kRadixTile = kRadixWarps * kRadixWarpItems;  // 4096
constexpr int kDigits = 256;

__device__ __forceinline__ uint64_t valid_count(uint64_t cap, const uint64_t *count_dev) {
    if (!count_dev) return cap;
    uint64_t c = *count_dev;
    return c < cap ? c : cap;
}

template <class K>
__global__ void __launch_bounds__(kRadixThreads)
    k_radix_hist(const K *__restrict__ keys, uint64_t cap, const uint64_t *__restrict__ count_dev,
                 int shift, uint32_t *__restrict__ hist, uint32_t tiles) {
    __shared__ uint32_t h[kDigits];
    uint64_t n = valid_count(cap, count_dev);
    h[threadIdx.x] = 0;
    __syncthreads();
    uint64_t base = (uint64_t)blockIdx.x * kRadixTile;
    if (base < n) {
        for (int k = 0; k < kRadixTile / kRadixThreads; k++) {
            uint64_t i = base + (uint64_t)k * kRadixThreads + threadIdx.x;
            if (i < n) atomicAdd(&h[(uint32_t)(keys[i] >> shift) & 0xffu], 1u);
        }
    }
    __syncthreads();
    hist[(uint64_t)threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

template <class K, bool kVals>
__global__ void __launch_bounds__(kRadixThreads)
    k_radix_scatter(const K *__restrict__ keys, const uint32_t *__restrict__ vals,
                    K *__restrict__ keys_out, uint32_t *__restrict__ vals_out, uint64_t cap,
                    const uint64_t *__restrict__ count_dev, int shift,
                    const uint64_t *__restrict__ offsets, uint32_t tiles) {
    __shared__ uint32_t s_wc[kRadixWarps][kDigits];
    __shared__ uint64_t s_base[kDigits];
    uint64_t n = valid_count(cap, count_dev);
    uint64_t tile_base = (uint64_t)blockIdx.x * kRadixTile;
    if (tile_base >= n) return;
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kRadixWarps * kDigits; i += kRadixThreads)
        (&s_wc[0][0])[i] = 0;
    __syncthreads();

    uint64_t wbase = tile_base + (uint64_t)warp * kRadixWarpItems;
    K key[kRadixRounds];
    uint32_t val[kRadixRounds];
    uint32_t rank[kRadixRounds];
    uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kRadixRounds; j++) {
        uint64_t idx = wbase + (uint64_t)j * 32 + lane;
        bool valid = idx < n;
        key[j] = valid ? keys[idx] : (K)0;
        if (kVals) val[j] = valid ? vals[idx] : 0u;
        uint32_t d = (uint32_t)(key[j] >> shift) & 0xffu;
        uint32_t active = __ballot_sync(0xffffffffu, valid);
        uint32_t old = 0, peers = 0;
        if (valid) {
            peers = __match_any_sync(active, d);
            old = s_wc[warp][d];
        }
        __syncwarp();
        if (valid && (peers & lt) == 0) s_wc[warp][d] = old + __popc(peers);
        __syncwarp();
        rank[j] = old + __popc(peers & lt);
    }
    __syncthreads();
    {
        uint32_t d = threadIdx.x;  // kRadixThreads == kDigits
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kRadixWarps; w++) {
            uint32_t c = s_wc[w][d];
            s_wc[w][d] = run;
            run += c;
        }
        s_base[d] = offsets[(uint64_t)d * tiles + blockIdx.x];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRadixRounds; j++) {
        uint64_t idx = wbase + (uint64_t)j * 32 + lane;
        if (idx < n) {
            uint32_t d = (uint32_t)(key[j] >> shift) & 0xffu;
            uint64_t pos = s_base[d] + s_wc[warp][d] + rank[j];
            keys_out[pos] = key[j];
            if (kVals) vals_out[pos] = val[j];
        }
    }
}

template <class K, bool kVals>
static bool radix_impl(Ctx &ctx, K *keys, K *keys_alt, uint32_t *vals, uint32_t *vals_alt,
                       uint64_t capacity, const uint64_t *count_dev, int bits) {
    if (capacity == 0 || bits <= 0) return false;
    uint32_t tiles = (uint32_t)((capacity + kRadixTile - 1) / kRadixTile);
    uint32_t *hist = ctx.alloc<uint32_t>((uint64_t)kDigits * tiles);
    uint64_t *offsets = ctx.alloc<uint64_t>((uint64_t)kDigits * tiles + 1);
    bool alt = false;
    for (int shift = 0; shift < bits; shift += 8) {
        K *kin = alt ? keys_alt : keys, *kout = alt ? keys : keys_alt;
        uint32_t *vin = alt ? vals_alt : vals, *vout = alt ? vals : vals_alt;
        k_radix_hist<K><<<tiles, kRadixThreads, 0, ctx.stream>>>(kin, capacity, count_dev, shift,
                                                                 hist, tiles);
        TC_LAUNCHED(ctx);
        scan_exclusive(ctx, hist, offsets, (uint64_t)kDigits * tiles);
        k_radix_scatter<K, kVals><<<tiles, kRadixThreads, 0, ctx.stream>>>(
            kin, vin, kout, vout, capacity, count_dev, shift, offsets, tiles);
        TC_LAUNCHED(ctx);
        alt = !alt;
    }
    return alt;
}

bool radix_sort(Ctx &ctx, uint64_t *keys, uint64_t *keys_alt, uint64_t capacity,
                const uint64_t *count_dev, int bits) {
    return radix_impl<uint64_t, false>(ctx, keys, keys_alt, nullptr, nullptr, capacity, count_dev,
                                       bits);
}

bool radix_sort_pairs(Ctx &ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                      uint32_t *vals_alt, uint64_t capacity, const uint64_t *count_dev, int bits) {
    return radix_impl<uint32_t, true>(ctx, keys, keys_alt, vals, vals_alt, capacity, count_dev,
                                      bits);
}

}  // namespace tc
