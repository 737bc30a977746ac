// segsort.cu -- a4: segmented sort of the oriented adjacency rows (north_star
// "segmented sort of the oriented adjacency lists"; needed when clean input rows
// are unsorted, SPEC S:209 requires sorted slices for the merge).
// Three tiers by row length:  <= 32: warp bitonic in registers;
// <= block_max (<= 8192): CTA bitonic in shared memory;  longer: CTA-local
// stable LSD radix sort (8-bit digits) through a global scratch buffer.
#include "block_scan.cuh"
#include "tc_internal.cuh"

namespace tc {

constexpr int kSegBlockThreads = 512;
constexpr uint32_t kSegSmemMax = 8192;

__global__ void k_seg_warp(const uint64_t *__restrict__ off, uint64_t n, uint32_t *__restrict__ col) {
    int lane = threadIdx.x & 31;
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t u = warp; u < n; u += nwarps) {
        uint64_t b = off[u], len = off[u + 1] - b;
        if (len < 2 || len > 32) continue;
        uint32_t x = lane < len ? col[b + lane] : kEmpty;
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
                bool asc = (lane & k) == 0, lower = (lane & j) == 0;
                x = (lower == asc) ? min(x, y) : max(x, y);
            }
        }
        if (lane < len) col[b + lane] = x;
    }
}

__global__ void __launch_bounds__(kSegBlockThreads)
    k_seg_block(const uint64_t *__restrict__ off, uint64_t n, uint32_t *__restrict__ col,
                uint32_t block_max) {
    extern __shared__ uint32_t s[];
    for (uint64_t u = blockIdx.x; u < n; u += gridDim.x) {
        uint64_t b = off[u], len = off[u + 1] - b;
        if (len <= 32 || len > block_max) continue;
        uint32_t P = 64;
        while (P < len) P <<= 1;
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) s[i] = i < len ? col[b + i] : kEmpty;
        __syncthreads();
        for (uint32_t k = 2; k <= P; k <<= 1) {
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                    uint32_t ixj = i ^ j;
                    if (ixj > i) {
                        bool asc = (i & k) == 0;
                        uint32_t a = s[i], c = s[ixj];
                        if ((a > c) == asc) {
                            s[i] = c;
                            s[ixj] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) col[b + i] = s[i];
        __syncthreads();
    }
}

// CTA-local stable radix sort of one long row, 4 passes of 8 bits, ping-pong
// between the row and the same range of `scratch` (even pass count: ends in col).
__global__ void __launch_bounds__(kSegBlockThreads)
    k_seg_radix(const uint64_t *__restrict__ off, uint64_t n, uint32_t *__restrict__ col,
                uint32_t *__restrict__ scratch, uint32_t block_max) {
    constexpr int W = kSegBlockThreads / 32;
    __shared__ uint32_t s_hist[256];
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_wc[W][256];
    __shared__ uint32_t s_scan[W];
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t lt = (1u << lane) - 1u;
    for (uint64_t u = blockIdx.x; u < n; u += gridDim.x) {
        uint64_t b = off[u], len = off[u + 1] - b;
        if (len <= block_max) continue;
        for (int pass = 0; pass < 4; pass++) {
            int shift = 8 * pass;
            uint32_t *src = (pass & 1) ? scratch + b : col + b;
            uint32_t *dst = (pass & 1) ? col + b : scratch + b;
            if (threadIdx.x < 256) s_hist[threadIdx.x] = 0;
            __syncthreads();
            for (uint64_t i = threadIdx.x; i < len; i += blockDim.x)
                atomicAdd(&s_hist[(src[i] >> shift) & 0xffu], 1u);
            __syncthreads();
            if (threadIdx.x < 256) {
                // exclusive scan of 256 digit counts by warps 0..7
                uint32_t h = s_hist[threadIdx.x];
                uint32_t inc = warp_inclusive_scan<SumOp>(h);
                if (lane == 31) s_scan[warp] = inc;
                s_base[threadIdx.x] = inc - h;
            }
            __syncthreads();
            if (threadIdx.x < 256) {
                uint32_t add = 0;
                for (int w = 0; w < warp; w++) add += s_scan[w];
                s_base[threadIdx.x] += add;
            }
            __syncthreads();
            for (uint64_t c0 = 0; c0 < len; c0 += blockDim.x) {
                for (int i = threadIdx.x; i < W * 256; i += blockDim.x) (&s_wc[0][0])[i] = 0;
                __syncthreads();
                uint64_t idx = c0 + threadIdx.x;
                bool valid = idx < len;
                uint32_t x = valid ? src[idx] : 0u, d = (x >> shift) & 0xffu;
                uint32_t active = __ballot_sync(0xffffffffu, valid), peers = 0, rank = 0;
                if (valid) {
                    peers = __match_any_sync(active, d);
                    rank = __popc(peers & lt);
                    if ((peers & lt) == 0) s_wc[warp][d] = __popc(peers);
                }
                __syncthreads();
                if (threadIdx.x < 256) {  // per digit: exclusive prefix over warps
                    uint32_t run = 0;
                    for (int w = 0; w < W; w++) {
                        uint32_t cnt = s_wc[w][threadIdx.x];
                        s_wc[w][threadIdx.x] = run;
                        run += cnt;
                    }
                    s_hist[threadIdx.x] = run;  // this chunk's count per digit
                }
                __syncthreads();
                if (valid) dst[s_base[d] + s_wc[warp][d] + rank] = x;
                __syncthreads();
                if (threadIdx.x < 256) s_base[threadIdx.x] += s_hist[threadIdx.x];
                __syncthreads();
            }
        }
    }
}

void segmented_sort(Ctx &ctx, uint64_t n, const uint64_t *off, uint32_t *col, uint64_t m_cap,
                    uint32_t block_max) {
    if (block_max == 0 || block_max > kSegSmemMax) block_max = kSegSmemMax;
    if (block_max < 32) block_max = 32;
    int grid = ctx.persistent_grid(4);
    k_seg_warp<<<grid, 256, 0, ctx.stream>>>(off, n, col);
    TC_LAUNCHED(ctx);
    uint32_t P = 64;
    while (P < block_max) P <<= 1;
    size_t smem = (size_t)P * sizeof(uint32_t);
    TC_CUDA(cudaFuncSetAttribute(k_seg_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    k_seg_block<<<grid, kSegBlockThreads, smem, ctx.stream>>>(off, n, col, block_max);
    TC_LAUNCHED(ctx);
    uint32_t *scratch = ctx.alloc<uint32_t>(m_cap);
    k_seg_radix<<<ctx.persistent_grid(1), kSegBlockThreads, 0, ctx.stream>>>(off, n, col, scratch,
                                                                              block_max);
    TC_LAUNCHED(ctx);
}

}  // namespace tc
