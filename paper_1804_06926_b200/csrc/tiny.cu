// tiny.cu -- the whole method in ONE kernel launch for small graphs (n <= 1024).
//
// The paper notes that on small graphs the step overheads dominate (the filter's
// "overhead causes a slowdown on road networks and small scale-free graphs"); the general
// pipeline launches ~60 kernels.  For n <= 1024 one CTA holds the whole graph as an n x n
// adjacency bitmap in shared memory (n^2 / 8 bytes, 128 KB at n = 1024) and runs every step
// of Alg. 2 on it:
//   a1 clean      -- each arc u -> v, u != v, sets bits (u, v) and (v, u): duplicates and
//                    antiparallel arcs collapse, self-loops are dropped (Table 1);
//   a2 degree     -- d(v) = popcount of row v;
//   a3 filter     -- row u keeps the neighbours v with rank(v) > rank(u), rank = (d, id)
//                    (DESIGN reading R2): row u becomes N+(u) as a bitmap;
//   a6 intersect  -- every oriented edge (u, v) adds popc(N+(u) & N+(v)) (both rows, word
//                    by word; w in N+(v) already has rank(w) > rank(v));
//   a7 reduce     -- per-lane sums, warp shuffles, one atomicAdd for the CTA.
// Per-vertex counts credit u, v and every common w (shared-memory counters).  Vertex ids
// stay the input's (no relabelling is needed: the rank test is a comparison).  Plain counts
// and per-vertex counts only; every other entry point uses the general pipeline.
#include "tc_internal.cuh"

namespace tc {

constexpr uint32_t kTinyThreads = 1024;

__device__ __forceinline__ bool tiny_rank_less(const uint32_t *deg, uint32_t u, uint32_t v) {
    return deg[u] < deg[v] || (deg[u] == deg[v] && u < v);
}

__global__ void __launch_bounds__(kTinyThreads)
    k_tiny(const uint64_t *__restrict__ rowptr, const uint32_t *__restrict__ col, uint32_t n,
           uint64_t *__restrict__ out_m, uint64_t *__restrict__ total, uint64_t *__restrict__ pv) {
    extern __shared__ __align__(16) uint32_t smem[];
    const uint32_t words = (n + 31) / 32;            // row length
    uint32_t *A = smem;                              // n x words adjacency bitmap
    uint32_t *deg = A + (size_t)n * words;           // d(v)
    uint32_t *tv = deg + n;                          // per-vertex counters (pv != nullptr)
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t kWarps = kTinyThreads / 32;
    for (uint32_t i = tid; i < n * words; i += kTinyThreads) A[i] = 0u;
    for (uint32_t i = tid; i < n; i += kTinyThreads) tv[i] = 0u;
    __syncthreads();
    // a1: one warp per row of the input CSR, lanes over its arcs
    for (uint32_t u = warp; u < n; u += kWarps) {
        const uint64_t b = rowptr[u], e = rowptr[u + 1];
        for (uint64_t k = b + lane; k < e; k += 32) {
            const uint32_t v = col[k];
            if (v == u) continue;
            atomicOr(&A[(size_t)u * words + (v >> 5)], 1u << (v & 31));
            atomicOr(&A[(size_t)v * words + (u >> 5)], 1u << (u & 31));
        }
    }
    __syncthreads();
    // a2: degrees (warp per row)
    for (uint32_t u = warp; u < n; u += kWarps) {
        uint32_t c = 0;
        for (uint32_t w = lane; w < words; w += 32) c += __popc(A[(size_t)u * words + w]);
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) deg[u] = c;
    }
    __syncthreads();
    // a3: keep the higher-ranked neighbours (one thread per row word); m from the kept bits
    uint32_t kept = 0;
    for (uint32_t i = tid; i < n * words; i += kTinyThreads) {
        const uint32_t u = i / words, w0 = (i - u * words) * 32;
        uint32_t bits = A[i], keep = 0;
        while (bits) {
            const uint32_t b = __ffs(bits) - 1;
            bits &= bits - 1;
            if (tiny_rank_less(deg, u, w0 + b)) keep |= 1u << b;
        }
        kept += __popc(keep);
        // (rows are only read after the barrier below, so the in-place write is safe)
        A[i] = keep;
    }
    __syncthreads();
    // a6 + a7: warp per source u, lanes over words; for every v in N+(u) add the AND counts
    uint64_t acc = 0;
    for (uint32_t u = warp; u < n; u += kWarps) {
        const uint32_t *Pu = A + (size_t)u * words;
        uint32_t cu = 0;
        for (uint32_t wv = 0; wv < words; wv++) {
            uint32_t vb = Pu[wv];   // broadcast read: the same word in every lane
            while (vb) {
                const uint32_t v = wv * 32 + __ffs(vb) - 1;
                vb &= vb - 1;
                const uint32_t *Pv = A + (size_t)v * words;
                uint32_t c = 0;
                for (uint32_t w = lane; w < words; w += 32) {
                    uint32_t x = Pu[w] & Pv[w];
                    c += __popc(x);
                    if (pv)
                        while (x) {
                            atomicAdd(&tv[w * 32 + __ffs(x) - 1], 1u);
                            x &= x - 1;
                        }
                }
                acc += c;
                if (pv) {
                    c = __reduce_add_sync(0xffffffffu, c);
                    if (lane == 0 && c) atomicAdd(&tv[v], c);
                    cu += c;
                }
            }
        }
        if (pv && lane == 0 && cu) atomicAdd(&tv[u], cu);
    }
    __shared__ uint64_t s_red[32];
    const uint64_t t = block_sum_u64(acc, s_red);
    const uint64_t mm = block_sum_u64(kept, s_red);
    if (tid == 0) {
        *total = t;
        *out_m = mm;
    }
    if (pv)
        for (uint32_t i = tid; i < n; i += kTinyThreads) pv[i] = tv[i];
}

size_t tiny_smem_bytes(uint64_t n) {
    const uint64_t words = (n + 31) / 32;
    return (size_t)(n * words + 2 * n) * sizeof(uint32_t);
}

void tiny_count(Ctx &ctx, uint64_t n, const uint64_t *rowptr, const uint32_t *col,
                uint64_t *total_dev, uint64_t *pv_dev, uint64_t *m_dev) {
    const size_t smem = tiny_smem_bytes(n);
    TC_CUDA(cudaFuncSetAttribute(k_tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_tiny<<<1, kTinyThreads, smem, ctx.stream>>>(rowptr, col, (uint32_t)n, m_dev, total_dev, pv_dev);
    TC_LAUNCHED(ctx);
}

}  // namespace tc
