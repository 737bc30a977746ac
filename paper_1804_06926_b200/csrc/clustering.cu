// clustering.cu -- NEXT-1: local clustering coefficients, wedge
// count and the sum behind the average clustering, from the per-vertex triangle
// counts t (rank ids, a7) and the cleaned degrees d = d+ + d- (the oriented CSR and
// its transpose).  "With little modification, we could also use [it] to compute
// clustering coefficient and transitivity"; conventions in
// include/tc.h (reading R14).
//
// c(v) = 2 t / (d (d - 1)) is one correctly rounded fp64 division of exact integers
// (2t < 2^53, d (d-1) < 2^53), so it is bit-identical to any IEEE evaluation of the
// same expression.  Wedges are exact (uint64).  The sum of c(v) is reduced in a
// fixed order (per-thread strided sums, fixed-shape block trees, then one block over
// the per-block partials), so it is deterministic for a given grid.
#include "tc_internal.cuh"

namespace tc {

constexpr int kCcThreads = 256;

__device__ __forceinline__ void block_reduce_fixed(uint64_t &w, double &s, uint64_t *sw, double *ss) {
    sw[threadIdx.x] = w;
    ss[threadIdx.x] = s;
    __syncthreads();
    for (int h = kCcThreads / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            sw[threadIdx.x] += sw[threadIdx.x + h];
            ss[threadIdx.x] += ss[threadIdx.x + h];
        }
        __syncthreads();
    }
    w = sw[0];
    s = ss[0];
}

__global__ void __launch_bounds__(kCcThreads)
    k_cc(const uint64_t *__restrict__ off, const uint64_t *__restrict__ in_off,
         const uint32_t *__restrict__ order, const uint64_t *__restrict__ t, uint64_t n,
         double *__restrict__ cc, uint64_t *__restrict__ part_w, double *__restrict__ part_s) {
    __shared__ uint64_t sw[kCcThreads];
    __shared__ double ss[kCcThreads];
    uint64_t w = 0;
    double s = 0.0;
    for (uint64_t x = (uint64_t)blockIdx.x * kCcThreads + threadIdx.x; x < n;
         x += (uint64_t)gridDim.x * kCcThreads) {
        uint64_t d = (off[x + 1] - off[x]) + (in_off[x + 1] - in_off[x]);
        uint64_t pairs = d * (d - 1);   // 2 * C(d, 2); 0 for d < 2 (d = 0: 0 * (2^64-1) = 0)
        double c = d >= 2 ? (2.0 * (double)t[x]) / (double)pairs : 0.0;
        if (cc) cc[order[x]] = c;
        w += pairs / 2;
        s += c;
    }
    block_reduce_fixed(w, s, sw, ss);
    if (threadIdx.x == 0) {
        part_w[blockIdx.x] = w;
        part_s[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(kCcThreads)
    k_cc_final(const uint64_t *__restrict__ part_w, const double *__restrict__ part_s, int parts,
               uint64_t *__restrict__ out) {
    __shared__ uint64_t sw[kCcThreads];
    __shared__ double ss[kCcThreads];
    uint64_t w = 0;
    double s = 0.0;
    for (int i = threadIdx.x; i < parts; i += kCcThreads) {
        w += part_w[i];
        s += part_s[i];
    }
    block_reduce_fixed(w, s, sw, ss);
    if (threadIdx.x == 0) {
        out[0] = w;
        out[1] = __double_as_longlong(s);
    }
}

void clustering(Ctx &ctx, const Oriented &g, const uint64_t *t_new, double *cc, uint64_t *out2) {
    const int grid = ctx.persistent_grid(4);
    uint64_t *part_w = ctx.alloc<uint64_t>(grid);
    double *part_s = ctx.alloc<double>(grid);
    k_cc<<<grid, kCcThreads, 0, ctx.stream>>>(g.off, g.in_off, g.order, t_new, g.n, cc, part_w, part_s);
    TC_LAUNCHED(ctx);
    k_cc_final<<<1, kCcThreads, 0, ctx.stream>>>(part_w, part_s, grid, out2);
    TC_LAUNCHED(ctx);
}

}  // namespace tc
