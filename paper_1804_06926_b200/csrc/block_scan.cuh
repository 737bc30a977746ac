// block_scan.cuh -- warp-shuffle block scans (one value per thread).
#pragma once
#include <stdint.h>

namespace tc {

struct SumOp {
    using T = uint32_t;
    static __device__ __forceinline__ T identity() { return 0u; }
    static __device__ __forceinline__ T apply(T a, T b) { return a + b; }
};
struct SumOp64 {
    using T = uint64_t;
    static __device__ __forceinline__ T identity() { return 0ull; }
    static __device__ __forceinline__ T apply(T a, T b) { return a + b; }
};
struct MaxOp {
    using T = uint32_t;
    static __device__ __forceinline__ T identity() { return 0u; }
    static __device__ __forceinline__ T apply(T a, T b) { return a > b ? a : b; }
};

template <class Op>
__device__ __forceinline__ typename Op::T warp_inclusive_scan(typename Op::T v) {
    int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        typename Op::T y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = Op::apply(v, y);
    }
    return v;
}

// Exclusive block scan; `scratch` holds blockDim.x/32 values; optional total.
// Must be called by every thread of the block; ends with a __syncthreads().
template <class Op>
__device__ __forceinline__ typename Op::T block_exclusive_scan(typename Op::T v,
                                                                typename Op::T *scratch,
                                                                typename Op::T *total = nullptr) {
    using T = typename Op::T;
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    T inc = warp_inclusive_scan<Op>(v);
    if (lane == 31) scratch[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nwarps ? scratch[lane] : Op::identity();
        T wi = warp_inclusive_scan<Op>(w);
        if (lane < nwarps) scratch[lane] = wi;  // inclusive warp totals
    }
    __syncthreads();
    T warp_prefix = warp == 0 ? Op::identity() : scratch[warp - 1];
    T excl = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) excl = Op::identity();
    T result = Op::apply(warp_prefix, excl);
    if (total) *total = scratch[nwarps - 1];
    __syncthreads();
    return result;
}

}  // namespace tc
