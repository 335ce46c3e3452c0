// Device-side building blocks shared by every kernel of libgapsafe_b200.
//
// Determinism: every reduction here has a fixed shape (per-thread strided
// accumulation in ascending index order, xor-butterfly inside a warp, warps
// combined in ascending warp order), so results are bit-identical run to run
// (the reference's own run-to-run identity test, pkg/tests/test_path.py:124-131).
// No floating-point atomics anywhere.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gs {

constexpr int kWarp = 32;
constexpr double kU = 1.1102230246251565e-16;   // unit roundoff 2^-53

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;   // a + b == b + a bitwise, so every lane holds the same value
}

__device__ __forceinline__ double warp_sum_ru(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_ru(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// (value, index) max with smallest-index tie break (design_matrix.py:160-174).
__device__ __forceinline__ void argmax_merge(double& v, int64_t& i, double v2, int64_t i2) {
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__device__ __forceinline__ void warp_argmax(double& v, int64_t& i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        long long i2 = __shfl_xor_sync(0xffffffffu, (long long)i, o);
        argmax_merge(v, i, v2, (int64_t)i2);
    }
}

// Block sum, same value returned to every thread.  `red` must hold >= 32
// doubles and may be reused after the call returns (trailing barrier).
__device__ __forceinline__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < nw; ++k) s += red[k];
    __syncthreads();
    return s;
}

__device__ __forceinline__ double block_sum_ru(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum_ru(v);
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < nw; ++k) s = __dadd_ru(s, red[k]);
    __syncthreads();
    return s;
}

template <typename T> __device__ __forceinline__ double to_d(T x) { return (double)x; }

// gamma_n bound for an n-term dot product in any summation order (with or
// without FMA): |fl(x.v) - x.v| <= gamma * sum|x_r v_r|.
__host__ __device__ inline double gamma_n(int64_t n) {
    double nu = (double)(n + 40) * kU;    // +36u: the Gram-window consumer's final summations
    return nu / (1.0 - nu) * 1.0001;
}

}  // namespace gs
