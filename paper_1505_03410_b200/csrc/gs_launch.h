// Launchers of the persistent solver kernels: one translation unit per
// (storage type, rows per lane) -- gs_solve_inst.cu compiled with -D flags --
// so the heavy template instantiations compile in parallel; gs_launch.cu
// dispatches on R.  Every function returns a cudaError_t.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace gs {
struct SolveDev;
struct BatchOut;
}  // namespace gs

#define GS_DECLARE_R(SUF, R)                                                                                  \
    cudaError_t gs_launch_solve_##SUF##_r##R(cudaStream_t st, const gs::SolveDev* dprobs, int G, int nprob,          \
                                             size_t smem);                                                        \
    cudaError_t gs_launch_cdpass_##SUF##_r##R(cudaStream_t st, const gs::SolveDev* dprobs, size_t smem);             \
    cudaError_t gs_launch_batch_##SUF##_r##R(cudaStream_t st, gs::SolveDev* dprobs, const gs::BatchOut* douts,       \
                                             int B, size_t smem);
#define GS_DECLARE_LAUNCHERS(SUF)                                                                              \
    GS_DECLARE_R(SUF, 1) GS_DECLARE_R(SUF, 2) GS_DECLARE_R(SUF, 4) GS_DECLARE_R(SUF, 5) GS_DECLARE_R(SUF, 8) GS_DECLARE_R(SUF, 48)    \
    cudaError_t gs_launch_solve_##SUF(int R, cudaStream_t st, const gs::SolveDev* dprobs, int G, int nprob,        \
                                      size_t smem);                                                            \
    cudaError_t gs_launch_cdpass_##SUF(int R, cudaStream_t st, const gs::SolveDev* dprobs, size_t smem);           \
    cudaError_t gs_launch_batch_##SUF(int R, cudaStream_t st, gs::SolveDev* dprobs, const gs::BatchOut* douts, int B,  \
                                      size_t smem);                                                            \
    cudaError_t gs_launch_screen_full_##SUF(cudaStream_t st, const gs::SolveDev* dprobs, double radius, int grid,  \
                                            size_t smem);

GS_DECLARE_LAUNCHERS(f64)
GS_DECLARE_LAUNCHERS(f32)
#undef GS_DECLARE_LAUNCHERS
#undef GS_DECLARE_R
