// Run-time dispatch on the rows-per-lane template parameter R to the
// per-(type, R) launchers of gs_solve_inst.cu.
#include "gs_launch.h"

#define GS_DISPATCH(SUF)                                                                                        \
    cudaError_t gs_launch_solve_##SUF(int R, cudaStream_t st, const gs::SolveDev* dprobs, int G, int nprob,      \
                                      size_t smem) {                                                          \
        switch (R) {                                                                                          \
            case 1: return gs_launch_solve_##SUF##_r1(st, dprobs, G, nprob, smem);                            \
            case 2: return gs_launch_solve_##SUF##_r2(st, dprobs, G, nprob, smem);                            \
            case 4: return gs_launch_solve_##SUF##_r4(st, dprobs, G, nprob, smem);                            \
            case 5: return gs_launch_solve_##SUF##_r5(st, dprobs, G, nprob, smem);                            \
            case 8: return gs_launch_solve_##SUF##_r8(st, dprobs, G, nprob, smem);                            \
            default: return gs_launch_solve_##SUF##_r48(st, dprobs, G, nprob, smem);                          \
        }                                                                                                     \
    }                                                                                                         \
    cudaError_t gs_launch_cdpass_##SUF(int R, cudaStream_t st, const gs::SolveDev* dprobs, size_t smem) {        \
        switch (R) {                                                                                          \
            case 1: return gs_launch_cdpass_##SUF##_r1(st, dprobs, smem);                                     \
            case 2: return gs_launch_cdpass_##SUF##_r2(st, dprobs, smem);                                     \
            case 4: return gs_launch_cdpass_##SUF##_r4(st, dprobs, smem);                                     \
            case 5: return gs_launch_cdpass_##SUF##_r5(st, dprobs, smem);                                     \
            case 8: return gs_launch_cdpass_##SUF##_r8(st, dprobs, smem);                                     \
            default: return gs_launch_cdpass_##SUF##_r48(st, dprobs, smem);                                   \
        }                                                                                                     \
    }                                                                                                         \
    cudaError_t gs_launch_batch_##SUF(int R, cudaStream_t st, gs::SolveDev* dprobs, const gs::BatchOut* douts,   \
                                      int B, size_t smem) {                                                   \
        switch (R) {                                                                                          \
            case 1: return gs_launch_batch_##SUF##_r1(st, dprobs, douts, B, smem);                            \
            case 2: return gs_launch_batch_##SUF##_r2(st, dprobs, douts, B, smem);                            \
            case 4: return gs_launch_batch_##SUF##_r4(st, dprobs, douts, B, smem);                            \
            case 5: return gs_launch_batch_##SUF##_r5(st, dprobs, douts, B, smem);                            \
            case 8: return gs_launch_batch_##SUF##_r8(st, dprobs, douts, B, smem);                            \
            default: return cudaErrorInvalidValue;     /* batched problems: n <= 1792 */                       \
        }                                                                                                     \
    }

GS_DISPATCH(f64)
GS_DISPATCH(f32)
