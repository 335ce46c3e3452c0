// Instantiates the persistent solver kernels for storage type GS_T and
// defines the gs_launch_*_<GS_SUF> launchers declared in gs_launch.h.
#include "gs_launch.h"
#include "gs_solve.cuh"

using namespace gs;

#define GS_CAT2(a, b) a##b
#define GS_CAT(a, b) GS_CAT2(a, b)

namespace {
constexpr int kThreads = 256;

template <int R>
cudaError_t solve_R(cudaStream_t st, const SolveDev* dprobs, int G, int nprob, size_t smem) {
    auto kern = k_solve<GS_T, R>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int G_ = G;
    void* args[] = {(void*)&dprobs, (void*)&G_};
    return cudaLaunchCooperativeKernel((void*)kern, dim3((unsigned)(G * nprob)), dim3(kThreads), args, smem, st);
}

template <int R>
cudaError_t cdpass_R(cudaStream_t st, const SolveDev* dprobs, size_t smem) {
    auto kern = k_cd_pass_prod<GS_T, R>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<1, kThreads, smem, st>>>(dprobs);
    return cudaGetLastError();
}

template <int R>
cudaError_t batch_R(cudaStream_t st, SolveDev* dprobs, const BatchOut* douts, int B, size_t smem) {
    auto kern = k_batch_path<GS_T, R>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int* next = nullptr;
    e = cudaMallocAsync((void**)&next, sizeof(int), st);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(next, 0, sizeof(int), st);
    const int grid = B < sms ? B : sms;
    kern<<<(unsigned)grid, kThreads, smem, st>>>(dprobs, douts, B, next);
    e = cudaGetLastError();
    cudaFreeAsync(next, st);
    return e;
}
}  // namespace

cudaError_t GS_CAT(gs_launch_solve_, GS_SUF)(int R, cudaStream_t st, const SolveDev* dprobs, int G, int nprob,
                                             size_t smem) {
    switch (R) {
        case 1: return solve_R<1>(st, dprobs, G, nprob, smem);
        case 2: return solve_R<2>(st, dprobs, G, nprob, smem);
        case 4: return solve_R<4>(st, dprobs, G, nprob, smem);
        case 8: return solve_R<8>(st, dprobs, G, nprob, smem);
        default: return solve_R<48>(st, dprobs, G, nprob, smem);
    }
}

cudaError_t GS_CAT(gs_launch_cdpass_, GS_SUF)(int R, cudaStream_t st, const SolveDev* dprobs, size_t smem) {
    switch (R) {
        case 1: return cdpass_R<1>(st, dprobs, smem);
        case 2: return cdpass_R<2>(st, dprobs, smem);
        case 4: return cdpass_R<4>(st, dprobs, smem);
        case 8: return cdpass_R<8>(st, dprobs, smem);
        default: return cdpass_R<48>(st, dprobs, smem);
    }
}

cudaError_t GS_CAT(gs_launch_batch_, GS_SUF)(int R, cudaStream_t st, SolveDev* dprobs, const BatchOut* douts, int B,
                                             size_t smem) {
    switch (R) {
        case 1: return batch_R<1>(st, dprobs, douts, B, smem);
        case 2: return batch_R<2>(st, dprobs, douts, B, smem);
        case 4: return batch_R<4>(st, dprobs, douts, B, smem);
        case 8: return batch_R<8>(st, dprobs, douts, B, smem);
        default: return cudaErrorInvalidValue;     // batched problems: n <= 1792
    }
}

cudaError_t GS_CAT(gs_launch_screen_full_, GS_SUF)(cudaStream_t st, const SolveDev* dprobs, double radius, int grid,
                                                   size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(k_screen_full<GS_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_screen_full<GS_T><<<(unsigned)grid, kThreads, smem, st>>>(dprobs, radius);
    return cudaGetLastError();
}
