// Instantiates the persistent solver kernels for storage type GS_T and rows
// per lane GS_R, and defines the gs_launch_*_<GS_SUF>_r<GS_R> launchers
// declared in gs_launch.h.  build() compiles this file once per (type, R)
// with -DGS_T=... -DGS_SUF=... -DGS_R=..., so the heavy instantiations build
// in parallel; gs_launch.cu dispatches on R at run time.
#include "gs_launch.h"
#include "gs_solve.cuh"

using namespace gs;

#define GS_CAT2(a, b) a##b
#define GS_CAT(a, b) GS_CAT2(a, b)
#define GS_NAME(base) GS_CAT(GS_CAT(GS_CAT(base, GS_SUF), _r), GS_R)

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

cudaError_t GS_NAME(gs_launch_solve_)(cudaStream_t st, const SolveDev* dprobs, int G, int nprob, size_t smem) {
    return solve_R<GS_R>(st, dprobs, G, nprob, smem);
}

cudaError_t GS_NAME(gs_launch_cdpass_)(cudaStream_t st, const SolveDev* dprobs, size_t smem) {
    return cdpass_R<GS_R>(st, dprobs, smem);
}

cudaError_t GS_NAME(gs_launch_batch_)(cudaStream_t st, SolveDev* dprobs, const BatchOut* douts, int B, size_t smem) {
#if GS_R <= 8
    return batch_R<GS_R>(st, dprobs, douts, B, smem);
#else
    (void)st; (void)dprobs; (void)douts; (void)B; (void)smem;
    return cudaErrorInvalidValue;     // batched problems: n <= 1792
#endif
}

#if GS_R == 1
cudaError_t GS_CAT(gs_launch_screen_full_, GS_SUF)(cudaStream_t st, const SolveDev* dprobs, double radius, int grid,
                                                   size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(k_screen_full<GS_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_screen_full<GS_T><<<(unsigned)grid, kThreads, smem, st>>>(dprobs, radius);
    return cudaGetLastError();
}
#endif
