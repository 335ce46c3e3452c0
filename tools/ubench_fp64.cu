// Microbenchmarks that size the CD chain on B200: dependent-latency and
// per-SM throughput of DFMA / DADD.RU / SHFL(double) / LDS.64 / named barrier /
// smem polling handshake between two warps.  One CTA, clock64() deltas.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ubench_fp64 tools/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(long long* out, double seed, int iters) {
    __shared__ double sm[1024];
    __shared__ volatile int flag[2];
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 1024; i += blockDim.x) sm[i] = seed + i;
    if (tid < 2) flag[tid] = 0;
    __syncthreads();
    double a = seed, b = seed * 0.5;
    long long t0, t1;
    // 1. dependent DFMA
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, 0.999999, b);
    t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0);
    // 2. dependent DADD.RU
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a = __dadd_ru(a, b);
    t1 = clock64();
    if (tid == 0) out[1] = (t1 - t0);
    // 3. dependent shfl.xor of a double + add (butterfly level)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1 + (i & 15));
    t1 = clock64();
    if (tid == 0) out[2] = (t1 - t0);
    // 4. dependent LDS.64 (pointer chase through smem indices)
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { double v = sm[idx]; idx = ((int)v) & 1023; }
    t1 = clock64();
    if (tid == 0) out[3] = (t1 - t0);
    a += idx;
    // 5. full warp_sum (5 butterfly levels) dependent
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double v = a;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        a = v * 1e-3;
    }
    t1 = clock64();
    if (tid == 0) out[4] = (t1 - t0);
    // 6. division chain as in the CD (q0=g*iv; r=fma(-q0,ns,g); q=fma(r,iv,q0); z=b+q; ST)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const double q0 = a * 0.37, r = fma(-q0, 2.7, a), q = fma(r, 0.37, q0), z = b + q;
        a = z > 0.1 ? z - 0.1 : (z < -0.1 ? z + 0.1 : 0.0);
        a += 1.0;
    }
    t1 = clock64();
    if (tid == 0) out[5] = (t1 - t0);
    // 7. named barrier among 4 warps (only warps 0..3 take part)
    if (tid < 128) {
        t0 = clock64();
        for (int i = 0; i < iters; ++i) asm volatile("bar.sync 1, 128;" ::: "memory");
        t1 = clock64();
        if (tid == 0) out[6] = (t1 - t0);
    }
    __syncthreads();
    // 8. ping-pong through smem flags between warp 0 and warp 1 (round trip)
    if (tid == 0) {
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            flag[0] = i + 1;
            while (flag[1] != i + 1) {}
        }
        t1 = clock64();
        out[7] = (t1 - t0);
    } else if (tid == 32) {
        for (int i = 0; i < iters; ++i) {
            while (flag[0] != i + 1) {}
            flag[1] = i + 1;
        }
    }
    __syncthreads();
    if (tid == 0) out[15] = (long long)a;
}

// throughput: every warp runs independent DFMA chains (8 per thread)
__global__ void k_tput(long long* out, double seed, int iters, int mode) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + k;
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) {
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 0.999999, 1e-7);
    } else {
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] += __shfl_xor_sync(0xffffffffu, a[k], 1 + k);
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (s == 12345.678) out[1] = 1;
}

int main() {
    long long *d, h[16];
    cudaMalloc(&d, 16 * sizeof(long long));
    const int iters = 4096;
    k_lat<<<1, 256>>>(d, 1.0, iters);
    k_lat<<<1, 256>>>(d, 1.0, iters);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[] = {"DFMA dep", "DADD.RU dep", "shfl.xor f64 + DADD dep", "LDS.64 chase", "warp_sum (5 lvl) + DMUL",
                           "div-chain+ST+DADD", "bar.sync 1,128", "smem ping-pong roundtrip"};
    for (int i = 0; i < 8; ++i) printf("%-28s %8.1f cycles\n", names[i], (double)h[i] / iters);
    for (int mode = 0; mode < 2; ++mode)
        for (int threads = 128; threads <= 1024; threads *= 2) {
            k_tput<<<1, threads>>>(d, 1.0, iters, mode);
            cudaMemcpy(h, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
            const double ops = (double)threads * iters * 8;
            printf("%s threads=%4d: %.2f %s/clk/SM\n", mode ? "SHFL.f64+DADD" : "DFMA", threads, ops / h[0],
                   mode ? "lane-shfl" : "FMA");
        }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
