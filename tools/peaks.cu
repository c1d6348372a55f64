// peaks.cu -- issue-rate microbenchmarks for the roofline denominators of the
// CUDA-core (popc) path on sm_100a: POPC and LOP3 per clock per SM.  One CTA of
// 1024 threads per SM, 8 independent dependency chains per thread; cycles are
// read with clock64() inside each CTA, so the result is per SM clock and does
// not depend on the (DVFS) frequency.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024) popc_rate(uint32_t* out, long long* cyc, int iters) {
    uint32_t x[8];
    uint32_t acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 0x9E3779B9u + i * 0x85EBCA6Bu + blockIdx.x; acc[i] = 0; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { acc[i] += __popc(x[i]); x[i] ^= acc[i]; }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i] ^ x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(1024) lop3_rate(uint32_t* out, long long* cyc, int iters) {
    uint32_t a[8], b = threadIdx.x * 7u + 1u, c = blockIdx.x * 13u + 5u;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0x9E3779B9u + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t r;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a[i]), "r"(b), "r"(c));
            a[i] = r;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 1024, iters = 4096;
    uint32_t* out; long long* cyc;
    cudaMalloc(&out, sizeof(uint32_t) * sms * threads);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    long long* h = new long long[sms];
    double rates[2];
    for (int which = 0; which < 2; ++which) {
        for (int rep = 0; rep < 3; ++rep) {
            if (which == 0) popc_rate<<<sms, threads>>>(out, cyc, iters);
            else lop3_rate<<<sms, threads>>>(out, cyc, iters);
        }
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        double mean = 0;
        for (int i = 0; i < sms; ++i) mean += (double)h[i];
        mean /= sms;
        rates[which] = (double)threads * iters * 8 / mean;   // ops per clock per SM
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"sms\": %d, \"popc_per_clk_per_sm\": %.3f, \"lop3_per_clk_per_sm\": %.3f, \"cuda\": \"%s\"}\n",
           sms, rates[0], rates[1], cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
