// Microbenchmark: cost per iteration of the MMA-issuer's per-tile synchronisation
// ops (try_wait on a completed mbarrier phase, tcgen05.fence::after_thread_sync,
// tcgen05.commit) issued by one thread, no MMAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void kern(int mode, int iters, long long* out) {
    __shared__ __align__(8) uint64_t bar[8];
    __shared__ uint32_t tptr;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        // complete phase 0 of bar[0] (so parity-0 waits return at once)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[0])) : "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tptr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; ++i) {
            if (mode & 1)
                asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, %1;\n\t@!p bra W_%=;\n\t}"
                             ::"r"(smem_u32(&bar[0])), "r"(1000000u) : "memory");
            if (mode & 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (mode & 4)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(smem_u32(&bar[1 + (i & 3)])) : "memory");
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tptr));
    if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
    long long* d; cudaMalloc(&d, 8);
    const char* names[] = {"none", "wait", "fence", "wait+fence", "commit", "wait+commit", "fence+commit", "all"};
    for (int mode = 0; mode < 8; ++mode) {
        const int it = 10000;
        kern<<<1, 64>>>(mode, it, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-14s %.1f cycles/iter  %s\n", names[mode], (double)h / it, cudaGetErrorString(e));
    }
    return 0;
}
