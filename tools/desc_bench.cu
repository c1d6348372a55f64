// Microbenchmark: tcgen05.mma kind::i8 cycles per MMA when every MMA reads a
// different A window (tap-offset pattern of conv_tz: 5 K-slice pairs per tile,
// tiles 2 KB apart), for 16-byte-misaligned vs 128-byte-aligned A starts.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)8 << 32) | (1ull << 46);
}
constexpr int SMEM = 200 * 1024;

__global__ void __launch_bounds__(128, 1) kern(int n, int align, int reps, int ntile, long long* cyc, int commit_every, int dstride) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bar2[8];
    __shared__ uint32_t tptr;
    for (int i = threadIdx.x; i < SMEM / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(i, i * 3, 0, 1);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tptr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t d = tptr;
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 150 * 1024);
    // tap offsets of a W = 256 plane (Po = 257): rows dy*257 + dx, paired as in conv_tz
    const int P = 257;
    int offs[5] = {0, 2, 257 + 1, 2 * 257, 2 * 257 + 2};
    int lbos[5] = {1, P - 2, 1, 1, 1};
    if (align) for (int i = 0; i < 5; ++i) { offs[i] = (offs[i] + 7) & ~7; lbos[i] = (lbos[i] + 7) & ~7; }
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    long long t0 = 0, t1 = 0;
    const int nw = dstride >= 3 ? 2 : 1;
    const bool exact = dstride == 4;
    if (threadIdx.x < 32 * nw) {
        const int w = threadIdx.x >> 5;
        uint32_t pred = 0;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
        __syncwarp();
        t0 = clock64();
        if (pred) {
            for (int r = 0; r < reps; ++r)
                for (int t = w; t < ntile; t += nw) {
                    if (commit_every < 0) {   // a per-tile wait on an already completed barrier phase
                        asm volatile("{\n\t.reg .pred p;\nWT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1;\n\t@!p bra WT_%=;\n\t}"
                                     ::"r"(smem_u32(&bar2[0])) : "memory");
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    }
#pragma unroll
                    for (int m = 0; m < 5; ++m)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                                     ::"r"(exact ? d + t * 48 : d + (t % 2) * 256 * (dstride == 0) + (t % 8) * 48 * (dstride == 1) + (t % 4) * 128 * (dstride == 2)), "l"(desc(sa + t * 2048 + offs[m] * 16, lbos[m] * 16)),
                                     "l"(exact ? desc(sb + m * 2560, 1280) : desc(sb + m * 2 * n * 16, n * 16)), "r"(idesc), "r"(1) : "memory");
                    if (commit_every != 0 && (commit_every < 0 || (t % commit_every) == 0))
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                     ::"r"(smem_u32(&bar2[1 + (t & 3)])) : "memory");
                }
            if (w == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        }
        __syncwarp();
        if (w == 0) asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        t1 = clock64();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    long long* dc; cudaMalloc(&dc, 148 * 8);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    for (int n : {48}) for (int ds : {3, 4}) for (int ce : {0, 1, -1}) { const int align = 0;
        const int reps = 40, ntile = 10;
        kern<<<148, 128, SMEM>>>(n, align, reps, ntile, dc, ce, ds);
        cudaError_t e = cudaDeviceSynchronize();
        long long hc[148]; cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
        double mean = 0; for (long long x : hc) mean += x; mean /= 148;
        printf("N=%3d dstride-mode %d commit every %2d tiles: %.1f cyc/MMA  (%s)\n", n, ds, ce, mean / (reps * ntile * 5),
               cudaGetErrorString(e));
    }
    return 0;
}
