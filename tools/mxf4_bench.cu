// Microbenchmark: tcgen05.mma kind::mxf4 (E2M1 x E2M1, unit UE8M0 scales, M = 128, K = 64) throughput
// (cycles per instruction) vs N, one CTA per SM; mode 1: two issuing warps into two accumulators.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) bench(long long* out, int n, int swz, int reps, int a_lbo) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tptr;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
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
    uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 64 * 1024);
    uint64_t ad, bd;
    if (swz) {  // 128B swizzle K-major: SBO = 1024 (8 rows x 128 B), LBO ignored (1)
        ad = ((uint64_t)((sa >> 4) & 0x3FFF)) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
        bd = ((uint64_t)((sb >> 4) & 0x3FFF)) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
    } else {    // no swizzle: rows 16 B apart, SBO = 128, K-halves LBO apart
        ad = ((uint64_t)((sa >> 4) & 0x3FFF)) | ((uint64_t)((a_lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
        bd = ((uint64_t)((sb >> 4) & 0x3FFF)) | ((uint64_t)(((n * 16) >> 4) & 0x3FFF) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
    }
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x < 32) {
        uint32_t pred = 0;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
        __syncwarp();
        t0 = clock64();
        if (pred) {
            for (int r = 0; r < reps; ++r) {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                             ::"r"(d), "l"(ad + ((r & 3) * 2)), "l"(bd + ((r & 3) * 2)), "r"(idesc), "r"(r),
                             "r"(d + 480), "r"(d + 496) : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        }
        __syncwarp();
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        t1 = clock64();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
    }
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
    long long* out; cudaMalloc(&out, 148 * sizeof(long long));
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    long long h[148];
    const int reps = 2048;
    int ns[] = {64, 128, 192, 256};
    for (int swz = 0; swz < 2; ++swz)
        for (int lbo : {2048, 2064}) {
            if (swz && lbo != 2048) continue;
            for (int n : ns) {
                bench<<<148, 128, 160 * 1024>>>(out, n, swz, reps, lbo);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
                double mean = 0; for (int i = 0; i < 148; ++i) mean += h[i]; mean /= 148;
                double cyc = mean / reps;
                printf("swz=%d a_lbo=%d N=%3d: %.1f cyc/MMA (ideal %.1f)  MAC/clk/SM=%.0f  %s\n", swz, lbo, n, cyc,
                       128.0 * n * 64 / 16384, 128.0 * n * 64 / cyc, cudaGetErrorString(e));
                if (e != cudaSuccess) return 1;
            }
        }
    return 0;
}
