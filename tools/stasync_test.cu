// Minimal probe: st.async into own-CTA smem with mbarrier complete_tx, launched
// as 1-CTA clusters via cudaLaunchKernelEx with large dynamic smem.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k(uint32_t* out, int use_big) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    uint32_t* buf = reinterpret_cast<uint32_t*>(smem);
    uint32_t bar_a = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(blockDim.x * 16));
    uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf + 4 * threadIdx.x));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                 ::"r"(dst), "r"(threadIdx.x), "r"(1u), "r"(2u), "r"(blockIdx.x), "r"(bar_a) : "memory");
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(bar_a) : "memory");
    out[blockIdx.x * blockDim.x + threadIdx.x] = buf[4 * ((threadIdx.x + 1) % blockDim.x)] + buf[4 * threadIdx.x + 3];
}

int main() {
    const int blocks = 148, threads = 128;
    uint32_t* out; cudaMalloc(&out, blocks * threads * 4);
    cudaMemset(out, 0xFF, blocks * threads * 4);
    for (int big = 0; big < 2; ++big) {
        size_t smem = big ? 200 * 1024 : 4096;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        printf("setattr %s\n", cudaGetErrorString(e));
        for (int cl = 1; cl >= 1; --cl) {
            cudaMemset(out, 0xFF, blocks * threads * 4);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 1; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr; cfg.numAttrs = cl;
            e = cudaLaunchKernelEx(&cfg, k, out, big);
            cudaError_t e2 = cudaDeviceSynchronize();
            uint32_t h[4]; cudaMemcpy(h, out + threads * 3, 16, cudaMemcpyDeviceToHost);
            printf("smem=%zu cluster=%d launch=%s sync=%s out=%u %u %u %u (expect %u %u ...)\n", smem, cl,
                   cudaGetErrorString(e), cudaGetErrorString(e2), h[0], h[1], h[2], h[3], 1 + 3 + 0, 2 + 3 + 1);
            if (e2 != cudaSuccess) return 1;
        }
    }
    return 0;
}
