// Microtest: tcgen05.mma kind::i8 with the A descriptor start at arbitrary
// 16-byte row offsets and arbitrary (even overlapping) LBO, no-swizzle K-major.
// (1) correctness vs a host reference; (2) cycles per MMA vs start alignment.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
constexpr int AROWS = 2048;              // A region rows (16 B each) = 32 KB
constexpr int SMEM = AROWS * 16 + 256 * 32 + 1024;

// A: int8 [AROWS][16]; B: [2][N][16]; D[m][n] = sum_h sum_j A[r0 + m + h*lbo/16][j] * B[h][n][j]
__global__ void __launch_bounds__(128, 1) kern(const int8_t* A, const int8_t* B, int* D, int n, int r0, int lbo,
                                              int reps, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tptr;
    uint8_t* sa = smem; uint8_t* sb = smem + AROWS * 16;
    for (int i = threadIdx.x; i < AROWS; i += 128) reinterpret_cast<uint4*>(sa)[i] = reinterpret_cast<const uint4*>(A)[i];
    for (int i = threadIdx.x; i < 2 * n; i += 128) reinterpret_cast<uint4*>(sb)[i] = reinterpret_cast<const uint4*>(B)[i];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tptr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t d = tptr;
    const uint64_t ad = desc(smem_u32(sa) + 16 * r0, lbo, 128);
    const uint64_t bd = desc(smem_u32(sb), n * 16, 128);
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x < 32) {
        uint32_t pred = 0;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
        __syncwarp();
        t0 = clock64();
        if (pred) {
            for (int r = 0; r < reps; ++r)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(0) : "memory");
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        }
        __syncwarp();
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        t1 = clock64();
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // read back: warp w reads lanes 32w..32w+31, n columns
    const int w = threadIdx.x >> 5;
    for (int c = 0; c < n; c += 16) {
        int v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(d + ((uint32_t)(32 * w) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (blockIdx.x == 0)
            for (int i = 0; i < 16; ++i) D[threadIdx.x * n + c + i] = v[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(d));
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    std::vector<int8_t> hA(AROWS * 16), hB(2 * 256 * 16);
    srand(1);
    for (auto& v : hA) v = (int8_t)(rand() % 3 - 1);
    for (auto& v : hB) v = (int8_t)(rand() % 3 - 1);
    int8_t *dA, *dB; int* dD; long long* dc;
    cudaMalloc(&dA, hA.size()); cudaMalloc(&dB, hB.size()); cudaMalloc(&dD, 128 * 256 * 4); cudaMalloc(&dc, 148 * 8);
    cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    struct Case { int n, r0, lbo; };
    Case cases[] = {{48, 0, 2048}, {48, 1, 2048}, {48, 3, 2048}, {48, 0, 16}, {48, 5, 16}, {48, 1, 16 * 257},
                    {48, 7, 16 * 255}, {16, 0, 2048}, {16, 3, 16}, {32, 2, 16 * 130}, {64, 0, 2048}, {64, 1, 16},
                    {96, 0, 2048}, {96, 3, 16 * 129}, {144, 0, 2048}, {144, 1, 16}, {192, 0, 2048}, {192, 5, 16 * 129}};
    int bad_total = 0;
    for (auto c : cases) {
        const int reps = 1;
        kern<<<1, 128, SMEM>>>(dA, dB, dD, c.n, c.r0, c.lbo, reps, dc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<int> hD(128 * c.n);
        cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < 128; ++m)
            for (int nn = 0; nn < c.n; ++nn) {
                int ref = 0;
                for (int h = 0; h < 2; ++h)
                    for (int j = 0; j < 16; ++j)
                        ref += hA[(c.r0 + m + h * c.lbo / 16) * 16 + j] * hB[(h * c.n + nn) * 16 + j];
                bad += ref != hD[m * c.n + nn];
            }
        bad_total += bad;
        // timing: 148 CTAs, 4096 back-to-back MMAs
        const int R = 4096;
        kern<<<148, 128, SMEM>>>(dA, dB, dD, c.n, c.r0, c.lbo, R, dc);
        cudaDeviceSynchronize();
        long long hc[148]; cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
        double mean = 0; for (long long x : hc) mean += x; mean /= 148;
        printf("N=%3d r0=%d lbo=%5d: mismatches %d / %d   %.1f cyc/MMA\n", c.n, c.r0, c.lbo, bad, 128 * c.n, mean / R);
    }
    printf(bad_total ? "FAIL\n" : "ALL OK\n");
    return bad_total != 0;
}
