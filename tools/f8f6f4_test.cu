// Microtest (round-2 groundwork): tcgen05.mma kind::f8f6f4 with E2M1 operands
// and f16 or f32 accumulators, on ternary values {-1,0,+1}.  Which smem placement of the
// E2M1 codes the MMA reads (found: 16 codes packed in the first 8 bytes of each 16-byte
// row), whether f16 accumulation of small integers is exact (yes), how
// f16 results sit in TMEM (low half of a column; .pack::16b loads pair them), and cycles
// per 128xNx32 MMA.
// usage: f8f6f4_test  (prints one line per (placement, D format, N))
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)8 << 32) | (1ull << 46);
}
// kind::f8f6f4: D format [4:5] (0 f16, 1 f32), A / B format [7:9] / [10:12] (E2M1 = 5)
__host__ __device__ constexpr uint32_t idesc_f8f6f4(int n, int dfmt) {
    return ((uint32_t)dfmt << 4) | (5u << 7) | (5u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) kern(const uint8_t* A, const uint8_t* B, uint32_t* D, int n, int dfmt, int reps,
                                               long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tptr;
    uint8_t* sa = smem;              // [2 halves][128 rows][16 B]
    uint8_t* sb = smem + 4096;       // [2 halves][n rows][16 B]
    for (int i = threadIdx.x; i < 4096 / 16; i += 128) reinterpret_cast<uint4*>(sa)[i] = reinterpret_cast<const uint4*>(A)[i];
    for (int i = threadIdx.x; i < 2 * n; i += 128) reinterpret_cast<uint4*>(sb)[i] = reinterpret_cast<const uint4*>(B)[i];
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
    const int w = threadIdx.x >> 5;
    const uint64_t ad = desc(smem_u32(sa), 2048);
    const uint64_t bd = desc(smem_u32(sb), n * 16);
    const uint32_t idesc = idesc_f8f6f4(n, dfmt);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x < 32) {
        uint32_t pred = 0;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
        __syncwarp();
        t0 = clock64();
        if (pred) {
            for (int r = 0; r < reps; ++r)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(d + (r & 1) * 256 * (reps > 1)), "l"(ad), "l"(bd), "r"(idesc), "r"(0) : "memory");
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        }
        __syncwarp();
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        t1 = clock64();
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < n; c += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(d + ((uint32_t)(32 * w) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (blockIdx.x == 0)
            for (int i = 0; i < 16; ++i) D[threadIdx.x * n + c + i] = v[i];
    }
    if (dfmt == 0 && blockIdx.x == 0) {   // the first 16 f16 columns, two per register (.pack::16b)
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(d + ((uint32_t)(32 * w) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 8; ++i) D[128 * n + threadIdx.x * 8 + i] = v[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static uint8_t fp4(int v) { return v == 1 ? 0x2 : (v == -1 ? 0xA : 0x0); }

int main() {
    for (int shift : {8}) {   // 0 / 4: E2M1 code at bit `shift` of a byte; 8: 16 codes packed in the first 8 bytes of each 16-byte row
        for (int dfmt : {1, 0}) {         // f32, f16 accumulators
            for (int n : {48, 96}) {
                std::vector<int> a(128 * 32), b(n * 32);
                srand(11 + n);
                for (auto& v : a) v = rand() % 3 - 1;
                for (auto& v : b) v = rand() % 3 - 1;
                std::vector<uint8_t> A(4096, 0), B(2 * n * 16, 0);
                auto put = [&](std::vector<uint8_t>& M, size_t row0, int k, int v) {
                    if (shift == 8) M[row0 + (k % 16) / 2] |= fp4(v) << (4 * (k & 1));
                    else M[row0 + (k % 16)] = fp4(v) << shift;
                };
                for (int r = 0; r < 128; ++r)
                    for (int k = 0; k < 32; ++k) put(A, (k / 16) * 2048 + r * 16, k, a[r * 32 + k]);
                for (int r = 0; r < n; ++r)
                    for (int k = 0; k < 32; ++k) put(B, (size_t)(k / 16) * n * 16 + r * 16, k, b[r * 32 + k]);
                uint8_t *dA, *dB; uint32_t* dD; long long* dc;
                cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, 128 * n * 4 + 128 * 8 * 4); cudaMalloc(&dc, 148 * 8);
                cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
                cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
                cudaMemset(dD, 0, 128 * n * 4);
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
                kern<<<1, 128, 64 * 1024>>>(dA, dB, dD, n, dfmt, 1, dc);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("shift %d dfmt %d N=%d error %s\n", shift, dfmt, n, cudaGetErrorString(e)); return 1; }
                std::vector<uint32_t> D(128 * n + 128 * 8);
                cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
                int bad32 = 0, badlo = 0, badpk = 0;
                for (int m = 0; m < 128; ++m)
                    for (int j = 0; j < n; ++j) {
                        int ref = 0;
                        for (int k = 0; k < 32; ++k) ref += a[m * 32 + k] * b[j * 32 + k];
                        float f32v; memcpy(&f32v, &D[m * n + j], 4);
                        if ((float)ref != f32v) { if (bad32 < 2 && dfmt == 1 && n == 48) printf("    m=%d j=%d ref %d got %g (0x%08x)\n", m, j, ref, f32v, D[m * n + j]); ++bad32; }
                        __half hl = __ushort_as_half((unsigned short)(D[m * n + j] & 0xFFFF));
                        if ((float)ref != __half2float(hl)) ++badlo;
                        // packed: two f16 per column (element j in column j/2, half j%2)
                        __half hp = __ushort_as_half((unsigned short)((D[m * n + j / 2] >> (16 * (j & 1))) & 0xFFFF));
                        if ((float)ref != __half2float(hp)) ++badpk;
                    }
                int badp16 = -1;
                if (dfmt == 0) {   // .pack::16b: register i of row m holds columns 2i (low) and 2i+1 (high)
                    badp16 = 0;
                    for (int m = 0; m < 128; ++m)
                        for (int j = 0; j < 16; ++j) {
                            int ref = 0;
                            for (int k = 0; k < 32; ++k) ref += a[m * 32 + k] * b[j * 32 + k];
                            const uint32_t r32 = D[128 * n + m * 8 + j / 2];
                            __half h = __ushort_as_half((unsigned short)((r32 >> (16 * (j & 1))) & 0xFFFF));
                            if ((float)ref != __half2float(h)) ++badp16;
                        }
                    printf("    .pack::16b load of 16 f16 columns: mismatches %d of %d\n", badp16, 128 * 16);
                }
                const int R = 4096;
                kern<<<148, 128, 64 * 1024>>>(dA, dB, dD, n, dfmt, R, dc);
                e = cudaDeviceSynchronize();
                long long hc[148]; cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
                double mean = 0; for (long long x : hc) mean += x; mean /= 148;
                printf("code<<%d D=%s N=%2d: mismatches as f32 %d, as f16 (low half) %d, as packed f16 %d of %d; %.1f cyc/MMA  %s\n",
                       shift, dfmt ? "f32" : "f16", n, bad32, badlo, badpk, 128 * n, mean / R, cudaGetErrorString(e));
                cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
            }
        }
    }
    return 0;
}
