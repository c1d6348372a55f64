// Exhaustive check of expand16_f4 (ternary sign/mask lanes -> FP4 E2M1 nibbles) against the
// lane-by-lane definition: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/f4check tools/f4_expand_check.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1801_09449_b200/csrc/tc_ptx.cuh"
using namespace tn;
__global__ void k(int* bad) {
    // exhaustive over 16-lane (s, m) pairs restricted to canonical: s subset of m
    for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < 65536; m += gridDim.x * blockDim.x) {
        for (uint32_t sv = 0; sv < 65536; sv += 97) {   // a spread of sign words
            const uint32_t s = sv & m;
            const uint2 r = expand16_f4(s, m, 0);
            for (int i = 0; i < 16; ++i) {
                const uint32_t nib = ((i < 8 ? r.x : r.y) >> (4 * (i & 7))) & 0xF;
                const uint32_t want = ((m >> i) & 1) ? (((s >> i) & 1) ? 0x2u : 0xAu) : 0u;
                if (nib != want) atomicAdd(bad, 1);
            }
            // sh = 16 on a 32-bit word
            const uint2 r2 = expand16_f4(s << 16 | 0x1234u, m << 16 | 0xFFFFu, 16);
            if (r2.x != r.x || r2.y != r.y) atomicAdd(bad, 1);
        }
    }
}
int main() { int* d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4); k<<<256, 256>>>(d); int h = -1; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost); printf("bad %d\n", h); return h != 0; }
