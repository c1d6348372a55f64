// tc_ptx.cuh -- inline-PTX helpers shared by the tcgen05 conv kernels (sm_100a):
// mbarriers, tcgen05.mma kind::i8 / commit / ld / st, UMMA descriptors, bulk
// copies, and the 2-bit -> int8 ternary expansion.  Internal; not part of the ABI.
#pragma once

#include <cstdint>

namespace tn {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Wait for the phase with the given parity to complete.  The suspend-time hint
// lets the hardware park the warp until the phase completes instead of
// re-polling: with 17+ warps per SM, spinning waiters were ~25 % of all issued
// instructions (ncu), stealing issue slots from the warps doing the work.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TN_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra TN_WAIT_%=;\n\t}" ::"r"(a), "r"(parity), "r"(1000000u) : "memory");
}
// Plain polling wait (no suspend-time hint).
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TN_WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TN_WAITS_%=;\n\t}" ::"r"(a), "r"(parity) : "memory");
}
// 16 ternary lanes (bits sh..sh+15 of a sign / mask word pair) -> 16 FP4 E2M1 nibbles:
// +1 -> 0x2 (1.0), -1 -> 0xA (-1.0), 0 -> 0x0; nibble k = lane k (k even in the low
// nibble of byte k/2, the element order of packed e2m1 operands).
// 8 lanes -> a PRMT selector whose nibble k is the lane pair (2k+1, 2k) of x (bits 0..7)
__device__ __forceinline__ uint32_t pair_selector(uint32_t x) {
    x &= 0xFFu;
    x = (x | (x << 4)) & 0x0F0Fu;
    return (x | (x << 2)) & 0x3333u;
}
__device__ __forceinline__ uint2 expand16_f4(uint32_t s, uint32_t m, int sh) {
    const uint32_t mm = m >> sh, nn = (m & ~s) >> sh;
    // byte k of the result = FP4 lanes 2k (low nibble) and 2k+1: each lane pair picks one
    // of four bytes with PRMT -- mask: {00, 02, 20, 22}, negative: {00, 08, 80, 88}
    const uint32_t lo = __byte_perm(0x22200200u, 0u, pair_selector(mm)) |
                        __byte_perm(0x88800800u, 0u, pair_selector(nn));
    const uint32_t hi = __byte_perm(0x22200200u, 0u, pair_selector(mm >> 8)) |
                        __byte_perm(0x88800800u, 0u, pair_selector(nn >> 8));
    return make_uint2(lo, hi);
}
// The same for a canonical 16-channel word pair (bits 16..31 of s and m zero, reading R4):
// the mask and negative bytes of each lane octet are gathered into one register by PRMT
// and spread to their PRMT selectors together (19 instructions instead of 31).
__device__ __forceinline__ uint2 expand16_f4_c16(uint32_t s, uint32_t m) {
    const uint32_t nn = m & ~s;
    uint32_t x = __byte_perm(m, nn, 0x6420u);     // [m.b0, 0, nn.b0, 0]
    uint32_t y = __byte_perm(m, nn, 0x6521u);     // [m.b1, 0, nn.b1, 0]
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    y = (y | (y << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;             // low half: mask selector, high half: negative
    y = (y | (y << 2)) & 0x33333333u;
    const uint32_t lo = __byte_perm(0x22200200u, 0u, x) | __byte_perm(0x88800800u, 0u, x >> 16);
    const uint32_t hi = __byte_perm(0x22200200u, 0u, y) | __byte_perm(0x88800800u, 0u, y >> 16);
    return make_uint2(lo, hi);
}
// All 32 lanes of a sign / mask word pair -> 32 FP4 nibbles (16 bytes; word w = lanes 8w..8w+7).
// The bytes of m and of the negative set nn go two per register into 16-bit lanes, are spread
// to selector nibbles together, and each output word is two PRMTs (39 instructions instead of
// the 60 of two expand16_f4 calls).
__device__ __forceinline__ uint4 expand32_f4(uint32_t s, uint32_t m) {
    const uint32_t nn = m & ~s;
    uint32_t a = m & 0x00FF00FFu, b = (m >> 8) & 0x00FF00FFu;       // m bytes 0|2, 1|3
    uint32_t c = nn & 0x00FF00FFu, d = (nn >> 8) & 0x00FF00FFu;     // nn bytes 0|2, 1|3
    a = (a | (a << 4)) & 0x0F0F0F0Fu;
    b = (b | (b << 4)) & 0x0F0F0F0Fu;
    c = (c | (c << 4)) & 0x0F0F0F0Fu;
    d = (d | (d << 4)) & 0x0F0F0F0Fu;
    a = (a | (a << 2)) & 0x33333333u;
    b = (b | (b << 2)) & 0x33333333u;
    c = (c | (c << 2)) & 0x33333333u;
    d = (d | (d << 2)) & 0x33333333u;
    uint4 r;
    r.x = __byte_perm(0x22200200u, 0u, a) | __byte_perm(0x88800800u, 0u, c);
    r.y = __byte_perm(0x22200200u, 0u, b) | __byte_perm(0x88800800u, 0u, d);
    r.z = __byte_perm(0x22200200u, 0u, a >> 16) | __byte_perm(0x88800800u, 0u, c >> 16);
    r.w = __byte_perm(0x22200200u, 0u, b >> 16) | __byte_perm(0x88800800u, 0u, d >> 16);
    return r;
}
__device__ __forceinline__ void tc_mma_mxf4(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, 1, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb)
        : "memory");
}
// The same with the accumulate flag (0: D = A x B, overwriting the accumulator).
__device__ __forceinline__ void tc_mma_mxf4_acc(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate)
        : "memory");
}
// Accumulator-start ("bias") B rows: an MMA of an A tile of constants (E2M1 1.0 in the first
// 32-element K half, 6.0 in the second; int8: 1 everywhere) with these rows writes v into
// every accumulator of the row's output channel, so a new output's block is initialised by
// the tensor core in the MMA stream itself.  E2M1: v = s0 + 6 s1 with s0, s1 sums of 32
// E2M1 codes (multiples of 1/2, |s1| <= 192: |v| <= 1344); int8: v = sum of 32 int8.
// Byte b of K half h of a start row (v = s0 + 6 s1, s1 the multiple of 1/2 nearest v / 6, so
// |s0| <= 3/2): the half's 32 E2M1 codes are as many 6.0 as fit, then the remainder as one or two
// codes (2.5 = 2 + .5, 3.5 = 3 + .5, 4.5 = 4 + .5, 5 = 4 + 1, 5.5 = 4 + 1.5); element 2j in the low
// nibble of byte j.
__device__ __forceinline__ uint32_t e2m1_start_nibble(float s, int j) {
    const uint32_t neg = s < 0.0f ? 8u : 0u;
    const int a2 = static_cast<int>(fabsf(s) * 2.0f + 0.25f);   // |s| in halves
    const int n6 = a2 / 12, rem = a2 - 12 * n6;
    const uint32_t first = static_cast<uint32_t>(0x666655443210ull >> (4 * rem)) & 0xFu;
    const uint32_t second = static_cast<uint32_t>(0x321010100000ull >> (4 * rem)) & 0xFu;
    const uint32_t c = j < n6 ? 7u : (j == n6 ? first : (j == n6 + 1 ? second : 0u));
    return c ? (c | neg) : 0u;
}
__device__ __forceinline__ uint8_t e2m1_start_byte(float v, int h, int b) {
    const float s1 = rintf(v / 3.0f) * 0.5f;
    const float s = h ? s1 : v - 6.0f * s1;
    return static_cast<uint8_t>(e2m1_start_nibble(s, 2 * b) | (e2m1_start_nibble(s, 2 * b + 1) << 4));
}
// Element j of 32 int8 summing to v (|v| <= 32 * 127): 127s first, then the remainder.
__device__ __forceinline__ uint8_t i8_start_byte(int v, int j) {
    const int a = v < 0 ? -v : v;
    const int t = max(0, min(127, a - 127 * j));
    return static_cast<uint8_t>(static_cast<int8_t>(v < 0 ? -t : t));
}
// Instruction descriptor for kind::mxf4: E2M1 x E2M1, UE8M0 scales, K-major, M = 128, N, K = 64.
__host__ __device__ constexpr uint32_t idesc_mxf4(int n) {
    return (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
}

// Programmatic dependent launch: the conv kernels are launched with
// programmatic stream serialisation, so a layer's setup (filter-bank expansion,
// barriers, TMEM) overlaps the previous layer's tail; every thread waits for
// the previous grid (and its memory) before touching activations.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Thresholds clamped to +-2^20: |acc| <= 27 * 64 < 2^12, so a threshold beyond that
// acts exactly like the INT32 sentinels (always / never), while acc - hi, lo - hi
// and their float images stay exact and cannot overflow.
__device__ __forceinline__ int clamp_threshold(int t) { return max(-(1 << 20), min(t, 1 << 20)); }

// Waits / commits on a barrier given by its shared-memory address.
__device__ __forceinline__ void mbar_wait_addr(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TN_WAITA_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra TN_WAITA_%=;\n\t}" ::"r"(a), "r"(parity), "r"(1000000u) : "memory");
}
__device__ __forceinline__ void tc_commit_addr(uint32_t a) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// UMMA shared-memory descriptor, K-major, no swizzle (canonical "interleave"
// layout: 8-row x 16-byte core matrices; rows 16 B apart, 8-row groups SBO
// apart, the two 16-byte K halves of a K=32 instruction LBO apart).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) |
           (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// Instruction descriptor: s32 accumulate, s8 x s8, both K-major, M=128, N.
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | ((128u >> 4) << 24);
}

// 16 ternary lanes (bits sh..sh+15 of a sign / mask word pair) -> 16 int8.
__device__ __forceinline__ uint4 expand16(uint32_t s, uint32_t m, int sh) {
    const uint32_t mm = m >> sh, nn = (m & ~s) >> sh;
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t mb = (((mm >> (4 * i)) & 0xFu) * 0x00204081u) & 0x01010101u;
        const uint32_t nb = (((nn >> (4 * i)) & 0xFu) * 0x00204081u) & 0x01010101u;
        o[i] = mb + nb * 0xFEu;          // +1 -> 0x01, -1 -> 0xFF, 0 -> 0x00
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// Shared-memory loads / stores by 32-bit shared-window address.
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint2 v) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared (async proxy), completion as tx bytes on bar.
// bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const int (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
// 16 columns of one value (one source register for all 16 operands)
__device__ __forceinline__ void tmem_st16_fill(uint32_t taddr, int v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint64_t umma_desc_lbo(uint32_t saddr, uint32_t lbo) { return umma_desc(saddr, lbo, 128); }

}  // namespace
}  // namespace tn
