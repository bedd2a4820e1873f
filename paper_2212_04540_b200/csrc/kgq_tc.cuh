// kgq_tc.cuh -- minimal tcgen05 / TMEM / mbarrier helpers (sm_100a, inline PTX).
//
// Operand layout used everywhere here: K-major, SWIZZLE_NONE ("interleaved")
// canonical UMMA layout.  A row-major R x K fp32 tile is stored as 16-byte
// core-matrix rows: element (r, k) lives at byte
//     (k/4) * LBO + (r/8) * 128 + (r%8) * 16 + (k%4) * 4,      LBO = R/8 * 128,
// i.e. 8x(4 fp32) core matrices, 8-row groups 128 B apart (SBO = 128) and
// 4-column chunks LBO apart.  One kind::tf32 MMA consumes K = 8 (two chunks).
#pragma once
#include "kgq_common.cuh"

namespace kgq {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__host__ __device__ constexpr uint32_t tile_off(int r, int k, int rows) {
    return (uint32_t)((k >> 2) * (rows / 8) * 128 + (r >> 3) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

// Shared-memory matrix descriptor (SWIZZLE_NONE, K-major), Blackwell version 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;                     // version = 1 (sm100)
    // base_offset = 0, lbo_mode = 0, layout_type = SWIZZLE_NONE (0)
    return d;
}

// Instruction descriptor: kind::tf32, D fp32, A/B K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)            // c_format F32
         | (2u << 7)            // a_format TF32
         | (2u << 10)           // b_format TF32
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}
// Same with the operand majorness bits (15: A MN-major, 16: B MN-major).
__host__ __device__ constexpr uint32_t idesc_tf32_major(int M, int N, bool a_mn, bool b_mn) {
    return idesc_tf32(M, N) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16);
}

// ---- 128-byte-swizzled row-major tiles ------------------------------------
// A [rows][D] fp32 tile is stored as D/32 column blocks of rows x 128 B (each
// block 1024-B aligned); inside a block row r's 16-byte chunk j sits at chunk
// j ^ (r & 7) (the SWIZZLE_128B pattern).  The same bytes serve as a K-major
// operand (rows = M/N, columns = K: e.g. G as A of dH = G . theta^T) and as an
// MN-major operand (rows = K, columns = M/N: H and G of dtheta = H^T . G), so
// each operand is staged once, with 16-byte stores.
__host__ __device__ constexpr uint32_t sw128_off(int r, int c, int rows) {
    return (uint32_t)((c >> 5) * rows * 128 + r * 128 + ((((c & 31) >> 2) ^ (r & 7)) << 4) + (c & 3) * 4);
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return smem_desc(saddr, lbo, sbo) | ((uint64_t)2 << 61);      // layout type SWIZZLE_128B
}
// K-major view, K step s (8 tf32 columns): block s/4, 32 B per step inside the row.
__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t base, int s, int rows) {
    return sw128_desc(base + (uint32_t)((s >> 2) * rows * 128 + (s & 3) * 32), 16, 1024);
}
// MN-major view, K step s (8 rows): 1024 B per step; MN atoms (column blocks) LBO apart.
__device__ __forceinline__ uint64_t mnmajor_sw128_desc(uint32_t base, int s, int rows) {
    return sw128_desc(base + (uint32_t)(s * 1024), (uint32_t)(rows * 128), 1024);
}

// ---- MN-major tf32 operands: SWIZZLE_128B_BASE32B ---------------------------
// The one MN-major smem form kind::tf32 accepts: row-major [rows][32-column
// blocks], 128-B rows, the 32-B granule j of row r stored at granule j ^ (r & 3);
// blocks rows * 128 B apart (LBO), 4-row K atoms 512 B apart (SBO).
__host__ __device__ constexpr uint32_t b32_off(int r, int c, int rows) {
    return (uint32_t)((c >> 5) * rows * 128 + r * 128 + ((((c & 31) >> 3) ^ (r & 3)) << 5) + (c & 7) * 4);
}
__device__ __forceinline__ uint64_t mnmajor_b32_desc(uint32_t base, int s, int rows, uint32_t sbo = 512) {
    return smem_desc(base + (uint32_t)(s * 1024), (uint32_t)(rows * 128), sbo) | ((uint64_t)1 << 61);
}

// D (+)= A . B with A read from TMEM (lanes = M rows, one tf32 per column), B a smem descriptor.
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
        :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 32 lanes x 16 consecutive 32-bit columns from 16 registers per thread.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
           "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
           "r"(v[15]) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
        :: "r"(taddr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]),
           "f"(v[7]) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *mbar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}"
                 :: "r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// 32 lanes x 16 consecutive fp32 columns -> 16 registers per thread (no wait).
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void commit(uint64_t *mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(mbar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n"
        :: "r"(smem_u32(mbar)), "r"(parity) : "memory");
}

// polling with a short sleep between tries: for producer / MMA threads that
// share an SM sub-partition with the warps they wait for
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *mbar, uint32_t parity) {
    uint32_t ok;
    for (;;) {
        asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                     "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(smem_u32(mbar)), "r"(parity) : "memory");
        if (ok) break;
        __nanosleep(64);
    }
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Warp-wide TMEM allocation (one warp calls); writes the base to *dst.
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(dst)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t base, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(base), "r"(ncols) : "memory");
}

// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

// 3xTF32 split: hi = RNA-tf32(x), lo = x - hi (exact in fp32).
__device__ __forceinline__ void split_tf32(float x, float &hi, float &lo) {
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    hi = __uint_as_float(h);
    lo = __fsub_rn(x, hi);
}

// 3xTF32 split in 3 integer/float instructions: hi = x rounded to the nearest
// tf32 (ties away, as cvt.rna; finite x), lo = x - hi (exact).  kind::tf32
// then reads hi exactly and lo truncated: |error| <= 2^-22 |x|.
__device__ __forceinline__ void split_tf32_fast(float x, float &hi, float &lo) {
    hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
    lo = __fsub_rn(x, hi);
}

// D[M x N] (+)= A[M x 64] . B[64 x N] in 3xTF32 (lo*hi + hi*lo + hi*hi),
// A/B given as hi/lo tiles in the interleaved layout.  Single thread issues.
template <int M, int N, int K>
__device__ __forceinline__ void mma_3xtf32(uint32_t tmem_d, const float *ah, const float *al,
                                           const float *bh, const float *bl) {
    constexpr uint32_t LBO_A = (M / 8) * 128, LBO_B = (N / 8) * 128;
    constexpr uint32_t idesc = idesc_tf32(M, N);
    const uint32_t sah = smem_u32(ah), sal = smem_u32(al), sbh = smem_u32(bh), sbl = smem_u32(bl);
    uint32_t acc = 0;
#pragma unroll
    for (int pass = 0; pass < 3; pass++) {
        const uint32_t sa = pass == 0 ? sal : sah;
        const uint32_t sb = pass == 1 ? sbl : sbh;
#pragma unroll
        for (int s = 0; s < K / 8; s++) {
            mma_tf32(tmem_d, smem_desc(sa + 2 * s * LBO_A, LBO_A, 128),
                     smem_desc(sb + 2 * s * LBO_B, LBO_B, 128), idesc, acc);
            acc = 1;
        }
    }
}

}  // namespace tc
}  // namespace kgq
