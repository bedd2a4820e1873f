// kgq_backward_tc.cu -- the fused layer backward (tape.py:217-225) on the
// 5th-generation tensor cores for d = 64:
//
//   g_j = (g_read + g_e) * mask;  dH = g_j . theta^T;  dtheta += Hhat^T . g_j
//
// One CTA (512 threads) per SM walks 128-row tiles.  All threads stage the
// tile: thread t owns row t/4 and column quads 4j + (t&3), forms g_j and the
// IEEE-dequantized
// Hhat in registers and writes their 3xTF32 hi/lo splits into shared memory in
// the K-major interleaved layout (kgq_tc.cuh) three times over:
//   Ag  (r, k=c)        A of dH       (M = 128 rows, K = 64)
//   Ah' (i=c, k=r)      A of dtheta   (M = 64,       K = 128 rows)
//   Bg' (j=c, k=r)      B of dtheta   (N = 64,       K = 128 rows)
// theta^T's split (B of dH, B(n,k) = theta[n][k]) is staged once per CTA.
// One elected thread issues 3 x 8 MMAs for dH into TMEM columns [0, 64) and
// 3 x 16 MMAs accumulating dtheta into columns [64, 128) across the CTA's
// tiles, then commits to an mbarrier; the 8 warps drain dH with tcgen05.ld.
// The M = 64 dtheta accumulator lives in TMEM lanes 32q + (0..15) for rows
// 16q..16q+15 (probed: tools/tc_probe/m64_layout.cu).  Per-CTA dtheta
// partials are reduced in a fixed order (reduce_partials_bwd_kernel).
// 3xTF32 = hi*hi + hi*lo + lo*hi with fp32 accumulation: fp32-level accuracy
// (the reference's BLAS GEMMs are tolerance-compared).
#include "kgq_tc.cuh"

namespace kgq {

constexpr int kTcRows = 128;
constexpr int kTcD = 64;

// The transposed operands (k = row) use a padded K-quad stride LBO_T = 1040 B
// (1024 + 16): with thread (row r, column quads 2j+h) the 32 scalar stores of
// a warp then hit 32 distinct banks.  Ag is written with 128-bit stores.
constexpr uint32_t kLboT = 1040;
constexpr uint32_t kLboA = 2080;     // Ag K-quad stride: 2048 + 32 B spreads a row's 4 quarter-threads
constexpr int kBtcThreads = 512;     // 4 threads per row: 16 warps keep more loads in flight
struct BwdTcSmem {
    static constexpr int AG = ((kTcD / 4 - 1) * kLboA + 2048) / 4;          // Ag hi or lo (floats)
    static constexpr int AT = ((kTcRows / 4 - 1) * kLboT + 1024) / 4;      // Ah'/Bg' hi or lo (floats)
    static constexpr int TH = kTcD * kTcD;
    static constexpr size_t bytes = (size_t)(2 * TH + 2 * AG + 4 * AT) * sizeof(float);   // 226.9 KB
};
__device__ __forceinline__ uint32_t toff_t(int c, int r) {   // (row c, k = r), padded K-quad stride
    return (uint32_t)((r >> 2) * kLboT + (c >> 3) * 128 + (c & 7) * 16 + (r & 3) * 4);
}

template <int BITS>
__global__ void __launch_bounds__(kBtcThreads, 1)
layer_backward_tc_kernel(const float *__restrict__ g_read, const float *__restrict__ g_e,
                         const uint32_t *__restrict__ mask, const uint8_t *__restrict__ codes,
                         const float *__restrict__ ranges, const float *__restrict__ offsets,
                         int64_t rows, const float *__restrict__ theta, float *__restrict__ dh,
                         float *__restrict__ partial) {
    constexpr int M = kTcRows, D = kTcD, RB = D * BITS / 8;
    constexpr uint32_t CM = BITS >= 32 ? 0xFFFFFFFFu : (1u << BITS) - 1u;
    constexpr int NCW = BITS >= 32 ? 1 : 2 * BITS;      // code words per row held in registers
    extern __shared__ __align__(128) float tsm[];
    float *th_hi = tsm, *th_lo = tsm + BwdTcSmem::TH;
    float *ag_hi = tsm + 2 * BwdTcSmem::TH, *ag_lo = ag_hi + BwdTcSmem::AG;
    float *ah_hi = ag_lo + BwdTcSmem::AG, *ah_lo = ah_hi + BwdTcSmem::AT;
    float *bg_hi = ah_lo + BwdTcSmem::AT, *bg_lo = bg_hi + BwdTcSmem::AT;
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;

    // theta^T split: B(n, k) = theta[n][k]
    for (int i = t; i < D * D; i += kBtcThreads) {
        const int n = i / D, k = i % D;
        float hi, lo;
        tc::split_tf32(__ldg(theta + i), hi, lo);
        th_hi[tc::tile_off(n, k, D) / 4] = hi;
        th_lo[tc::tile_off(n, k, D) / 4] = lo;
    }
    if (t == 0) tc::mbar_init(&mbar, 1);
    if (warp == 0) tc::tmem_alloc(&tmem_base, 128);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;

    // staging: thread owns row r = t/4 and the column quads 4j + h (j = 0..3)
    const int r = t >> 2, h = t & 3;
    uint32_t phase = 0;
    bool first = true;
    const int64_t n_tiles = (rows + M - 1) / M;
    // register prefetch of one tile's inputs (issued while the previous
    // tile's MMAs run, so the loads overlap the tensor-core work)
    float4 pa[4], pe[4];
    float prg = 0.f, pzz = 0.f;
    uint32_t pm0 = 0u, pm1 = 0u, pcw[NCW];
    float4 ph[BITS == 32 ? 4 : 1];                       // pass-through: the fp32 H quads
    auto load = [&](int64_t tl) {
        const int64_t row = tl * M + r;
        const bool ok = tl < n_tiles && row < rows;
        prg = (ok && BITS != 32) ? __ldg(ranges + row) : 0.f;
        pzz = (ok && BITS != 32) ? __ldg(offsets + row) : 0.f;
        pm0 = ok ? __ldg(mask + row * 2) : 0u;
        pm1 = ok ? __ldg(mask + row * 2 + 1) : 0u;
        if (BITS == 32) {
            const float4 *h4 = reinterpret_cast<const float4 *>(codes) + row * (D / 4);
#pragma unroll
            for (int j = 0; j < (BITS == 32 ? 4 : 1); j++) ph[j] = ok ? __ldg(h4 + 4 * j + h) : make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            const uint32_t *crow = reinterpret_cast<const uint32_t *>(codes + row * RB);
#pragma unroll
            for (int w = 0; w < NCW; w++) pcw[w] = ok ? __ldg(crow + w) : 0u;
        }
        const float4 *gr4 = reinterpret_cast<const float4 *>(g_read + row * D);
        const float4 *ge4 = reinterpret_cast<const float4 *>(g_e + row * D);
#pragma unroll
        for (int j = 0; j < 4; j++) {
            pa[j] = (ok && g_read) ? __ldg(gr4 + 4 * j + h) : make_float4(0.f, 0.f, 0.f, 0.f);
            pe[j] = (ok && g_e) ? __ldg(ge4 + 4 * j + h) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    load(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t row = tile * M + r;
        const bool ok = row < rows;
        // ---- 1. stage g_j and Hhat (hi/lo, three layouts) from the prefetched registers ----
        {
            const float rg = prg, zz = pzz;
            // b <= 2: the row's 2^b reconstruction values once (IEEE, lut_entry),
            // then a select per element instead of the division sequence
            float lut[BITS <= 2 ? (1 << BITS) : 1];
            if constexpr (BITS <= 2) {
#pragma unroll
                for (int c = 0; c < (1 << BITS); c++) lut[c] = lut_entry<BITS>(rg, zz, c);
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const float av[4] = {pa[j].x, pa[j].y, pa[j].z, pa[j].w}, ev[4] = {pe[j].x, pe[j].y, pe[j].z, pe[j].w};
                float gh[4], gl[4];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int c = 16 * j + 4 * h + q;
                    // g = g_read + g_e in the reference's routing order (tape.py:204-209)
                    const float g = (g_read && g_e) ? __fadd_rn(av[q], ev[q]) : (g_read ? av[q] : ev[q]);
                    const uint32_t mw = c < 32 ? pm0 : pm1;
                    const float gj = __fmul_rn(g, ((mw >> (c & 31)) & 1u) ? 1.0f : 0.0f);
                    const int bp = c * BITS;
                    const uint32_t code = BITS == 32 ? 0u : (pcw[(bp >> 5) % NCW] >> (bp & 31)) & CM;
                    float hv;
                    if (BITS == 32) {
                        const float4 hq = ph[BITS == 32 ? j : 0];
                        hv = q == 0 ? hq.x : q == 1 ? hq.y : q == 2 ? hq.z : hq.w;
                    } else if (BITS == 1) hv = code ? lut[BITS <= 2 ? 1 : 0] : lut[0];
                    else if (BITS == 2) hv = (code & 2u) ? ((code & 1u) ? lut[BITS == 2 ? 3 : 0] : lut[BITS == 2 ? 2 : 0])
                                                     : ((code & 1u) ? lut[BITS <= 2 ? 1 : 0] : lut[0]);
                    else hv = lut_entry<BITS <= 8 ? BITS : 8>(rg, zz, (int)code);
                    hv = ok ? hv : 0.0f;
                    float hh, hl;
                    tc::split_tf32(gj, gh[q], gl[q]);
                    tc::split_tf32(hv, hh, hl);
                    const uint32_t ob = toff_t(c, r) / 4;              // Ah', Bg' (c, k=r)
                    bg_hi[ob] = gh[q]; bg_lo[ob] = gl[q];
                    ah_hi[ob] = hh; ah_lo[ob] = hl;
                }
                const uint32_t oa = ((4 * j + h) * kLboA + (r >> 3) * 128 + (r & 7) * 16) / 4;   // Ag (r, quad)
                *reinterpret_cast<float4 *>(ag_hi + oa) = make_float4(gh[0], gh[1], gh[2], gh[3]);
                *reinterpret_cast<float4 *>(ag_lo + oa) = make_float4(gl[0], gl[1], gl[2], gl[3]);
            }
        }
        tc::fence_proxy_async();
        __syncthreads();
        // ---- 2. MMAs: dH (cols 0..63), dtheta accumulate (cols 64..127) ----
        if (t == 0) {
            tc::fence_after();
            {   // dH: A = Ag (K-quad stride kLboA), B = theta^T split (standard stride)
                constexpr uint32_t idA = tc::idesc_tf32(M, D), LBO_B = (D / 8) * 128;
                const uint32_t gah = tc::smem_u32(ag_hi), gal = tc::smem_u32(ag_lo);
                const uint32_t tbh = tc::smem_u32(th_hi), tbl = tc::smem_u32(th_lo);
                uint32_t acc0 = 0;
#pragma unroll
                for (int pass = 0; pass < 3; pass++) {
                    const uint32_t sa = pass == 0 ? gal : gah;
                    const uint32_t sb = pass == 1 ? tbl : tbh;
#pragma unroll
                    for (int st = 0; st < D / 8; st++) {
                        tc::mma_tf32(tmem, tc::smem_desc(sa + 2 * st * kLboA, kLboA, 128),
                                     tc::smem_desc(sb + 2 * st * LBO_B, LBO_B, 128), idA, acc0);
                        acc0 = 1u;
                    }
                }
            }
            constexpr uint32_t LBO = kLboT;                          // padded K-quad stride
            constexpr uint32_t idesc = tc::idesc_tf32(D, D);         // M = 64, N = 64
            const uint32_t sah = tc::smem_u32(ah_hi), sal = tc::smem_u32(ah_lo);
            const uint32_t sbh = tc::smem_u32(bg_hi), sbl = tc::smem_u32(bg_lo);
            uint32_t acc = first ? 0u : 1u;
#pragma unroll
            for (int pass = 0; pass < 3; pass++) {
                const uint32_t sa = pass == 0 ? sal : sah;
                const uint32_t sb = pass == 1 ? sbl : sbh;
#pragma unroll
                for (int s = 0; s < M / 8; s++) {
                    tc::mma_tf32(tmem + 64, tc::smem_desc(sa + 2 * s * LBO, LBO, 128),
                                 tc::smem_desc(sb + 2 * s * LBO, LBO, 128), idesc, acc);
                    acc = 1u;
                }
            }
            tc::commit(&mbar);
        }
        first = false;
        load(tile + gridDim.x);                     // next tile's inputs, in flight during the MMAs
        tc::mbar_wait(&mbar, phase);
        phase ^= 1u;
        tc::fence_after();
        // ---- 3. drain dH: warp w < 8 -> lanes 32*(w%4).., columns 32*(w/4).. ----
        if (warp < 8) {
            const int q = warp & 3, cb = (warp >> 2) * 32;
            float v[32];
            tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)cb, v);
            const int64_t orow = tile * M + 32 * q + lane;
            if (orow < rows) {
                float4 *dst = reinterpret_cast<float4 *>(dh + orow * D + cb);
#pragma unroll
                for (int j = 0; j < 8; j++) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
        }
        tc::fence_before();
        __syncthreads();
    }
    // ---- dtheta partial of this CTA: rows i = 16q + l live in lanes 32q + l ----
    if (warp < 4) {
        float *dst = partial + (int64_t)blockIdx.x * D * D;
#pragma unroll
        for (int cb = 0; cb < 64; cb += 32) {
            float v[32];
            if (first) {
#pragma unroll
                for (int j = 0; j < 32; j++) v[j] = 0.0f;     // no tile: zero partial
            } else {
                tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + 64u + (uint32_t)cb, v);
            }
            if (lane < 16) {
                float4 *o = reinterpret_cast<float4 *>(dst + (16 * warp + lane) * D + cb);
#pragma unroll
                for (int j = 0; j < 8; j++) o[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free(tmem, 128);
}

}  // namespace kgq

using namespace kgq;

// Launch helper used by kgq_layer_backward_f32 (kgq_backward.cu) for d = 64.
int kgq_launch_layer_backward_tc(const float *g_read, const float *g_e, const uint32_t *mask,
                                 const uint8_t *codes, const float *ranges, const float *offsets,
                                 int64_t rows, int32_t bits, const float *theta, float *dh,
                                 float *partial, int grid, cudaStream_t s) {
    static bool attr[33] = {false};
#define KGQ_BTC(B) do {                                                                            \
        if (!attr[B]) {                                                                            \
            cudaError_t e = cudaFuncSetAttribute(layer_backward_tc_kernel<B>,                        \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                                 (int)BwdTcSmem::bytes);                            \
            if (e != cudaSuccess) return kgq_set_cuda_error(e);                                    \
            attr[B] = true;                                                                        \
        }                                                                                          \
        layer_backward_tc_kernel<B><<<grid, kBtcThreads, BwdTcSmem::bytes, s>>>(g_read, g_e, mask, codes, \
                                                                        ranges, offsets, rows, theta, dh, partial); \
    } while (0)
    switch (bits) {
        case 1: KGQ_BTC(1); break;
        case 2: KGQ_BTC(2); break;
        case 4: KGQ_BTC(4); break;
        case 8: KGQ_BTC(8); break;
        default: KGQ_BTC(32); break;
    }
#undef KGQ_BTC
    return KGQ_OK;
}
