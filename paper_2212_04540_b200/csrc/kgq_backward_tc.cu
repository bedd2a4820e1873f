// kgq_backward_tc.cu -- the fused layer backward (tape.py:217-225) on the
// 5th-generation tensor cores for d = 64:
//
//   g_j = (g_read + g_e) * mask;  dH = g_j . theta^T;  dtheta += Hhat^T . g_j
//
// One persistent CTA per SM walks 128-row tiles, warp-specialized and
// pipelined so that the staging of one tile overlaps the MMAs of the previous:
//
// * 16 staging warps in two groups.  Warp w covers TMEM lane quadrant w % 4
//   (rows 32 (w % 4) .. + 31 of the tile, thread = row) and columns
//   16 (w / 4) .. + 15.  Group g = (w % 4) / 2 owns rows [64 g, 64 g + 64) of
//   every tile and its own shared-memory slot.  g_read and g_e arrive by TMA
//   (one 64-row x 32-column SWIZZLE_128B box per array and column half, per
//   group, issued one tile ahead as soon as the group has read the previous
//   one; rows past the end read as zeros); the per-row mask bits, codes, R, Z
//   come by register prefetch one tile ahead.  A thread reads its row's slice
//   (LDS.128, conflict-free through the swizzle), forms g_j and the
//   IEEE-dequantized Hhat, splits both into 3xTF32 hi/lo (hi = x itself, lo =
//   x - trunc_tf32(x)) and writes
//     - Hhat hi|lo and g_j hi|lo into its group's slot as MN-major
//       SWIZZLE_128B_BASE32B tiles (row-major 128-B rows, the layout
//       kind::tf32 reads MN-major; kgq_tc.cuh b32_off), 16-byte stores; lanes
//       with bit 2 set write the two halves of each 32-B granule in swapped
//       order so a quarter-warp's eight stores hit eight distinct bank groups;
//     - g_j hi|lo into TMEM (tcgen05.st, lane = row): the A operand of dH.
//   then arrives on its slot's `full` barrier, and drains the previous tile's
//   dH rows (tcgen05.ld -> 64-B row stores).
// * 1 MMA warp: per tile, per group slot: dtheta += [Hhat_hi | Hhat_lo]^T .
//   [g_hi | g_lo] as 8 MMAs M = 128, N = 128, K = 8 (both operands MN-major,
//   the hi/lo halves stacked along M and N, so one accumulator collects all
//   four products: hi.hi, hi.lo, lo.hi and lo.lo), commit -> the slot's
//   `empty` barrier; then dH = g_j . theta^T with A from TMEM (3 passes x 8
//   MMAs M = 128, N = 64: lo.hi + hi.lo + hi.hi, theta^T split staged once in
//   SWIZZLE_128B K-major) into a double-buffered TMEM accumulator, commit ->
//   `dhdone` (which also frees that tile's TMEM A buffer).
// TMEM (512 columns): dtheta accumulator [0,128), dH buffers [128,192) and
// [192,256), A buffers (hi 64 | lo 64) [256,384) and [384,512).
// At the end the four 64x64 quadrants of the dtheta accumulator are summed
// per CTA in a fixed order; reduce_partials_bwd_kernel (kgq_backward.cu)
// reduces the per-CTA partials in a fixed order (deterministic).
// 3xTF32 with fp32 accumulation: fp32-level accuracy (the reference's BLAS
// GEMMs are tolerance-compared).
#include "kgq_tma.cuh"

namespace kgq {

constexpr int kTcRows = 128;
constexpr int kTcD = 64;
constexpr int kBtcThreads = 544;            // 16 staging warps + 1 MMA warp
struct BwdTcSmem {
    static constexpr uint32_t SLOT = 64 * 1024;      // one group's 64 rows: Hhi, Hlo, Ghi, Glo (2 x 8 KB each)
    static constexpr uint32_t TH = 16 * 1024;        // theta split hi or lo (64 x 64 fp32, SW128 K-major)
    static constexpr uint32_t IN = 32 * 1024;        // one group's TMA stage: g_read, g_e (2 x 8 KB boxes each)
    static constexpr uint32_t INB = 2 * SLOT + 2 * TH;
    static constexpr uint32_t BAR = INB + 2 * IN;
    static constexpr size_t bytes = (size_t)BAR + 128 + 1024;   // + barriers + alignment slack (225.1 KB)
};
constexpr uint32_t kTmAcc = 0, kTmDh = 128, kTmA = 256;

template <int BITS>
__global__ void __launch_bounds__(kBtcThreads, 1)
layer_backward_tc_kernel(const __grid_constant__ CUtensorMap tm_gr, const __grid_constant__ CUtensorMap tm_ge,
                         int has_gr, int has_ge, const int32_t *__restrict__ gr_map,
                         const float *__restrict__ gr_rows, const uint32_t *__restrict__ mask, const uint8_t *__restrict__ codes,
                         const float *__restrict__ ranges, const float *__restrict__ offsets,
                         int64_t rows, const float *__restrict__ theta, float *__restrict__ dh,
                         float *__restrict__ partial) {
    constexpr int D = kTcD, M = kTcRows, RB = D * BITS / 8;
    constexpr uint32_t CM = BITS >= 32 ? 0xFFFFFFFFu : (1u << BITS) - 1u;
    constexpr int NCW = BITS >= 32 ? 1 : (16 * BITS + 31) / 32;     // code words of a 16-column slice
    extern __shared__ uint8_t tsm_raw[];
    uint8_t *sm = tsm_raw + ((1024u - (tc::smem_u32(tsm_raw) & 1023u)) & 1023u);   // stays a shared-space pointer
    float *thh = reinterpret_cast<float *>(sm + 2 * BwdTcSmem::SLOT);
    float *thl = reinterpret_cast<float *>(sm + 2 * BwdTcSmem::SLOT + BwdTcSmem::TH);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + BwdTcSmem::BAR);
    uint64_t *full = bar, *empty = bar + 2, *dhdone = bar + 4, *dhempty = bar + 6, *ldfull = bar + 8;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 10);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;

    // theta^T split, B of dH: B(n, k) = theta[n][k]
    {
        constexpr int PER = (D * D + kBtcThreads - 1) / kBtcThreads;
        float tv[PER];
#pragma unroll
        for (int k = 0; k < PER; k++) tv[k] = t + k * kBtcThreads < D * D ? __ldg(theta + t + k * kBtcThreads) : 0.f;
#pragma unroll
        for (int k = 0; k < PER; k++) {
            const int i = t + k * kBtcThreads;
            if (i < D * D) {
                const uint32_t o = tc::sw128_off(i / D, i % D, D) / 4;
                tc::split_tf32_fast(tv[k], thh[o], thl[o]);
            }
        }
    }
    if (t == 0) {
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(full + i, 256);
            tc::mbar_init(empty + i, 1);
            tc::mbar_init(dhdone + i, 1);
            tc::mbar_init(dhempty + i, 512);
            tc::mbar_init(ldfull + i, 1);
        }
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t n_tiles = (rows + M - 1) / M;
    const int nj = (int)((n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);   // >= 1 (grid <= n_tiles)

    if (warp == 16) {
        // ------------------------------ MMA issuer ------------------------------
        if (lane == 0) {
            constexpr uint32_t id_th = tc::idesc_tf32_major(128, 128, true, true);
            constexpr uint32_t id_dh = tc::idesc_tf32(128, 64);
            const uint32_t sbase = tc::smem_u32(sm);
            const uint32_t bh = tc::smem_u32(thh), bl = tc::smem_u32(thl);
            for (int j = 0; j < nj; j++) {
                for (int g = 0; g < 2; g++) {
                    tc::mbar_wait(full + g, (uint32_t)(j & 1));
                    tc::fence_after();
                    const uint32_t base = sbase + g * BwdTcSmem::SLOT;
#pragma unroll
                    for (int s = 0; s < 8; s++)
                        tc::mma_tf32(tmem + kTmAcc, tc::mnmajor_b32_desc(base, s, 64),
                                     tc::mnmajor_b32_desc(base + 32768, s, 64), id_th, (j | g | s) != 0);
                    tc::commit(empty + g);
                }
                const int b = j & 1;
                if (j >= 2) {
                    tc::mbar_wait(dhempty + b, (uint32_t)(((j >> 1) - 1) & 1));
                    tc::fence_after();
                }
                const uint32_t ab = tmem + kTmA + 128u * b, dd = tmem + kTmDh + 64u * b;
#pragma unroll
                for (int p = 0; p < 3; p++) {          // lo.hi, hi.lo, hi.hi
                    const uint32_t ao = p == 0 ? 64u : 0u;
                    const uint32_t bs = p == 1 ? bl : bh;
#pragma unroll
                    for (int s = 0; s < 8; s++)
                        tc::mma_tf32_ts(dd, ab + ao + 8u * s, tc::kmajor_sw128_desc(bs, s, D), id_dh, (p | s) != 0);
                }
                tc::commit(dhdone + b);
            }
        }
        __syncwarp();
    } else {
        // --------------------------- staging / drain ---------------------------
        const int q = warp & 3, cq = warp >> 2, g = q >> 1;
        const int r_tile = 32 * q + lane;            // row within the tile (= TMEM lane)
        const int r_unit = 32 * (q & 1) + lane;      // row within the group's 64-row unit
        const int sw = (lane >> 2) & 1;              // granule-half swap (bank spread)
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        float *slot = reinterpret_cast<float *>(sm + g * BwdTcSmem::SLOT);
        // block offsets (floats) inside the slot: Hhi blocks 0,1; Hlo 2,3; Ghi 4,5; Glo 6,7 (8 KB each)
        const int blk = cq >> 1;
        const int cbase = 16 * (cq & 1);             // first column inside the 32-column block
        float4 pa[4], pe[4];
        float prg = 0.f, pzz = 0.f;
        uint32_t pm = 0u, pcw[NCW];
        int32_t pslot = -1;                          // compact g_read: this row's slot (-1: zero)
        float4 ph[BITS == 32 ? 4 : 1];
        const uint8_t *instage = sm + BwdTcSmem::INB + g * BwdTcSmem::IN;
        const bool issuer = (warp == 2 * g) && lane == 0;   // first warp of the group
        const int in_bytes = (has_gr ? 16384 : 0) + (has_ge ? 16384 : 0);
        auto row_of = [&](int jj) {
            return ((int64_t)blockIdx.x + (int64_t)jj * gridDim.x) * M + r_tile;
        };
        // TMA: the group's 64 rows of tile jj (g_read boxes at +0 / +8 KB, g_e at +16 / +24 KB)
        auto issue_in = [&](int jj) {
            const int r0 = (int)(((int64_t)blockIdx.x + (int64_t)jj * gridDim.x) * M + 64 * g);
            tma::expect_tx(ldfull + g, (uint32_t)in_bytes);
            if (has_gr) {
                tma::load_2d(const_cast<uint8_t *>(instage), &tm_gr, 0, r0, ldfull + g);
                tma::load_2d(const_cast<uint8_t *>(instage) + 8192, &tm_gr, 32, r0, ldfull + g);
            }
            if (has_ge) {
                tma::load_2d(const_cast<uint8_t *>(instage) + 16384, &tm_ge, 0, r0, ldfull + g);
                tma::load_2d(const_cast<uint8_t *>(instage) + 24576, &tm_ge, 32, r0, ldfull + g);
            }
        };
        // the per-row scalars (and, at b = 32, the raw H slice) by register prefetch
        auto load_small = [&](int jj) {
            const int64_t row = row_of(jj);
            const bool ok = jj < nj && row < rows;
            prg = (ok && BITS != 32) ? __ldg(ranges + row) : 0.f;
            pzz = (ok && BITS != 32) ? __ldg(offsets + row) : 0.f;
            pm = ok ? __ldg(mask + row * 2 + (cq >> 1)) : 0u;        // raw word: bits 16 (cq & 1) ..
            pslot = (ok && gr_map) ? __ldg(gr_map + row) : -1;
            if constexpr (BITS == 1) {
                pcw[0] = ok ? (uint32_t)__ldg(reinterpret_cast<const uint16_t *>(codes + row * RB) + cq) : 0u;
            } else if constexpr (BITS != 32) {
                const uint32_t *cw = reinterpret_cast<const uint32_t *>(codes + row * RB) + cq * NCW;
#pragma unroll
                for (int w = 0; w < NCW; w++) pcw[w] = ok ? __ldg(cw + w) : 0u;
            } else {
                const float4 *h4 = reinterpret_cast<const float4 *>(codes) + row * (D / 4) + 4 * cq;
#pragma unroll
                for (int i = 0; i < 4; i++) ph[i] = ok ? __ldg(h4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        auto drain = [&](int jj) {
            const int b = jj & 1;
            tc::mbar_wait(dhdone + b, (uint32_t)((jj >> 1) & 1));
            tc::fence_after();
            uint32_t v[16];
            tc::tmem_ld16_nowait(tmem + lane_addr + kTmDh + 64u * b + 16u * cq, v);
            tc::tmem_ld_wait();
            tc::fence_before();
            tc::mbar_arrive(dhempty + b);
            // 4 x 4 transpose of 16-byte chunks inside each quad of lanes (two
            // xor-shuffle rounds): lane 4a + k then holds chunk k of rows
            // 4a .. 4a + 3, so each store instruction writes 8 rows x 64
            // contiguous bytes (8 L1 tag lookups instead of 32 for thread = row)
            const int k = lane & 3;
#pragma unroll
            for (int rd = 2; rd >= 1; rd >>= 1) {
                const bool up = (k & rd) != 0;
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    if (c & rd) continue;                       // pairs (c, c + rd)
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const uint32_t send = up ? v[4 * c + e] : v[4 * (c + rd) + e];
                        const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, rd);
                        if (up) v[4 * c + e] = recv;
                        else v[4 * (c + rd) + e] = recv;
                    }
                }
            }
            const int64_t row0 = ((int64_t)blockIdx.x + (int64_t)jj * gridDim.x) * M + 32 * q + (lane & ~3);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int64_t row = row0 + i;
                if (row < rows)
                    reinterpret_cast<float4 *>(dh + row * D)[4 * cq + k] =
                        make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                    __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
            }
        };
        if (issuer) issue_in(0);
        load_small(0);
        for (int j = 0; j < nj; j++) {
            const float rg = prg, zz = pzz;
            const uint32_t mw = (pm >> (16 * (cq & 1))) & 0xFFFFu;
            const int32_t grs = pslot;                   // compact g_read slot of this row
            uint32_t cw[NCW];
#pragma unroll
            for (int w = 0; w < NCW; w++) cw[w] = pcw[w];
            float4 hq4[BITS == 32 ? 4 : 1];
            if constexpr (BITS == 32) {
#pragma unroll
                for (int i = 0; i < 4; i++) hq4[i] = ph[i];
            }
            load_small(j + 1);
            // this tile's g_read / g_e slice from the TMA stage, then the stage is refilled
            tc::mbar_wait(ldfull + g, (uint32_t)(j & 1));
            {
                const int bx = cq >> 1;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const uint32_t o = bx * 8192 + tma::box_off(r_unit, 16 * (cq & 1) + 4 * i);
                    pa[i] = has_gr ? *reinterpret_cast<const float4 *>(instage + o)
                          : (grs >= 0 ? __ldg(reinterpret_cast<const float4 *>(gr_rows + (int64_t)grs * D) + 4 * cq + i)
                                       : make_float4(0.f, 0.f, 0.f, 0.f));
                    pe[i] = has_ge ? *reinterpret_cast<const float4 *>(instage + 16384 + o) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            tma::named_sync(1 + g, 256);
            if (issuer && j + 1 < nj) {
                tc::fence_proxy_async();           // generic reads of the stage before the async-proxy refill
                issue_in(j + 1);
            }
            // b <= 2: the row's 2^b IEEE dequantized values (K2's arithmetic) once,
            // then a select per element; b = 4 / 8: Hhat = Z + c * (R / B) with one
            // FFMA per element (<= 2 ulp from K2's value).  The FFMA form at b <= 2
            // is 2 % faster but its errors are coherent across rows (same code, same
            // error): Last-FM theta after 10 steps drifts 5e-5 from the reference vs
            // 2e-6 with the exact values, so b <= 2 keeps them.
            const float rb = __fmul_rn(rg, 1.0f / (float)((1u << (BITS < 32 ? BITS : 1)) - 1u));
            float lut[BITS <= 2 ? (1 << BITS) : 1];
            if constexpr (BITS <= 2) {
#pragma unroll
                for (int c = 0; c < (1 << BITS); c++) lut[c] = lut_entry<BITS>(rg, zz, c);
            }
            // slot free (dtheta MMAs of the previous tile done), TMEM A buffer free (dH of tile j-2 done)
            if (j >= 1) tc::mbar_wait(empty + g, (uint32_t)((j - 1) & 1));
            const int b = j & 1;
            if (j >= 2) tc::mbar_wait(dhdone + b, (uint32_t)(((j >> 1) - 1) & 1));
            tc::fence_after();
#pragma unroll
            for (int pr = 0; pr < 2; pr++) {          // chunk pairs (2 pr, 2 pr + 1): 8 columns
                float gh[8], gl[8], hh[8], hl[8];
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const int i = 2 * pr + u;
                    const float av[4] = {pa[i].x, pa[i].y, pa[i].z, pa[i].w};
                    const float ev[4] = {pe[i].x, pe[i].y, pe[i].z, pe[i].w};
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int c = 4 * i + e;                 // column inside the 16-column slice
                        // g = g_read + g_e in the reference's routing order (tape.py:204-209)
                        const bool read = has_gr || gr_map;          // compact g_read: absent rows are +0
                        const float gv = (read && has_ge) ? __fadd_rn(av[e], ev[e]) : (read ? av[e] : ev[e]);
                        const float gj = ((mw >> c) & 1u) ? gv : 0.0f;   // relu backward (sign of 0 immaterial: GEMM operand)
                        float hv;
                        if constexpr (BITS == 32) {
                            const float4 hq = hq4[BITS == 32 ? i : 0];
                            hv = e == 0 ? hq.x : e == 1 ? hq.y : e == 2 ? hq.z : hq.w;
                        } else {
                            const int bp = c * BITS;
                            const uint32_t code = (cw[(bp >> 5) % NCW] >> (bp & 31)) & CM;
                            if constexpr (BITS == 1) hv = code ? lut[BITS <= 2 ? 1 : 0] : lut[0];
                            else if constexpr (BITS == 2)
                                hv = (code & 2u) ? ((code & 1u) ? lut[BITS == 2 ? 3 : 0] : lut[BITS == 2 ? 2 : 0])
                                                 : ((code & 1u) ? lut[BITS <= 2 ? 1 : 0] : lut[0]);
                            else hv = __fmaf_rn(__uint2float_rn(code), rb, zz);
                        }
                        tc::split_tf32_fast(gj, gh[4 * u + e], gl[4 * u + e]);
                        tc::split_tf32_fast(hv, hh[4 * u + e], hl[4 * u + e]);
                    }
                }
                // smem: logical chunk (2 pr + u) ^ sw at instruction u
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const int src = u ^ sw;                        // which chunk's registers (0/1 of the pair)
                    const int col = cbase + 4 * (2 * pr + src);    // its first column in the block
                    const uint32_t o = tc::b32_off(r_unit, col, 64) / 4;
                    auto pick = [&](const float *v) {
                        return make_float4(src ? v[4] : v[0], src ? v[5] : v[1], src ? v[6] : v[2], src ? v[7] : v[3]);
                    };
                    *reinterpret_cast<float4 *>(slot + (0 + blk) * 2048 + o) = pick(hh);
                    *reinterpret_cast<float4 *>(slot + (2 + blk) * 2048 + o) = pick(hl);
                    *reinterpret_cast<float4 *>(slot + (4 + blk) * 2048 + o) = pick(gh);
                    *reinterpret_cast<float4 *>(slot + (6 + blk) * 2048 + o) = pick(gl);
                }
                // TMEM A: g_j hi at columns 16 cq + 8 pr, lo 64 further
                const uint32_t ta = tmem + lane_addr + kTmA + 128u * b + 16u * cq + 8u * pr;
                tc::tmem_st8(ta, gh);
                tc::tmem_st8(ta + 64u, gl);
            }
            tc::tmem_st_wait();
            tc::fence_proxy_async();
            tc::fence_before();
            tc::mbar_arrive(full + g);
            if (j >= 1) drain(j - 1);
        }
        drain(nj - 1);
    }

    // ---- dtheta partial of this CTA: sum of the accumulator's four 64x64 quadrants ----
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    float *red = reinterpret_cast<float *>(sm);            // [128][65] (slot memory is free now; padded rows)
    if (warp < 4) {
        float v0[32], v1[32];
#pragma unroll
        for (int cb = 0; cb < 64; cb += 32) {
            tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + kTmAcc + cb, v0);
            tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + kTmAcc + 64 + cb, v1);
#pragma unroll
            for (int c = 0; c < 32; c++) red[(32 * warp + lane) * 65 + cb + c] = __fadd_rn(v0[c], v1[c]);
        }
    }
    tc::fence_before();
    __syncthreads();
    float *dst = partial + (int64_t)blockIdx.x * D * D;
    for (int i = t; i < D * D; i += kBtcThreads)
        dst[i] = __fadd_rn(red[(i / D) * 65 + i % D], red[(i / D + 64) * 65 + i % D]);
    if (warp == 0) tc::tmem_free(tmem, 512);
}


// ---------------------------------------------------------------------------
// d = 128 (the configs[4] width).  TMEM cannot hold a 128-column G operand
// (hi + lo) next to the 128 x 128 dtheta accumulator and a dH accumulator, so
// dH is computed transposed, dH^T = theta . G^T, with theta (hi | lo) as the
// TMEM A operand, loaded once per CTA (lanes = n), and G as a K-major
// SWIZZLE_128B smem operand; dtheta = Hhat^T . G as three MMAs per K step
// (hi.hi, hi.lo, lo.hi) into one 128 x 128 accumulator, both operands MN-major
// SWIZZLE_128B_BASE32B.  TMEM: theta hi [0,128), lo [128,256), dtheta
// [256,384), four 32-column dH^T buffers [384,512).
// Units of 32 rows (two smem slots of 96 KB: Hhat hi/lo, G hi/lo MN-major,
// G hi/lo K-major; one 32 KB TMA stage of g_read / g_e), 16 staging warps
// (warp w: rows 8 (w % 4) + lane % 8, columns 8 (lane / 8 + 4 (w / 4)) .. +8,
// so a quarter-warp writes 8 consecutive rows of one column chunk: conflict-
// free through the swizzles, with the BASE32B granule halves swapped on lanes
// with bit 2 set) + 1 MMA warp.  The drain reads dH^T (lanes = n, columns =
// unit rows): each tcgen05.ld column is one dH row segment, stored 128 B wide.
// ---------------------------------------------------------------------------
constexpr int kT8U = 32;                   // rows per unit
struct Bwd128Smem {
    static constexpr uint32_t OP = kT8U * 128 * 4;     // one [32][128] fp32 operand (16 KB)
    static constexpr uint32_t SLOT = 6 * OP;           // HH HL GH GL (MN-major) KH KL (K-major)
    static constexpr uint32_t IN = 2 * OP;             // TMA stage: g_read, g_e
    static constexpr uint32_t BAR = 2 * SLOT + IN;
    static constexpr size_t bytes = (size_t)BAR + 128 + 1024;     // 225.1 KB
};
constexpr uint32_t kT8Th = 0, kT8Acc = 256, kT8Dh = 384;

template <int BITS>
__global__ void __launch_bounds__(kBtcThreads, 1)
layer_backward_tc128_kernel(const __grid_constant__ CUtensorMap tm_gr, const __grid_constant__ CUtensorMap tm_ge,
                            int has_gr, int has_ge, const uint32_t *__restrict__ mask,
                            const uint8_t *__restrict__ codes, const float *__restrict__ ranges,
                            const float *__restrict__ offsets, int64_t rows, const float *__restrict__ theta,
                            float *__restrict__ dh, float *__restrict__ partial) {
    constexpr int D = 128, U = kT8U, RB = D * BITS / 8;
    constexpr uint32_t CM = BITS >= 32 ? 0xFFFFFFFFu : (1u << BITS) - 1u;
    constexpr int CW = BITS >= 32 ? 1 : (8 * BITS + 31) / 32;       // code words of an 8-column chunk
    using S = Bwd128Smem;
    extern __shared__ uint8_t t8_raw[];
    uint8_t *sm = t8_raw + ((1024u - (tc::smem_u32(t8_raw) & 1023u)) & 1023u);
    uint8_t *instage = sm + 2 * S::SLOT;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S::BAR);
    uint64_t *full = bar, *empty = bar + 2, *dhfull = bar + 4, *dhempty = bar + 8, *infull = bar + 12;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 13);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;

    if (t == 0) {
        for (int i = 0; i < 2; i++) { tc::mbar_init(full + i, 512); tc::mbar_init(empty + i, 1); }
        for (int i = 0; i < 4; i++) { tc::mbar_init(dhfull + i, 1); tc::mbar_init(dhempty + i, 512); }
        tc::mbar_init(infull, 1);
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    // theta (hi | lo) into TMEM as the A operand of dH^T: lane n holds theta[n][0..128)
    if (warp < 4) {
        const int n = 32 * warp + lane;
        const float4 *src = reinterpret_cast<const float4 *>(theta + n * D);
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + kT8Th;
#pragma unroll
        for (int cb = 0; cb < D; cb += 8) {
            const float4 v0 = __ldg(src + cb / 4), v1 = __ldg(src + cb / 4 + 1);
            const float xs[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
            float hi[8], lo[8];
#pragma unroll
            for (int e = 0; e < 8; e++) tc::split_tf32_fast(xs[e], hi[e], lo[e]);
            tc::tmem_st8(ta + (uint32_t)cb, hi);
            tc::tmem_st8(ta + 128u + (uint32_t)cb, lo);
        }
        tc::tmem_st_wait();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const int64_t n_units = (rows + U - 1) / U;
    const int nj = (int)((n_units - blockIdx.x + gridDim.x - 1) / gridDim.x);     // >= 1 (grid <= n_units)
    auto unit_row0 = [&](int j) { return ((int64_t)blockIdx.x + (int64_t)j * gridDim.x) * U; };

    if (warp == 16) {
        // ------------------------------ MMA issuer ------------------------------
        if (lane == 0) {
            constexpr uint32_t id_th = tc::idesc_tf32_major(128, 128, true, true);
            constexpr uint32_t id_dh = tc::idesc_tf32(128, U);
            for (int j = 0; j < nj; j++) {
                const int s = j & 1, b = j & 3;
                tc::mbar_wait(full + s, (uint32_t)((j >> 1) & 1));
                if (j >= 4) tc::mbar_wait(dhempty + b, (uint32_t)(((j >> 2) - 1) & 1));
                tc::fence_after();
                const uint32_t base = tc::smem_u32(sm + s * S::SLOT);
                const uint32_t hh = base, hl = base + S::OP, gh = base + 2 * S::OP, gl = base + 3 * S::OP;
                const uint32_t kh = base + 4 * S::OP, kl = base + 5 * S::OP;
#pragma unroll
                for (int ks = 0; ks < U / 8; ks++) {       // dtheta += Hhat^T G: hi.hi, hi.lo, lo.hi
                    const uint32_t acc0 = (j | ks) != 0;
                    tc::mma_tf32(tmem + kT8Acc, tc::mnmajor_b32_desc(hh, ks, U), tc::mnmajor_b32_desc(gh, ks, U),
                                 id_th, acc0);
                    tc::mma_tf32(tmem + kT8Acc, tc::mnmajor_b32_desc(hh, ks, U), tc::mnmajor_b32_desc(gl, ks, U),
                                 id_th, 1u);
                    tc::mma_tf32(tmem + kT8Acc, tc::mnmajor_b32_desc(hl, ks, U), tc::mnmajor_b32_desc(gh, ks, U),
                                 id_th, 1u);
                }
                const uint32_t dd = tmem + kT8Dh + 32u * b;
#pragma unroll
                for (int p = 0; p < 3; p++) {                 // dH^T = theta G^T: lo.hi, hi.lo, hi.hi
                    const uint32_t ta = tmem + kT8Th + (p == 0 ? 128u : 0u);
                    const uint32_t gb = p == 1 ? kl : kh;
#pragma unroll
                    for (int ks = 0; ks < D / 8; ks++)
                        tc::mma_tf32_ts(dd, ta + 8u * ks, tc::kmajor_sw128_desc(gb, ks, U), id_dh, (p | ks) != 0);
                }
                tc::commit(empty + s);
                tc::commit(dhfull + b);
            }
        }
        __syncwarp();
    } else {
        // --------------------------- staging / drain ---------------------------
        const int r = (lane & 7) + 8 * (warp & 3);          // row in the unit
        const int ck = (lane >> 3) + 4 * (warp >> 2);       // 8-column chunk
        const int c0 = 8 * ck;
        const int sw = (lane >> 2) & 1;                     // BASE32B granule-half swap
        const bool issuer = t == 0;
        float prg = 0.f, pzz = 0.f;
        uint32_t pm = 0u, pcw[CW];
        float4 ph[BITS == 32 ? 2 : 1];
        auto load_small = [&](int jj) {
            const int64_t row = unit_row0(jj) + r;
            const bool ok = jj < nj && row < rows;
            prg = (ok && BITS != 32) ? __ldg(ranges + row) : 0.f;
            pzz = (ok && BITS != 32) ? __ldg(offsets + row) : 0.f;
            pm = ok ? __ldg(mask + row * 4 + (c0 >> 5)) : 0u;
            if constexpr (BITS == 32) {
                const float4 *h4 = reinterpret_cast<const float4 *>(codes) + row * (D / 4) + c0 / 4;
                ph[0] = ok ? __ldg(h4) : make_float4(0.f, 0.f, 0.f, 0.f);
                ph[BITS == 32 ? 1 : 0] = ok ? __ldg(h4 + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
            } else if constexpr (BITS == 1) {
                pcw[0] = ok ? (uint32_t)__ldg(codes + row * RB + ck) : 0u;
            } else if constexpr (BITS == 2) {
                pcw[0] = ok ? (uint32_t)__ldg(reinterpret_cast<const uint16_t *>(codes + row * RB) + ck) : 0u;
            } else {
                const uint32_t *cw = reinterpret_cast<const uint32_t *>(codes + row * RB) + ck * CW;
#pragma unroll
                for (int w = 0; w < CW; w++) pcw[w] = ok ? __ldg(cw + w) : 0u;
            }
        };
        const int in_bytes = (has_gr ? 16384 : 0) + (has_ge ? 16384 : 0);
        auto issue_in = [&](int jj) {
            const int r0 = (int)unit_row0(jj);
            tma::expect_tx(infull, (uint32_t)in_bytes);
#pragma unroll
            for (int bx = 0; bx < 4; bx++) {
                if (has_gr) tma::load_2d(instage + bx * 4096, &tm_gr, 32 * bx, r0, infull);
                if (has_ge) tma::load_2d(instage + 16384 + bx * 4096, &tm_ge, 32 * bx, r0, infull);
            }
        };
        auto drain = [&](int jj) {
            const int b = jj & 3;
            tc::mbar_wait(dhfull + b, (uint32_t)((jj >> 2) & 1));
            tc::fence_after();
            // warp w: lanes n = 32 (w % 4) + lane, unit rows 8 (w / 4) .. + 8
            const int q = warp & 3, rb = 8 * (warp >> 2);
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                           "=r"(v[7])
                         : "r"(tmem + ((uint32_t)(32 * q) << 16) + kT8Dh + 32u * b + (uint32_t)rb));
            tc::tmem_ld_wait();
            tc::fence_before();
            tc::mbar_arrive(dhempty + b);
            const int64_t r0 = unit_row0(jj);
#pragma unroll
            for (int i = 0; i < 8; i++)
                if (r0 + rb + i < rows) dh[(r0 + rb + i) * D + 32 * q + lane] = __uint_as_float(v[i]);
        };
        if (issuer) issue_in(0);
        load_small(0);
        for (int j = 0; j < nj; j++) {
            const int s = j & 1;
            const float rg = prg, zz = pzz;
            const uint32_t mw = (pm >> (c0 & 31)) & 0xFFu;
            uint32_t cw[CW];
#pragma unroll
            for (int w = 0; w < CW; w++) cw[w] = pcw[w];
            float4 hq4[BITS == 32 ? 2 : 1];
            if constexpr (BITS == 32) { hq4[0] = ph[0]; hq4[BITS == 32 ? 1 : 0] = ph[BITS == 32 ? 1 : 0]; }
            load_small(j + 1);
            // g_read / g_e chunk from the TMA stage, then the stage is refilled
            tc::mbar_wait(infull, (uint32_t)(j & 1));
            float4 a4[2], e4[2];
            {
                const uint32_t o = (c0 >> 5) * 4096 + tma::box_off(r, c0 & 31);
                const uint32_t o1 = (c0 >> 5) * 4096 + tma::box_off(r, (c0 & 31) + 4);
                a4[0] = has_gr ? *reinterpret_cast<const float4 *>(instage + o) : make_float4(0.f, 0.f, 0.f, 0.f);
                a4[1] = has_gr ? *reinterpret_cast<const float4 *>(instage + o1) : make_float4(0.f, 0.f, 0.f, 0.f);
                e4[0] = has_ge ? *reinterpret_cast<const float4 *>(instage + 16384 + o) : make_float4(0.f, 0.f, 0.f, 0.f);
                e4[1] = has_ge ? *reinterpret_cast<const float4 *>(instage + 16384 + o1) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            tma::named_sync(1, 512);
            if (issuer && j + 1 < nj) {
                tc::fence_proxy_async();
                issue_in(j + 1);
            }
            const float rb = __fmul_rn(rg, 1.0f / (float)((1u << (BITS < 32 ? BITS : 1)) - 1u));
            float lut[BITS <= 2 ? (1 << BITS) : 1];
            if constexpr (BITS <= 2) {
#pragma unroll
                for (int c = 0; c < (1 << BITS); c++) lut[c] = lut_entry<BITS>(rg, zz, c);
            }
            float gh[8], gl[8], hh[8], hl[8];
#pragma unroll
            for (int e = 0; e < 8; e++) {
                const float av = e < 4 ? (e == 0 ? a4[0].x : e == 1 ? a4[0].y : e == 2 ? a4[0].z : a4[0].w)
                                       : (e == 4 ? a4[1].x : e == 5 ? a4[1].y : e == 6 ? a4[1].z : a4[1].w);
                const float ev = e < 4 ? (e == 0 ? e4[0].x : e == 1 ? e4[0].y : e == 2 ? e4[0].z : e4[0].w)
                                       : (e == 4 ? e4[1].x : e == 5 ? e4[1].y : e == 6 ? e4[1].z : e4[1].w);
                // g = g_read + g_e in the reference's routing order (tape.py:204-209)
                const float gv = (has_gr && has_ge) ? __fadd_rn(av, ev) : (has_gr ? av : ev);
                const float gj = ((mw >> e) & 1u) ? gv : 0.0f;
                float hv;
                if constexpr (BITS == 32) {
                    const float4 hq = hq4[BITS == 32 ? (e >> 2) : 0];
                    const int q4 = e & 3;
                    hv = q4 == 0 ? hq.x : q4 == 1 ? hq.y : q4 == 2 ? hq.z : hq.w;
                } else {
                    const int bp = e * BITS;
                    const uint32_t code = (cw[(bp >> 5) % CW] >> (bp & 31)) & CM;
                    if constexpr (BITS == 1) hv = code ? lut[BITS <= 2 ? 1 : 0] : lut[0];
                    else if constexpr (BITS == 2)
                        hv = (code & 2u) ? ((code & 1u) ? lut[BITS == 2 ? 3 : 0] : lut[BITS == 2 ? 2 : 0])
                                         : ((code & 1u) ? lut[BITS <= 2 ? 1 : 0] : lut[0]);
                    else hv = __fmaf_rn(__uint2float_rn(code), rb, zz);
                }
                tc::split_tf32_fast(gj, gh[e], gl[e]);
                tc::split_tf32_fast(hv, hh[e], hl[e]);
            }
            // slot s free once the MMAs of unit j-2 are done
            if (j >= 2) tc::mbar_wait(empty + s, (uint32_t)(((j >> 1) - 1) & 1));
            uint8_t *slot = sm + s * S::SLOT;
#pragma unroll
            for (int u = 0; u < 2; u++) {               // MN-major: granule half u ^ sw
                const int src = u ^ sw;
                const uint32_t o = tc::b32_off(r, c0 + 4 * src, U);
                auto pick = [&](const float *v) {
                    return make_float4(src ? v[4] : v[0], src ? v[5] : v[1], src ? v[6] : v[2], src ? v[7] : v[3]);
                };
                *reinterpret_cast<float4 *>(slot + o) = pick(hh);
                *reinterpret_cast<float4 *>(slot + S::OP + o) = pick(hl);
                *reinterpret_cast<float4 *>(slot + 2 * S::OP + o) = pick(gh);
                *reinterpret_cast<float4 *>(slot + 3 * S::OP + o) = pick(gl);
            }
#pragma unroll
            for (int u = 0; u < 2; u++) {               // K-major SW128 copy of G (B of dH^T)
                const uint32_t o = tc::sw128_off(r, c0 + 4 * u, U);
                *reinterpret_cast<float4 *>(slot + 4 * S::OP + o) =
                    make_float4(gh[4 * u], gh[4 * u + 1], gh[4 * u + 2], gh[4 * u + 3]);
                *reinterpret_cast<float4 *>(slot + 5 * S::OP + o) =
                    make_float4(gl[4 * u], gl[4 * u + 1], gl[4 * u + 2], gl[4 * u + 3]);
            }
            tc::fence_proxy_async();
            tc::mbar_arrive(full + s);
            if (j >= 1) drain(j - 1);
        }
        drain(nj - 1);
    }
    // ---- dtheta partial of this CTA: lane i = row i, 128 columns ----
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp < 4) {
        float *dst = partial + (int64_t)blockIdx.x * D * D + (int64_t)(32 * warp + lane) * D;
#pragma unroll
        for (int cb = 0; cb < D; cb += 32) {
            float v[32];
            tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + kT8Acc + (uint32_t)cb, v);
#pragma unroll
            for (int k4 = 0; k4 < 8; k4++)
                reinterpret_cast<float4 *>(dst + cb)[k4] = make_float4(v[4 * k4], v[4 * k4 + 1], v[4 * k4 + 2], v[4 * k4 + 3]);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free(tmem, 512);
}

}  // namespace kgq

using namespace kgq;

// Launch helper used by kgq_layer_backward_f32 (kgq_backward.cu) for d = 64.
int kgq_launch_layer_backward_tc(const float *g_read, const float *g_e, const uint32_t *mask,
                                 const uint8_t *codes, const float *ranges, const float *offsets,
                                 int64_t rows, int32_t d, int32_t bits, const float *theta, float *dh,
                                 float *partial, int grid, cudaStream_t s, const int32_t *gr_map,
                                 const float *gr_rows) {
    static bool attr[33] = {false}, attr128[33] = {false};
    CUtensorMap tgr, tge;
    const float *any = g_read ? g_read : (g_e ? g_e : gr_rows);    // an unused map still needs an address
    const uint32_t box_rows = d == 128 ? (uint32_t)kT8U : 64u;
    if (!tma::make_rowmajor_f32(&tgr, g_read ? g_read : any, (uint64_t)rows, (uint64_t)d, box_rows) ||
        !tma::make_rowmajor_f32(&tge, g_e ? g_e : any, (uint64_t)rows, (uint64_t)d, box_rows))
        return KGQ_ERR_CUDA;
    const int hr = g_read ? 1 : 0, he = g_e ? 1 : 0;
    if (d == 128) {
#define KGQ_BTC8(B) do {                                                                           \
        if (!attr128[B]) {                                                                         \
            cudaError_t e = cudaFuncSetAttribute(layer_backward_tc128_kernel<B>,                     \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                                 (int)Bwd128Smem::bytes);                           \
            if (e != cudaSuccess) return kgq_set_cuda_error(e);                                    \
            attr128[B] = true;                                                                     \
        }                                                                                          \
        layer_backward_tc128_kernel<B><<<grid, kBtcThreads, Bwd128Smem::bytes, s>>>(tgr, tge, hr, he, mask, \
                                                                codes, ranges, offsets, rows, theta, dh, partial); \
    } while (0)
        switch (bits) {
            case 1: KGQ_BTC8(1); break;
            case 2: KGQ_BTC8(2); break;
            case 4: KGQ_BTC8(4); break;
            case 8: KGQ_BTC8(8); break;
            default: KGQ_BTC8(32); break;
        }
#undef KGQ_BTC8
        return KGQ_OK;
    }
#define KGQ_BTC(B) do {                                                                            \
        if (!attr[B]) {                                                                            \
            cudaError_t e = cudaFuncSetAttribute(layer_backward_tc_kernel<B>,                        \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                                 (int)BwdTcSmem::bytes);                            \
            if (e != cudaSuccess) return kgq_set_cuda_error(e);                                    \
            attr[B] = true;                                                                        \
        }                                                                                          \
        layer_backward_tc_kernel<B><<<grid, kBtcThreads, BwdTcSmem::bytes, s>>>(tgr, tge, hr, he, gr_map, gr_rows, \
                                                                        mask, codes, ranges, offsets, rows, theta, dh, \
                                                                        partial); \
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
