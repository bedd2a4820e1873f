// kgq_quant.cu -- fused per-group quantize+pack (K1) and unpack+dequantize (K2)
// for sm_100a.  Semantics: reference quantize.py:177-247 (see include/kgq.h).
//
// Fast kernels (group G in {32,64,128,256}, 16-byte aligned buffers):
//   * 4 threads per group, 8 groups per warp.  Thread j of a group owns the
//     float4 j of every 16-element block of the group (element 16i+4j+e), so a
//     warp-wide 128-bit load covers 8 x 64 contiguous bytes (fully used
//     sectors), and min/max needs only two xor-shuffles.
//   * fp32 math reproduces numpy bit-for-bit: a = x - Z, q = a / R (IEEE,
//     hoisted reciprocal + Markstein correction, kgq_common.cuh), s = q * B,
//     clip, then the code.  Stochastic rounding uses code = ceil(s - u),
//     which equals floor(s) + [u < frac] exactly; ceil(s - u) is formed with
//     round-up FP adds, and the magic constant 1.5*2^23 turns it into an
//     integer in the low mantissa bits with no F2I conversion.
//   * Codes are staged per warp in shared memory and leave as coalesced
//     16-byte stores.  R, Z leave as one fp32 each per group.
// Generic kernels (any G, any alignment, caller noise): warp per group.
#include "kgq_common.cuh"

namespace kgq {

#ifndef KGQ_QRING_KB
#define KGQ_QRING_KB 64                // quantize prefetch ring per CTA
#endif
constexpr int kWarps = 8;              // warps per CTA
constexpr int kThreads = kWarps * 32;

// Thread geometry of the fast quantizer: a G-element group is handled by T
// threads (T = 2 or 4); thread j owns float4 q in [j*Q, j*Q+Q) (Q = 4/T) of
// every 16-element block, so one warp-wide 128-bit load covers 32/T groups
// with fully used sectors and the noise calls (which pair float4 q of blocks
// 2p and 2p+1) are never split across threads.
template <int G, int T>
struct Geo {
    static constexpr int NBLK = G / 16;     // 16-element blocks per group
    static constexpr int Q = 4 / T;         // float4 per block per thread
    static constexpr int NF = NBLK * Q;     // float4 per thread
    static constexpr int GPW = 32 / T;      // groups per warp tile
    // cp.async ring depth: <= 64 KB of prefetch slots per CTA
    static constexpr int S = (NF * 512 * kWarps * 2 <= KGQ_QRING_KB * 1024) ? (KGQ_QRING_KB * 1024) / (NF * 512 * kWarps) : 1;
};

// Codes of the NF float4 a thread owns, 4*BITS bits per float4 (LSB-first).
// GUARD=false: the group passed group_div_unguarded (no per-element check).
template <int G, int T, int BITS, int MODE, bool GUARD>
__device__ __forceinline__ void quant_pieces(const float4 (&v)[Geo<G, T>::NF], float z, const DivR &dv,
                                             const FastKey &fk, uint64_t gglob, int j,
                                             uint64_t seed, uint64_t tid,
                                             uint32_t (&piece)[Geo<G, T>::NF]) {
    using GE = Geo<G, T>;
    constexpr float Bf = (float)PackInfo<BITS>::B;
    const uint32_t kc = MODE == KGQ_ROUND_SR_FAST ? carrier_const() : 0u;
#pragma unroll
    for (int p = 0; p < GE::NBLK / 2; p++) {
#pragma unroll
        for (int qq = 0; qq < GE::Q; qq++) {
            const int q = j * GE::Q + qq;
            uint4 rnd = make_uint4(0, 0, 0, 0);
            if (MODE == KGQ_ROUND_SR_FAST) rnd = fast_call(fk, gglob, (uint32_t)(4 * p + q));
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int i = 2 * p + h;
                const int f = i * GE::Q + qq;
                u64x4 r64 = {0, 0, 0, 0};
                if (MODE == KGQ_ROUND_SR_COMPAT)
                    r64 = philox4x64_10(gglob * (uint64_t)(G / 4) + (uint64_t)(4 * i + q) + 1ull,
                                        0, 0, 0, seed, tid);
                const float xs[4] = {v[f].x, v[f].y, v[f].z, v[f].w};
                const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
                const uint64_t cw[4] = {r64.x, r64.y, r64.z, r64.w};
                uint32_t acc = 0;
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const float a = __fsub_rn(xs[e], z);
                    const float qv = GUARD ? div_a(dv, a) : div_a_unguarded(dv, a);
                    float s = __fmul_rn(qv, Bf);
                    // R = inf (an inf in the group, or a range that overflows):
                    // inf/inf scales to NaN, which numpy casts to code 0
                    if (GUARD && !(s == s)) s = 0.0f;
                    const float uf = h ? u16_carrier_hi(rw[e], kc) : u16_carrier_lo(rw[e], kc);
                    acc += code_bits<MODE>(s, uf, cw[e] >> 11) << (BITS * e);
                }
                piece[f] = acc - magic_sum4<BITS>();
            }
        }
    }
}

// Unguarded groups (the common case) on packed fp32 pairs: the same IEEE
// sequence as quant_pieces<..., false> -- a = x - Z, q0 = a*y, e = a - R*q0,
// q = q0 + y*e, s = q*B, then the code -- two elements per FADD2 / FMUL2 /
// FFMA2, so about half the FP issue slots (K1 is issue-bound).
template <int G, int T, int BITS, int MODE>
__device__ __forceinline__ void quant_pieces_x2(const float4 (&v)[Geo<G, T>::NF], float z, const DivR &dv,
                                                const FastKey &fk, uint64_t gglob, int j,
                                                uint64_t seed, uint64_t tid,
                                                uint32_t (&piece)[Geo<G, T>::NF]) {
    using GE = Geo<G, T>;
    constexpr float Bf = (float)PackInfo<BITS>::B;
    const uint32_t kc = MODE == KGQ_ROUND_SR_FAST ? carrier_const() : 0u;
    const f32x2 mz = pk2(-z, -z), y2 = pk2(dv.y, dv.y), mr2 = pk2(-dv.r, -dv.r), B2 = pk2(Bf, Bf);
    const f32x2 mu2 = pk2(-0x1p-16f, -0x1p-16f), mg2 = pk2(kMagic + 128.0f, kMagic + 128.0f);
#pragma unroll
    for (int p = 0; p < GE::NBLK / 2; p++) {
#pragma unroll
        for (int qq = 0; qq < GE::Q; qq++) {
            const int q = j * GE::Q + qq;
            uint4 rnd = make_uint4(0, 0, 0, 0);
            if (MODE == KGQ_ROUND_SR_FAST) rnd = fast_call(fk, gglob, (uint32_t)(4 * p + q));
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int i = 2 * p + h;
                const int f = i * GE::Q + qq;
                u64x4 r64 = {0, 0, 0, 0};
                if (MODE == KGQ_ROUND_SR_COMPAT)
                    r64 = philox4x64_10(gglob * (uint64_t)(G / 4) + (uint64_t)(4 * i + q) + 1ull,
                                        0, 0, 0, seed, tid);
                const f32x2 xv[2] = {pk2(v[f].x, v[f].y), pk2(v[f].z, v[f].w)};
                const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
                const uint64_t cw[4] = {r64.x, r64.y, r64.z, r64.w};
                uint32_t cb[4];
#pragma unroll
                for (int e2 = 0; e2 < 2; e2++) {
                    const f32x2 a = add2_rn(xv[e2], mz);
                    const f32x2 q0 = mul2_rn(a, y2);
                    const f32x2 er = fma2_rn(mr2, q0, a);
                    const f32x2 qv = fma2_rn(y2, er, q0);
                    const f32x2 sc = mul2_rn(qv, B2);
                    if (MODE == KGQ_ROUND_NEAREST) {
                        // scalar magic adds: ptxas contracts mul.rn.f32x2 + add.rn.f32x2
                        // into one FFMA2 (a single rounding), which would change rint(s)
                        uint32_t s0, s1;
                        upk2u(sc, s0, s1);
                        cb[2 * e2] = code_bits<MODE>(__uint_as_float(s0), 0.f, 0);
                        cb[2 * e2 + 1] = code_bits<MODE>(__uint_as_float(s1), 0.f, 0);
                    } else if (MODE == KGQ_ROUND_SR_FAST) {
                        const uint32_t u0 = h ? __byte_perm(rw[2 * e2], kc, 0x7632) : __byte_perm(rw[2 * e2], kc, 0x7610);
                        const uint32_t u1 = h ? __byte_perm(rw[2 * e2 + 1], kc, 0x7632)
                                              : __byte_perm(rw[2 * e2 + 1], kc, 0x7610);
                        const f32x2 x1 = fma2_ru(pk2u(u0, u1), mu2, sc);   // RU(s - 128 - u)
                        upk2u(add2_ru(x1, mg2), cb[2 * e2], cb[2 * e2 + 1]);
                    } else {
                        uint32_t s0, s1;
                        upk2u(sc, s0, s1);
                        cb[2 * e2] = code_bits<MODE>(__uint_as_float(s0), 0.f, cw[2 * e2] >> 11);
                        cb[2 * e2 + 1] = code_bits<MODE>(__uint_as_float(s1), 0.f, cw[2 * e2 + 1] >> 11);
                    }
                }
                uint32_t acc = cb[0];
#pragma unroll
                for (int e = 1; e < 4; e++) acc += cb[e] << (BITS * e);
                piece[f] = acc - magic_sum4<BITS>();
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K1: fast fused quantize + pack.
// ---------------------------------------------------------------------------
// One warp tile (GPW groups) from the NF float4 each lane holds: min / max,
// the codes (packed, staged in shared memory, 16-byte coalesced stores) and
// R, Z.  FULL tiles (all but at most one per launch) skip every bounds check.
template <int G, int T, int BITS, int MODE, bool FULL>
__device__ __forceinline__ void quant_tile(const float4 (&v)[Geo<G, T>::NF], int64_t tile, int64_t n_groups,
                                           int lane, int j, int gw, uint8_t *st, const FastKey &fk,
                                           uint64_t seed, uint64_t tid, int64_t group_offset,
                                           uint8_t *__restrict__ codes, float *__restrict__ ranges,
                                           float *__restrict__ offsets) {
    using GE = Geo<G, T>;
    constexpr int NF = GE::NF, Q = GE::Q, GPW = GE::GPW;
    constexpr int GB = G * BITS / 8;              // packed bytes per group
    constexpr int PW = 4 * BITS * Q;              // packed bits per thread per block
    constexpr int TB = GPW * GB;                  // packed bytes per tile (multiple of 16)
    const int64_t g = tile * GPW + gw;
    float mn = fmin_nan(fmin_nan(v[0].x, v[0].y), fmin_nan(v[0].z, v[0].w));
    float mx = fmax_nan(fmax_nan(v[0].x, v[0].y), fmax_nan(v[0].z, v[0].w));
#pragma unroll
    for (int f = 1; f < NF; f++) {
        mn = fmin_nan(mn, fmin_nan(fmin_nan(v[f].x, v[f].y), fmin_nan(v[f].z, v[f].w)));
        mx = fmax_nan(mx, fmax_nan(fmax_nan(v[f].x, v[f].y), fmax_nan(v[f].z, v[f].w)));
    }
#pragma unroll
    for (int o = 1; o < T; o <<= 1) {
        mn = fmin_nan(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax_nan(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const float z = mn;
    const float r = __fsub_rn(mx, mn);
    const DivR dv = make_div(r);
    const uint64_t gglob = (uint64_t)(group_offset + g);

    uint32_t piece[NF];
    if (r > 0.0f) {
        if (group_div_unguarded(dv, z))
#ifndef KGQ_NO_X2
            quant_pieces_x2<G, T, BITS, MODE>(v, z, dv, fk, gglob, j, seed, tid, piece);
#else
            quant_pieces<G, T, BITS, MODE, false>(v, z, dv, fk, gglob, j, seed, tid, piece);
#endif
        else
            quant_pieces<G, T, BITS, MODE, true>(v, z, dv, fk, gglob, j, seed, tid, piece);
    } else {
#pragma unroll
        for (int f = 0; f < NF; f++) piece[f] = 0;   // R == 0 -> scaled 0 -> code 0
    }

    // stage the packed codes: the thread's Q float4 of block i are PW
    // contiguous bits at byte (16i + 4jQ) * BITS / 8 of the group
    uint8_t *gst = st + gw * GB;
#pragma unroll
    for (int i = 0; i < GE::NBLK; i++) {
        const int off = (16 * i + 4 * j * Q) * BITS / 8;
        if (PW == 64) {
            *reinterpret_cast<uint2 *>(gst + off) = make_uint2(piece[i * Q], piece[i * Q + 1]);
        } else {
            uint32_t w = piece[i * Q];
            if constexpr (Q == 2) w |= piece[i * Q + 1] << (4 * BITS);
            if (PW == 32) *reinterpret_cast<uint32_t *>(gst + off) = w;
            else if (PW == 16) *reinterpret_cast<uint16_t *>(gst + off) = (uint16_t)w;
            else if (PW == 8) gst[off] = (uint8_t)w;
            else {  // PW == 4 (T=4, BITS=1): pair lanes j, j^1 into one byte
                const uint32_t other = __shfl_xor_sync(0xffffffffu, w, 1);
                if ((j & 1) == 0) gst[off] = (uint8_t)(w | (other << 4));
            }
        }
    }
    __syncwarp();
    uint8_t *dst = codes + tile * TB;
    if (FULL) {
        constexpr int NCH = TB / 16;
#pragma unroll
        for (int k = 0; k < (NCH + 31) / 32; k++) {
            const int c = lane + 32 * k;
            if (NCH % 32 == 0 || c < NCH)
                *reinterpret_cast<uint4 *>(dst + 16 * c) = *reinterpret_cast<const uint4 *>(st + 16 * c);
        }
        // R and Z: one store per lane (j = 0 -> R, j = 1 -> Z)
        if (j < 2) (j ? offsets : ranges)[g] = j ? z : r;
    } else {
        const int nvalid = (int)imin64(GPW, n_groups - tile * GPW);
        const int nbytes = nvalid * GB;
        if ((nbytes & 15) == 0) {
            for (int b = lane * 16; b < nbytes; b += 32 * 16)
                *reinterpret_cast<uint4 *>(dst + b) = *reinterpret_cast<const uint4 *>(st + b);
        } else {
            for (int b = lane * 4; b < nbytes; b += 32 * 4)
                *reinterpret_cast<uint32_t *>(dst + b) = *reinterpret_cast<const uint32_t *>(st + b);
        }
        if (gw < nvalid && j < 2) (j ? offsets : ranges)[g] = j ? z : r;
    }
    __syncwarp();
}

template <int G, int T, int BITS, int MODE>
__global__ void __launch_bounds__(kThreads)
quantize_fast_kernel(const float *__restrict__ x, int64_t n_groups, uint8_t *__restrict__ codes,
                     float *__restrict__ ranges, float *__restrict__ offsets, uint64_t seed,
                     uint64_t tid, const uint64_t *__restrict__ tid_base, int64_t group_offset) {
    if (tid_base) tid += __ldg(tid_base);          // graph replays advance the key on device
    using GE = Geo<G, T>;
    constexpr int NF = GE::NF, Q = GE::Q, GPW = GE::GPW, S = GE::S;
    constexpr int GB = G * BITS / 8;
    __shared__ __align__(16) uint8_t stage[kWarps][GPW * GB];
    // cp.async ring: each lane streams its own float4s for the next S-1 full
    // tiles into private shared-memory slots (no cross-lane sharing -> no barriers).
    extern __shared__ __align__(16) float4 pf_raw[];   // [kWarps][S][NF][32]
    auto pf = reinterpret_cast<float4 (*)[S][NF][32]>(pf_raw);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane % T, gw = lane / T;
    uint8_t *st = stage[warp];
    const FastKey fk = make_fast_key(seed, tid);

    const int64_t n_full = n_groups / GPW;             // full tiles
    const int64_t stride = (int64_t)gridDim.x * kWarps;
    const int64_t tile0 = (int64_t)blockIdx.x * kWarps + warp;
    const float4 *xb = reinterpret_cast<const float4 *>(x) + j * Q + gw * (G / 4);
    int64_t pnext = tile0;                             // next full tile to prefetch
    auto issue = [&](int s) {                          // one commit group per tile (possibly empty)
        if (pnext < n_full) {
            const float4 *src = xb + pnext * (GPW * G / 4);
#pragma unroll
            for (int i = 0; i < GE::NBLK; i++)
#pragma unroll
                for (int qq = 0; qq < Q; qq++) cp_async16(&pf[warp][s][i * Q + qq][lane], src + 4 * i + qq);
        }
        cp_async_commit();
        pnext += stride;
    };
    if (S > 1) {
#pragma unroll
        for (int k = 0; k < S - 1; k++) issue(k);
    }
    int cur = 0;
    int64_t tile = tile0;
    for (; tile < n_full; tile += stride) {
        float4 v[NF];
        if (S > 1) {
            cp_async_wait<(S > 1 ? S - 2 : 0)>();
#pragma unroll
            for (int f = 0; f < NF; f++) v[f] = pf[warp][cur][f][lane];
            issue(cur == 0 ? S - 1 : cur - 1);
            cur = (cur + 1 == S) ? 0 : cur + 1;
        } else {
            const float4 *src = xb + tile * (GPW * G / 4);
#pragma unroll
            for (int i = 0; i < GE::NBLK; i++)
#pragma unroll
                for (int qq = 0; qq < Q; qq++) v[i * Q + qq] = ldg_stream(src + 4 * i + qq);
        }
        quant_tile<G, T, BITS, MODE, true>(v, tile, n_groups, lane, j, gw, st, fk, seed, tid, group_offset,
                                          codes, ranges, offsets);
    }
    if (S > 1) cp_async_wait<0>();
    // the partial last tile (at most one per launch): guarded direct loads;
    // lanes past the end compute on zeros and store nothing
    if (tile * GPW < n_groups) {
        const int64_t g = tile * GPW + gw;
        const bool valid = g < n_groups;
        const float4 *src = xb + tile * (GPW * G / 4);
        float4 v[NF];
#pragma unroll
        for (int i = 0; i < GE::NBLK; i++)
#pragma unroll
            for (int qq = 0; qq < Q; qq++)
                v[i * Q + qq] = valid ? ldg_stream(src + 4 * i + qq) : make_float4(0.f, 0.f, 0.f, 0.f);
        quant_tile<G, T, BITS, MODE, false>(v, tile, n_groups, lane, j, gw, st, fk, seed, tid, group_offset,
                                           codes, ranges, offsets);
    }
}

// ---------------------------------------------------------------------------
// K1 generic: one warp per group, any G / alignment / mode (incl. caller noise).
// Each lane owns whole output bytes, so no packing races.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
quantize_generic_kernel(const float *__restrict__ x, int64_t n_groups, int G, int bits, int mode,
                        uint64_t seed, uint64_t tid, const uint64_t *__restrict__ tid_base,
                        int64_t group_offset,
                        const double *__restrict__ noise, uint8_t *__restrict__ codes,
                        float *__restrict__ ranges, float *__restrict__ offsets) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int GB = (G * bits + 7) / 8;
    const float Bf = (float)((1u << bits) - 1u);
    if (tid_base) tid += __ldg(tid_base);
    const FastKey fk = make_fast_key(seed, tid);
    for (int64_t g = warp_id; g < n_groups; g += n_warps) {
        const float *row = x + g * (int64_t)G;
        float mn = INFINITY, mx = -INFINITY;
        for (int k = lane; k < G; k += 32) {
            mn = fmin_nan(mn, row[k]);
            mx = fmax_nan(mx, row[k]);
        }
        mn = warp_min(mn, 32);
        mx = warp_max(mx, 32);
        const float z = mn, r = __fsub_rn(mx, mn);
        const uint64_t gglob = (uint64_t)(group_offset + g);
        const int per_byte = 8 / bits;
        for (int bi = lane; bi < GB; bi += 32) {
            uint32_t byte = 0;
            for (int t = 0; t < per_byte; t++) {
                const int k = bi * per_byte + t;
                if (k >= G) break;
                uint32_t code = 0;
                if (r > 0.0f) {
                    float s = __fmul_rn(__fdiv_rn(__fsub_rn(row[k], z), r), Bf);
                    s = fminf(fmaxf(s, 0.0f), Bf);     // NaN (inf/inf) -> 0, numpy's cast
                    if (mode == KGQ_ROUND_NEAREST) {
                        code = (uint32_t)rintf(s);
                    } else {
                        const float fl = floorf(s);
                        const float frac = __fsub_rn(s, fl);
                        double u;
                        if (mode == KGQ_ROUND_SR_FAST)
                            u = (double)fast_u16(fk, gglob, k) * (1.0 / 65536.0);
                        else if (mode == KGQ_ROUND_SR_COMPAT)
                            u = (double)compat_raw53(seed, tid, gglob, G, k) * 0x1p-53;
                        else
                            u = noise[g * (int64_t)G + k];
                        code = (uint32_t)fl + ((u < (double)frac) ? 1u : 0u);
                    }
                }
                byte |= code << (t * bits);
            }
            codes[g * (int64_t)GB + bi] = (uint8_t)byte;
        }
        if (lane == 0) {
            ranges[g] = r;
            offsets[g] = z;
        }
    }
}

// ---------------------------------------------------------------------------
// K2: fast unpack + dequantize.  out = (R*c)/B + Z (fp32, IEEE), R==0 -> Z.
// bits <= 4: per-group table of the B+1 reconstruction values in smem
// (computed once with IEEE division), one LDS per element.
// bits == 8: arithmetic with the hoisted-reciprocal division.
// ---------------------------------------------------------------------------
// Per-group outputs of one warp tile (8 groups) from staged codes + table.
template <int G, int BITS, int T>
__device__ __forceinline__ void dequant_tile_store(const uint8_t *gst, const float *lt, float r, float z,
                                                   float4 *dst, int j) {
    constexpr int NB = G / (4 * T);     // float4 per thread: thread j owns float4 T*i + j
    constexpr int NL = (BITS <= 4) ? (1 << BITS) : 1;
    constexpr float Bf = (float)PackInfo<BITS>::B;
    DivR dB;
    if (BITS == 8) dB = make_div(Bf);
    const bool rfast = (r >= 0x1p-100f) && (r <= 0x1p100f);
    if (BITS == 8 && rfast) {
        const Dq8 k8 = make_dq8(r, z, dB.y);
#pragma unroll
        for (int i = 0; i < NB; i++)
            stg_stream(dst + T * i + j, dq8_word(k8, *reinterpret_cast<const uint32_t *>(gst + 4 * (T * i + j))));
        return;
    }
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int f = T * i + j;        // float4 index in the group: codes 4f .. 4f+3
        uint32_t piece;
        if (BITS == 8) piece = *reinterpret_cast<const uint32_t *>(gst + 4 * f);
        else if (BITS == 4) piece = *reinterpret_cast<const uint16_t *>(gst + 2 * f);
        else if (BITS == 2) piece = gst[f];
        else piece = (gst[f >> 1] >> (4 * (f & 1))) & 0xFu;
        float o[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const uint32_t c = (piece >> (BITS * e)) & PackInfo<BITS>::B;
            if (NL > 1) {
                o[e] = lt[c];
            } else {
                if (r == 0.0f) { o[e] = z; continue; }
                const float cf = __fsub_rn(__uint_as_float(0x4B000000u | c), 8388608.0f);
                const float t = __fmul_rn(r, cf);
                float qv;
                if (rfast) {
                    const float q0 = __fmul_rn(t, dB.y);
                    const float er = __fmaf_rn(-Bf, q0, t);
                    qv = __fmaf_rn(dB.y, er, q0);
                } else {
                    qv = __fdiv_rn(t, Bf);
                }
                o[e] = __fadd_rn(qv, z);
            }
        }
        stg_stream(dst + f, make_float4(o[0], o[1], o[2], o[3]));
    }
}

// K2: T lanes per group (T = 4 at G <= 128, 8 at G = 256), 32/T groups per
// warp tile; thread j of a group owns float4 T*i + j, so one store
// instruction writes T*16-byte pieces of 32/T groups (T = 8 at G = 256: whole
// 128-byte lines).
template <int G, int BITS, int T>
__global__ void __launch_bounds__(kThreads)
dequantize_t4_kernel(const uint8_t *__restrict__ codes, const float *__restrict__ ranges,
                     const float *__restrict__ offsets, int64_t n_groups, float *__restrict__ out) {
    constexpr int GPW = 32 / T;                         // groups per warp tile
    constexpr int GB = G * BITS / 8;
    constexpr int TB = GPW * GB;             // code bytes per warp tile
    constexpr int NCH = TB / 16;                        // uint4 chunks per tile
    constexpr int CPL = (NCH + 31) / 32;                // chunks per lane
    constexpr int NL = (BITS <= 4) ? (1 << BITS) : 1;   // table entries per group
    constexpr int LS = (NL == 16) ? 17 : NL;            // padded stride (bank spread)
    __shared__ __align__(16) uint8_t stage[kWarps][TB];
    __shared__ float lut[kWarps][GPW * LS];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane % T, gw = lane / T;
    uint8_t *st = stage[warp];
    float *lt = lut[warp] + gw * LS;

    const int64_t n_full = n_groups / GPW;   // full tiles (software-pipelined)
    const int64_t stride = (int64_t)gridDim.x * kWarps;
    int64_t tile = (int64_t)blockIdx.x * kWarps + warp;

    // prefetch registers: this lane's code chunks + its group's (R, Z)
    uint4 cw[CPL];
    float r_n = 0.f, z_n = 0.f;
    auto prefetch = [&](int64_t t) {
        const uint4 *src = reinterpret_cast<const uint4 *>(codes + t * TB);
#pragma unroll
        for (int k = 0; k < CPL; k++)
            if (lane + 32 * k < NCH) cw[k] = __ldg(src + lane + 32 * k);
        r_n = __ldg(ranges + t * GPW + gw);
        z_n = __ldg(offsets + t * GPW + gw);
    };
    if (tile < n_full) prefetch(tile);
    for (; tile < n_full; tile += stride) {
#pragma unroll
        for (int k = 0; k < CPL; k++)
            if (lane + 32 * k < NCH) reinterpret_cast<uint4 *>(st)[lane + 32 * k] = cw[k];
        const float r = r_n, z = z_n;
        if (NL > 1) {
#pragma unroll
            for (int c = j; c < NL; c += T) lt[c] = lut_entry<BITS>(r, z, c);
        }
        // prefetch after the table: a slow-path division call would otherwise
        // force the in-flight loads to retire
        if (tile + stride < n_full) prefetch(tile + stride);
        __syncwarp();
        const int64_t g = tile * GPW + gw;
        dequant_tile_store<G, BITS, T>(st + gw * GB, lt, r, z, reinterpret_cast<float4 *>(out) + g * (G / 4), j);
        __syncwarp();
    }
    // the last partial tile (at most one in the grid)
    if (n_groups % GPW && (int64_t)blockIdx.x * kWarps + warp == n_full % stride) {
        const int64_t g0 = n_full * GPW;
        const int nvalid = (int)(n_groups - g0);
        const uint8_t *srcc = codes + g0 * GB;
        for (int b = lane * 4; b < nvalid * GB; b += 32 * 4)
            *reinterpret_cast<uint32_t *>(st + b) = __ldg(reinterpret_cast<const uint32_t *>(srcc + b));
        const bool valid = gw < nvalid;
        const float r = valid ? __ldg(ranges + g0 + gw) : 0.f;
        const float z = valid ? __ldg(offsets + g0 + gw) : 0.f;
        if (NL > 1) {
            for (int c = j; c < NL; c += T) lt[c] = lut_entry<BITS>(r, z, c);
        }
        __syncwarp();
        if (valid)
            dequant_tile_store<G, BITS, T>(st + gw * GB, lt, r, z,
                                        reinterpret_cast<float4 *>(out) + (g0 + gw) * (G / 4), j);
    }
}

__global__ void dequantize_generic_kernel(const uint8_t *__restrict__ codes,
                                          const float *__restrict__ ranges,
                                          const float *__restrict__ offsets, int64_t n_groups,
                                          int G, int bits, float *__restrict__ out) {
    const int GB = (G * bits + 7) / 8;
    const float Bf = (float)((1u << bits) - 1u);
    const uint32_t mask = (1u << bits) - 1u;
    const int64_t n = n_groups * (int64_t)G;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = idx / G;
        const int k = (int)(idx - g * G);
        const int bit = k * bits;
        const uint32_t c = (codes[g * GB + (bit >> 3)] >> (bit & 7)) & mask;
        const float r = ranges[g], z = offsets[g];
        out[idx] = (r == 0.0f) ? z : __fadd_rn(__fdiv_rn(__fmul_rn(r, (float)c), Bf), z);
    }
}

// ---------------------------------------------------------------------------
// Noise export (parity seam) and pack/unpack of raw codes.
// ---------------------------------------------------------------------------
__global__ void fast_noise_kernel(uint64_t seed, uint64_t tid, int64_t group_offset,
                                  int64_t n_groups, int G, uint16_t *__restrict__ out) {
    const FastKey fk = make_fast_key(seed, tid);
    const int64_t n = n_groups * (int64_t)G;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = idx / G;
        out[idx] = (uint16_t)fast_u16(fk, (uint64_t)(group_offset + g), (int)(idx - g * G));
    }
}

__global__ void compat_noise_kernel(uint64_t seed, uint64_t tid, int64_t group_offset,
                                    int64_t n_groups, int G, uint64_t *__restrict__ out) {
    const int64_t n = n_groups * (int64_t)G;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = idx / G;
        out[idx] = compat_raw53(seed, tid, (uint64_t)(group_offset + g), G, (int)(idx - g * G));
    }
}

__global__ void pack_codes_kernel(const uint8_t *__restrict__ codes, int64_t rows, int cols,
                                  int bits, uint8_t *__restrict__ packed, int32_t *overflow) {
    const int RB = (cols * bits + 7) / 8;
    const int per_byte = 8 / bits;
    const int64_t n = rows * (int64_t)RB;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = idx / RB;
        const int bi = (int)(idx - row * RB);
        uint32_t byte = 0;
        for (int t = 0; t < per_byte; t++) {
            const int k = bi * per_byte + t;
            if (k >= cols) break;
            const uint32_t c = codes[row * cols + k];
            if (c >> bits) atomicOr(overflow, 1);
            byte |= (c & ((1u << bits) - 1u)) << (t * bits);
        }
        packed[idx] = (uint8_t)byte;
    }
}

__global__ void unpack_codes_kernel(const uint8_t *__restrict__ packed, int64_t rows, int cols,
                                    int bits, uint8_t *__restrict__ codes) {
    const int RB = (cols * bits + 7) / 8;
    const int64_t n = rows * (int64_t)cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = idx / cols;
        const int k = (int)(idx - row * cols);
        const int bit = k * bits;
        codes[idx] = (uint8_t)((packed[row * RB + (bit >> 3)] >> (bit & 7)) & ((1u << bits) - 1u));
    }
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
static inline bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

static inline int grid_for(int64_t work_items, int per_block, int max_blocks_per_sm) {
    int64_t b = (work_items + per_block - 1) / per_block;
    const int64_t cap = (int64_t)kSMs * max_blocks_per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// T = threads per group: 4 (registers and the prefetch ring stay small;
// -DKGQ_T64_2 builds the 2-thread variant for G = 64: measured 58 % vs 81 %
// of the HBM peak on configs[1], so 4 stays).
template <int G> struct PickT { static constexpr int T = 4; };
#ifdef KGQ_T64_2   // A/B switch: 2 threads per 64-element group
template <> struct PickT<64> { static constexpr int T = 2; };
#endif

template <int G, int BITS, int MODE>
static void launch_quant_t4(const float *x, int64_t n_groups, uint8_t *codes, float *ranges,
                            float *offsets, uint64_t seed, uint64_t tid, const uint64_t *tid_base,
                            int64_t goff, cudaStream_t s) {
    constexpr int T = PickT<G>::T;
    using GE = Geo<G, T>;
    const int64_t tiles = (n_groups + GE::GPW - 1) / GE::GPW;
#ifndef KGQ_QGRID_PER_SM
#define KGQ_QGRID_PER_SM 8   // 3 / 6: -1..-3 %; 12 / 16 / 32: within noise of 8 (configs[1])
#endif
    const int grid = grid_for(tiles, kWarps, KGQ_QGRID_PER_SM);
    const size_t smem = GE::S > 1 ? (size_t)kWarps * GE::S * GE::NF * 32 * sizeof(float4) : 0;
    if (smem > 0) {   // dynamic + static smem may exceed the 48 KB default
        static unsigned attr_set = 0;   // per template instance, bit per device
        int dev = 0;
        cudaGetDevice(&dev);
        if (!(attr_set & (1u << (dev & 31)))) {
            cudaFuncSetAttribute(quantize_fast_kernel<G, T, BITS, MODE>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr_set |= 1u << (dev & 31);
        }
    }
    quantize_fast_kernel<G, T, BITS, MODE><<<grid, kThreads, smem, s>>>(x, n_groups, codes, ranges,
                                                                       offsets, seed, tid, tid_base, goff);
}

template <int G, int BITS>
static bool dispatch_quant_mode(int mode, const float *x, int64_t n_groups, uint8_t *codes,
                                float *ranges, float *offsets, uint64_t seed, uint64_t tid,
                                const uint64_t *tb, int64_t goff, cudaStream_t s) {
    switch (mode) {
        case KGQ_ROUND_NEAREST:
            launch_quant_t4<G, BITS, KGQ_ROUND_NEAREST>(x, n_groups, codes, ranges, offsets, seed, tid, tb, goff, s);
            return true;
        case KGQ_ROUND_SR_FAST:
            launch_quant_t4<G, BITS, KGQ_ROUND_SR_FAST>(x, n_groups, codes, ranges, offsets, seed, tid, tb, goff, s);
            return true;
        case KGQ_ROUND_SR_COMPAT:
            launch_quant_t4<G, BITS, KGQ_ROUND_SR_COMPAT>(x, n_groups, codes, ranges, offsets, seed, tid, tb, goff, s);
            return true;
        default:
            return false;
    }
}

template <int G>
static bool dispatch_quant_bits(int bits, int mode, const float *x, int64_t n_groups,
                                uint8_t *codes, float *ranges, float *offsets, uint64_t seed,
                                uint64_t tid, const uint64_t *tb, int64_t goff, cudaStream_t s) {
    switch (bits) {
        case 1: return dispatch_quant_mode<G, 1>(mode, x, n_groups, codes, ranges, offsets, seed, tid, tb, goff, s);
        case 2: return dispatch_quant_mode<G, 2>(mode, x, n_groups, codes, ranges, offsets, seed, tid, tb, goff, s);
        case 4: return dispatch_quant_mode<G, 4>(mode, x, n_groups, codes, ranges, offsets, seed, tid, tb, goff, s);
        case 8: return dispatch_quant_mode<G, 8>(mode, x, n_groups, codes, ranges, offsets, seed, tid, tb, goff, s);
    }
    return false;
}

template <int G>
static bool dispatch_dequant_bits(int bits, const uint8_t *codes, const float *ranges,
                                  const float *offsets, int64_t n_groups, float *out,
                                  cudaStream_t s) {
    // lanes per group, from A/B runs on 16M x 128: 8 at G = 256 (whole 128-byte
    // lines per store instruction; beats both 4 lanes, which scatter 64-byte
    // pieces 1 KB apart and stall on the store queue, and a warp per group,
    // which has too little work per warp in flight), 4 below
#ifndef KGQ_DQ_T256
#define KGQ_DQ_T256 8
#endif
    constexpr int T = G >= 256 ? KGQ_DQ_T256 : 4;
    const int64_t tiles = (n_groups + 32 / T - 1) / (32 / T);
    const int grid = grid_for(tiles, kWarps, 8);
    switch (bits) {
        case 1: dequantize_t4_kernel<G, 1, T><<<grid, kThreads, 0, s>>>(codes, ranges, offsets, n_groups, out); return true;
        case 2: dequantize_t4_kernel<G, 2, T><<<grid, kThreads, 0, s>>>(codes, ranges, offsets, n_groups, out); return true;
        case 4: dequantize_t4_kernel<G, 4, T><<<grid, kThreads, 0, s>>>(codes, ranges, offsets, n_groups, out); return true;
        case 8: dequantize_t4_kernel<G, 8, T><<<grid, kThreads, 0, s>>>(codes, ranges, offsets, n_groups, out); return true;
    }
    return false;
}

}  // namespace kgq

using namespace kgq;

static inline bool bits_ok(int bits) { return bits == 1 || bits == 2 || bits == 4 || bits == 8; }

extern "C" int kgq_quantize_f32(const float *x, int64_t n_groups, int32_t group, int32_t bits,
                                int32_t rounding, uint64_t seed, uint64_t tensor_id,
                                const uint64_t *tid_base, int64_t group_offset,
                                const double *noise, uint8_t *codes,
                                float *ranges, float *offsets, void *stream) {
    if (!bits_ok(bits)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (group < 1 || n_groups < 0 || rounding < 0 || rounding > 3 || group_offset < 0)
        return KGQ_ERR_INVALID_ARG;
    if (rounding == KGQ_ROUND_SR_NOISE && !noise) return KGQ_ERR_INVALID_ARG;
    if (n_groups == 0) return KGQ_OK;
    if (!x || !codes || !ranges || !offsets) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const bool fast_ok = rounding != KGQ_ROUND_SR_NOISE && aligned16(x) && aligned16(codes) &&
                         (group == 32 || group == 64 || group == 128 || group == 256);
    bool done = false;
    if (fast_ok) {
        switch (group) {
            case 32: done = dispatch_quant_bits<32>(bits, rounding, x, n_groups, codes, ranges, offsets, seed, tensor_id, tid_base, group_offset, s); break;
            case 64: done = dispatch_quant_bits<64>(bits, rounding, x, n_groups, codes, ranges, offsets, seed, tensor_id, tid_base, group_offset, s); break;
            case 128: done = dispatch_quant_bits<128>(bits, rounding, x, n_groups, codes, ranges, offsets, seed, tensor_id, tid_base, group_offset, s); break;
            case 256: done = dispatch_quant_bits<256>(bits, rounding, x, n_groups, codes, ranges, offsets, seed, tensor_id, tid_base, group_offset, s); break;
        }
    }
    if (!done) {
        const int grid = grid_for(n_groups, kWarps, 8);
        quantize_generic_kernel<<<grid, kThreads, 0, s>>>(x, n_groups, group, bits, rounding, seed,
                                                          tensor_id, tid_base, group_offset, noise,
                                                          codes, ranges, offsets);
    }
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_dequantize_f32(const uint8_t *codes, const float *ranges, const float *offsets,
                                  int64_t n_groups, int32_t group, int32_t bits, float *out,
                                  void *stream) {
    if (!bits_ok(bits)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (group < 1 || n_groups < 0) return KGQ_ERR_INVALID_ARG;
    if (n_groups == 0) return KGQ_OK;
    if (!codes || !ranges || !offsets || !out) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const bool fast_ok = aligned16(codes) && aligned16(out) &&
                         (group == 32 || group == 64 || group == 128 || group == 256);
    bool done = false;
    if (fast_ok) {
        switch (group) {
            case 32: done = dispatch_dequant_bits<32>(bits, codes, ranges, offsets, n_groups, out, s); break;
            case 64: done = dispatch_dequant_bits<64>(bits, codes, ranges, offsets, n_groups, out, s); break;
            case 128: done = dispatch_dequant_bits<128>(bits, codes, ranges, offsets, n_groups, out, s); break;
            case 256: done = dispatch_dequant_bits<256>(bits, codes, ranges, offsets, n_groups, out, s); break;
        }
    }
    if (!done) {
        const int grid = grid_for(n_groups * (int64_t)group, 256, 8);
        dequantize_generic_kernel<<<grid, 256, 0, s>>>(codes, ranges, offsets, n_groups, group, bits, out);
    }
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_fast_noise_u16(uint64_t seed, uint64_t tensor_id, int64_t group_offset,
                                  int64_t n_groups, int32_t group, uint16_t *out, void *stream) {
    if (group < 1 || n_groups < 0 || group_offset < 0 || (!out && n_groups)) return KGQ_ERR_INVALID_ARG;
    if (n_groups == 0) return KGQ_OK;
    const int grid = grid_for(n_groups * (int64_t)group, 256, 8);
    fast_noise_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(seed, tensor_id, group_offset, n_groups, group, out);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_compat_noise_raw53(uint64_t seed, uint64_t tensor_id, int64_t group_offset,
                                      int64_t n_groups, int32_t group, uint64_t *out, void *stream) {
    if (group < 1 || n_groups < 0 || group_offset < 0 || (!out && n_groups)) return KGQ_ERR_INVALID_ARG;
    if (n_groups == 0) return KGQ_OK;
    const int grid = grid_for(n_groups * (int64_t)group, 256, 8);
    compat_noise_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(seed, tensor_id, group_offset, n_groups, group, out);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_pack_codes(const uint8_t *codes, int64_t rows, int32_t cols, int32_t bits,
                              uint8_t *packed, int32_t *overflow, void *stream) {
    if (!bits_ok(bits)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (rows < 0 || cols < 0 || !overflow) return KGQ_ERR_INVALID_ARG;
    if (rows == 0 || cols == 0) return KGQ_OK;
    const int64_t n = rows * (int64_t)((cols * bits + 7) / 8);
    pack_codes_kernel<<<grid_for(n, 256, 8), 256, 0, (cudaStream_t)stream>>>(codes, rows, cols, bits, packed, overflow);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_unpack_codes(const uint8_t *packed, int64_t rows, int32_t cols, int32_t bits,
                                uint8_t *codes, void *stream) {
    if (!bits_ok(bits)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (rows < 0 || cols < 0) return KGQ_ERR_INVALID_ARG;
    if (rows == 0 || cols == 0) return KGQ_OK;
    unpack_codes_kernel<<<grid_for(rows * (int64_t)cols, 256, 8), 256, 0, (cudaStream_t)stream>>>(packed, rows, cols, bits, codes);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
