// kgq_graph.cu -- KG neighbour aggregation (K4 CSR SpMM) and the fused
// per-layer forward (spmm -> quantize H -> H.theta -> relu -> mask) on sm_100a.
//
// Exactness: every output element is accumulated in ascending column order
// as acc = acc + a*x with separate mul and add -- the order scipy's
// csr_matvecs uses (tensorops.py:8-12, 37-50) -- so results are bit-identical
// to the reference.  Only the LOADS are reordered/prefetched; the per-element
// add chain is never split, so rows cannot be divided across threads along
// the nonzero axis.  What we parallelise instead is (a) rows, (b) features.
//
// Schedule (row_order = rows by decreasing degree, n_heavy = #rows above
// kHeavy nonzeros; both built once per graph by the host):
//  * heavy rows (the first n_heavy of row_order): one CTA per row.  Thread t
//    owns feature t and runs that feature's sequential chain; all 256
//    threads stream the row's neighbour rows into a P-stage shared-memory
//    ring with cp.async (32 neighbours per stage), with the next stage's
//    column ids prefetched into registers one iteration ahead, so a 6k-nonzero
//    hub row costs ~nnz/(P*32) memory latencies instead of ~nnz/8.
//  * light rows: row groups.  A row is owned by LPR = d/8 lanes and a warp
//    works on RPW = 32/LPR rows of similar degree at once.  Lane gl owns the
//    two float4 at features 32p+4q and 32p+16+4q (p = gl>>2, q = gl&3): one
//    neighbour row is one 128-bit load per lane, and those 8 features are
//    the 8 elements of fast-noise call 4p+q (one Philox call per lane in the
//    fused quantizer).  The next column ids are prefetched while the current
//    neighbour rows are gathered.
#include "kgq_common.cuh"
#include "kgq_tma.cuh"
#include <type_traits>

namespace kgq {

constexpr int kCH = 32;             // neighbours per ring stage (heavy path)

// The CSR column ids / values and the SpMM output are streamed once per call;
// loading / storing them evict-first (.cs) keeps the gathered embedding table
// resident in L2 (table + CSR + output exceed the 126 MB L2 at Amazon shape).
#ifndef KGQ_SPMM_CS
#define KGQ_SPMM_CS 1
#endif
#if KGQ_SPMM_CS
#define KGQ_LD_STREAM(p) __ldcs(p)
#define KGQ_ST_STREAM(p, v) __stcs((p), (v))
#else
#define KGQ_LD_STREAM(p) __ldg(p)
#define KGQ_ST_STREAM(p, v) (*(p) = (v))
#endif

template <int D>
struct RG {
    static constexpr int LPR = D / 8;      // lanes per row (light path)
    static constexpr int RPW = 32 / LPR;   // rows per warp
    // heavy-path ring: P stages of kCH neighbour rows (<= 32 KB) + values
    static constexpr int P = (32 * 1024) / (kCH * D * 4) > 4 ? 4 : (32 * 1024) / (kCH * D * 4);
    static constexpr int NI = kCH * D / 4 / 256;           // cp.async per thread per stage
    // + column-id / value blocks: 2 x 256 ids and values (8 stages each),
    // streamed with cp.async a block ahead so no id load is on the chain
    static constexpr size_t ring_bytes = (size_t)P * kCH * (D + 1) * 4 + 2 * 256 * 8;
};

// ---------------------------------------------------------------------------
// Light path: one row per LPR-lane group (all lanes of the warp call this
// together; the nonzero loop runs to the warp's longest row with per-row
// predicates so shuffles stay convergent).
// ---------------------------------------------------------------------------
// Feature layout of the two float4 a lane owns:
//  NOISE_LAYOUT (fused layer): float4 f0 = 8(gl>>2) + (gl&3) and f0 + 4, so a
//    lane's 8 features are one fast-noise call;
//  contiguous (plain SpMM): float4 gl and gl + LPR, so each warp-wide load
//    touches whole 128-byte lines of every row (half the L1 tag lookups of
//    the noise layout, whose two loads each touch half of the same lines).
template <int D, bool NOISE_LAYOUT>
__device__ __forceinline__ int rg_f4a(int gl) {
    return NOISE_LAYOUT ? 8 * (gl >> 2) + (gl & 3) : gl;
}
template <int D, bool NOISE_LAYOUT>
__device__ __forceinline__ int rg_f4b(int gl) {
    return NOISE_LAYOUT ? 8 * (gl >> 2) + (gl & 3) + 4 : gl + RG<D>::LPR;
}

#ifndef KGQ_SPMM_BATCH
#define KGQ_SPMM_BATCH 1    // neighbour rows per batch in the light path: 1 (48 registers, 5 CTAs/SM)
                            // measured 13 % faster than 4 and 2 (tools/spmm_ab.py A/B builds)
#endif
#ifdef KGQ_SPMM_NOALLOC
// gathered rows are almost never re-hit in L1 (4 % hit rate): do not allocate
__device__ __forceinline__ float4 ldg_noalloc(const float4 *p) {
    float4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
#endif
// seg_beg / seg_end (both or neither): the row's nonzeros [seg_beg[row],
// seg_end[row]) only, continuing the running sums the caller put in acc
// (a source-block phase of the pipelined SpMM); else the whole row from 0.
template <int D, bool NOISE_LAYOUT = true, int BATCH = 4>
__device__ __forceinline__ void rg_spmm_row(const int32_t *__restrict__ indptr,
                                            const int32_t *__restrict__ indices,
                                            const float *__restrict__ vals,
                                            const float *__restrict__ x, int64_t row, bool active,
                                            int gl, float4 (&acc)[2],
                                            const int32_t *__restrict__ seg_beg = nullptr,
                                            const int32_t *__restrict__ seg_end = nullptr) {
    constexpr int LPR = RG<D>::LPR;
    if (!seg_beg) acc[0] = acc[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    int32_t beg = 0, end = 0;
    if (active) {
        beg = __ldg((seg_beg ? seg_beg : indptr) + row);
        end = seg_end ? __ldg(seg_end + row) : __ldg(indptr + row + 1);
    }
    const int len = end - beg;
    int maxlen = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    const int fa = rg_f4a<D, NOISE_LAYOUT>(gl), fb = rg_f4b<D, NOISE_LAYOUT>(gl);
    f32x2 ap[4] = {pk2(acc[0].x, acc[0].y), pk2(acc[0].z, acc[0].w), pk2(acc[1].x, acc[1].y), pk2(acc[1].z, acc[1].w)};
    int32_t nx_col = 0;
    float nx_val = 0.0f;
    if (gl < len) {
        nx_col = KGQ_LD_STREAM(indices + beg + gl);
        nx_val = KGQ_LD_STREAM(vals + beg + gl);
    }
    for (int base = 0; base < maxlen; base += LPR) {
        const int cnt = min(LPR, len - base);         // may be <= 0 for short rows
        const int32_t my_col = nx_col;
        const float my_val = nx_val;
        if (gl < len - base - LPR) {                  // prefetch the next LPR column ids
            nx_col = KGQ_LD_STREAM(indices + beg + base + LPR + gl);
            nx_val = KGQ_LD_STREAM(vals + beg + base + LPR + gl);
        }
#pragma unroll
        for (int t = 0; t < LPR; t += BATCH) {
            float4 xa[BATCH], xb[BATCH];
            float av[BATCH];
#pragma unroll
            for (int u = 0; u < BATCH; u++) {
                const int32_t col = __shfl_sync(0xffffffffu, my_col, t + u, LPR);
                av[u] = __shfl_sync(0xffffffffu, my_val, t + u, LPR);
                if (t + u < cnt) {
                    const float4 *xr = reinterpret_cast<const float4 *>(x + (int64_t)col * D);
#ifdef KGQ_SPMM_NOALLOC
                    xa[u] = ldg_noalloc(xr + fa);
                    xb[u] = ldg_noalloc(xr + fb);
#else
                    xa[u] = __ldg(xr + fa);
                    xb[u] = __ldg(xr + fb);
#endif
                }
            }
#pragma unroll
            for (int u = 0; u < BATCH; u++) {
                if (t + u < cnt) {
                    // acc = acc + a * x with separate roundings: scalar products,
                    // packed adds (FADD2, the same per-lane rounding); a packed
                    // multiply would be contracted into FFMA2 by ptxas
                    const float a = av[u];
                    ap[0] = add2_rn(ap[0], pk2(__fmul_rn(a, xa[u].x), __fmul_rn(a, xa[u].y)));
                    ap[1] = add2_rn(ap[1], pk2(__fmul_rn(a, xa[u].z), __fmul_rn(a, xa[u].w)));
                    ap[2] = add2_rn(ap[2], pk2(__fmul_rn(a, xb[u].x), __fmul_rn(a, xb[u].y)));
                    ap[3] = add2_rn(ap[3], pk2(__fmul_rn(a, xb[u].z), __fmul_rn(a, xb[u].w)));
                }
            }
        }
    }
    uint32_t w0, w1;
    upk2u(ap[0], w0, w1); acc[0].x = __uint_as_float(w0); acc[0].y = __uint_as_float(w1);
    upk2u(ap[1], w0, w1); acc[0].z = __uint_as_float(w0); acc[0].w = __uint_as_float(w1);
    upk2u(ap[2], w0, w1); acc[1].x = __uint_as_float(w0); acc[1].y = __uint_as_float(w1);
    upk2u(ap[3], w0, w1); acc[1].z = __uint_as_float(w0); acc[1].w = __uint_as_float(w1);
}

// ---------------------------------------------------------------------------
// Heavy path: one row per CTA (256 threads).  Thread t < D ends with H[row][t].
// ring: P stages x kCH rows x D floats, then P x kCH values.
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ float heavy_spmm_row(const int32_t *__restrict__ indptr,
                                                const int32_t *__restrict__ indices,
                                                const float *__restrict__ vals,
                                                const float *__restrict__ x, int64_t row,
                                                float *ring, const int32_t *__restrict__ seg_beg = nullptr,
                                                const int32_t *__restrict__ seg_end = nullptr,
                                                float acc0 = 0.0f) {
    constexpr int P = RG<D>::P, NI = RG<D>::NI;
    constexpr int SPB = 256 / kCH;                  // stages per id block
    float *xs = ring;                               // [P][kCH][D]
    float *vs = ring + P * kCH * D;                 // [P][kCH]
    int32_t *ids = reinterpret_cast<int32_t *>(vs + P * kCH);   // [2][256]
    float *vls = reinterpret_cast<float *>(ids + 512);           // [2][256]
    const int t = threadIdx.x;
    const int32_t beg = __ldg((seg_beg ? seg_beg : indptr) + row);
    const int32_t end = seg_end ? __ldg(seg_end + row) : __ldg(indptr + row + 1);
    const int n = end - beg;
    const int nch = (n + kCH - 1) / kCH;
    auto load_block = [&](int b) {                  // ids/values of stages [b*SPB, (b+1)*SPB)
        const int k = b * 256 + t;
        if (k < n) {
            cp_async4(ids + (b & 1) * 256 + t, indices + beg + k);
            cp_async4(vls + (b & 1) * 256 + t, vals + beg + k);
        }
    };
    auto issue = [&](int c) {                       // data of stage c (ids already in smem)
        const int st = c % P;
        if (c < nch) {
            const int32_t *blk = ids + ((c / SPB) & 1) * 256 + (c % SPB) * kCH;
#pragma unroll
            for (int m = 0; m < NI; m++) {
                const int i = t + 256 * m, r = i / (D / 4), f4 = i % (D / 4);
                if (c * kCH + r < n)
                    cp_async16(xs + (st * kCH + r) * D + f4 * 4, x + (int64_t)blk[r] * D + f4 * 4);
            }
            if (t < kCH) vs[st * kCH + t] = (c * kCH + t < n) ? vls[((c / SPB) & 1) * 256 + (c % SPB) * kCH + t] : 0.0f;
        }
        cp_async_commit();
    };
    // prologue: id blocks 0 and 1, then the first P-1 stages
    load_block(0);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    load_block(1);
#pragma unroll
    for (int c = 0; c < P - 1; c++) issue(c);
    float acc = acc0;
    for (int c = 0; c < nch; c++) {
        cp_async_wait<P - 2>();
        __syncthreads();
        // chunk c+P-1 opens id block kb: block kb-1 is fully issued, so its
        // buffer takes block kb+1 (landing long before chunk 8(kb+1) issues)
        const int cn = c + P - 1;
        if (cn % SPB == 0 && cn >= SPB) load_block(cn / SPB + 1);
        const int st = c % P;
        if (t < D) {
            const int cnt = min(kCH, n - c * kCH);
            const float *xr = xs + st * kCH * D + t;
            const float *vr = vs + st * kCH;
            if (cnt == kCH) {       // full stage: all products first (independent LDS), then the chain
                float pr[kCH];
#pragma unroll
                for (int r = 0; r < kCH; r++) pr[r] = __fmul_rn(vr[r], xr[r * D]);
#pragma unroll
                for (int r = 0; r < kCH; r++) acc = __fadd_rn(acc, pr[r]);
            } else {
                for (int r = 0; r < cnt; r++) acc = __fadd_rn(acc, __fmul_rn(vr[r], xr[r * D]));
            }
        }
        __syncthreads();
        issue(cn);
    }
    cp_async_wait<0>();
    __syncthreads();
    return acc;
}

#ifndef KGQ_SPMM_MINB
#define KGQ_SPMM_MINB 3     // register cap 80; with KGQ_SPMM_BATCH 1 ptxas needs 48 (5 CTAs/SM resident)
#endif
// SEG: one source-block phase of the pipelined SpMM -- each scheduled row
// continues its ascending-column chain over its nonzeros [seg_beg, seg_end)
// from the running sums already in out (zeroed before the first phase), so
// the last phase leaves exactly the chain of the whole row.
template <int D, bool SEG = false, int BATCH = KGQ_SPMM_BATCH>
__global__ void __launch_bounds__(256, KGQ_SPMM_MINB)
spmm_kernel(const int32_t *__restrict__ indptr, const int32_t *__restrict__ indices,
            const float *__restrict__ vals, int64_t n_rows, const int32_t *__restrict__ row_order,
            int64_t n_heavy, const float *__restrict__ x, float *__restrict__ out,
            const int32_t *__restrict__ seg_beg = nullptr, const int32_t *__restrict__ seg_end = nullptr) {
    constexpr int LPR = RG<D>::LPR, RPW = RG<D>::RPW;
    extern __shared__ __align__(16) float dyn[];
    if ((int64_t)blockIdx.x < n_heavy) {
        const int64_t row = __ldg(row_order + blockIdx.x);
        const float a0 = (SEG && threadIdx.x < D) ? out[row * D + threadIdx.x] : 0.0f;
        const float h = heavy_spmm_row<D>(indptr, indices, vals, x, row, dyn, SEG ? seg_beg : nullptr,
                                          SEG ? seg_end : nullptr, a0);
        if (threadIdx.x < D) out[row * D + threadIdx.x] = h;
        return;
    }
    const int lane = threadIdx.x & 31;
    const int gl = lane % LPR, grp = lane / LPR;
    const int64_t lb = (int64_t)blockIdx.x - n_heavy;
    const int64_t nlb = (int64_t)gridDim.x - n_heavy;
    const int64_t warp = lb * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nw = nlb * (blockDim.x >> 5);
    const int64_t n_light = n_rows - n_heavy;
    const int fa = rg_f4a<D, false>(gl), fb = rg_f4b<D, false>(gl);
    for (int64_t base = warp * RPW; base < n_light; base += nw * RPW) {
        const int64_t slot = base + grp;
        const bool active = slot < n_light;
        const int64_t row = active ? (row_order ? (int64_t)__ldg(row_order + n_heavy + slot) : slot) : 0;
        float4 acc[2];
        if (SEG) {
            const float4 *o = reinterpret_cast<const float4 *>(out + row * D);
            acc[0] = active ? o[fa] : make_float4(0.f, 0.f, 0.f, 0.f);
            acc[1] = active ? o[fb] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        rg_spmm_row<D, false, BATCH>(indptr, indices, vals, x, row, active, gl, acc,
                                              SEG ? seg_beg : nullptr, SEG ? seg_end : nullptr);
        if (active) {
            float4 *o = reinterpret_cast<float4 *>(out + row * D);
            KGQ_ST_STREAM(o + fa, acc[0]);
            KGQ_ST_STREAM(o + fb, acc[1]);
        }
    }
}

// any d: warp per row, features strided by 32, same ordering.
__global__ void __launch_bounds__(256)
spmm_generic_kernel(const int32_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                    const float *__restrict__ vals, int64_t n_rows, const float *__restrict__ x,
                    int d, float *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= n_rows) return;
    const int32_t beg = indptr[row], end = indptr[row + 1];
    for (int f = lane; f < d; f += 32) {
        float acc = 0.0f;
        for (int32_t jj = beg; jj < end; jj++)
            acc = __fadd_rn(acc, __fmul_rn(vals[jj], x[(int64_t)indices[jj] * d + f]));
        out[row * d + f] = acc;
    }
}

// Quantize one light row held by its LPR-lane group (group = the row; the
// same arithmetic and noise as kgq_quantize_f32) and store codes, R, Z.
template <int D, int BITS, int MODE>
__device__ __forceinline__ void light_row_quantize(const float4 (&h)[2], bool active, int64_t row,
                                                   int gl, const FastKey &fk, uint64_t seed,
                                                   uint64_t tid, int64_t row_offset,
                                                   uint8_t *__restrict__ codes,
                                                   float *__restrict__ ranges,
                                                   float *__restrict__ offsets) {
    constexpr int LPR = RG<D>::LPR;
    constexpr float Bf = (float)((1u << BITS) - 1u);
    constexpr int RB = D * BITS / 8;
    const int p = gl >> 2, q = gl & 3;
    const int f0 = 8 * p + q;
        // ---- quantize H (group = this row) ----
    float mn = fminf(fminf(fminf(h[0].x, h[0].y), fminf(h[0].z, h[0].w)),
                     fminf(fminf(h[1].x, h[1].y), fminf(h[1].z, h[1].w)));
    float mx = fmaxf(fmaxf(fmaxf(h[0].x, h[0].y), fmaxf(h[0].z, h[0].w)),
                     fmaxf(fmaxf(h[1].x, h[1].y), fmaxf(h[1].z, h[1].w)));
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const float z = mn, r = __fsub_rn(mx, mn);
    const DivR dv = make_div(r);
    const uint64_t gglob = (uint64_t)(row_offset + row);
    uint32_t piece[2] = {0u, 0u};
    if (r > 0.0f) {
        const uint32_t kc = MODE == KGQ_ROUND_SR_FAST ? carrier_const() : 0u;
        uint4 rnd = make_uint4(0, 0, 0, 0);
        if (MODE == KGQ_ROUND_SR_FAST) rnd = fast_call(fk, gglob, (uint32_t)(4 * p + q));
        const bool unguarded = group_div_unguarded(dv, z);
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
            u64x4 r64 = {0, 0, 0, 0};
            if (MODE == KGQ_ROUND_SR_COMPAT)
                r64 = philox4x64_10(gglob * (uint64_t)(D / 4) + (uint64_t)(f0 + 4 * hh) + 1ull,
                                    0, 0, 0, seed, tid);
            const float xs[4] = {h[hh].x, h[hh].y, h[hh].z, h[hh].w};
            const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
            const uint64_t cw[4] = {r64.x, r64.y, r64.z, r64.w};
            uint32_t acc = 0;
#pragma unroll
            for (int el = 0; el < 4; el++) {
                const float a = __fsub_rn(xs[el], z);
                const float qv = unguarded ? div_a_unguarded(dv, a) : div_a(dv, a);
                const float s = __fmul_rn(qv, Bf);
                const float uf = hh ? u16_carrier_hi(rw[el], kc) : u16_carrier_lo(rw[el], kc);
                acc += code_bits<MODE>(s, uf, cw[el] >> 11) << (BITS * el);
            }
            piece[hh] = acc - magic_sum4<BITS>();
        }
    }
    // pieces: 4*BITS bits at element offsets 4*f0 and 4*(f0+4) of the row
    {
        uint8_t *rc = codes + row * RB;
        if (BITS == 1) {   // nibbles: pair lanes q, q^1 into bytes
            const uint32_t o0 = __shfl_xor_sync(0xffffffffu, piece[0], 1);
            const uint32_t o1 = __shfl_xor_sync(0xffffffffu, piece[1], 1);
            if (active && (q & 1) == 0) {
                rc[(4 * f0) / 8] = (uint8_t)(piece[0] | (o0 << 4));
                rc[(4 * (f0 + 4)) / 8] = (uint8_t)(piece[1] | (o1 << 4));
            }
        } else if (active) {
#pragma unroll
            for (int hh = 0; hh < 2; hh++) {
                const int off = (4 * (f0 + 4 * hh)) * BITS / 8;
                if (BITS == 2) rc[off] = (uint8_t)piece[hh];
                else if (BITS == 4) *reinterpret_cast<uint16_t *>(rc + off) = (uint16_t)piece[hh];
                else *reinterpret_cast<uint32_t *>(rc + off) = piece[hh];
            }
        }
    }
    if (active && gl == 0) {
        ranges[row] = r;
        offsets[row] = z;
    }
}

// Heavy row (one CTA): bit-exact SpMM streamed through the smem ring, then
// quantize / J = H.theta (FFMA, theta in smem) / relu / mask for that row.
template <int D, int BITS, int MODE>
__device__ __forceinline__ void heavy_layer_row(const int32_t *__restrict__ indptr,
                                                const int32_t *__restrict__ indices,
                                                const float *__restrict__ vals,
                                                const float *__restrict__ e, int64_t row,
                                                const float *th, float *ring, float (*red)[8],
                                                float *hrow, const FastKey &fk, uint64_t seed,
                                                uint64_t tid, int64_t row_offset,
                                                uint8_t *__restrict__ codes,
                                                float *__restrict__ ranges,
                                                float *__restrict__ offsets,
                                                float *__restrict__ e_next,
                                                uint32_t *__restrict__ mask,
                                                float *__restrict__ h_out) {
    constexpr float Bf = (float)((1u << BITS) - 1u);
    constexpr int RB = D * BITS / 8;
    constexpr int LPW = 32 / BITS;
        // ------------------------- heavy row: CTA -------------------------
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const float h = heavy_spmm_row<D>(indptr, indices, vals, e, row, ring);
    const bool own = t < D;                     // warps 0 .. D/32-1 hold the row
    if (own && h_out) h_out[row * D + t] = h;
    float mn = own ? h : INFINITY, mx = own ? h : -INFINITY;
    mn = warp_min(mn, 32);
    mx = warp_max(mx, 32);
    if (lane == 0) { red[0][wid] = mn; red[1][wid] = mx; }
    if (own) hrow[t] = h;
    __syncthreads();
    mn = red[0][0];
    mx = red[1][0];
#pragma unroll
    for (int w = 1; w < D / 32; w++) { mn = fminf(mn, red[0][w]); mx = fmaxf(mx, red[1][w]); }
    const float z = mn, r = __fsub_rn(mx, mn);
    const uint64_t gglob = (uint64_t)(row_offset + row);
    if (own) {
        uint32_t code = 0;
        if (r > 0.0f) {
            const DivR dv = make_div(r);
            const float s = __fmul_rn(div_a(dv, __fsub_rn(h, z)), Bf);
            float uf = 0.0f;
            uint64_t raw53 = 0;
            if (MODE == KGQ_ROUND_SR_FAST) uf = u16_carrier(fast_u16(fk, gglob, t));
            if (MODE == KGQ_ROUND_SR_COMPAT) raw53 = compat_raw53(seed, tid, gglob, D, t);
            code = code_bits<MODE>(s, uf, raw53) - kMagicBits;
        }
        // feature t = 32*wid + lane: word (t*BITS)/32 collects LPW lanes
        const uint32_t mine = code << ((lane % LPW) * BITS);
        const int wib = lane / LPW;
#pragma unroll
        for (int w = 0; w < 32 / LPW; w++) {
            const uint32_t word = __reduce_or_sync(0xffffffffu, wib == w ? mine : 0u);
            if (lane == w)
                reinterpret_cast<uint32_t *>(codes + row * RB)[wid * (32 / LPW) + w] = word;
        }
        if (t == 0) {
            ranges[row] = r;
            offsets[row] = z;
        }
        float j = 0.0f;
#pragma unroll 8
        for (int k = 0; k < D; k++) j = __fmaf_rn(hrow[k], th[k * D + t], j);
        const bool pos = j > 0.0f;
        const uint32_t bal = __ballot_sync(0xffffffffu, pos);
        e_next[row * D + t] = relu_nan(j);
        if (lane == 0) mask[row * (D / 32) + wid] = bal;
    }
}

// Epilogue of the light path for the warp's RPW rows (slots base..base+RPW-1
// of the schedule): quantize H (group = the row), J = H . theta (ascending k,
// FFMA), E' = relu(J), mask words.  Shared by the fused layer kernel (H from
// the SpMM registers) and the split epilogue kernel (H loaded from memory).
template <int D, int BITS, int MODE>
__device__ __forceinline__ void light_epilogue(const float4 (&h)[2], bool active, int64_t row,
                                               int64_t base, int64_t n_light,
                                               const int32_t *__restrict__ row_order, int64_t n_heavy,
                                               const float *th, float *hst, const FastKey &fk,
                                               uint64_t seed, uint64_t tid, int64_t row_offset,
                                               uint8_t *__restrict__ codes, float *__restrict__ ranges,
                                               float *__restrict__ offsets, float *__restrict__ e_next,
                                               uint32_t *__restrict__ mask) {
    constexpr int LPR = RG<D>::LPR, RPW = RG<D>::RPW;
    const int lane = threadIdx.x & 31;
    const int gl = lane % LPR, grp = lane / LPR;
    const int p = gl >> 2, q = gl & 3;
    const int f0 = 8 * p + q;
    light_row_quantize<D, BITS, MODE>(h, active, row, gl, fk, seed, tid, row_offset, codes,
                                      ranges, offsets);
        // ---- J = H . theta (ascending k, FFMA) ----
        // The warp's RPW rows are staged k-major in smem (hs[k][RPW]); lane l
        // then computes columns l + 32c of all RPW rows: per k one broadcast
        // LDS of H[.][k], D/32 conflict-free LDS of theta[k][.], 8 FFMA.
        {
            float *hs = hst + (threadIdx.x >> 5) * (D * RPW);
#pragma unroll
            for (int hh = 0; hh < 2; hh++) {
                const int k0 = 4 * (f0 + 4 * hh);
                hs[(k0 + 0) * RPW + grp] = hh ? h[1].x : h[0].x;
                hs[(k0 + 1) * RPW + grp] = hh ? h[1].y : h[0].y;
                hs[(k0 + 2) * RPW + grp] = hh ? h[1].z : h[0].z;
                hs[(k0 + 3) * RPW + grp] = hh ? h[1].w : h[0].w;
            }
            __syncwarp();
            constexpr int NCB = D / 32;
            float jacc[RPW][NCB];
#pragma unroll
            for (int rr = 0; rr < RPW; rr++)
#pragma unroll
                for (int c = 0; c < NCB; c++) jacc[rr][c] = 0.0f;
#pragma unroll 8
            for (int k = 0; k < D; k++) {
                float hk[RPW];
                if (RPW == 4) {
                    const float4 v4 = *reinterpret_cast<const float4 *>(hs + k * RPW);
                    hk[0] = v4.x; hk[1] = v4.y; hk[2] = v4.z; hk[3] = v4.w;
                } else {
#pragma unroll
                    for (int rr = 0; rr < RPW; rr++) hk[rr] = hs[k * RPW + rr];
                }
#pragma unroll
                for (int c = 0; c < NCB; c++) {
                    const float tk = th[k * D + lane + 32 * c];
#pragma unroll
                    for (int rr = 0; rr < RPW; rr++) jacc[rr][c] = __fmaf_rn(hk[rr], tk, jacc[rr][c]);
                }
            }
            // ---- relu + mask: ballot over lanes gives mask word c of row rr ----
            const int64_t base_slot = base;
#pragma unroll
            for (int rr = 0; rr < RPW; rr++) {
                const int64_t sl = base_slot + rr;
                const bool act = sl < n_light;
                const int64_t rrow = act ? (row_order ? (int64_t)__ldg(row_order + n_heavy + sl) : sl) : 0;
#pragma unroll
                for (int c = 0; c < NCB; c++) {
                    const float jv = jacc[rr][c];
                    const uint32_t bal = __ballot_sync(0xffffffffu, jv > 0.0f);
                    if (act) {
                        e_next[rrow * D + lane + 32 * c] = relu_nan(jv);
                        if (lane == 0) mask[rrow * (D / 32) + c] = bal;
                    }
                }
            }
            __syncwarp();
        }
}

// ---------------------------------------------------------------------------
// Fused layer forward: H = A_hat.E (bit-exact), quantize H on chip (group =
// d; the same arithmetic and noise as kgq_quantize_f32), J = H.theta (theta
// in smem, FFMA over ascending k), E' = relu(J), mask = J > 0.  H and J never
// reach HBM.  Dynamic smem: theta (D*D fp32) then the heavy-path ring.
// ---------------------------------------------------------------------------
template <int D, int BITS, int MODE>
__global__ void __launch_bounds__(256)
layer_forward_kernel(const int32_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                     const float *__restrict__ vals, int64_t n_rows,
                     const int32_t *__restrict__ row_order, int64_t n_heavy,
                     const float *__restrict__ e, const float *__restrict__ theta, uint64_t seed,
                     uint64_t tid, const uint64_t *__restrict__ tid_base, int64_t row_offset,
                     uint8_t *__restrict__ codes,
                     float *__restrict__ ranges, float *__restrict__ offsets,
                     float *__restrict__ e_next, uint32_t *__restrict__ mask,
                     float *__restrict__ h_out) {
    constexpr int LPR = RG<D>::LPR, RPW = RG<D>::RPW;
    extern __shared__ __align__(16) float dyn[];
    float *th = dyn;                                // [D][D]
    float *ring = dyn + D * D;                      // heavy-path staging
    __shared__ float red[2][8];
    __shared__ float hrow[D];
    __shared__ __align__(16) float hst[8 * 256];   // per-warp k-major H staging (D * RPW = 256)
    for (int i = threadIdx.x; i < D * D / 4; i += blockDim.x)
        reinterpret_cast<float4 *>(th)[i] = __ldg(reinterpret_cast<const float4 *>(theta) + i);
    __syncthreads();
    if (tid_base) tid += __ldg(tid_base);          // graph replays advance the key on device
    const FastKey fk = make_fast_key(seed, tid);

    if ((int64_t)blockIdx.x < n_heavy) {
        heavy_layer_row<D, BITS, MODE>(indptr, indices, vals, e, __ldg(row_order + blockIdx.x), th,
                                       ring, red, hrow, fk, seed, tid, row_offset, codes, ranges,
                                       offsets, e_next, mask, h_out);
        return;
    }

    // ------------------------- light rows: row groups -----------------------
    const int lane = threadIdx.x & 31;
    const int gl = lane % LPR, grp = lane / LPR;
    const int p = gl >> 2, q = gl & 3;
    const int f0 = 8 * p + q;                       // float4 index of my first four features
    const int64_t lb = (int64_t)blockIdx.x - n_heavy;
    const int64_t nlb = (int64_t)gridDim.x - n_heavy;
    const int64_t warp = lb * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nw = nlb * (blockDim.x >> 5);
    const int64_t n_light = n_rows - n_heavy;

    for (int64_t base = warp * RPW; base < n_light; base += nw * RPW) {
        const int64_t slot = base + grp;
        const bool active = slot < n_light;
        const int64_t row = active ? (row_order ? (int64_t)__ldg(row_order + n_heavy + slot) : slot) : 0;
        float4 h[2];
        rg_spmm_row<D>(indptr, indices, vals, e, row, active, gl, h);
        if (active && h_out) {
            float4 *o = reinterpret_cast<float4 *>(h_out + row * D);
            o[f0] = h[0];
            o[f0 + 4] = h[1];
        }
        light_epilogue<D, BITS, MODE>(h, active, row, base, n_light, row_order, n_heavy, th, hst, fk, seed,
                                      tid, row_offset, codes, ranges, offsets, e_next, mask);
    }
}

// Split layer forward, part 2 (after spmm_kernel wrote H).  Tiles of
// ROWS = 4096/d rows per CTA:
//  1. each warp loads RPW rows at a time in the fused kernel's lane layout
//     (LPR = d/8 lanes per row, a lane's 8 features = one fast-noise call) and
//     quantizes them with the same code (light_row_quantize), then stages H
//     k-major in smem;
//  2. J = H.theta as a register-blocked FFMA GEMM: thread (tr, tc) owns rows
//     4tr..4tr+3 x columns 4tc..4tc+3, per k one LDS.128 of H and one of theta
//     for 16 FFMA; every J element is the same ascending-k fmaf chain from 0
//     as in the fused kernel, so E_next and the mask are bit-identical;
//  3. relu, float4 stores, mask words from 8-lane nibble ORs.
template <int D>
struct EpiTile {
    static constexpr int ROWS = 4096 / D;    // 128 / 64 / 32 rows for d = 32 / 64 / 128
    static constexpr int TC = D / 4;         // column groups
    static constexpr int TR = 256 / TC;      // row groups (= ROWS / 4)
    static constexpr int RS = ROWS + 4;      // padded k-major row stride
    static constexpr size_t smem = ((size_t)D * D + (size_t)D * RS) * sizeof(float);
};

// Occupancy: plain __launch_bounds__(256) gives 64 registers (4 CTAs/SM).
// -DKGQ_EPI_MINB=n asks for n CTAs/SM at d <= 64 (fast/nearest modes): 5 is
// faster in the warm layer loop of tools/spmm_ab.py (60 vs 67 us) but not
// inside the captured training step (1.345 vs 1.332 ms); an explicit 1 lets
// ptxas take 91 registers (2 CTAs/SM) and costs the step ~3 % (1.368 ms).
#ifdef KGQ_EPI_MINB
#define KGQ_EPI_BOUNDS __launch_bounds__(256, (D <= 64 && MODE != KGQ_ROUND_SR_COMPAT) ? KGQ_EPI_MINB : 1)
#else
#define KGQ_EPI_BOUNDS __launch_bounds__(256)
#endif
template <int D, int BITS, int MODE>
__global__ void KGQ_EPI_BOUNDS
layer_epilogue_kernel(const float *hin, int64_t n_rows, const float *__restrict__ theta,
                      uint64_t seed, uint64_t tid, const uint64_t *__restrict__ tid_base,
                      int64_t row_offset, uint8_t *__restrict__ codes, float *__restrict__ ranges,
                      float *__restrict__ offsets, float *e_next,
                      uint32_t *__restrict__ mask) {
    using ET = EpiTile<D>;
    constexpr int LPR = RG<D>::LPR, RPW = RG<D>::RPW, ROWS = ET::ROWS, RS = ET::RS, TC = ET::TC;
    static_assert(ET::TR * 4 == ROWS, "tile geometry");
    extern __shared__ __align__(16) float epi_smem[];
    float *th = epi_smem;                    // [D][D]
    float *hs = epi_smem + D * D;            // [D][RS], k-major
    for (int i = threadIdx.x; i < D * D / 4; i += blockDim.x)
        reinterpret_cast<float4 *>(th)[i] = __ldg(reinterpret_cast<const float4 *>(theta) + i);
    if (tid_base) tid += __ldg(tid_base);
    const FastKey fk = make_fast_key(seed, tid);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int gl = lane % LPR, grp = lane / LPR;
    const int fa = rg_f4a<D, true>(gl), fb = rg_f4b<D, true>(gl);
    const int tc = t % TC, tr = t / TC;
    const int64_t n_tiles = (n_rows + ROWS - 1) / ROWS;
    constexpr int NP = ROWS / (8 * RPW);            // passes per tile (2)
    // register prefetch: the next pass's two float4 are in flight while the
    // current pass quantizes (and, across tiles, while the GEMM runs)
    float4 nh[2];
    auto fetch = [&](int64_t tl, int ps) {
        const int64_t rw = tl * ROWS + (ps * 8 + warp) * RPW + grp;
        if (tl < n_tiles && rw < n_rows) {
            const float4 *src = reinterpret_cast<const float4 *>(hin + rw * D);
            nh[0] = __ldcg(src + fa);       // coherent loads: E' may be written over H
            nh[1] = __ldcg(src + fb);       // (functional.EPILOGUE_IN_PLACE), tile by tile
        } else {
            nh[0] = nh[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    fetch(blockIdx.x, 0);
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t r0 = tile * ROWS;
        // ---- 1. load + quantize + stage (ROWS / (8 * RPW) = 2 passes) ----
#pragma unroll
        for (int pass = 0; pass < NP; pass++) {
            const int lr = (pass * 8 + warp) * RPW + grp;
            const int64_t row = r0 + lr;
            const bool active = row < n_rows;
            float4 h[2] = {nh[0], nh[1]};
            if (pass + 1 < NP) fetch(tile, pass + 1);
            else fetch(tile + gridDim.x, 0);
            if constexpr (BITS != 32)   // b = 32: pass-through context (H itself), nothing to quantize
            light_row_quantize<D, BITS, MODE>(h, active, active ? row : 0, gl, fk, seed, tid, row_offset,
                                              codes, ranges, offsets);
            const float hv[8] = {h[0].x, h[0].y, h[0].z, h[0].w, h[1].x, h[1].y, h[1].z, h[1].w};
#pragma unroll
            for (int e = 0; e < 4; e++) {
                hs[(4 * fa + e) * RS + lr] = hv[e];
                hs[(4 * fb + e) * RS + lr] = hv[4 + e];
            }
        }
        __syncthreads();
        // ---- 2. J tile = H . theta, ascending k ----
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) acc[i][j] = 0.0f;
#pragma unroll 8
        for (int k = 0; k < D; k++) {
            const float4 a4 = *reinterpret_cast<const float4 *>(hs + k * RS + 4 * tr);
            const float4 b4 = *reinterpret_cast<const float4 *>(th + k * D + 4 * tc);
            const float av[4] = {a4.x, a4.y, a4.z, a4.w};
            const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
        }
        // ---- 3. relu, E_next, mask (columns 32c..32c+31 = lanes with tc in [8c, 8c+8)) ----
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int64_t row = r0 + 4 * tr + i;
            uint32_t nib = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) nib |= (acc[i][j] > 0.0f ? 1u : 0u) << j;
            uint32_t word = nib << (4 * (tc & 7));
            word |= __shfl_xor_sync(0xffffffffu, word, 1);
            word |= __shfl_xor_sync(0xffffffffu, word, 2);
            word |= __shfl_xor_sync(0xffffffffu, word, 4);
            if (row < n_rows) {
                *reinterpret_cast<float4 *>(e_next + row * D + 4 * tc) =
                    make_float4(relu_nan(acc[i][0]), relu_nan(acc[i][1]), relu_nan(acc[i][2]), relu_nan(acc[i][3]));
                if ((tc & 7) == 0) mask[row * (D / 32) + (tc >> 3)] = word;
            }
        }
        __syncthreads();
    }
}


// Split layer forward, part 2 on the tensor cores (K6t, d in {32, 64}): the
// same per-row quantization as layer_epilogue_kernel (light_row_quantize, one
// LPR-lane group per row), then J = H . theta as a tcgen05 GEMM -- H split
// into TF32 hi/lo and staged in the K-major interleaved UMMA layout, theta
// staged once per CTA, 3xTF32 (hi.hi + hi.lo + lo.hi, fp32-level accuracy)
// into a TMEM accumulator of 128 lanes x D columns issued by one thread --
// and a TMEM drain that applies relu and writes the mask words; the E_next
// rows go through shared memory (the H-hi tile, free once the MMAs are done,
// rewritten in the SWIZZLE_128B box layout: conflict-free for thread = row)
// and leave as TMA tensor stores, so no thread-per-row global stores.
// J differs from the FFMA chain of the fused kernel in the last bits (another
// summation order, as OpenBLAS's differs from both): split and fused agree to
// fp32 rounding, not bitwise (tests/test_gpu_train.py).
template <int D>
struct EpiTc {
    static constexpr int M = 128;                                   // rows per tile
    static constexpr size_t smem = (size_t)(2 * M * D + 2 * D * D) * sizeof(float) + 1024;
};

template <int D, int BITS, int MODE>
__global__ void __launch_bounds__(256)
layer_epilogue_tc_kernel(const float *hin, int64_t n_rows, const float *__restrict__ theta,
                         uint64_t seed, uint64_t tid, const uint64_t *__restrict__ tid_base,
                         int64_t row_offset, uint8_t *__restrict__ codes, float *__restrict__ ranges,
                         float *__restrict__ offsets, const __grid_constant__ CUtensorMap tm_out,
                         uint32_t *__restrict__ mask) {
    constexpr int M = EpiTc<D>::M;
    constexpr int LPR = RG<D>::LPR, RPW = RG<D>::RPW;
    constexpr int NP = M / (8 * RPW);               // load/quantize passes per tile
    constexpr uint32_t TCOLS = D < 32 ? 32 : D;
    extern __shared__ uint8_t tc_smem_raw[];
    uint8_t *smb = tc_smem_raw + ((1024u - (tc::smem_u32(tc_smem_raw) & 1023u)) & 1023u);
    float *ah = reinterpret_cast<float *>(smb), *al = ah + M * D;   // H tile hi / lo [M x D]
    float *bh = ah + 2 * M * D, *bl = bh + D * D;                   // theta^T hi / lo: B(n, k) = theta[k][n]
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int gl = lane % LPR, grp = lane / LPR;
    const int fa = rg_f4a<D, true>(gl), fb = rg_f4b<D, true>(gl);

    {   // theta^T split: all loads first (one latency), then the stores
        constexpr int PER = D * D / 256;
        float tv[PER];
#pragma unroll
        for (int k = 0; k < PER; k++) {
            const int i = t + 256 * k, n = i / D, kk = i % D;
            tv[k] = __ldg(theta + kk * D + n);
        }
#pragma unroll
        for (int k = 0; k < PER; k++) {
            const int i = t + 256 * k, n = i / D, kk = i % D;
            tc::split_tf32_fast(tv[k], bh[tc::tile_off(n, kk, D) / 4], bl[tc::tile_off(n, kk, D) / 4]);
        }
    }
    if (t == 0) tc::mbar_init(&mbar, 1);
    if (warp == 0) tc::tmem_alloc(&tmem_base, TCOLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;
    if (tid_base) tid += __ldg(tid_base);
    const FastKey fk = make_fast_key(seed, tid);

    const int64_t n_tiles = (n_rows + M - 1) / M;
    float4 nh[2];
    auto fetch = [&](int64_t tl, int ps) {
        const int64_t rw = tl * M + (ps * 8 + warp) * RPW + grp;
        if (tl < n_tiles && rw < n_rows) {
            const float4 *src = reinterpret_cast<const float4 *>(hin + rw * D);
            nh[0] = __ldcg(src + fa);       // coherent loads: E' may be written over H
            nh[1] = __ldcg(src + fb);       // (functional.EPILOGUE_IN_PLACE), tile by tile
        } else {
            nh[0] = nh[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    fetch(blockIdx.x, 0);
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t r0 = tile * M;
        // the previous tile's E_next store must have finished reading the H-hi tile
        if (t == 0) tma::store_wait_read<0>();
        __syncthreads();
        // ---- 1. load + quantize + split/stage (register prefetch one pass ahead) ----
#pragma unroll
        for (int pass = 0; pass < NP; pass++) {
            const int lr = (pass * 8 + warp) * RPW + grp;
            const int64_t row = r0 + lr;
            const bool active = row < n_rows;
            float4 h[2] = {nh[0], nh[1]};
            if (pass + 1 < NP) fetch(tile, pass + 1);
            else fetch(tile + gridDim.x, 0);
            if constexpr (BITS != 32)
            light_row_quantize<D, BITS, MODE>(h, active, active ? row : 0, gl, fk, seed, tid, row_offset,
                                              codes, ranges, offsets);
#pragma unroll
            for (int hf = 0; hf < 2; hf++) {
                const float xs[4] = {h[hf].x, h[hf].y, h[hf].z, h[hf].w};
                float hi[4], lo[4];
#pragma unroll
                for (int e = 0; e < 4; e++) tc::split_tf32_fast(xs[e], hi[e], lo[e]);
                const uint32_t off = tc::tile_off(lr, 4 * (hf ? fb : fa), M) / 4;
                *reinterpret_cast<float4 *>(ah + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<float4 *>(al + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
        }
        tc::fence_proxy_async();
        __syncthreads();
        // ---- 2. J = H . theta on the tensor cores ----
        if (t == 0) {
            tc::fence_after();
            tc::mma_3xtf32<M, D, D>(tmem, ah, al, bh, bl);
            tc::commit(&mbar);
        }
        tc::mbar_wait(&mbar, phase);
        phase ^= 1u;
        tc::fence_after();
        // ---- 3. drain: warp w -> TMEM lanes 32*(w%4).. (its rows), columns 32*(w/4)..;
        //         relu into the E_next box stage (the H-hi tile), mask words ----
        if (warp < 4 * (D / 32)) {
            const int q = warp & 3, cb = 32 * (warp >> 2);
            float v[32];
            tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)cb, v);
            const int rr = 32 * q + lane;
            const int64_t row = r0 + rr;
            uint32_t word = 0;
#pragma unroll
            for (int c = 0; c < 32; c++) {
                word |= (v[c] > 0.0f ? 1u : 0u) << c;
                v[c] = relu_nan(v[c]);
            }
            uint8_t *box = reinterpret_cast<uint8_t *>(ah) + (cb >> 5) * (M * 128);
#pragma unroll
            for (int j = 0; j < 8; j++)
                *reinterpret_cast<float4 *>(box + tma::box_off(rr, 4 * j)) =
                    make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            if (row < n_rows) mask[row * (D / 32) + (cb >> 5)] = word;
        }
        tc::fence_before();
        tc::fence_proxy_async();
        __syncthreads();
        if (t == 0) {
#pragma unroll
            for (int cb = 0; cb < D; cb += 32)
                tma::store_2d(&tm_out, reinterpret_cast<uint8_t *>(ah) + (cb >> 5) * (M * 128), cb, (int)r0);
            tma::store_commit();
        }
    }
    if (t == 0) tma::store_wait<0>();
    __syncthreads();
    if (warp == 0) tc::tmem_free(tmem, TCOLS);
}



// K6t at d = 64, thread = row (`layer_epilogue_tc64_kernel`): persistent CTA,
// warp-specialized -- warp 0 streams H tiles (128 rows x 64 fp32, two
// SWIZZLE_128B boxes) by TMA through a 3-stage ring; warp 1 issues J = H .
// theta (3xTF32: 3 passes x 8 kind::tf32 MMAs, M = 128, N = 64, A = H hi|lo
// from TMEM, B = theta^T split in smem); two sets of 4 row warps (set s takes
// tiles j = s mod 2, so one set quantizes while the other waits for its MMAs)
// where thread = row = TMEM lane: it reads its row from the stage
// (conflict-free through the swizzle), quantizes it whole in registers -- the
// same arithmetic and the same fast-noise words per element as
// light_row_quantize / K1 (element k: call 4(k>>5) + ((k>>2)&3), word k&3,
// half (k>>4)&1), so codes and R/Z are bit-identical -- writes its 16-byte code
// row and R/Z, puts H hi|lo into TMEM (tcgen05.st) and, once the MMAs are
// done, drains J: relu, the two mask words, E' into the set's box stage for a
// TMA tensor store.  No shuffles, no cross-lane reductions, no thread-per-row
// global loads or stores.

// The rare exact path of layer_epilogue_tc64_kernel: one row's codes with the
// checked division (div_a), x re-read from the SWIZZLE_128B stage.
template <int BITS, int MODE, int D = 64, int C0 = 0, int NC = 8>
__device__ __noinline__ void tc64_row_codes_exact(const uint8_t *hst, int r, float z, DivR dv, FastKey fk,
                                                 uint64_t gglob, uint64_t seed, uint64_t tid, uint32_t *cw) {
    // calls [C0, C0 + NC) -> code words [(C0 / 4) BITS, ...) of the row, written from cw[0]
    constexpr int NW = NC * BITS / 4, W0 = (C0 / 4) * BITS;
    constexpr float Bf = (float)((1u << BITS) - 1u);
    const uint32_t kc = MODE == KGQ_ROUND_SR_FAST ? carrier_const() : 0u;
    for (int w = 0; w < NW; w++) cw[w] = 0u;
#pragma unroll 1
    for (int c = C0; c < C0 + NC; c++) {
        uint4 rnd = make_uint4(0, 0, 0, 0);
        if (MODE == KGQ_ROUND_SR_FAST) rnd = fast_call(fk, gglob, (uint32_t)c);
        const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
#pragma unroll 1
        for (int h = 0; h < 2; h++) {
            const int k0 = 32 * (c >> 2) + 4 * (c & 3) + 16 * h;
            u64x4 r64 = {0, 0, 0, 0};
            if (MODE == KGQ_ROUND_SR_COMPAT)
                r64 = philox4x64_10(gglob * (uint64_t)(D / 4) + (uint64_t)(k0 >> 2) + 1ull, 0, 0, 0, seed, tid);
            const uint64_t cw64[4] = {r64.x, r64.y, r64.z, r64.w};
            const float4 v = *reinterpret_cast<const float4 *>(hst + (k0 >> 5) * (128 * 128) + tma::box_off(r, k0 & 31));
            const float xs[4] = {v.x, v.y, v.z, v.w};
            uint32_t acc = 0;
#pragma unroll
            for (int el = 0; el < 4; el++) {
                const float sv = __fmul_rn(div_a(dv, __fsub_rn(xs[el], z)), Bf);
                const float uf = h ? u16_carrier_hi(rw[el], kc) : u16_carrier_lo(rw[el], kc);
                acc += code_bits<MODE>(sv, uf, cw64[el] >> 11) << (BITS * el);
            }
            const int bit = k0 * BITS;
            cw[(bit >> 5) - W0] |= (acc - magic_sum4<BITS>()) << (bit & 31);
        }
    }
}

constexpr int kE2Stages = 3;
constexpr int kE2Threads = 320;             // TMA warp, MMA warp, 2 x 4 row warps
struct Epi64Smem {
    static constexpr uint32_t TH = 64 * 64 * 4;          // theta^T hi or lo (16 KB)
    static constexpr uint32_t HS = 128 * 64 * 4;         // one H tile (32 KB)
    static constexpr uint32_t ES = 128 * 64 * 4;         // one E' tile stage (32 KB)
    static constexpr uint32_t RING = 2 * TH;
    static constexpr uint32_t EST = RING + kE2Stages * HS;
    static constexpr uint32_t BAR = EST + 2 * ES;
    static constexpr size_t bytes = (size_t)BAR + 128 + 1024;
};
// TMEM: A (H hi | lo) of set s at 128 s, J of set s at 256 + 64 s
constexpr uint32_t kE2A = 0, kE2J = 256;

template <int BITS, int MODE>
__global__ void __launch_bounds__(kE2Threads, 1)
layer_epilogue_tc64_kernel(const __grid_constant__ CUtensorMap tm_h, int64_t n_rows, const float *__restrict__ theta,
                           uint64_t seed, uint64_t tid, const uint64_t *__restrict__ tid_base, int64_t row_offset,
                           uint8_t *__restrict__ codes, float *__restrict__ ranges, float *__restrict__ offsets,
                           const __grid_constant__ CUtensorMap tm_out, uint32_t *__restrict__ mask) {
    constexpr int D = 64, M = 128, RB = D * BITS / 8;
    constexpr int NW = BITS >= 32 ? 1 : 2 * BITS;                 // 32-bit code words per row
    constexpr float Bf = (float)((1u << (BITS < 32 ? BITS : 1)) - 1u);
    using S = Epi64Smem;
    extern __shared__ uint8_t e2_raw[];
    uint8_t *sm = e2_raw + ((1024u - (tc::smem_u32(e2_raw) & 1023u)) & 1023u);
    float *thh = reinterpret_cast<float *>(sm), *thl = reinterpret_cast<float *>(sm + S::TH);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S::BAR);
    uint64_t *hfull = bar, *hempty = bar + kE2Stages, *afull = bar + 2 * kE2Stages, *dfull = afull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(dfull + 2);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    // theta^T split (B of J = H . theta): B(n, k) = theta[k][n], K-major SWIZZLE_128B
    {
        constexpr int PER = (D * D + kE2Threads - 1) / kE2Threads;
        float tv[PER];
#pragma unroll
        for (int k = 0; k < PER; k++) {                 // coalesced: i = kk * D + n -> B(n, kk)
            const int i = t + kE2Threads * k;
            tv[k] = i < D * D ? __ldg(theta + i) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < PER; k++) {
            const int i = t + kE2Threads * k;
            if (i < D * D) {
                const uint32_t o = tc::sw128_off(i % D, i / D, D) / 4;
                tc::split_tf32_fast(tv[k], thh[o], thl[o]);
            }
        }
    }
    if (t == 0) {
        for (int i = 0; i < kE2Stages; i++) { tc::mbar_init(hfull + i, 1); tc::mbar_init(hempty + i, 128); }
        for (int i = 0; i < 2; i++) { tc::mbar_init(afull + i, 128); tc::mbar_init(dfull + i, 1); }
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t n_tiles = (n_rows + M - 1) / M;
    const int nj = (int)((n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);   // >= 1 (grid <= n_tiles)
    auto tile_of = [&](int j) { return (int64_t)blockIdx.x + (int64_t)j * gridDim.x; };

    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------
        if (lane == 0) {
            for (int j = 0; j < nj; j++) {
                const int st = j % kE2Stages;
                if (j >= kE2Stages) tc::mbar_wait_sleep(hempty + st, (uint32_t)((j / kE2Stages - 1) & 1));
                uint8_t *dst = sm + S::RING + st * S::HS;
                tma::expect_tx(hfull + st, S::HS);
                const int r0 = (int)(tile_of(j) * M);
                tma::load_2d(dst, &tm_h, 0, r0, hfull + st);
                tma::load_2d(dst + S::HS / 2, &tm_h, 32, r0, hfull + st);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------ MMA issuer ------------------------------
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_tf32(M, D);
            const uint32_t bh = tc::smem_u32(thh), bl = tc::smem_u32(thl);
            for (int j = 0; j < nj; j++) {
                const int s = j & 1;
                tc::mbar_wait(afull + s, (uint32_t)((j >> 1) & 1));
                tc::fence_after();
                const uint32_t ab = tmem + kE2A + 128u * s, dd = tmem + kE2J + 64u * s;
#pragma unroll
                for (int p = 0; p < 3; p++) {          // lo.hi, hi.lo, hi.hi
                    const uint32_t ao = p == 0 ? 64u : 0u;
                    const uint32_t bs = p == 1 ? bl : bh;
#pragma unroll
                    for (int ks = 0; ks < D / 8; ks++)
                        tc::mma_tf32_ts(dd, ab + ao + 8u * ks, tc::kmajor_sw128_desc(bs, ks, D), idesc, (p | ks) != 0);
                }
                tc::commit(dfull + s);
            }
        }
        __syncwarp();
    } else {
        // --------------------------- row warps (thread = row) ---------------------------
        const int s = (warp - 2) >> 2, q = warp & 3;
        const int r = 32 * q + lane;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        uint8_t *estage = sm + S::EST + s * S::ES;
        if (tid_base) tid += __ldg(tid_base);
        const FastKey fk = make_fast_key(seed, tid);
        const bool leader = q == 0 && lane == 0;
        for (int j = s; j < nj; j += 2) {
            const int st = j % kE2Stages;
            const int64_t row = tile_of(j) * M + r;
            const bool active = row < n_rows;
            tc::mbar_wait(hfull + st, (uint32_t)((j / kE2Stages) & 1));
            float x[D];
            const uint8_t *hst = sm + S::RING + st * S::HS;
#pragma unroll
            for (int c4 = 0; c4 < D / 4; c4++) {
                const float4 v = *reinterpret_cast<const float4 *>(hst + (c4 >> 3) * (S::HS / 2) + tma::box_off(r, 4 * c4));
                x[4 * c4] = v.x; x[4 * c4 + 1] = v.y; x[4 * c4 + 2] = v.z; x[4 * c4 + 3] = v.w;
            }
            // ---- H hi | lo into TMEM (A of J), first, so the MMAs run while the row is quantized ----
            {
                const uint32_t ta = tmem + lane_addr + kE2A + 128u * s;
#pragma unroll
                for (int cb = 0; cb < D; cb += 8) {
                    float hi[8], lo[8];
#pragma unroll
                    for (int e = 0; e < 8; e++) tc::split_tf32_fast(x[cb + e], hi[e], lo[e]);
                    tc::tmem_st8(ta + (uint32_t)cb, hi);
                    tc::tmem_st8(ta + 64u + (uint32_t)cb, lo);
                }
                tc::tmem_st_wait();
                tc::fence_before();
                tc::mbar_arrive(afull + s);
            }
            if constexpr (BITS != 32) {
                // ---- quantize the row (light_row_quantize's arithmetic and noise) ----
                // min / max as a tree (exact, order-free); the division as the
                // Markstein fast path for every element with a per-row flag for
                // the rare elements outside its window, which then redo the row
                // with the checked division (no per-element branch)
                float mn4[4], mx4[4];                 // four interleaved chains
#pragma unroll
                for (int u = 0; u < 4; u++) { mn4[u] = x[u]; mx4[u] = x[u]; }
#pragma unroll
                for (int k = 4; k < D; k++) { mn4[k & 3] = fminf(mn4[k & 3], x[k]); mx4[k & 3] = fmaxf(mx4[k & 3], x[k]); }
                const float z = fminf(fminf(mn4[0], mn4[1]), fminf(mn4[2], mn4[3]));
                const float rr = __fsub_rn(fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])), z);
                const DivR dv = make_div(rr);
                const uint64_t gglob = (uint64_t)(row_offset + row);
                uint32_t cw[NW];
#pragma unroll
                for (int w = 0; w < NW; w++) cw[w] = 0u;
                if (rr > 0.0f) {
                    bool slow = !dv.fast;
                    const uint32_t kc = MODE == KGQ_ROUND_SR_FAST ? carrier_const() : 0u;
#pragma unroll
                    for (int c = 0; c < 8; c++) {           // fast-noise call c: elements 32(c>>2) + 4(c&3) + w + 16h
                        uint4 rnd = make_uint4(0, 0, 0, 0);
                        if (MODE == KGQ_ROUND_SR_FAST) rnd = fast_call(fk, gglob, (uint32_t)c);
                        const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            const int k0 = 32 * (c >> 2) + 4 * (c & 3) + 16 * h;      // 4 consecutive elements
                            u64x4 r64 = {0, 0, 0, 0};
                            if (MODE == KGQ_ROUND_SR_COMPAT)
                                r64 = philox4x64_10(gglob * (uint64_t)(D / 4) + (uint64_t)(k0 >> 2) + 1ull, 0, 0, 0,
                                                    seed, tid);
                            const uint64_t cw64[4] = {r64.x, r64.y, r64.z, r64.w};
                            uint32_t acc = 0;
#pragma unroll
                            for (int el = 0; el < 4; el++) {
                                const float a = __fsub_rn(x[k0 + el], z);
                                slow |= (__float_as_uint(a) - 1u) < dv.thr_m1;      // 0 < a < threshold
                                const float sv = __fmul_rn(div_a_unguarded(dv, a), Bf);
                                const float uf = h ? u16_carrier_hi(rw[el], kc) : u16_carrier_lo(rw[el], kc);
                                acc += code_bits<MODE>(sv, uf, cw64[el] >> 11) << (BITS * el);
                            }
                            const uint32_t piece = acc - magic_sum4<BITS>();
                            const int bit = k0 * BITS;
                            cw[bit >> 5] |= piece << (bit & 31);
                        }
                    }
                    // rare: an element outside the Markstein window -> the row again with the
                    // checked division (x re-read from the stage, one element at a time)
                    if (slow)
                        tc64_row_codes_exact<BITS, MODE>(hst, r, z, dv, fk, gglob, seed, tid, cw);
                }
                if (active) {
                    uint32_t *crow = reinterpret_cast<uint32_t *>(codes + row * RB);
                    if constexpr (NW % 4 == 0) {
#pragma unroll
                        for (int w = 0; w < NW; w += 4)
                            *reinterpret_cast<uint4 *>(crow + w) = make_uint4(cw[w], cw[w + 1], cw[w + 2], cw[w + 3]);
                    } else {
#pragma unroll
                        for (int w = 0; w < NW; w++) crow[w] = cw[w];
                    }
                    ranges[row] = rr;
                    offsets[row] = z;
                }
            }
            tc::mbar_arrive(hempty + st);                 // the stage is no longer read
            // ---- drain J: relu, mask words, E' into the box stage ----
            if (leader) tma::store_wait_read<0>();          // previous tile's E' store has read the stage
            tma::named_sync(1 + s, 128);
            tc::mbar_wait(dfull + s, (uint32_t)((j >> 1) & 1));
            tc::fence_after();
#pragma unroll
            for (int cb = 0; cb < D; cb += 32) {
                float v[32];
                tc::tmem_ld32(tmem + lane_addr + kE2J + 64u * s + (uint32_t)cb, v);
                uint32_t word = 0;
#pragma unroll
                for (int c = 0; c < 32; c++) {
                    word |= (v[c] > 0.0f ? 1u : 0u) << c;
                    v[c] = relu_nan(v[c]);
                }
                uint8_t *box = estage + (cb >> 5) * (M * 128);
#pragma unroll
                for (int e = 0; e < 8; e++)
                    *reinterpret_cast<float4 *>(box + tma::box_off(r, 4 * e)) =
                        make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
                if (active) mask[row * (D / 32) + (cb >> 5)] = word;
            }
            tc::fence_before();
            tc::fence_proxy_async();
            tma::named_sync(1 + s, 128);
            if (leader) {
                tma::store_2d(&tm_out, estage, 0, (int)(tile_of(j) * M));
                tma::store_2d(&tm_out, estage + M * 128, 32, (int)(tile_of(j) * M));
                tma::store_commit();
            }
        }
        if (leader) tma::store_wait<0>();
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_free(tmem, 512);
}

}  // namespace kgq

using namespace kgq;

#ifndef KGQ_SPMM_BATCH_BIG
#define KGQ_SPMM_BATCH_BIG 2
#endif
// The gathered table is taken to be HBM-resident when the output block alone
// exceeds 96 MB (the table is at least the block); KGQ_SPMM_BIG=0/1 forces
// the choice (read once).
static bool spmm_big_table(int64_t n_rows, int d) {
    static int force = -2;
    if (force == -2) {
        const char *e = getenv("KGQ_SPMM_BIG");
        force = e ? (e[0] == '1' ? 1 : 0) : -1;
    }
    if (force >= 0) return force == 1;
    return n_rows * (int64_t)d * 4 > ((int64_t)96 << 20);
}

static inline int light_blocks(int64_t n_light, int rpw, int per_sm) {
    int64_t warps = (n_light + rpw - 1) / rpw;
    int64_t b = (warps + 7) / 8;
    const int64_t cap = (int64_t)kSMs * per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

template <typename K>
static cudaError_t ensure_smem(K kern, size_t smem) {
    if (smem <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int D, bool SEG = false>
static int launch_spmm(const int32_t *indptr, const int32_t *indices, const float *vals,
                       int64_t n_rows, const int32_t *row_order, int64_t n_heavy, const float *x,
                       float *out, cudaStream_t s, const int32_t *seg_beg = nullptr,
                       const int32_t *seg_end = nullptr) {
    const size_t smem = n_heavy ? RG<D>::ring_bytes : 0;
    static size_t smem_set = 0, smem_set_big = 0;
    const int grid = (int)n_heavy + light_blocks(n_rows - n_heavy, RG<D>::RPW, 16);
    if (spmm_big_table(n_rows, D)) {
        // gathered rows come from HBM, not L2: keep more neighbour rows in
        // flight per row group (Little's law on the DRAM latency)
        if (smem > smem_set_big) {
            cudaError_t ea = ensure_smem(spmm_kernel<D, SEG, KGQ_SPMM_BATCH_BIG>, smem);
            if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
            smem_set_big = smem;
        }
        spmm_kernel<D, SEG, KGQ_SPMM_BATCH_BIG><<<grid, 256, smem, s>>>(indptr, indices, vals, n_rows, row_order,
                                                                       n_heavy, x, out, seg_beg, seg_end);
        return KGQ_OK;
    }
    if (smem > smem_set) {
        cudaError_t ea = ensure_smem(spmm_kernel<D, SEG>, smem);
        if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
        smem_set = smem;
    }
    spmm_kernel<D, SEG><<<grid, 256, smem, s>>>(indptr, indices, vals, n_rows, row_order, n_heavy, x, out,
                                                seg_beg, seg_end);
    return KGQ_OK;
}

extern "C" int kgq_spmm_csr_seg_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                                    int64_t n_slots, const int32_t *row_order, int64_t n_heavy,
                                    const int32_t *seg_beg, const int32_t *seg_end, const float *x, int32_t d,
                                    float *out, void *stream) {
    if (n_slots < 0 || n_heavy < 0 || n_heavy > n_slots) return KGQ_ERR_INVALID_ARG;
    if (n_slots == 0) return KGQ_OK;
    if (!indptr || !indices || !vals || !row_order || !seg_beg || !seg_end || !x || !out) return KGQ_ERR_INVALID_ARG;
    if ((((uintptr_t)x) | ((uintptr_t)out)) & 15u) return KGQ_ERR_MISALIGNED;
    cudaStream_t s = (cudaStream_t)stream;
    int st;
    if (d == 32) st = launch_spmm<32, true>(indptr, indices, vals, n_slots, row_order, n_heavy, x, out, s, seg_beg, seg_end);
    else if (d == 64) st = launch_spmm<64, true>(indptr, indices, vals, n_slots, row_order, n_heavy, x, out, s, seg_beg, seg_end);
    else if (d == 128) st = launch_spmm<128, true>(indptr, indices, vals, n_slots, row_order, n_heavy, x, out, s, seg_beg, seg_end);
    else return KGQ_ERR_INVALID_ARG;
    if (st != KGQ_OK) return st;
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_spmm_csr_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                                int64_t n_rows, const int32_t *row_order, int64_t n_heavy,
                                const float *x, int32_t d, float *out, void *stream) {
    if (n_rows < 0 || d < 1 || n_heavy < 0 || n_heavy > n_rows) return KGQ_ERR_INVALID_ARG;
    if (n_heavy && !row_order) return KGQ_ERR_INVALID_ARG;
    if (n_rows == 0) return KGQ_OK;
    if (!indptr || !out || !x) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const bool vec = ((((uintptr_t)x) | ((uintptr_t)out)) & 15u) == 0;
    int st = KGQ_OK;
    if (vec && d == 32) st = launch_spmm<32>(indptr, indices, vals, n_rows, row_order, n_heavy, x, out, s);
    else if (vec && d == 64) st = launch_spmm<64>(indptr, indices, vals, n_rows, row_order, n_heavy, x, out, s);
    else if (vec && d == 128) st = launch_spmm<128>(indptr, indices, vals, n_rows, row_order, n_heavy, x, out, s);
    else {
        int64_t b = (n_rows + 7) / 8;
        spmm_generic_kernel<<<(int)(b < 0x7fffffff ? b : 0x7fffffff), 256, 0, s>>>(indptr, indices, vals, n_rows, x, d, out);
    }
    if (st != KGQ_OK) return st;
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

template <int D, int BITS>
static int launch_layer(int rounding, const int32_t *indptr, const int32_t *indices, const float *vals,
                        int64_t n_rows, const int32_t *row_order, int64_t n_heavy, const float *e,
                        const float *theta, uint64_t seed, uint64_t tid, const uint64_t *tid_base,
                        int64_t row_offset, uint8_t *codes, float *ranges, float *offsets,
                        float *e_next, uint32_t *mask, float *h_out, cudaStream_t s) {
    const size_t smem = (size_t)D * D * sizeof(float) + (n_heavy ? RG<D>::ring_bytes : 0);
    void (*kern)(const int32_t *, const int32_t *, const float *, int64_t, const int32_t *, int64_t,
                 const float *, const float *, uint64_t, uint64_t, const uint64_t *, int64_t,
                 uint8_t *, float *, float *, float *, uint32_t *, float *);
    switch (rounding) {
        case KGQ_ROUND_NEAREST: kern = layer_forward_kernel<D, BITS, KGQ_ROUND_NEAREST>; break;
        case KGQ_ROUND_SR_FAST: kern = layer_forward_kernel<D, BITS, KGQ_ROUND_SR_FAST>; break;
        case KGQ_ROUND_SR_COMPAT: kern = layer_forward_kernel<D, BITS, KGQ_ROUND_SR_COMPAT>; break;
        default: return KGQ_ERR_INVALID_ARG;
    }
    static size_t smem_set[3] = {0, 0, 0};   // per instance: largest attribute already set
    if (smem > smem_set[rounding]) {
        cudaError_t ea = ensure_smem(kern, smem);
        if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
        smem_set[rounding] = smem;
    }
    const int grid = (int)n_heavy + light_blocks(n_rows - n_heavy, RG<D>::RPW, 8);
    kern<<<grid, 256, smem, s>>>(indptr, indices, vals, n_rows, row_order, n_heavy, e, theta, seed,
                                 tid, tid_base, row_offset, codes, ranges, offsets, e_next, mask, h_out);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

// K6t (tcgen05 J) is the default for d in {32, 64}; KGQ_EPI_FFMA=1 in the
// environment selects the FFMA epilogue (bit-identical to the fused kernel).
static bool epi_use_tc(int d) {
    const char *e = getenv("KGQ_EPI_FFMA");      // read per launch (host side, cheap)
    return !(e && e[0] == '1') && (d == 32 || d == 64 || d == 128);
}


template <int BITS>
static int launch_epilogue_tc64(int rounding, const float *h, int64_t n_rows, const float *theta, uint64_t seed,
                                uint64_t tid, const uint64_t *tid_base, int64_t row_offset, uint8_t *codes,
                                float *ranges, float *offsets, float *e_next, uint32_t *mask, cudaStream_t s) {
    void (*kern)(const CUtensorMap, int64_t, const float *, uint64_t, uint64_t, const uint64_t *, int64_t,
                 uint8_t *, float *, float *, const CUtensorMap, uint32_t *);
    switch (rounding) {
        case KGQ_ROUND_NEAREST: kern = layer_epilogue_tc64_kernel<BITS, KGQ_ROUND_NEAREST>; break;
        case KGQ_ROUND_SR_FAST: kern = layer_epilogue_tc64_kernel<BITS, KGQ_ROUND_SR_FAST>; break;
        case KGQ_ROUND_SR_COMPAT: kern = layer_epilogue_tc64_kernel<BITS, KGQ_ROUND_SR_COMPAT>; break;
        default: return KGQ_ERR_INVALID_ARG;
    }
    static bool smem_set[3] = {false, false, false};
    if (!smem_set[rounding]) {
        cudaError_t ea = ensure_smem(kern, Epi64Smem::bytes);
        if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
        smem_set[rounding] = true;
    }
    CUtensorMap tm_h, tm_out;
    if (!tma::make_rowmajor_f32(&tm_h, h, (uint64_t)n_rows, 64, 128) ||
        !tma::make_rowmajor_f32(&tm_out, e_next, (uint64_t)n_rows, 64, 128))
        return KGQ_ERR_CUDA;
    const int64_t tiles = (n_rows + 127) / 128;
    const int grid = (int)(tiles < kSMs ? tiles : kSMs);
    kern<<<grid, kE2Threads, Epi64Smem::bytes, s>>>(tm_h, n_rows, theta, seed, tid, tid_base, row_offset, codes,
                                                    ranges, offsets, tm_out, mask);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}


// K6t at d = 128 (`layer_epilogue_tc128_kernel`).  theta^T (hi | lo) cannot
// sit in smem beside the tiles (128 KB), so J is computed transposed,
// J^T = theta^T . H^T, with theta^T hi | lo as the TMEM A operand (loaded once
// per CTA, lane = output column n) and H itself as the B operand: the TMA
// stage (two 64 KB... four 128-row x 32-column SWIZZLE_128B boxes) *is* a
// K-major SW128 operand, read as hi by the MMA (kind::tf32 ignores the low
// mantissa bits), so only H_lo = H - trunc_tf32(H) is written, by the row
// warps.  3 passes (theta_lo.H, theta_hi.H_lo, theta_hi.H) x 16 K steps, M =
// 128 (n), N = 128 (rows), into one of two TMEM accumulators.
// Warps: 0 TMA, 1 MMA, 2-9 row warps (thread = row: min / max in a first pass
// over the stage, then the quantization of the row -- same arithmetic and
// noise words as light_row_quantize / K1 -- streaming float4s from the stage,
// and H_lo), 6-9 drain warps (thread = output column n: each tcgen05.ld gives
// 32 rows of J for that column; relu; the mask words by ballot over the 32
// columns of the warp; E' rows stored 128 B per warp instruction).
constexpr int kE8Threads = 448;
struct Epi128Smem {
    static constexpr uint32_t HS = 128 * 128 * 4;        // one H tile (64 KB): 4 boxes of 16 KB
    static constexpr uint32_t LO = 2 * HS;               // H_lo (64 KB) after the 2-stage ring
    static constexpr uint32_t BAR = 3 * HS;
    static constexpr size_t bytes = (size_t)BAR + 96 + 2 * 512 * 4 + 1024;
};
constexpr uint32_t kE8Th = 0, kE8J = 256;             // TMEM: theta^T hi [0,128) lo [128,256); J^T 2 x 128

template <int BITS, int MODE>
__global__ void __launch_bounds__(kE8Threads, 1)
layer_epilogue_tc128_kernel(const __grid_constant__ CUtensorMap tm_h, int64_t n_rows, const float *__restrict__ theta,
                            uint64_t seed, uint64_t tid, const uint64_t *__restrict__ tid_base, int64_t row_offset,
                            uint8_t *__restrict__ codes, float *__restrict__ ranges, float *__restrict__ offsets,
                            float *__restrict__ e_next, uint32_t *__restrict__ mask) {
    constexpr int D = 128, M = 128, RB = D * BITS / 8;
    constexpr int NW = BITS >= 32 ? 1 : 4 * BITS;                 // 32-bit code words per row
    constexpr float Bf = (float)((1u << (BITS < 32 ? BITS : 1)) - 1u);
    using S = Epi128Smem;
    extern __shared__ uint8_t e8_raw[];
    uint8_t *sm = e8_raw + ((1024u - (tc::smem_u32(e8_raw) & 1023u)) & 1023u);
    uint8_t *lo_buf = sm + S::LO;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S::BAR);
    uint64_t *hfull = bar, *hempty = bar + 2, *lofull = bar + 4, *loempty = bar + 5, *jfull = bar + 6, *jempty = bar + 8;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 10);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t == 0) {
        for (int i = 0; i < 2; i++) { tc::mbar_init(hfull + i, 1); tc::mbar_init(hempty + i, 1); }
        tc::mbar_init(lofull, 256);
        tc::mbar_init(loempty, 1);
        for (int i = 0; i < 2; i++) { tc::mbar_init(jfull + i, 1); tc::mbar_init(jempty + i, 128); }
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    // theta^T hi | lo into TMEM: lane n holds A(n, k) = theta[k][n], k = 0..127
    if (warp >= 2 && warp < 10) {                    // 8 warps: lane quadrant warp % 4, k half (warp - 2) / 4
        const int n = 32 * (warp & 3) + lane, k0 = 64 * ((warp - 2) >> 2);
        const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + kE8Th + (uint32_t)k0;
        float tv[64];                                // all loads in flight at once (L2 latency once)
#pragma unroll
        for (int e = 0; e < 64; e++) tv[e] = __ldg(theta + (k0 + e) * D + n);
#pragma unroll
        for (int kb = 0; kb < 64; kb += 8) {
            float hi[8], lo[8];
#pragma unroll
            for (int e = 0; e < 8; e++) tc::split_tf32_fast(tv[kb + e], hi[e], lo[e]);
            tc::tmem_st8(ta + (uint32_t)kb, hi);
            tc::tmem_st8(ta + 128u + (uint32_t)kb, lo);
        }
        tc::tmem_st_wait();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const int64_t n_tiles = (n_rows + M - 1) / M;
    const int nj = (int)((n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);   // >= 1 (grid <= n_tiles)
    auto tile_of = [&](int j) { return (int64_t)blockIdx.x + (int64_t)j * gridDim.x; };

    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------
        if (lane == 0) {
            for (int j = 0; j < nj; j++) {
                const int st = j & 1;
                if (j >= 2) tc::mbar_wait_sleep(hempty + st, (uint32_t)(((j >> 1) - 1) & 1));
                uint8_t *dst = sm + st * S::HS;
                tma::expect_tx(hfull + st, S::HS);
                const int r0 = (int)(tile_of(j) * M);
#pragma unroll
                for (int bx = 0; bx < 4; bx++) tma::load_2d(dst + bx * (S::HS / 4), &tm_h, 32 * bx, r0, hfull + st);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------ MMA issuer ------------------------------
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_tf32(128, 128);
            const uint32_t lob = tc::smem_u32(lo_buf);
            for (int j = 0; j < nj; j++) {
                const int st = j & 1, b = j & 1;
                tc::mbar_wait(hfull + st, (uint32_t)((j >> 1) & 1));
                tc::mbar_wait(lofull, (uint32_t)(j & 1));
                if (j >= 2) tc::mbar_wait(jempty + b, (uint32_t)(((j >> 1) - 1) & 1));
                tc::fence_after();
                const uint32_t hb = tc::smem_u32(sm + st * S::HS);
                const uint32_t dd = tmem + kE8J + 128u * b;
#pragma unroll
                for (int p = 0; p < 3; p++) {                 // theta_lo.H, theta_hi.H_lo, theta_hi.H
                    const uint32_t ta = tmem + kE8Th + (p == 0 ? 128u : 0u);
                    const uint32_t bsrc = p == 1 ? lob : hb;
#pragma unroll
                    for (int ks = 0; ks < D / 8; ks++)
                        tc::mma_tf32_ts(dd, ta + 8u * ks, tc::kmajor_sw128_desc(bsrc, ks, M), idesc, (p | ks) != 0);
                }
                tc::commit(hempty + st);
                tc::commit(loempty);
                tc::commit(jfull + b);
            }
        }
        __syncwarp();
    } else if (warp < 10) {
        // ------------------- row warps (thread = half a row: 64 columns) -------------------
        const int q = warp & 3, half = (warp - 2) >> 2, r = 32 * q + lane;
        constexpr int HW = NW / 2 > 0 ? NW / 2 : 1;                     // code words per half row
        float *mm = reinterpret_cast<float *>(bar + 12);               // [2 parity][2 half][2 min|max][128]
        if (tid_base) tid += __ldg(tid_base);
        const FastKey fk = make_fast_key(seed, tid);
        for (int j = 0; j < nj; j++) {
            const int st = j & 1;
            const int64_t row = tile_of(j) * M + r;
            const bool active = row < n_rows;
            tc::mbar_wait(hfull + st, (uint32_t)((j >> 1) & 1));
            const uint8_t *hst = sm + st * S::HS;
            float x[64];
#pragma unroll
            for (int c4 = 0; c4 < 16; c4++) {
                const int k = 64 * half + 4 * c4;
                const float4 v = *reinterpret_cast<const float4 *>(hst + (k >> 5) * (S::HS / 4) + tma::box_off(r, k & 31));
                x[4 * c4] = v.x; x[4 * c4 + 1] = v.y; x[4 * c4 + 2] = v.z; x[4 * c4 + 3] = v.w;
            }
            if (j >= 1) tc::mbar_wait(loempty, (uint32_t)((j - 1) & 1));      // MMA of j-1 read H_lo
#pragma unroll
            for (int c4 = 0; c4 < 16; c4++) {                              // H_lo for the MMA (H is the hi operand)
                const int k = 64 * half + 4 * c4;
                float lo4[4];
#pragma unroll
                for (int el = 0; el < 4; el++) {
                    const float xv = x[4 * c4 + el];
                    // x - trunc_tf32(x) has up to 13 significant bits; rounded to
                    // tf32 here so the MMA does not truncate it again (2^-22 |x|
                    // per product instead of 2^-20)
                    const float r = __fsub_rn(xv, __uint_as_float(__float_as_uint(xv) & 0xFFFFE000u));
                    lo4[el] = __uint_as_float((__float_as_uint(r) + 0x1000u) & 0xFFFFE000u);
                }
                *reinterpret_cast<float4 *>(lo_buf + (k >> 5) * (S::HS / 4) + tma::box_off(r, k & 31)) =
                    make_float4(lo4[0], lo4[1], lo4[2], lo4[3]);
            }
            tc::fence_proxy_async();
            tc::mbar_arrive(lofull);
            if constexpr (BITS != 32) {
                // min / max of the half (exact, order-free), then of the row through smem
                float mn4[4], mx4[4];
#pragma unroll
                for (int u = 0; u < 4; u++) { mn4[u] = x[u]; mx4[u] = x[u]; }
#pragma unroll
                for (int k = 4; k < 64; k++) { mn4[k & 3] = fminf(mn4[k & 3], x[k]); mx4[k & 3] = fmaxf(mx4[k & 3], x[k]); }
                float *mp = mm + (j & 1) * 512;
                mp[half * 256 + r] = fminf(fminf(mn4[0], mn4[1]), fminf(mn4[2], mn4[3]));
                mp[half * 256 + 128 + r] = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
                tma::named_sync(1, 256);
                const float z = fminf(mp[r], mp[256 + r]);
                const float rr = __fsub_rn(fmaxf(mp[128 + r], mp[384 + r]), z);
                const DivR dv = make_div(rr);
                const uint64_t gglob = (uint64_t)(row_offset + row);
                uint32_t cw[HW];
#pragma unroll
                for (int w = 0; w < HW; w++) cw[w] = 0u;
                if (rr > 0.0f) {
                    bool slow = !dv.fast;
                    const uint32_t kc = MODE == KGQ_ROUND_SR_FAST ? carrier_const() : 0u;
#pragma unroll
                    for (int cc = 0; cc < 8; cc++) {         // fast-noise call c = 8 half + cc
                        const int c = 8 * half + cc;
                        uint4 rnd = make_uint4(0, 0, 0, 0);
                        if (MODE == KGQ_ROUND_SR_FAST) rnd = fast_call(fk, gglob, (uint32_t)c);
                        const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            const int kl = 32 * (cc >> 2) + 4 * (cc & 3) + 16 * h;   // column within the half
                            u64x4 r64 = {0, 0, 0, 0};
                            if (MODE == KGQ_ROUND_SR_COMPAT)
                                r64 = philox4x64_10(gglob * (uint64_t)(D / 4) + (uint64_t)((64 * half + kl) >> 2) + 1ull,
                                                    0, 0, 0, seed, tid);
                            const uint64_t cw64[4] = {r64.x, r64.y, r64.z, r64.w};
                            uint32_t acc = 0;
#pragma unroll
                            for (int el = 0; el < 4; el++) {
                                const float a = __fsub_rn(x[kl + el], z);
                                slow |= (__float_as_uint(a) - 1u) < dv.thr_m1;      // 0 < a < threshold
                                const float sv = __fmul_rn(div_a_unguarded(dv, a), Bf);
                                const float uf = h ? u16_carrier_hi(rw[el], kc) : u16_carrier_lo(rw[el], kc);
                                acc += code_bits<MODE>(sv, uf, cw64[el] >> 11) << (BITS * el);
                            }
                            const int bit = kl * BITS;
                            cw[bit >> 5] |= (acc - magic_sum4<BITS>()) << (bit & 31);
                        }
                    }
                    if (slow) {
                        if (half == 0) tc64_row_codes_exact<BITS, MODE, 128, 0, 8>(hst, r, z, dv, fk, gglob, seed, tid, cw);
                        else tc64_row_codes_exact<BITS, MODE, 128, 8, 8>(hst, r, z, dv, fk, gglob, seed, tid, cw);
                    }
                }
                if (active) {
                    uint32_t *crow = reinterpret_cast<uint32_t *>(codes + row * RB) + HW * half;
                    if constexpr (HW % 4 == 0) {
#pragma unroll
                        for (int w = 0; w < HW; w += 4)
                            *reinterpret_cast<uint4 *>(crow + w) = make_uint4(cw[w], cw[w + 1], cw[w + 2], cw[w + 3]);
                    } else {
#pragma unroll
                        for (int w = 0; w < HW; w += 2)
                            *reinterpret_cast<uint2 *>(crow + w) = make_uint2(cw[w], cw[w + 1]);
                    }
                    if (half == 0) {
                        ranges[row] = rr;
                        offsets[row] = z;
                    }
                }
            }
        }
    } else {
        // --------------------------- drain warps (thread = column n) ---------------------------
        const int q = warp & 3, n = 32 * q + lane;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        for (int j = 0; j < nj; j++) {
            const int b = j & 1;
            tc::mbar_wait(jfull + b, (uint32_t)((j >> 1) & 1));
            tc::fence_after();
            const int64_t r0 = tile_of(j) * M;
#pragma unroll 1
            for (int cb = 0; cb < M; cb += 32) {
                float v[32];
                tc::tmem_ld32(tmem + lane_addr + kE8J + 128u * b + (uint32_t)cb, v);
                if (cb == M - 32) {
                    tc::fence_before();
                    tc::mbar_arrive(jempty + b);
                }
                uint32_t myword = 0;
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    const uint32_t bal = __ballot_sync(0xffffffffu, v[i] > 0.0f);   // row r0+cb+i, columns 32q..
                    if (lane == i) myword = bal;
                    const int64_t row = r0 + cb + i;
                    if (row < n_rows) e_next[row * D + n] = relu_nan(v[i]);
                }
                const int64_t row = r0 + cb + lane;
                if (row < n_rows) mask[row * (D / 32) + q] = myword;
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_free(tmem, 512);
}

template <int BITS>
static int launch_epilogue_tc128(int rounding, const float *h, int64_t n_rows, const float *theta, uint64_t seed,
                                 uint64_t tid, const uint64_t *tid_base, int64_t row_offset, uint8_t *codes,
                                 float *ranges, float *offsets, float *e_next, uint32_t *mask, cudaStream_t s) {
    void (*kern)(const CUtensorMap, int64_t, const float *, uint64_t, uint64_t, const uint64_t *, int64_t,
                 uint8_t *, float *, float *, float *, uint32_t *);
    switch (rounding) {
        case KGQ_ROUND_NEAREST: kern = layer_epilogue_tc128_kernel<BITS, KGQ_ROUND_NEAREST>; break;
        case KGQ_ROUND_SR_FAST: kern = layer_epilogue_tc128_kernel<BITS, KGQ_ROUND_SR_FAST>; break;
        case KGQ_ROUND_SR_COMPAT: kern = layer_epilogue_tc128_kernel<BITS, KGQ_ROUND_SR_COMPAT>; break;
        default: return KGQ_ERR_INVALID_ARG;
    }
    static bool smem_set[3] = {false, false, false};
    if (!smem_set[rounding]) {
        cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Epi128Smem::bytes);
        if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
        smem_set[rounding] = true;
    }
    CUtensorMap tm_h;
    if (!tma::make_rowmajor_f32(&tm_h, h, (uint64_t)n_rows, 128, 128)) return KGQ_ERR_CUDA;
    const int64_t tiles = (n_rows + 127) / 128;
    const int grid = (int)(tiles < kSMs ? tiles : kSMs);
    kern<<<grid, kE8Threads, Epi128Smem::bytes, s>>>(tm_h, n_rows, theta, seed, tid, tid_base, row_offset, codes,
                                                     ranges, offsets, e_next, mask);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

template <int D, int BITS>
static int launch_epilogue_tc(int rounding, const float *h, int64_t n_rows, const float *theta,
                              uint64_t seed, uint64_t tid, const uint64_t *tid_base, int64_t row_offset,
                              uint8_t *codes, float *ranges, float *offsets, float *e_next,
                              uint32_t *mask, cudaStream_t s) {
    if constexpr (D == 64) {
        if (!(getenv("KGQ_EPI_TC1") && getenv("KGQ_EPI_TC1")[0] == '1'))
            return launch_epilogue_tc64<BITS>(rounding, h, n_rows, theta, seed, tid, tid_base, row_offset, codes,
                                              ranges, offsets, e_next, mask, s);
    }
    const size_t smem = EpiTc<D>::smem;
    void (*kern)(const float *, int64_t, const float *, uint64_t, uint64_t, const uint64_t *, int64_t,
                 uint8_t *, float *, float *, const CUtensorMap, uint32_t *);
    switch (rounding) {
        case KGQ_ROUND_NEAREST: kern = layer_epilogue_tc_kernel<D, BITS, KGQ_ROUND_NEAREST>; break;
        case KGQ_ROUND_SR_FAST: kern = layer_epilogue_tc_kernel<D, BITS, KGQ_ROUND_SR_FAST>; break;
        case KGQ_ROUND_SR_COMPAT: kern = layer_epilogue_tc_kernel<D, BITS, KGQ_ROUND_SR_COMPAT>; break;
        default: return KGQ_ERR_INVALID_ARG;
    }
    static bool smem_set[3] = {false, false, false};
    if (!smem_set[rounding]) {
        cudaError_t ea = ensure_smem(kern, smem);
        if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
        smem_set[rounding] = true;
    }
    CUtensorMap tm_out;     // E_next rows leave by TMA: 128-row x 32-column boxes
    if (!tma::make_rowmajor_f32(&tm_out, e_next, (uint64_t)n_rows, (uint64_t)D, EpiTc<D>::M))
        return KGQ_ERR_CUDA;
    const int64_t tiles = (n_rows + EpiTc<D>::M - 1) / EpiTc<D>::M;
    const int64_t cap = (int64_t)kSMs * (D > 32 ? 2 : 4);
    const int grid = (int)(tiles < cap ? tiles : cap);
    kern<<<grid, 256, smem, s>>>(h, n_rows, theta, seed, tid, tid_base, row_offset, codes, ranges,
                                 offsets, tm_out, mask);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

template <int D, int BITS>
static int launch_epilogue(int rounding, const float *h, int64_t n_rows, const float *theta,
                           uint64_t seed, uint64_t tid, const uint64_t *tid_base, int64_t row_offset,
                           uint8_t *codes, float *ranges, float *offsets, float *e_next,
                           uint32_t *mask, cudaStream_t s) {
    if constexpr (D == 32 || D == 64) {
        if (epi_use_tc(D))
            return launch_epilogue_tc<D, BITS>(rounding, h, n_rows, theta, seed, tid, tid_base, row_offset,
                                               codes, ranges, offsets, e_next, mask, s);
    }
    if constexpr (D == 128) {
        if (epi_use_tc(D) && ((((uintptr_t)h) | ((uintptr_t)codes)) & 15u) == 0)
            return launch_epilogue_tc128<BITS>(rounding, h, n_rows, theta, seed, tid, tid_base, row_offset,
                                               codes, ranges, offsets, e_next, mask, s);
    }
    const size_t smem = EpiTile<D>::smem;
    void (*kern)(const float *, int64_t, const float *, uint64_t, uint64_t, const uint64_t *, int64_t,
                 uint8_t *, float *, float *, float *, uint32_t *);
    switch (rounding) {
        case KGQ_ROUND_NEAREST: kern = layer_epilogue_kernel<D, BITS, KGQ_ROUND_NEAREST>; break;
        case KGQ_ROUND_SR_FAST: kern = layer_epilogue_kernel<D, BITS, KGQ_ROUND_SR_FAST>; break;
        case KGQ_ROUND_SR_COMPAT: kern = layer_epilogue_kernel<D, BITS, KGQ_ROUND_SR_COMPAT>; break;
        default: return KGQ_ERR_INVALID_ARG;
    }
    static bool smem_set[3] = {false, false, false};
    if (!smem_set[rounding]) {
        cudaError_t ea = ensure_smem(kern, smem);
        if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
        smem_set[rounding] = true;
    }
    const int64_t tiles = (n_rows + EpiTile<D>::ROWS - 1) / EpiTile<D>::ROWS;
    const int64_t cap = (int64_t)kSMs * (D > 64 ? 2 : 6);
    const int grid = (int)(tiles < cap ? tiles : cap);
    kern<<<grid, 256, smem, s>>>(h, n_rows, theta, seed, tid, tid_base, row_offset, codes, ranges,
                                 offsets, e_next, mask);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

template <int D>
static int launch_layer_bits(int bits, int rounding, const int32_t *indptr, const int32_t *indices,
                             const float *vals, int64_t n_rows, const int32_t *row_order,
                             int64_t n_heavy, const float *e, const float *theta, uint64_t seed,
                             uint64_t tid, const uint64_t *tid_base, int64_t row_offset,
                             uint8_t *codes, float *ranges,
                             float *offsets, float *e_next, uint32_t *mask, float *h_out,
                             cudaStream_t s) {
#define KGQ_LAYER(B) launch_layer<D, B>(rounding, indptr, indices, vals, n_rows, row_order, n_heavy, e, \
                                        theta, seed, tid, tid_base, row_offset, codes, ranges, offsets, \
                                        e_next, mask, h_out, s)
    switch (bits) {
        case 1: return KGQ_LAYER(1);
        case 2: return KGQ_LAYER(2);
        case 4: return KGQ_LAYER(4);
        case 8: return KGQ_LAYER(8);
    }
#undef KGQ_LAYER
    return KGQ_ERR_UNSUPPORTED_BITS;
}

extern "C" int kgq_layer_forward_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                                     int64_t n_rows, const int32_t *row_order, int64_t n_heavy,
                                     const float *e, int32_t d, const float *theta, int32_t bits,
                                     int32_t rounding, uint64_t seed, uint64_t tensor_id,
                                     const uint64_t *tid_base, int64_t row_offset, uint8_t *codes,
                                     float *ranges,
                                     float *offsets, float *e_next, uint8_t *mask, float *h_out,
                                     void *stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (n_rows < 0 || row_offset < 0 || rounding < 0 || rounding > 2 || n_heavy < 0 || n_heavy > n_rows)
        return KGQ_ERR_INVALID_ARG;
    if (n_heavy && !row_order) return KGQ_ERR_INVALID_ARG;
    if (n_rows == 0) return KGQ_OK;
    if (!indptr || !e || !theta || !codes || !ranges || !offsets || !e_next || !mask)
        return KGQ_ERR_INVALID_ARG;
    if (((uintptr_t)mask & 3u) || ((uintptr_t)codes & 3u) || ((uintptr_t)e & 15u) ||
        ((uintptr_t)e_next & 15u) || ((uintptr_t)theta & 15u) || (h_out && ((uintptr_t)h_out & 15u)))
        return KGQ_ERR_MISALIGNED;
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *m32 = reinterpret_cast<uint32_t *>(mask);
    switch (d) {
        case 32: return launch_layer_bits<32>(bits, rounding, indptr, indices, vals, n_rows, row_order, n_heavy, e, theta, seed, tensor_id, tid_base, row_offset, codes, ranges, offsets, e_next, m32, h_out, s);
        case 64: return launch_layer_bits<64>(bits, rounding, indptr, indices, vals, n_rows, row_order, n_heavy, e, theta, seed, tensor_id, tid_base, row_offset, codes, ranges, offsets, e_next, m32, h_out, s);
        case 128: return launch_layer_bits<128>(bits, rounding, indptr, indices, vals, n_rows, row_order, n_heavy, e, theta, seed, tensor_id, tid_base, row_offset, codes, ranges, offsets, e_next, m32, h_out, s);
    }
    return KGQ_ERR_INVALID_ARG;
}

extern "C" int kgq_layer_epilogue_f32(const float *h, int64_t n_rows, int32_t d, const float *theta,
                                      int32_t bits, int32_t rounding, uint64_t seed, uint64_t tensor_id,
                                      const uint64_t *tid_base, int64_t row_offset, uint8_t *codes,
                                      float *ranges, float *offsets, float *e_next, uint8_t *mask,
                                      void *stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8 || bits == 32)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (n_rows < 0 || row_offset < 0 || rounding < 0 || rounding > 2) return KGQ_ERR_INVALID_ARG;
    if (n_rows == 0) return KGQ_OK;
    if (!h || !theta || !e_next || !mask) return KGQ_ERR_INVALID_ARG;
    if (bits != 32 && (!codes || !ranges || !offsets)) return KGQ_ERR_INVALID_ARG;
    if (((uintptr_t)mask & 3u) || ((uintptr_t)codes & 3u) || ((uintptr_t)h & 15u) ||
        ((uintptr_t)e_next & 15u) || ((uintptr_t)theta & 15u))
        return KGQ_ERR_MISALIGNED;
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *m32 = reinterpret_cast<uint32_t *>(mask);
#define KGQ_EPI(D, B) launch_epilogue<D, B>(rounding, h, n_rows, theta, seed, tensor_id, tid_base, row_offset, \
                                            codes, ranges, offsets, e_next, m32, s)
#define KGQ_EPI_BITS(D) switch (bits) { case 1: return KGQ_EPI(D, 1); case 2: return KGQ_EPI(D, 2); \
                                        case 4: return KGQ_EPI(D, 4); case 8: return KGQ_EPI(D, 8); \
                                        default: return KGQ_EPI(D, 32); }
    switch (d) {
        case 32: KGQ_EPI_BITS(32)
        case 64: KGQ_EPI_BITS(64)
        case 128: KGQ_EPI_BITS(128)
    }
#undef KGQ_EPI_BITS
#undef KGQ_EPI
    return KGQ_ERR_INVALID_ARG;
}
