// kgq_graph.cu -- KG neighbour aggregation (K4 CSR SpMM), ReLU + 1-bit mask
// (K5) and the fused per-layer forward (spmm -> quantize H -> H.theta -> relu
// -> mask) for sm_100a.
//
// Row-group layout (d in {32, 64, 128}): a row is owned by LPR = d/8 lanes and
// a warp works on RPW = 32/LPR rows at once.  Lane gl of a row group owns the
// two float4 at feature offsets 32p+4q and 32p+16+4q (p = gl>>2, q = gl&3):
// one neighbour row is gathered with one 128-bit load per lane (fully used
// sectors), and those 8 features are exactly the 8 elements of fast-noise
// call 4p+q, so the fused quantizer needs one Philox call per lane.
// Every output element is accumulated in ascending column order as
// acc = acc + a*x with separate mul and add -- the order scipy's csr_matvecs
// uses (tensorops.py:8-12, 37-50) -- so results are bit-identical; only the
// loads are reordered (4 neighbours x 2 float4 in flight per lane).
// Rows are visited in an optional degree-sorted order (row_order) so the RPW
// rows of a warp have similar lengths.
#include "kgq_common.cuh"

namespace kgq {

template <int D>
struct RG {
    static constexpr int LPR = D / 8;      // lanes per row
    static constexpr int RPW = 32 / LPR;   // rows per warp
};

// Sequential ascending-column accumulation of one row (bit-exact with scipy).
// All lanes of the warp must call this together: the nonzero loop runs to the
// warp's longest row with per-row predicates so shuffles stay convergent.
template <int D>
__device__ __forceinline__ void rg_spmm_row(const int32_t *__restrict__ indptr,
                                            const int32_t *__restrict__ indices,
                                            const float *__restrict__ vals,
                                            const float *__restrict__ x, int64_t row, bool active,
                                            int gl, float4 (&acc)[2]) {
    constexpr int LPR = RG<D>::LPR;
    acc[0] = acc[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    int32_t beg = 0, end = 0;
    if (active) {
        beg = __ldg(indptr + row);
        end = __ldg(indptr + row + 1);
    }
    int len = end - beg;
    int maxlen = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    const int f0 = 8 * (gl >> 2) + (gl & 3);
    for (int base = 0; base < maxlen; base += LPR) {
        const int cnt = min(LPR, len - base);         // may be <= 0 for short rows
        int32_t my_col = 0;
        float my_val = 0.0f;
        if (gl < cnt) {
            my_col = __ldg(indices + beg + base + gl);
            my_val = __ldg(vals + beg + base + gl);
        }
#pragma unroll
        for (int t = 0; t < LPR; t += 4) {
            float4 xa[4], xb[4];
            float av[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int32_t col = __shfl_sync(0xffffffffu, my_col, t + u, LPR);
                av[u] = __shfl_sync(0xffffffffu, my_val, t + u, LPR);
                if (t + u < cnt) {
                    const float4 *xr = reinterpret_cast<const float4 *>(x + (int64_t)col * D);
                    xa[u] = __ldg(xr + f0);
                    xb[u] = __ldg(xr + f0 + 4);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                if (t + u < cnt) {
                    const float a = av[u];
                    acc[0].x = __fadd_rn(acc[0].x, __fmul_rn(a, xa[u].x));
                    acc[0].y = __fadd_rn(acc[0].y, __fmul_rn(a, xa[u].y));
                    acc[0].z = __fadd_rn(acc[0].z, __fmul_rn(a, xa[u].z));
                    acc[0].w = __fadd_rn(acc[0].w, __fmul_rn(a, xa[u].w));
                    acc[1].x = __fadd_rn(acc[1].x, __fmul_rn(a, xb[u].x));
                    acc[1].y = __fadd_rn(acc[1].y, __fmul_rn(a, xb[u].y));
                    acc[1].z = __fadd_rn(acc[1].z, __fmul_rn(a, xb[u].z));
                    acc[1].w = __fadd_rn(acc[1].w, __fmul_rn(a, xb[u].w));
                }
            }
        }
    }
}

template <int D>
__global__ void __launch_bounds__(256)
spmm_rg_kernel(const int32_t *__restrict__ indptr, const int32_t *__restrict__ indices,
               const float *__restrict__ vals, int64_t n_rows, const int32_t *__restrict__ row_order,
               const float *__restrict__ x, float *__restrict__ out) {
    constexpr int LPR = RG<D>::LPR, RPW = RG<D>::RPW;
    const int lane = threadIdx.x & 31;
    const int gl = lane % LPR, grp = lane / LPR;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int f0 = 8 * (gl >> 2) + (gl & 3);
    for (int64_t base = warp * RPW; base < n_rows; base += nw * RPW) {
        const int64_t slot = base + grp;
        const bool active = slot < n_rows;
        const int64_t row = active ? (row_order ? (int64_t)__ldg(row_order + slot) : slot) : 0;
        float4 acc[2];
        rg_spmm_row<D>(indptr, indices, vals, x, row, active, gl, acc);
        if (active) {
            float4 *o = reinterpret_cast<float4 *>(out + row * D);
            o[f0] = acc[0];
            o[f0 + 4] = acc[1];
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

// spread the 8 bits of b so that bit k lands at bit 4k
__device__ __forceinline__ uint32_t spread4(uint32_t b) {
    b &= 0xFFu;
    b = (b | (b << 12)) & 0x000F000Fu;
    b = (b | (b << 6)) & 0x03030303u;
    b = (b | (b << 3)) & 0x11111111u;
    return b;
}

// relu + LSB-first flat bit mask.  A warp handles 128 elements per step:
// lane l loads float4 l; ballot e collects bit (4l+e); lanes 0..3 assemble
// the four 32-bit mask words.
__global__ void __launch_bounds__(256)
relu_mask_kernel(const float *__restrict__ x, int64_t n128, float *__restrict__ out,
                 uint32_t *__restrict__ mask) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < n128; c += nw) {
        const float4 v = ldg_stream(reinterpret_cast<const float4 *>(x) + c * 32 + lane);
        const uint32_t b0 = __ballot_sync(0xffffffffu, v.x > 0.0f);
        const uint32_t b1 = __ballot_sync(0xffffffffu, v.y > 0.0f);
        const uint32_t b2 = __ballot_sync(0xffffffffu, v.z > 0.0f);
        const uint32_t b3 = __ballot_sync(0xffffffffu, v.w > 0.0f);
        const float4 o = make_float4(v.x > 0.0f ? v.x : 0.0f, v.y > 0.0f ? v.y : 0.0f,
                                     v.z > 0.0f ? v.z : 0.0f, v.w > 0.0f ? v.w : 0.0f);
        stg_stream(reinterpret_cast<float4 *>(out) + c * 32 + lane, o);
        if (lane < 4) {
            const int sh = 8 * lane;
            const uint32_t w = spread4(b0 >> sh) | (spread4(b1 >> sh) << 1) |
                               (spread4(b2 >> sh) << 2) | (spread4(b3 >> sh) << 3);
            mask[c * 4 + lane] = w;
        }
    }
}

// tail / unaligned: thread per mask byte
__global__ void relu_mask_bytes_kernel(const float *__restrict__ x, int64_t start, int64_t n,
                                       float *__restrict__ out, uint8_t *__restrict__ mask) {
    const int64_t nb = (n - start + 7) / 8;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint32_t byte = 0;
        for (int t = 0; t < 8; t++) {
            const int64_t i = start + 8 * b + t;
            if (i >= n) break;
            const float v = x[i];
            out[i] = v > 0.0f ? v : 0.0f;
            byte |= (v > 0.0f ? 1u : 0u) << t;
        }
        mask[start / 8 + b] = (uint8_t)byte;
    }
}

// ReLU backward: out = g * float(mask bit) (tape.py:224-225: g * mask.to_bool())
__global__ void mask_apply_kernel(const float *__restrict__ g, const uint8_t *__restrict__ mask,
                                  int64_t n, float *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t bit = (mask[i >> 3] >> (i & 7)) & 1u;
        out[i] = __fmul_rn(g[i], bit ? 1.0f : 0.0f);
    }
}

__global__ void mask_apply_vec_kernel(const float4 *__restrict__ g, const uint8_t *__restrict__ mask,
                                      int64_t n4, float4 *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t m = (mask[i >> 1] >> (4 * (i & 1))) & 0xFu;
        const float4 v = ldg_stream(g + i);
        stg_stream(out + i, make_float4(__fmul_rn(v.x, (m & 1u) ? 1.0f : 0.0f),
                                        __fmul_rn(v.y, (m & 2u) ? 1.0f : 0.0f),
                                        __fmul_rn(v.z, (m & 4u) ? 1.0f : 0.0f),
                                        __fmul_rn(v.w, (m & 8u) ? 1.0f : 0.0f)));
    }
}

// ---------------------------------------------------------------------------
// Fused layer forward (row-group layout):
//   H = A_hat.E (bit-exact spmm), quantize H on chip (group = d; same
//   arithmetic and noise as kgq_quantize_f32: lane gl's 8 features are the 8
//   elements of call 4p+q), J = H.theta (theta in smem, FFMA, ascending k),
//   E' = relu(J), mask = J > 0.  H and J never reach HBM.
// ---------------------------------------------------------------------------
template <int D, int BITS, int MODE>
__global__ void __launch_bounds__(256)
layer_forward_kernel(const int32_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                     const float *__restrict__ vals, int64_t n_rows,
                     const int32_t *__restrict__ row_order, const float *__restrict__ e,
                     const float *__restrict__ theta, uint64_t seed, uint64_t tid,
                     int64_t row_offset, uint8_t *__restrict__ codes, float *__restrict__ ranges,
                     float *__restrict__ offsets, float *__restrict__ e_next,
                     uint32_t *__restrict__ mask, float *__restrict__ h_out) {
    constexpr int LPR = RG<D>::LPR, RPW = RG<D>::RPW;
    constexpr float Bf = (float)((1u << BITS) - 1u);
    constexpr int RB = D * BITS / 8;                // packed bytes per row
    extern __shared__ __align__(16) float th[];     // theta, D*D fp32 (64 KB at D=128)
    for (int i = threadIdx.x; i < D * D / 4; i += blockDim.x)
        reinterpret_cast<float4 *>(th)[i] = __ldg(reinterpret_cast<const float4 *>(theta) + i);
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int gl = lane % LPR, grp = lane / LPR;
    const int p = gl >> 2, q = gl & 3;
    const int f0 = 8 * p + q;                       // float4 index of my first four features
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const FastKey fk = make_fast_key(seed, tid);
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));

    for (int64_t base = warp * RPW; base < n_rows; base += nw * RPW) {
        const int64_t slot = base + grp;
        const bool active = slot < n_rows;
        const int64_t row = active ? (row_order ? (int64_t)__ldg(row_order + slot) : slot) : 0;
        float4 h[2];
        rg_spmm_row<D>(indptr, indices, vals, e, row, active, gl, h);
        if (active && h_out) {
            float4 *o = reinterpret_cast<float4 *>(h_out + row * D);
            o[f0] = h[0];
            o[f0 + 4] = h[1];
        }
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
                    const float uf = hh ? __uint2float_rn(rw[el] >> 16) : __uint2float_rn(rw[el] & 0xFFFFu);
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
        // ---- J = H . theta (ascending k, FFMA) ----
        float4 j0 = make_float4(0.f, 0.f, 0.f, 0.f), j1 = j0;
#pragma unroll 4
        for (int k = 0; k < D; k++) {
            const int src = 4 * (k >> 5) + ((k >> 2) & 3);      // lane owning H[k]
            const int hh = (k >> 4) & 1, el = k & 3;
            const float mine = hh ? (el == 0 ? h[1].x : el == 1 ? h[1].y : el == 2 ? h[1].z : h[1].w)
                                  : (el == 0 ? h[0].x : el == 1 ? h[0].y : el == 2 ? h[0].z : h[0].w);
            const float hk = __shfl_sync(0xffffffffu, mine, src, LPR);
            const float4 ta = reinterpret_cast<const float4 *>(th + k * D)[f0];
            const float4 tb = reinterpret_cast<const float4 *>(th + k * D)[f0 + 4];
            j0.x = __fmaf_rn(hk, ta.x, j0.x); j0.y = __fmaf_rn(hk, ta.y, j0.y);
            j0.z = __fmaf_rn(hk, ta.z, j0.z); j0.w = __fmaf_rn(hk, ta.w, j0.w);
            j1.x = __fmaf_rn(hk, tb.x, j1.x); j1.y = __fmaf_rn(hk, tb.y, j1.y);
            j1.z = __fmaf_rn(hk, tb.z, j1.z); j1.w = __fmaf_rn(hk, tb.w, j1.w);
        }
        // ---- relu + mask (word p of the row: nibble 4q and 16+4q) ----
        uint32_t w = (j0.x > 0.f ? 1u : 0u) | (j0.y > 0.f ? 2u : 0u) | (j0.z > 0.f ? 4u : 0u) |
                     (j0.w > 0.f ? 8u : 0u);
        w <<= 4 * q;
        w |= ((j1.x > 0.f ? 1u : 0u) | (j1.y > 0.f ? 2u : 0u) | (j1.z > 0.f ? 4u : 0u) |
              (j1.w > 0.f ? 8u : 0u)) << (16 + 4 * q);
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        if (active) {
            float4 *o = reinterpret_cast<float4 *>(e_next + row * D);
            o[f0] = make_float4(j0.x > 0.f ? j0.x : 0.f, j0.y > 0.f ? j0.y : 0.f,
                                j0.z > 0.f ? j0.z : 0.f, j0.w > 0.f ? j0.w : 0.f);
            o[f0 + 4] = make_float4(j1.x > 0.f ? j1.x : 0.f, j1.y > 0.f ? j1.y : 0.f,
                                    j1.z > 0.f ? j1.z : 0.f, j1.w > 0.f ? j1.w : 0.f);
            if (q == 0) mask[row * (D / 32) + p] = w;
        }
        (void)gmask;
    }
}

}  // namespace kgq

using namespace kgq;

static inline int persistent_blocks(int64_t warps_needed, int per_sm) {
    int64_t b = (warps_needed + 7) / 8;
    const int64_t cap = (int64_t)kSMs * per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

extern "C" int kgq_spmm_csr_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                                int64_t n_rows, const int32_t *row_order, const float *x, int32_t d,
                                float *out, void *stream) {
    if (n_rows < 0 || d < 1) return KGQ_ERR_INVALID_ARG;
    if (n_rows == 0) return KGQ_OK;
    if (!indptr || !out || !x) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const bool vec = ((((uintptr_t)x) | ((uintptr_t)out)) & 15u) == 0;
    if (vec && d == 32) {
        spmm_rg_kernel<32><<<persistent_blocks((n_rows + 7) / 8, 16), 256, 0, s>>>(indptr, indices, vals, n_rows, row_order, x, out);
    } else if (vec && d == 64) {
        spmm_rg_kernel<64><<<persistent_blocks((n_rows + 3) / 4, 16), 256, 0, s>>>(indptr, indices, vals, n_rows, row_order, x, out);
    } else if (vec && d == 128) {
        spmm_rg_kernel<128><<<persistent_blocks((n_rows + 1) / 2, 16), 256, 0, s>>>(indptr, indices, vals, n_rows, row_order, x, out);
    } else {
        int64_t b = (n_rows + 7) / 8;
        spmm_generic_kernel<<<(int)(b < 0x7fffffff ? b : 0x7fffffff), 256, 0, s>>>(indptr, indices, vals, n_rows, x, d, out);
    }
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
extern "C" int kgq_relu_mask_f32(const float *x, int64_t n, float *out, uint8_t *mask, void *stream) {
    if (n < 0) return KGQ_ERR_INVALID_ARG;
    if (n == 0) return KGQ_OK;
    if (!x || !out || !mask) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    int64_t n128 = 0;
    if ((((uintptr_t)x | (uintptr_t)out) & 15u) == 0 && ((uintptr_t)mask & 3u) == 0) n128 = n / 128;
    if (n128) {
        int64_t blocks = (n128 + 7) / 8;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        relu_mask_kernel<<<(int)blocks, 256, 0, s>>>(x, n128, out, reinterpret_cast<uint32_t *>(mask));
    }
    const int64_t start = n128 * 128;
    if (start < n) {
        const int64_t nb = (n - start + 7) / 8;
        int64_t blocks = (nb + 255) / 256;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        relu_mask_bytes_kernel<<<(int)blocks, 256, 0, s>>>(x, start, n, out, mask);
    }
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_mask_apply_f32(const float *g, const uint8_t *mask, int64_t n, float *out,
                                  void *stream) {
    if (n < 0) return KGQ_ERR_INVALID_ARG;
    if (n == 0) return KGQ_OK;
    if (!g || !mask || !out) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if ((n & 3) == 0 && (((uintptr_t)g | (uintptr_t)out) & 15u) == 0) {
        const int64_t n4 = n / 4;
        int64_t blocks = (n4 + 255) / 256;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        mask_apply_vec_kernel<<<(int)blocks, 256, 0, s>>>(reinterpret_cast<const float4 *>(g), mask, n4,
                                                          reinterpret_cast<float4 *>(out));
    } else {
        int64_t blocks = (n + 255) / 256;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        mask_apply_kernel<<<(int)blocks, 256, 0, s>>>(g, mask, n, out);
    }
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

template <int D, int BITS>
static int launch_layer(int rounding, const int32_t *indptr, const int32_t *indices, const float *vals,
                        int64_t n_rows, const int32_t *row_order, const float *e, const float *theta,
                        uint64_t seed, uint64_t tid, int64_t row_offset, uint8_t *codes, float *ranges,
                        float *offsets, float *e_next, uint32_t *mask, float *h_out,
                        cudaStream_t s) {
    const size_t smem = (size_t)D * D * sizeof(float);
    const int blocks = persistent_blocks((n_rows + RG<D>::RPW - 1) / RG<D>::RPW, 8);
    void (*kern)(const int32_t *, const int32_t *, const float *, int64_t, const int32_t *,
                 const float *, const float *, uint64_t, uint64_t, int64_t, uint8_t *, float *,
                 float *, float *, uint32_t *, float *);
    switch (rounding) {
        case KGQ_ROUND_NEAREST: kern = layer_forward_kernel<D, BITS, KGQ_ROUND_NEAREST>; break;
        case KGQ_ROUND_SR_FAST: kern = layer_forward_kernel<D, BITS, KGQ_ROUND_SR_FAST>; break;
        case KGQ_ROUND_SR_COMPAT: kern = layer_forward_kernel<D, BITS, KGQ_ROUND_SR_COMPAT>; break;
        default: return KGQ_ERR_INVALID_ARG;
    }
    if (smem > 48 * 1024) {
        cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
    }
    kern<<<blocks, 256, smem, s>>>(indptr, indices, vals, n_rows, row_order, e, theta, seed, tid,
                                   row_offset, codes, ranges, offsets, e_next, mask, h_out);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

template <int D>
static int launch_layer_bits(int bits, int rounding, const int32_t *indptr, const int32_t *indices,
                             const float *vals, int64_t n_rows, const int32_t *row_order,
                             const float *e, const float *theta,
                             uint64_t seed, uint64_t tid, int64_t row_offset, uint8_t *codes,
                             float *ranges, float *offsets, float *e_next, uint32_t *mask,
                             float *h_out, cudaStream_t s) {
    switch (bits) {
        case 1: return launch_layer<D, 1>(rounding, indptr, indices, vals, n_rows, row_order, e, theta, seed, tid, row_offset, codes, ranges, offsets, e_next, mask, h_out, s);
        case 2: return launch_layer<D, 2>(rounding, indptr, indices, vals, n_rows, row_order, e, theta, seed, tid, row_offset, codes, ranges, offsets, e_next, mask, h_out, s);
        case 4: return launch_layer<D, 4>(rounding, indptr, indices, vals, n_rows, row_order, e, theta, seed, tid, row_offset, codes, ranges, offsets, e_next, mask, h_out, s);
        case 8: return launch_layer<D, 8>(rounding, indptr, indices, vals, n_rows, row_order, e, theta, seed, tid, row_offset, codes, ranges, offsets, e_next, mask, h_out, s);
    }
    return KGQ_ERR_UNSUPPORTED_BITS;
}

extern "C" int kgq_layer_forward_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                                     int64_t n_rows, const int32_t *row_order, const float *e,
                                     int32_t d, const float *theta,
                                     int32_t bits, int32_t rounding, uint64_t seed,
                                     uint64_t tensor_id, int64_t row_offset, uint8_t *codes,
                                     float *ranges, float *offsets, float *e_next, uint8_t *mask,
                                     float *h_out, void *stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (n_rows < 0 || row_offset < 0 || rounding < 0 || rounding > 2) return KGQ_ERR_INVALID_ARG;
    if (n_rows == 0) return KGQ_OK;
    if (!indptr || !e || !theta || !codes || !ranges || !offsets || !e_next || !mask)
        return KGQ_ERR_INVALID_ARG;
    if (((uintptr_t)mask & 3u) || ((uintptr_t)codes & 3u) || ((uintptr_t)e & 15u) ||
        ((uintptr_t)e_next & 15u) || ((uintptr_t)theta & 15u) || (h_out && ((uintptr_t)h_out & 15u)))
        return KGQ_ERR_MISALIGNED;
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *m32 = reinterpret_cast<uint32_t *>(mask);
    switch (d) {
        case 32: return launch_layer_bits<32>(bits, rounding, indptr, indices, vals, n_rows, row_order, e, theta, seed, tensor_id, row_offset, codes, ranges, offsets, e_next, m32, h_out, s);
        case 64: return launch_layer_bits<64>(bits, rounding, indptr, indices, vals, n_rows, row_order, e, theta, seed, tensor_id, row_offset, codes, ranges, offsets, e_next, m32, h_out, s);
        case 128: return launch_layer_bits<128>(bits, rounding, indptr, indices, vals, n_rows, row_order, e, theta, seed, tensor_id, row_offset, codes, ranges, offsets, e_next, m32, h_out, s);
    }
    return KGQ_ERR_INVALID_ARG;
}
