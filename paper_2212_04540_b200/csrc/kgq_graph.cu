// kgq_graph.cu -- KG neighbour aggregation (K4 CSR SpMM), ReLU + 1-bit mask
// (K5) and the fused per-layer forward (spmm -> quantize H -> H.theta -> relu
// -> mask) for sm_100a.
//
// SpMM is warp-per-row: lane l owns features l + 32c, the row's nonzeros are
// fetched 32 at a time with one coalesced load and broadcast by shuffles, and
// each output element is accumulated in ascending column order as
// acc = acc + a*x with separate mul and add -- the exact order scipy's
// csr_matvecs uses (tensorops.py:8-12, 37-50), so results are bit-identical.
// Up to 8 neighbour rows are in flight per warp to hide L2 latency.
#include "kgq_common.cuh"

namespace kgq {

// Sequential accumulation over the nonzeros of row `row` for the NC feature
// chunks a lane owns (feature l + 32c).  Bit-exact with scipy.
template <int NC>
__device__ __forceinline__ void spmm_row_acc(const int32_t *__restrict__ indptr,
                                             const int32_t *__restrict__ indices,
                                             const float *__restrict__ vals,
                                             const float *__restrict__ x, int d, int64_t row,
                                             int lane, float (&acc)[NC]) {
#pragma unroll
    for (int c = 0; c < NC; c++) acc[c] = 0.0f;
    const int32_t beg = __ldg(indptr + row), end = __ldg(indptr + row + 1);
    for (int32_t base = beg; base < end; base += 32) {
        const int cnt = min(32, end - base);
        int32_t my_col = 0;
        float my_val = 0.0f;
        if (lane < cnt) {
            my_col = __ldg(indices + base + lane);
            my_val = __ldg(vals + base + lane);
        }
        int t = 0;
        for (; t + 8 <= cnt; t += 8) {
            float xv[8][NC];
            float av[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int32_t col = __shfl_sync(0xffffffffu, my_col, t + u);
                av[u] = __shfl_sync(0xffffffffu, my_val, t + u);
                const float *xr = x + (int64_t)col * d + lane;
#pragma unroll
                for (int c = 0; c < NC; c++) xv[u][c] = __ldg(xr + 32 * c);
            }
#pragma unroll
            for (int u = 0; u < 8; u++)
#pragma unroll
                for (int c = 0; c < NC; c++) acc[c] = __fadd_rn(acc[c], __fmul_rn(av[u], xv[u][c]));
        }
        for (; t < cnt; t++) {
            const int32_t col = __shfl_sync(0xffffffffu, my_col, t);
            const float a = __shfl_sync(0xffffffffu, my_val, t);
            const float *xr = x + (int64_t)col * d + lane;
#pragma unroll
            for (int c = 0; c < NC; c++) acc[c] = __fadd_rn(acc[c], __fmul_rn(a, __ldg(xr + 32 * c)));
        }
    }
}

template <int NC>
__global__ void __launch_bounds__(256)
spmm_warp_row_kernel(const int32_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                     const float *__restrict__ vals, int64_t n_rows, const float *__restrict__ x,
                     float *__restrict__ out) {
    constexpr int d = 32 * NC;
    const int lane = threadIdx.x & 31;
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= n_rows) return;
    float acc[NC];
    spmm_row_acc<NC>(indptr, indices, vals, x, d, row, lane, acc);
    float *o = out + row * d + lane;
#pragma unroll
    for (int c = 0; c < NC; c++) o[32 * c] = acc[c];
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
// Fused layer forward, one warp per row:
//   H = A_hat.E (bit-exact spmm), quantize H on chip (group = d, same
//   arithmetic and noise as kgq_quantize_f32), J = H.theta (theta in smem,
//   FFMA, ascending k), E' = relu(J), mask = J > 0.
// Lane l owns features l + 32c, so ballot c is mask word c directly and the
// packed code word for 32/BITS consecutive features is an OR-reduction over
// the lanes that own them.
// ---------------------------------------------------------------------------
template <int NC, int BITS, int MODE>
__global__ void __launch_bounds__(256)
layer_forward_kernel(const int32_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                     const float *__restrict__ vals, int64_t n_rows, const float *__restrict__ e,
                     const float *__restrict__ theta, uint64_t seed, uint64_t tid,
                     int64_t row_offset, uint8_t *__restrict__ codes, float *__restrict__ ranges,
                     float *__restrict__ offsets, float *__restrict__ e_next,
                     uint32_t *__restrict__ mask, float *__restrict__ h_out) {
    constexpr int d = 32 * NC;
    constexpr float Bf = (float)((1u << BITS) - 1u);
    constexpr int LPW = 32 / BITS;                 // lanes (codes) per 32-bit word
    extern __shared__ float th[];   // theta, d*d fp32 (dynamic: 64 KB at d=128)
    for (int i = threadIdx.x; i < d * d; i += blockDim.x) th[i] = theta[i];
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const FastKey fk = make_fast_key(seed, tid);

    for (int64_t row = warp0; row < n_rows; row += nw) {
        float h[NC];
        spmm_row_acc<NC>(indptr, indices, vals, e, d, row, lane, h);
        if (h_out) {
#pragma unroll
            for (int c = 0; c < NC; c++) h_out[row * d + lane + 32 * c] = h[c];
        }
        // ---- quantize H (group = this row) ----
        float mn = h[0], mx = h[0];
#pragma unroll
        for (int c = 1; c < NC; c++) { mn = fminf(mn, h[c]); mx = fmaxf(mx, h[c]); }
        mn = warp_min(mn, 32);
        mx = warp_max(mx, 32);
        const float z = mn, r = __fsub_rn(mx, mn);
        const DivR dv = make_div(r);
        const uint64_t gglob = (uint64_t)(row_offset + row);
#pragma unroll
        for (int c = 0; c < NC; c++) {
            const int k = lane + 32 * c;
            uint32_t code = 0;
            if (r > 0.0f) {
                const float s = __fmul_rn(div_a(dv, __fsub_rn(h[c], z)), Bf);
                uint32_t u16 = 0;
                uint64_t raw53 = 0;
                if (MODE == KGQ_ROUND_SR_FAST) {
                    // lanes 0..3 compute the four calls of this 32-feature chunk;
                    // lane l takes word l&3 of call (l>>2)&3, half (l>>4)&1.
                    uint4 o = make_uint4(0, 0, 0, 0);
                    if (lane < 4) o = fast_call(fk, gglob, (uint32_t)(4 * c + lane));
                    const int src = (lane >> 2) & 3;
                    const uint32_t w0 = __shfl_sync(0xffffffffu, o.x, src);
                    const uint32_t w1 = __shfl_sync(0xffffffffu, o.y, src);
                    const uint32_t w2 = __shfl_sync(0xffffffffu, o.z, src);
                    const uint32_t w3 = __shfl_sync(0xffffffffu, o.w, src);
                    const int wsel = lane & 3;
                    const uint32_t w = wsel == 0 ? w0 : wsel == 1 ? w1 : wsel == 2 ? w2 : w3;
                    u16 = (w >> (16 * ((lane >> 4) & 1))) & 0xFFFFu;
                } else if (MODE == KGQ_ROUND_SR_COMPAT) {
                    raw53 = compat_raw53(seed, tid, gglob, d, k);
                }
                code = code_bits<MODE>(s, __uint2float_rn(u16), raw53) - kMagicBits;
            } else if (MODE == KGQ_ROUND_SR_FAST) {
                // keep the shuffles convergent: nothing to do, code stays 0
            }
            // pack: word (k*BITS)/32 collects lanes with the same k/LPW
            const uint32_t mine = code << ((k % LPW) * BITS);
            const int wib = lane / LPW;               // word index within this chunk
#pragma unroll
            for (int w = 0; w < 32 / LPW; w++) {
                const uint32_t word = __reduce_or_sync(0xffffffffu, wib == w ? mine : 0u);
                if (lane == w) {
                    reinterpret_cast<uint32_t *>(codes + row * (d * BITS / 8))[c * (32 / LPW) + w] = word;
                }
            }
        }
        if (lane == 0) {
            ranges[row] = r;
            offsets[row] = z;
        }
        // ---- J = H . theta ----
        float j[NC];
#pragma unroll
        for (int c = 0; c < NC; c++) j[c] = 0.0f;
#pragma unroll
        for (int cc = 0; cc < NC; cc++) {
#pragma unroll 8
            for (int kl = 0; kl < 32; kl++) {
                const float hk = __shfl_sync(0xffffffffu, h[cc], kl);
                const float *trow = th + (32 * cc + kl) * d + lane;
#pragma unroll
                for (int c = 0; c < NC; c++) j[c] = __fmaf_rn(hk, trow[32 * c], j[c]);
            }
        }
        // ---- relu + mask ----
#pragma unroll
        for (int c = 0; c < NC; c++) {
            const bool pos = j[c] > 0.0f;
            const uint32_t bal = __ballot_sync(0xffffffffu, pos);
            e_next[row * d + lane + 32 * c] = pos ? j[c] : 0.0f;
            if (lane == 0) mask[row * NC + c] = bal;
        }
    }
}

}  // namespace kgq

using namespace kgq;

static inline int blocks_for_warps(int64_t warps) {
    int64_t b = (warps + 7) / 8;
    if (b < 1) b = 1;
    if (b > 0x7fffffff) b = 0x7fffffff;
    return (int)b;
}

extern "C" int kgq_spmm_csr_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                                int64_t n_rows, const float *x, int32_t d, float *out,
                                void *stream) {
    if (n_rows < 0 || d < 1) return KGQ_ERR_INVALID_ARG;
    if (n_rows == 0) return KGQ_OK;
    if (!indptr || !out || !x) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = blocks_for_warps(n_rows);
    switch (d) {
        case 32: spmm_warp_row_kernel<1><<<grid, 256, 0, s>>>(indptr, indices, vals, n_rows, x, out); break;
        case 64: spmm_warp_row_kernel<2><<<grid, 256, 0, s>>>(indptr, indices, vals, n_rows, x, out); break;
        case 128: spmm_warp_row_kernel<4><<<grid, 256, 0, s>>>(indptr, indices, vals, n_rows, x, out); break;
        case 256: spmm_warp_row_kernel<8><<<grid, 256, 0, s>>>(indptr, indices, vals, n_rows, x, out); break;
        default: spmm_generic_kernel<<<grid, 256, 0, s>>>(indptr, indices, vals, n_rows, x, d, out); break;
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

template <int NC, int BITS>
static int launch_layer(int rounding, const int32_t *indptr, const int32_t *indices, const float *vals,
                        int64_t n_rows, const float *e, const float *theta, uint64_t seed,
                        uint64_t tid, int64_t row_offset, uint8_t *codes, float *ranges,
                        float *offsets, float *e_next, uint32_t *mask, float *h_out,
                        cudaStream_t s) {
    constexpr int d = 32 * NC;
    const size_t smem = (size_t)d * d * sizeof(float);
    int64_t blocks = (n_rows + 7) / 8;
    if (blocks > (int64_t)kSMs * 8) blocks = (int64_t)kSMs * 8;
    if (blocks < 1) blocks = 1;
    void (*kern)(const int32_t *, const int32_t *, const float *, int64_t, const float *,
                 const float *, uint64_t, uint64_t, int64_t, uint8_t *, float *, float *, float *,
                 uint32_t *, float *);
    switch (rounding) {
        case KGQ_ROUND_NEAREST: kern = layer_forward_kernel<NC, BITS, KGQ_ROUND_NEAREST>; break;
        case KGQ_ROUND_SR_FAST: kern = layer_forward_kernel<NC, BITS, KGQ_ROUND_SR_FAST>; break;
        case KGQ_ROUND_SR_COMPAT: kern = layer_forward_kernel<NC, BITS, KGQ_ROUND_SR_COMPAT>; break;
        default: return KGQ_ERR_INVALID_ARG;
    }
    if (smem > 48 * 1024) {
        cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
    }
    kern<<<(int)blocks, 256, smem, s>>>(indptr, indices, vals, n_rows, e, theta, seed, tid, row_offset,
                                        codes, ranges, offsets, e_next, mask, h_out);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

template <int NC>
static int launch_layer_bits(int bits, int rounding, const int32_t *indptr, const int32_t *indices,
                             const float *vals, int64_t n_rows, const float *e, const float *theta,
                             uint64_t seed, uint64_t tid, int64_t row_offset, uint8_t *codes,
                             float *ranges, float *offsets, float *e_next, uint32_t *mask,
                             float *h_out, cudaStream_t s) {
    switch (bits) {
        case 1: return launch_layer<NC, 1>(rounding, indptr, indices, vals, n_rows, e, theta, seed, tid, row_offset, codes, ranges, offsets, e_next, mask, h_out, s);
        case 2: return launch_layer<NC, 2>(rounding, indptr, indices, vals, n_rows, e, theta, seed, tid, row_offset, codes, ranges, offsets, e_next, mask, h_out, s);
        case 4: return launch_layer<NC, 4>(rounding, indptr, indices, vals, n_rows, e, theta, seed, tid, row_offset, codes, ranges, offsets, e_next, mask, h_out, s);
        case 8: return launch_layer<NC, 8>(rounding, indptr, indices, vals, n_rows, e, theta, seed, tid, row_offset, codes, ranges, offsets, e_next, mask, h_out, s);
    }
    return KGQ_ERR_UNSUPPORTED_BITS;
}

extern "C" int kgq_layer_forward_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                                     int64_t n_rows, const float *e, int32_t d, const float *theta,
                                     int32_t bits, int32_t rounding, uint64_t seed,
                                     uint64_t tensor_id, int64_t row_offset, uint8_t *codes,
                                     float *ranges, float *offsets, float *e_next, uint8_t *mask,
                                     float *h_out, void *stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (n_rows < 0 || row_offset < 0 || rounding < 0 || rounding > 2) return KGQ_ERR_INVALID_ARG;
    if (n_rows == 0) return KGQ_OK;
    if (!indptr || !e || !theta || !codes || !ranges || !offsets || !e_next || !mask)
        return KGQ_ERR_INVALID_ARG;
    if (((uintptr_t)mask & 3u) || ((uintptr_t)codes & 3u)) return KGQ_ERR_MISALIGNED;
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *m32 = reinterpret_cast<uint32_t *>(mask);
    switch (d) {
        case 32: return launch_layer_bits<1>(bits, rounding, indptr, indices, vals, n_rows, e, theta, seed, tensor_id, row_offset, codes, ranges, offsets, e_next, m32, h_out, s);
        case 64: return launch_layer_bits<2>(bits, rounding, indptr, indices, vals, n_rows, e, theta, seed, tensor_id, row_offset, codes, ranges, offsets, e_next, m32, h_out, s);
        case 128: return launch_layer_bits<4>(bits, rounding, indptr, indices, vals, n_rows, e, theta, seed, tensor_id, row_offset, codes, ranges, offsets, e_next, m32, h_out, s);
    }
    return KGQ_ERR_INVALID_ARG;
}
