// kgq_gemm.cu -- K3: fused decompressor -> weight gradient (tape.py:219-222)
//   dtheta (+)= dequantize(ctx)^T @ g,   ctx = per-row quantized H [rows][d]
// The dequantized activation only ever exists in shared memory.
//
// Each CTA owns a fixed set of 32-row chunks (deterministic grid), stages the
// chunk's g rows (fp32) and its dequantized H rows (bit-exact with
// dequantize_tensor) in shared memory, and accumulates the full d x d product
// in registers: an 8x8 register tile per thread, (d/8)^2 threads per tile,
// 256/(d/8)^2 row slices per CTA.  Slices and CTAs are reduced in a fixed
// order, so the result is run-to-run deterministic.
#include "kgq_common.cuh"

namespace kgq {

constexpr int kGemmThreads = 256;
constexpr int kChunkRows = 64;

static inline int dq_gemm_grid(int64_t rows) {
    int64_t chunks = (rows + kChunkRows - 1) / kChunkRows;
    int64_t g = chunks < (int64_t)kSMs ? chunks : (int64_t)kSMs;   // 1 CTA per SM (135 regs)
    return g < 1 ? 1 : (int)g;
}

// Each CTA walks a fixed set of 64-row chunks.  The next chunk's g rows
// (float4), packed code bytes and (R, Z) are prefetched into registers while
// the current chunk is dequantized into shared memory (bit-exact with
// dequantize_tensor) and accumulated into 8x8 FFMA register tiles.
template <int D, int BITS>
__global__ void __launch_bounds__(kGemmThreads)
dequant_gemm_tn_kernel(const uint8_t *__restrict__ codes, const float *__restrict__ ranges,
                       const float *__restrict__ offsets, int64_t rows,
                       const float *__restrict__ g, float *__restrict__ partial) {
    constexpr int T8 = D / 8;               // 8x8 tiles per dimension
    constexpr int TT = T8 * T8;             // threads per full d x d tile
    constexpr int S = kGemmThreads / TT;    // row slices
    constexpr int RB = D * BITS / 8;        // packed bytes per row
    constexpr int GV = kChunkRows * D / 4 / kGemmThreads;   // g float4 per thread per chunk
    constexpr int CW = (kChunkRows * RB / 4 + kGemmThreads - 1) / kGemmThreads;  // code words per thread
    constexpr int EPT = kChunkRows * D / kGemmThreads;      // dequantized elements per thread
    constexpr uint32_t MASK = (1u << BITS) - 1u;
    extern __shared__ __align__(16) float sm[];
    float *hs = sm;                                          // [kChunkRows][D]
    float *gs = sm + kChunkRows * D;                         // [kChunkRows][D]
    uint32_t *cs = reinterpret_cast<uint32_t *>(gs + kChunkRows * D);   // [kChunkRows*RB/4]
    float *rz = reinterpret_cast<float *>(cs + kChunkRows * RB / 4);    // [2][kChunkRows]

    const int t = threadIdx.x;
    const int slice = t / TT, tt = t % TT;
    const int ti = tt / T8, tj = tt % T8;
    float acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 8; b++) acc[a][b] = 0.0f;

    const int64_t n_chunks = (rows + kChunkRows - 1) / kChunkRows;
    float4 pg[GV];
    uint32_t pc[CW];
    float pr = 0.f, pz = 0.f;
    auto prefetch = [&](int64_t ch) {
        const int64_t r0 = ch * kChunkRows;
        const int nr = (int)imin64(kChunkRows, rows - r0);
#pragma unroll
        for (int m = 0; m < GV; m++) {
            const int i = t + kGemmThreads * m, rr = (i * 4) / D;
            pg[m] = rr < nr ? __ldg(reinterpret_cast<const float4 *>(g + r0 * D) + i)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int m = 0; m < CW; m++) {
            const int i = t + kGemmThreads * m;
            pc[m] = (i < kChunkRows * RB / 4 && i * 4 < nr * RB)
                        ? __ldg(reinterpret_cast<const uint32_t *>(codes + r0 * RB) + i) : 0u;
        }
        if (t < kChunkRows) {
            pr = t < nr ? __ldg(ranges + r0 + t) : 0.f;
            pz = t < nr ? __ldg(offsets + r0 + t) : 0.f;
        }
    };
    int64_t ch = blockIdx.x;
    if (ch < n_chunks) prefetch(ch);
    for (; ch < n_chunks; ch += gridDim.x) {
        const int nr = (int)imin64(kChunkRows, rows - ch * kChunkRows);
#pragma unroll
        for (int m = 0; m < GV; m++) reinterpret_cast<float4 *>(gs)[t + kGemmThreads * m] = pg[m];
#pragma unroll
        for (int m = 0; m < CW; m++)
            if (t + kGemmThreads * m < kChunkRows * RB / 4) cs[t + kGemmThreads * m] = pc[m];
        if (t < kChunkRows) { rz[t] = pr; rz[kChunkRows + t] = pz; }
        __syncthreads();
        if (ch + gridDim.x < n_chunks) prefetch(ch + gridDim.x);
        // dequantize: (R*c)/B + Z, R == 0 -> Z (quantize.py:206-209); rows past the end -> 0
        {
            const int rr = (t * EPT) / D, k0 = (t * EPT) % D;
            const float r = rz[rr], z = rz[kChunkRows + rr];
            const uint8_t *cb = reinterpret_cast<const uint8_t *>(cs) + rr * RB;
#pragma unroll
            for (int e = 0; e < EPT; e++) {
                const int bit = (k0 + e) * BITS;
                const uint32_t c = (cb[bit >> 3] >> (bit & 7)) & MASK;
                hs[rr * D + k0 + e] = rr < nr ? lut_entry<BITS>(r, z, (int)c) : 0.0f;
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int rr = slice; rr < kChunkRows; rr += S) {
            const float4 a0 = *reinterpret_cast<const float4 *>(hs + rr * D + ti * 8);
            const float4 a1 = *reinterpret_cast<const float4 *>(hs + rr * D + ti * 8 + 4);
            const float4 b0 = *reinterpret_cast<const float4 *>(gs + rr * D + tj * 8);
            const float4 b1 = *reinterpret_cast<const float4 *>(gs + rr * D + tj * 8 + 4);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
                for (int b = 0; b < 8; b++) acc[a][b] = __fmaf_rn(av[a], bv[b], acc[a][b]);
        }
        __syncthreads();
    }
    // reduce the S slices in order (reuse the staging smem: needs D*D floats)
    float *red = sm;
    for (int s = 0; s < S; s++) {
        if (slice == s) {
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
                for (int b = 0; b < 8; b++) {
                    float *p = red + (ti * 8 + a) * D + tj * 8 + b;
                    *p = (s == 0) ? acc[a][b] : __fadd_rn(*p, acc[a][b]);
                }
        }
        __syncthreads();
    }
    float *dst = partial + (int64_t)blockIdx.x * D * D;
    for (int i = t; i < D * D; i += kGemmThreads) dst[i] = red[i];
}

// Fixed-order reduction of the per-CTA partials: 8 interleaved ascending
// chains (partials p = u mod 8) combined as ((0+1)+(2+3))+((4+5)+(6+7)) ->
// deterministic.  A CTA owns 32 consecutive outputs, warp u runs chain u.
__global__ void __launch_bounds__(256)
reduce_partials_kernel(const float *__restrict__ partial, int nparts, int dd,
                       float *__restrict__ out, int accumulate) {
    __shared__ float s8[8][32];
    const int c = threadIdx.x & 31, u = threadIdx.x >> 5;
    const int i = blockIdx.x * 32 + c;
    float acc = 0.0f;
    if (i < dd) {
#pragma unroll 4
        for (int p = u; p < nparts; p += 8) acc = __fadd_rn(acc, __ldg(partial + (int64_t)p * dd + i));
    }
    s8[u][c] = acc;
    __syncthreads();
    if (u == 0 && i < dd) {
        const float sum = __fadd_rn(__fadd_rn(__fadd_rn(s8[0][c], s8[1][c]), __fadd_rn(s8[2][c], s8[3][c])),
                                    __fadd_rn(__fadd_rn(s8[4][c], s8[5][c]), __fadd_rn(s8[6][c], s8[7][c])));
        out[i] = accumulate ? __fadd_rn(out[i], sum) : sum;
    }
}

// any d (correctness path): thread per output element, rows in order.
__global__ void dequant_gemm_generic_kernel(const uint8_t *__restrict__ codes,
                                            const float *__restrict__ ranges,
                                            const float *__restrict__ offsets, int64_t rows,
                                            int d, int bits, const float *__restrict__ g,
                                            float *__restrict__ out, int accumulate) {
    const int RB = (d * bits + 7) / 8;
    const float Bf = (float)((1u << bits) - 1u);
    const uint32_t mask = (1u << bits) - 1u;
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < d * d; o += gridDim.x * blockDim.x) {
        const int i = o / d, jj = o % d;
        float s = 0.0f;
        const int bit = i * bits;
        for (int64_t n = 0; n < rows; n++) {
            const uint32_t c = (codes[n * RB + (bit >> 3)] >> (bit & 7)) & mask;
            const float r = ranges[n], z = offsets[n];
            const float h = (r == 0.0f) ? z : __fadd_rn(__fdiv_rn(__fmul_rn(r, (float)c), Bf), z);
            s = __fmaf_rn(h, g[n * d + jj], s);
        }
        out[o] = accumulate ? __fadd_rn(out[o], s) : s;
    }
}

template <int D>
static int launch_dq_gemm(int bits, const uint8_t *codes, const float *ranges, const float *offsets,
                          int64_t rows, const float *g, float *partial, cudaStream_t s) {
    const int grid = dq_gemm_grid(rows);
    size_t smem = (size_t)2 * kChunkRows * D * sizeof(float) + (size_t)kChunkRows * D * bits / 8 +
                  2 * kChunkRows * sizeof(float);
    if (smem < (size_t)D * D * sizeof(float)) smem = (size_t)D * D * sizeof(float);
    void (*kern)(const uint8_t *, const float *, const float *, int64_t, const float *, float *);
    switch (bits) {
        case 1: kern = dequant_gemm_tn_kernel<D, 1>; break;
        case 2: kern = dequant_gemm_tn_kernel<D, 2>; break;
        case 4: kern = dequant_gemm_tn_kernel<D, 4>; break;
        case 8: kern = dequant_gemm_tn_kernel<D, 8>; break;
        default: return KGQ_ERR_UNSUPPORTED_BITS;
    }
    if (smem > 48 * 1024) {
        cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return kgq_set_cuda_error(ea);
    }
    kern<<<grid, kGemmThreads, smem, s>>>(codes, ranges, offsets, rows, g, partial);
    return KGQ_OK;
}

}  // namespace kgq

using namespace kgq;

extern "C" size_t kgq_dequant_gemm_workspace_bytes(int64_t rows, int32_t d) {
    if (d == 32 || d == 64 || d == 128) return (size_t)dq_gemm_grid(rows) * d * d * sizeof(float);
    return 0;
}

extern "C" int kgq_dequant_gemm_tn_f32(const uint8_t *codes, const float *ranges,
                                       const float *offsets, int64_t rows, int32_t d, int32_t bits,
                                       const float *g, float *dtheta, void *workspace,
                                       size_t workspace_bytes, int32_t accumulate, void *stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (rows < 0 || d < 1 || !dtheta) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (rows == 0) {
        if (!accumulate) {
            cudaError_t e = cudaMemsetAsync(dtheta, 0, (size_t)d * d * sizeof(float), s);
            if (e != cudaSuccess) return kgq_set_cuda_error(e);
        }
        return KGQ_OK;
    }
    if (!codes || !ranges || !offsets || !g) return KGQ_ERR_INVALID_ARG;
    const bool fast = (d == 32 || d == 64 || d == 128) && (((uintptr_t)g & 15u) == 0);
    if (fast) {
        const size_t need = kgq_dequant_gemm_workspace_bytes(rows, d);
        if (!workspace || workspace_bytes < need) return KGQ_ERR_INVALID_ARG;
        float *partial = reinterpret_cast<float *>(workspace);
        int st = KGQ_OK;
        switch (d) {
            case 32: st = launch_dq_gemm<32>(bits, codes, ranges, offsets, rows, g, partial, s); break;
            case 64: st = launch_dq_gemm<64>(bits, codes, ranges, offsets, rows, g, partial, s); break;
            case 128: st = launch_dq_gemm<128>(bits, codes, ranges, offsets, rows, g, partial, s); break;
        }
        if (st != KGQ_OK) return st;
        const int dd = d * d;
        reduce_partials_kernel<<<(dd + 31) / 32, 256, 0, s>>>(partial, dq_gemm_grid(rows), dd,
                                                                dtheta, accumulate);
    } else {
        dequant_gemm_generic_kernel<<<(d * d + 255) / 256, 256, 0, s>>>(
            codes, ranges, offsets, rows, d, bits, g, dtheta, accumulate);
    }
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
