// kgq_rowmm.cu -- out[rows][D] = A[rows][D] . theta (or theta^T) on the 5th-gen
// tensor cores (tcgen05, kind::tf32, 3xTF32 split for fp32-level accuracy).
// The dense d x d layer GEMMs of the backward pass (dH = g . theta^T,
// tape.py:223) run here.  One CTA per 128-row tile: 256 threads stage the
// tile (split hi/lo) into shared memory in the interleaved K-major layout,
// one thread issues 3 x D/8 MMAs into a TMEM accumulator (D fp32 columns),
// commits to an mbarrier, and all 8 warps drain TMEM with tcgen05.ld.
#include "kgq_tc.cuh"

namespace kgq {

template <int D, bool TRANS>
__global__ void __launch_bounds__(256)
rowmm_tc_kernel(const float *__restrict__ a, int64_t rows, const float *__restrict__ theta,
                float *__restrict__ out) {
    constexpr int M = 128;
    extern __shared__ __align__(128) float sm[];
    float *ah = sm, *al = sm + M * D;              // [M x D] each
    float *bh = sm + 2 * M * D, *bl = bh + D * D;  // [D x D] each (B(n, k), K-major)
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;

    // B(n, k) = theta[k][n] (out = A.theta) or theta[n][k] (out = A.theta^T)
    for (int i = t; i < D * D; i += 256) {
        const int n = i / D, k = i % D;
        const float x = TRANS ? __ldg(theta + n * D + k) : __ldg(theta + k * D + n);
        float hi, lo;
        tc::split_tf32(x, hi, lo);
        bh[tc::tile_off(n, k, D) / 4] = hi;
        bl[tc::tile_off(n, k, D) / 4] = lo;
    }
    if (t == 0) tc::mbar_init(&mbar, 1);
    if (warp == 0) tc::tmem_alloc(&tmem_base, D < 32 ? 32 : D);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;

    uint32_t phase = 0;
    const int64_t n_tiles = (rows + M - 1) / M;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t r0 = tile * M;
        // stage A: thread t -> row t/2, columns [ (t&1)*D/2, +D/2 )
        {
            const int r = t >> 1, c0 = (t & 1) * (D / 2);
            const bool ok = r0 + r < rows;
            const float4 *src = reinterpret_cast<const float4 *>(a + (r0 + r) * D + c0);
#pragma unroll
            for (int v = 0; v < D / 8; v++) {
                const float4 x = ok ? __ldg(src + v) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    float hi, lo;
                    tc::split_tf32(xs[e], hi, lo);
                    const uint32_t off = tc::tile_off(r, c0 + 4 * v + e, M) / 4;
                    ah[off] = hi;
                    al[off] = lo;
                }
            }
        }
        tc::fence_proxy_async();
        __syncthreads();
        if (t == 0) {
            tc::fence_after();
            tc::mma_3xtf32<M, D, D>(tmem, ah, al, bh, bl);
            tc::commit(&mbar);
        }
        tc::mbar_wait(&mbar, phase);
        phase ^= 1u;
        tc::fence_after();
        // drain: warp w reads TMEM lanes 32*(w%4).., columns (w/4)*32.. (D=32: warps 0-3 only)
        if (D >= 64 || warp < 4) {
            const int q = warp & 3, half = warp >> 2;
#pragma unroll
            for (int cb = half * 32; cb < D; cb += (D >= 64 ? 64 : 32)) {
                float v[32];
                tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)cb, v);
                const int64_t row = r0 + 32 * q + lane;
                if (row < rows) {
                    float4 *dst = reinterpret_cast<float4 *>(out + row * D + cb);
#pragma unroll
                    for (int j = 0; j < 8; j++)
                        dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                }
            }
        }
        tc::fence_before();
        __syncthreads();
    }
    if (warp == 0) tc::tmem_free(tmem, D < 32 ? 32 : D);
}

}  // namespace kgq

using namespace kgq;

template <int D, bool TR>
static int launch_rowmm(const float *a, int64_t rows, const float *theta, float *out, cudaStream_t s) {
    const size_t smem = (size_t)(2 * 128 * D + 2 * D * D) * sizeof(float);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(rowmm_tc_kernel<D, TR>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return kgq_set_cuda_error(e);
        attr = true;
    }
    int64_t tiles = (rows + 127) / 128;
    const int grid = (int)(tiles < (int64_t)kSMs * 2 ? tiles : (int64_t)kSMs * 2);
    rowmm_tc_kernel<D, TR><<<grid, 256, smem, s>>>(a, rows, theta, out);
    return KGQ_OK;
}

extern "C" int kgq_rowmm_f32(const float *a, int64_t rows, int32_t d, const float *theta,
                             int32_t transpose_theta, float *out, void *stream) {
    if (rows < 0) return KGQ_ERR_INVALID_ARG;
    if (d != 32 && d != 64) return KGQ_ERR_INVALID_ARG;       // caller falls back (cuBLAS)
    if (rows == 0) return KGQ_OK;
    if (!a || !theta || !out) return KGQ_ERR_INVALID_ARG;
    if ((((uintptr_t)a) | ((uintptr_t)out)) & 15u) return KGQ_ERR_MISALIGNED;
    cudaStream_t s = (cudaStream_t)stream;
    int st;
    if (d == 64) st = transpose_theta ? launch_rowmm<64, true>(a, rows, theta, out, s)
                                      : launch_rowmm<64, false>(a, rows, theta, out, s);
    else st = transpose_theta ? launch_rowmm<32, true>(a, rows, theta, out, s)
                              : launch_rowmm<32, false>(a, rows, theta, out, s);
    if (st != KGQ_OK) return st;
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
