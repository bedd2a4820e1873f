// kgq_backward.cu -- fused per-layer backward of the KGNN layer (tape.py:217-225,
// SURVEY.md 8(f) rank 1), d in {32, 64, 128}:
//
//   g_j   = (g_read + g_e) * mask                      (relu backward, tape.py:224-225)
//   dH    = g_j . theta^T                              (mm backward, tape.py:223)
//   dtheta += Hhat^T . g_j, Hhat = dequant(ctx)        (mm backward, tape.py:220-222)
//
// in one pass over the rows: g_j and the dequantized Hhat exist only in
// registers / shared memory.  Each CTA walks 32-row chunks (8 warps x 4 rows);
// lane l owns columns l + 32c.  dH uses theta^T staged in smem (broadcast
// LDS of g_j, conflict-free LDS of theta^T, FFMA); dtheta is accumulated in a
// TSxTS register tile per thread (TS = 4 for d <= 64, 8 for d = 128, so the
// d*d/TS^2 tiles fit 256 threads) over the CTA's rows and reduced across CTAs
// in a fixed order (deterministic).  dH then feeds the SpMM (A_hat^T = A_hat).
// Shared memory is dynamic: theta^T d*d + g_j, Hhat 2*32*d + g_j k-major 32*d
// floats (112 KB at d = 128).
#include "kgq_common.cuh"
#include <cstdlib>

namespace kgq {

constexpr int kBwdRows = 32;   // rows per chunk (8 warps x 4)

static inline int bwd_grid(int64_t rows) {
    int64_t chunks = (rows + kBwdRows - 1) / kBwdRows;
    int64_t g = chunks < (int64_t)kSMs * 2 ? chunks : (int64_t)kSMs * 2;
    return g < 1 ? 1 : (int)g;
}

template <int D>
struct BwdSmem {
    static constexpr size_t bytes = ((size_t)D * D + 3 * (size_t)kBwdRows * D) * sizeof(float);
};

#ifndef KGQ_BWD_MINB
#define KGQ_BWD_MINB 1
#endif
template <int D, int BITS>
#ifndef KGQ_BWD128_MINB
#define KGQ_BWD128_MINB 1
#endif
__global__ void __launch_bounds__(256, D > 64 ? KGQ_BWD128_MINB : KGQ_BWD_MINB)
layer_backward_kernel(const float *__restrict__ g_read, const float *__restrict__ g_e,
                      const uint32_t *__restrict__ mask, const uint8_t *__restrict__ codes,
                      const float *__restrict__ ranges, const float *__restrict__ offsets,
                      int64_t rows, const float *__restrict__ theta, float *__restrict__ dh,
                      float *__restrict__ partial) {
    constexpr int NC = D / 32;                     // columns per lane
    constexpr int RB = D * BITS / 8;
    constexpr uint32_t CM = BITS >= 32 ? 0xFFFFFFFFu : (1u << BITS) - 1u;
    constexpr int TS = D > 64 ? 8 : 4;             // dtheta register tile
    constexpr int TPD = D / TS;                    // tiles per dimension (TPD^2 <= 256)
    static_assert(TPD * TPD <= 256, "dtheta tiles exceed the CTA");
    extern __shared__ __align__(16) float bwd_smem[];
    float *tht = bwd_smem;                                                   // theta^T [D][D]
    auto gs = reinterpret_cast<float (*)[D]>(bwd_smem + D * D);              // g_j [32][D]
    auto hs = reinterpret_cast<float (*)[D]>(bwd_smem + D * D + kBwdRows * D);   // Hhat [32][D]
    auto gk = reinterpret_cast<float (*)[D][4]>(bwd_smem + D * D + 2 * kBwdRows * D);  // [8][D][4]
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int i = t; i < D * D; i += 256) {
        const int j = i / D, k = i % D;
        tht[k * D + j] = __ldg(theta + i);         // theta[j][k]
    }
    const bool owner = t < TPD * TPD;
    const int ti = (t / TPD) * TS, tj = (t % TPD) * TS;
    float acc[TS][TS];
#pragma unroll
    for (int a = 0; a < TS; a++)
#pragma unroll
        for (int b = 0; b < TS; b++) acc[a][b] = 0.0f;

    // register prefetch of one chunk: this warp's 4 rows, columns lane + 32c
    float pg[4][NC], pe[4][NC], pr[4], pz[4];
    uint32_t pm[4][NC], pc[4][NC];
    auto load = [&](int64_t ch) {
#pragma unroll
        for (int rr = 0; rr < 4; rr++) {
            const int64_t row = ch * kBwdRows + warp * 4 + rr;
            const bool ok = row < rows;
            pr[rr] = (ok && BITS != 32) ? __ldg(ranges + row) : 0.f;
            pz[rr] = (ok && BITS != 32) ? __ldg(offsets + row) : 0.f;
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const int col = lane + 32 * c;
                pg[rr][c] = (ok && g_read) ? __ldg(g_read + row * D + col) : 0.f;
                pe[rr][c] = (ok && g_e) ? __ldg(g_e + row * D + col) : 0.f;
                pm[rr][c] = ok ? __ldg(mask + row * (D / 32) + c) : 0u;
                const int b = col * BITS;
                if (BITS == 32)        // pass-through context: codes holds the fp32 H
                    pc[rr][c] = ok ? __float_as_uint(__ldg(reinterpret_cast<const float *>(codes) + row * D + col)) : 0u;
                else
                    pc[rr][c] = ok ? __ldg(codes + row * RB + (b >> 3)) : 0u;
            }
        }
    };
    __syncthreads();

    const int64_t n_chunks = (rows + kBwdRows - 1) / kBwdRows;
    int64_t ch = blockIdx.x;
    if (ch < n_chunks) load(ch);
    for (; ch < n_chunks; ch += gridDim.x) {
        // ---- stage g_j = (g_read + g_e) * mask and Hhat from the prefetched registers ----
#pragma unroll
        for (int rr = 0; rr < 4; rr++) {
            const int lr = warp * 4 + rr;
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const int col = lane + 32 * c;
                // g = g_read + g_e in the reference's routing order (tape.py:204-209)
                const float g = (g_read && g_e) ? __fadd_rn(pg[rr][c], pe[rr][c]) : (g_read ? pg[rr][c] : pe[rr][c]);
                const float gj = __fmul_rn(g, ((pm[rr][c] >> lane) & 1u) ? 1.0f : 0.0f);
                const int b = col * BITS;
                const uint32_t code = BITS == 32 ? 0u : (pc[rr][c] >> (b & 7)) & CM;
                gs[lr][col] = gj;
                gk[warp][col][rr] = gj;
                hs[lr][col] = BITS == 32 ? __uint_as_float(pc[rr][c]) : lut_entry<BITS <= 8 ? BITS : 8>(pr[rr], pz[rr], (int)code);
            }
        }
        if (ch + gridDim.x < n_chunks) load(ch + gridDim.x);
        __syncwarp();
        // ---- dH for the warp's 4 rows: dh[r][j] = sum_k g_j[r][k] theta[j][k] ----
        {
            float o[4][NC];
#pragma unroll
            for (int rr = 0; rr < 4; rr++)
#pragma unroll
                for (int c = 0; c < NC; c++) o[rr][c] = 0.0f;
#pragma unroll 8
            for (int k = 0; k < D; k++) {
                const float4 g4 = *reinterpret_cast<const float4 *>(&gk[warp][k][0]);
                const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    const float tk = tht[k * D + lane + 32 * c];
#pragma unroll
                    for (int rr = 0; rr < 4; rr++) o[rr][c] = __fmaf_rn(gv[rr], tk, o[rr][c]);
                }
            }
#pragma unroll
            for (int rr = 0; rr < 4; rr++) {
                const int64_t row = ch * kBwdRows + warp * 4 + rr;
                if (row < rows) {
#pragma unroll
                    for (int c = 0; c < NC; c++) dh[row * D + lane + 32 * c] = o[rr][c];
                }
            }
        }
        __syncthreads();
        // ---- dtheta += Hhat^T g_j over the chunk's 32 rows (rows past the end are 0) ----
        if (owner) {
#pragma unroll 4
            for (int rr = 0; rr < kBwdRows; rr++) {
                float av[TS], bv[TS];
#pragma unroll
                for (int v = 0; v < TS / 4; v++) {
                    const float4 a4 = *reinterpret_cast<const float4 *>(&hs[rr][ti + 4 * v]);
                    const float4 b4 = *reinterpret_cast<const float4 *>(&gs[rr][tj + 4 * v]);
                    av[4 * v] = a4.x; av[4 * v + 1] = a4.y; av[4 * v + 2] = a4.z; av[4 * v + 3] = a4.w;
                    bv[4 * v] = b4.x; bv[4 * v + 1] = b4.y; bv[4 * v + 2] = b4.z; bv[4 * v + 3] = b4.w;
                }
#pragma unroll
                for (int a = 0; a < TS; a++)
#pragma unroll
                    for (int b = 0; b < TS; b++) acc[a][b] = __fmaf_rn(av[a], bv[b], acc[a][b]);
            }
        }
        __syncthreads();
    }
    if (owner) {
        float *dst = partial + (int64_t)blockIdx.x * D * D;
#pragma unroll
        for (int a = 0; a < TS; a++)
#pragma unroll
            for (int v = 0; v < TS / 4; v++)
                *reinterpret_cast<float4 *>(dst + (ti + a) * D + tj + 4 * v) =
                    make_float4(acc[a][4 * v], acc[a][4 * v + 1], acc[a][4 * v + 2], acc[a][4 * v + 3]);
    }
}

// dtheta[i] = sum over the CTA partials in a fixed order: 32 interleaved
// ascending chains (partials p = c mod 32, c = the thread's chain), combined
// by a fixed pairwise tree.  A CTA (1024 threads) owns 32 consecutive outputs;
// each thread loads its <= ceil(nparts / 32) partials at once (coalesced
// 128-byte rows per warp), so the kernel is one load round trip deep.
__global__ void __launch_bounds__(1024)
reduce_partials_bwd_kernel(const float *__restrict__ partial, int nparts, int dd,
                           float *__restrict__ out, int accumulate) {
    __shared__ float s[32][33];
    const int o = threadIdx.x & 31, c = threadIdx.x >> 5;
    const int i = blockIdx.x * 32 + o;
    float acc = 0.0f;
    if (i < dd) {
        constexpr int KB = 8;
        for (int p0 = c; p0 < nparts; p0 += 32 * KB) {
            float v[KB];
#pragma unroll
            for (int k = 0; k < KB; k++) {
                const int p = p0 + 32 * k;
                v[k] = p < nparts ? __ldg(partial + (int64_t)p * dd + i) : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < KB; k++)
                if (p0 + 32 * k < nparts) acc = __fadd_rn(acc, v[k]);
        }
    }
    s[c][o] = acc;
    __syncthreads();
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        if (c < w) s[c][o] = __fadd_rn(s[c][o], s[c + w][o]);
        __syncthreads();
    }
    if (c == 0 && i < dd) out[i] = accumulate ? __fadd_rn(out[i], s[0][o]) : s[0][o];
}

}  // namespace kgq

using namespace kgq;

// d = 64 and 128: the tcgen05 kernels (kgq_backward_tc.cu) by default;
// KGQ_BWD_TC=0 selects the FFMA kernel below (read once).  Amazon shape,
// inside the training step: 31.1 us vs 110 us (d = 64); 105 vs 337 us (d = 128).
int kgq_launch_layer_backward_tc(const float *g_read, const float *g_e, const uint32_t *mask,
                                 const uint8_t *codes, const float *ranges, const float *offsets,
                                 int64_t rows, int32_t d, int32_t bits, const float *theta, float *dh,
                                 float *partial, int grid, cudaStream_t s, const int32_t *gr_map = nullptr,
                                 const float *gr_rows = nullptr);
static bool use_tc_backward() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("KGQ_BWD_TC");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

extern "C" size_t kgq_layer_backward_workspace_bytes(int64_t rows, int32_t d) {
    if (d != 32 && d != 64 && d != 128) return 0;
    return (size_t)bwd_grid(rows) * d * d * sizeof(float);
}

extern "C" int kgq_layer_backward_f32(const float *g_read, const float *g_e, const uint8_t *mask,
                                      const uint8_t *codes, const float *ranges,
                                      const float *offsets, int64_t rows, int32_t d, int32_t bits,
                                      const float *theta, float *dh, float *dtheta,
                                      void *workspace, size_t workspace_bytes, int32_t accumulate,
                                      void *stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8 || bits == 32)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (d != 32 && d != 64 && d != 128) return KGQ_ERR_INVALID_ARG;   // caller falls back (unfused)
    if (rows < 0) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (rows == 0) {
        if (!accumulate) {
            cudaError_t e = cudaMemsetAsync(dtheta, 0, (size_t)d * d * sizeof(float), s);
            if (e != cudaSuccess) return kgq_set_cuda_error(e);
        }
        return KGQ_OK;
    }
    if ((!g_read && !g_e) || !mask || !codes || !theta || !dh || !dtheta) return KGQ_ERR_INVALID_ARG;
    if (bits != 32 && (!ranges || !offsets)) return KGQ_ERR_INVALID_ARG;
    if (((uintptr_t)mask) & 3u) return KGQ_ERR_MISALIGNED;
    if (!workspace || workspace_bytes < kgq_layer_backward_workspace_bytes(rows, d))
        return KGQ_ERR_INVALID_ARG;
    int grid = bwd_grid(rows);
    float *partial = reinterpret_cast<float *>(workspace);
    const uint32_t *m32 = reinterpret_cast<const uint32_t *>(mask);
    const bool aligned16 = ((((uintptr_t)g_read) | ((uintptr_t)g_e) | ((uintptr_t)dh)) & 15u) == 0 &&
                           ((uintptr_t)codes & (bits == 32 ? 15u : 3u)) == 0;
    if ((d == 64 || d == 128) && aligned16 && use_tc_backward()) {
        const int64_t tiles = d == 128 ? (rows + 31) / 32 : (rows + 127) / 128;
        grid = (int)(tiles < kSMs ? tiles : kSMs);
        const int st = kgq_launch_layer_backward_tc(g_read, g_e, m32, codes, ranges, offsets, rows, d, bits,
                                                    theta, dh, partial, grid, s);
        if (st != KGQ_OK) return st;
        const int dd = d * d;
        reduce_partials_bwd_kernel<<<(dd + 31) / 32, 1024, 0, s>>>(partial, grid, dd, dtheta, accumulate);
        KGQ_LAUNCH_CHECK();
        return KGQ_OK;
    }
#define KGQ_BWD(D, B) do {                                                                          \
        static bool attr_set = false;   /* > 48 KB dynamic smem needs the opt-in once per instance */ \
        if (!attr_set) {                                                                          \
            cudaFuncSetAttribute(layer_backward_kernel<D, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)BwdSmem<D>::bytes);                                         \
            attr_set = true;                                                                      \
        }                                                                                         \
        layer_backward_kernel<D, B><<<grid, 256, BwdSmem<D>::bytes, s>>>(g_read, g_e, m32, codes, ranges, \
                                                                         offsets, rows, theta, dh, partial); \
    } while (0)
    if (d == 128) {
        switch (bits) { case 1: KGQ_BWD(128, 1); break; case 2: KGQ_BWD(128, 2); break;
                        case 4: KGQ_BWD(128, 4); break; case 8: KGQ_BWD(128, 8); break;
                        default: KGQ_BWD(128, 32); break; }
    } else if (d == 64) {
        switch (bits) { case 1: KGQ_BWD(64, 1); break; case 2: KGQ_BWD(64, 2); break;
                        case 4: KGQ_BWD(64, 4); break; case 8: KGQ_BWD(64, 8); break;
                        default: KGQ_BWD(64, 32); break; }
    } else {
        switch (bits) { case 1: KGQ_BWD(32, 1); break; case 2: KGQ_BWD(32, 2); break;
                        case 4: KGQ_BWD(32, 4); break; case 8: KGQ_BWD(32, 8); break;
                        default: KGQ_BWD(32, 32); break; }
    }
#undef KGQ_BWD
    const int dd = d * d;
    reduce_partials_bwd_kernel<<<(dd + 31) / 32, 1024, 0, s>>>(partial, grid, dd, dtheta, accumulate);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

// kgq_layer_backward_f32 with g_read in compact form (the readout gradient of a
// training batch touches ~3B of N rows): row r's g_read is gr_rows[gr_map[r]]
// when gr_map[r] >= 0, else +0.  Saves the dense N x d zero-fill and its reads
// in every layer.  d = 64 on the tensor-core kernel only (others:
// KGQ_ERR_INVALID_ARG, the host densifies).
extern "C" int kgq_layer_backward_rows_f32(const int32_t *gr_map, const float *gr_rows, const float *g_e,
                                           const uint8_t *mask, const uint8_t *codes, const float *ranges,
                                           const float *offsets, int64_t rows, int32_t d, int32_t bits,
                                           const float *theta, float *dh, float *dtheta, void *workspace,
                                           size_t workspace_bytes, int32_t accumulate, void *stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8 || bits == 32)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (d != 64 || rows < 1 || !use_tc_backward()) return KGQ_ERR_INVALID_ARG;
    if (!gr_map || !gr_rows || !mask || !codes || !theta || !dh || !dtheta) return KGQ_ERR_INVALID_ARG;
    if (bits != 32 && (!ranges || !offsets)) return KGQ_ERR_INVALID_ARG;
    if (((uintptr_t)mask) & 3u) return KGQ_ERR_MISALIGNED;
    if ((((uintptr_t)gr_rows) | ((uintptr_t)g_e) | ((uintptr_t)dh)) & 15u) return KGQ_ERR_MISALIGNED;
    if (((uintptr_t)codes) & (bits == 32 ? 15u : 3u)) return KGQ_ERR_MISALIGNED;
    if (!workspace || workspace_bytes < kgq_layer_backward_workspace_bytes(rows, d)) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tiles = (rows + 127) / 128;
    const int grid = (int)(tiles < kSMs ? tiles : kSMs);
    float *partial = reinterpret_cast<float *>(workspace);
    const int st = kgq_launch_layer_backward_tc(nullptr, g_e, reinterpret_cast<const uint32_t *>(mask), codes, ranges,
                                                offsets, rows, d, bits, theta, dh, partial, grid, s, gr_map, gr_rows);
    if (st != KGQ_OK) return st;
    const int dd = d * d;
    reduce_partials_bwd_kernel<<<(dd + 31) / 32, 1024, 0, s>>>(partial, grid, dd, dtheta, accumulate);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
