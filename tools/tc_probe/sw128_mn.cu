// Probe: kind::tf32 tcgen05 MMAs reading 128B-swizzled row-major fp32 tiles
// as K-major (A of dH = G . theta^T) and as MN-major (A and B of
// dtheta = H^T . G), the layouts the layer backward / epilogue kernels use.
// Inputs are small integers (exact in tf32), so results must be exact.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 sw128_mn.cu -o sw128_mn
#include "../../paper_2212_04540_b200/csrc/kgq_tc.cuh"
#include <cstdio>
#include <cstdlib>
#include <cmath>
using namespace kgq;

constexpr int R = 128;      // rows (K of dtheta, M of dH)

template <int D>
__global__ void probe(const float *g, const float *h, const float *th, float *dh, float *dth, int var) {
    extern __shared__ __align__(1024) uint8_t sm[];
    // tile layout: column block cb (32 cols) of a [rows][D] tile at cb * rows * 128 B
    float *gs = reinterpret_cast<float *>(sm);
    float *hs = reinterpret_cast<float *>(sm + R * D * 4);
    float *ts = reinterpret_cast<float *>(sm + 2 * R * D * 4);      // theta^T rows n, cols k
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tb;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < R * D; i += blockDim.x) {
        const int r = i / D, c = i % D;
        gs[tc::sw128_off(r, c, R) / 4] = g[i];
        hs[tc::sw128_off(r, c, R) / 4] = h[i];
    }
    for (int i = t; i < D * D; i += blockDim.x) {
        const int k = i / D, n = i % D;            // theta[k][n] -> B(n, k)
        ts[tc::sw128_off(n, k, D) / 4] = th[i];
    }
    if (t == 0) tc::mbar_init(&mbar, 1);
    if (warp == 0) tc::tmem_alloc(&tb, 256);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (t == 0) {
        // dH[r][n] = sum_k G[r][k] theta[k][n]: A = G K-major (M = 128), B = theta^T K-major (N = D)
        for (int s = 0; s < D / 8; s++) {
            const uint64_t ad = tc::kmajor_sw128_desc(tc::smem_u32(gs), s, R);
            const uint64_t bd = tc::kmajor_sw128_desc(tc::smem_u32(ts), s, D);
            tc::mma_tf32(tb, ad, bd, tc::idesc_tf32_major(R, D, false, false), s > 0);
        }
        // dtheta[i][j] = sum_r H[r][i] G[r][j]: A = H MN-major (M = D), B = G MN-major (N = D), K = R
        for (int s = 0; s < R / 8; s++) {
            uint64_t ad = tc::mnmajor_sw128_desc(tc::smem_u32(hs), s, R);
            uint64_t bd = tc::mnmajor_sw128_desc(tc::smem_u32(gs), s, R);
            if (var & 1) {   // swap LBO / SBO
                ad = tc::sw128_desc(tc::smem_u32(hs) + s * 1024, 1024, R * 128);
                bd = tc::sw128_desc(tc::smem_u32(gs) + s * 1024, 1024, R * 128);
            }
            if (var & 2) {   // SBO = stride of the 8-row groups measured in the atom, LBO 16
                ad = tc::sw128_desc(tc::smem_u32(hs) + s * 1024, R * 128, 1024) ;
                bd = tc::sw128_desc(tc::smem_u32(gs) + s * 1024, R * 128, 1024);
                ad = (ad & ~((uint64_t)7 << 61)) | ((uint64_t)2 << 61);
                bd = (bd & ~((uint64_t)7 << 61)) | ((uint64_t)2 << 61);
            }
            tc::mma_tf32(tb + 128, ad, bd, tc::idesc_tf32_major(D, D, !(var & 4), !(var & 4)), s > 0);
        }
        tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    for (int cb = 0; cb < D; cb += 32) {
        float v[32];
        tc::tmem_ld32(tb + ((uint32_t)(32 * warp) << 16) + cb, v);
        for (int j = 0; j < 32; j++) dh[(32 * warp + lane) * D + cb + j] = v[j];
        tc::tmem_ld32(tb + ((uint32_t)(32 * warp) << 16) + 128 + cb, v);
        for (int j = 0; j < 32; j++) dth[(32 * warp + lane) * D + cb + j] = v[j];
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free(tb, 256);
}

template <int D>
static int run(int var) {
    const size_t nG = R * D, nT = D * D;
    float *hg = (float *)malloc(nG * 4), *hh = (float *)malloc(nG * 4), *ht = (float *)malloc(nT * 4);
    float *odh = (float *)malloc(R * D * 4), *odt = (float *)malloc(128 * D * 4);
    srand(1);
    for (size_t i = 0; i < nG; i++) { hg[i] = (float)(rand() % 9 - 4); hh[i] = (float)(rand() % 7 - 3); }
    for (size_t i = 0; i < nT; i++) ht[i] = (float)(rand() % 5 - 2);
    float *dg, *dh_, *dt, *ddh, *ddt;
    cudaMalloc(&dg, nG * 4); cudaMalloc(&dh_, nG * 4); cudaMalloc(&dt, nT * 4);
    cudaMalloc(&ddh, R * D * 4); cudaMalloc(&ddt, 128 * D * 4);
    cudaMemcpy(dg, hg, nG * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dh_, hh, nG * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, ht, nT * 4, cudaMemcpyHostToDevice);
    const size_t smem = (2 * nG + nT) * 4 + 1024;
    cudaFuncSetAttribute(probe<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaMemset(ddt, 0xff, 128 * D * 4);
    probe<D><<<1, 128, smem>>>(dg, dh_, dt, ddh, ddt, var);
    cudaError_t e = cudaDeviceSynchronize();
    printf("D=%d var %d err %s\n", D, var, cudaGetErrorString(e));
    cudaMemcpy(odh, ddh, R * D * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(odt, ddt, 128 * D * 4, cudaMemcpyDeviceToHost);
    int bad_dh = 0, bad_dt = 0;
    for (int r = 0; r < R; r++)
        for (int n = 0; n < D; n++) {
            double s = 0;
            for (int k = 0; k < D; k++) s += (double)hg[r * D + k] * ht[k * D + n];
            if (odh[r * D + n] != (float)s) { if (bad_dh < 4) printf("dH[%d][%d] %g vs %g\n", r, n, odh[r * D + n], s); bad_dh++; }
        }
    // M = D accumulator lanes: D = 128 -> lane i; D = 64 -> lane 32*(i/16) + i%16
    for (int i = 0; i < D; i++)
        for (int j = 0; j < D; j++) {
            double s = 0;
            for (int r = 0; r < R; r++) s += (double)hh[r * D + i] * hg[r * D + j];
            const int lane = D == 128 ? i : 32 * (i / 16) + i % 16;
            if (odt[lane * D + j] != (float)s) { if (bad_dt < 4) printf("dT[%d][%d] %g vs %g\n", i, j, odt[lane * D + j], s); bad_dt++; }
        }
    printf("D=%d dH mismatches %d / %d, dtheta mismatches %d / %d\n", D, bad_dh, R * D, bad_dt, D * D);
    return bad_dh + bad_dt;
}

int main() {
    int bad = 0;
    for (int var = 0; var < 8; var++) { bad += run<128>(var); }
    bad += run<64>(0);
    printf(bad ? "FAIL\n" : "PASS\n");
    return bad ? 1 : 0;
}
