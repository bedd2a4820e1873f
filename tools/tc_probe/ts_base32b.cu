// Probe for the layer-backward v2 operand forms (exact small-integer inputs):
//  (1) kind::tf32 with BOTH operands MN-major in SWIZZLE_128B_BASE32B layout
//      (the only MN-major form CUTLASS allows for 32-bit types): row-major
//      [rows][32-col blocks], 128-B rows, 32-B granule j of row r stored at
//      j ^ (r & 3).  D[i][j] = sum_r A[r][i] B[r][j], M = N = 128 (four
//      32-column blocks each, LBO apart), K = 64 rows (8 K-steps of 1024 B).
//  (2) A from TMEM (tcgen05.st by thread = row), B K-major SWIZZLE_128B:
//      D[r][n] = sum_k A[r][k] T[n][k], M = 128, N = 64, K = 64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 ts_base32b.cu -o ts_base32b.bin
#include "../../paper_2212_04540_b200/csrc/kgq_tc.cuh"
#include <cstdio>
#include <cstdlib>
using namespace kgq;

constexpr int KR = 64;     // rows (K) of (1)
constexpr int MN = 128;    // M = N of (1)

__global__ void probe(const float *a, const float *b, const float *g, const float *th, float *d1, float *d2,
                      int sbo) {
    extern __shared__ __align__(1024) uint8_t sm[];
    float *as = reinterpret_cast<float *>(sm);                       // [KR][MN] BASE32B
    float *bs = reinterpret_cast<float *>(sm + KR * MN * 4);         // [KR][MN] BASE32B
    float *ts = reinterpret_cast<float *>(sm + 2 * KR * MN * 4);     // theta^T [64][64] SW128 K-major
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tb;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < KR * MN; i += blockDim.x) {
        const int r = i / MN, c = i % MN;
        as[tc::b32_off(r, c, KR) / 4] = a[i];
        bs[tc::b32_off(r, c, KR) / 4] = b[i];
    }
    for (int i = t; i < 64 * 64; i += blockDim.x) {
        const int k = i / 64, n = i % 64;
        ts[tc::sw128_off(n, k, 64) / 4] = th[i];
    }
    if (t == 0) tc::mbar_init(&mbar, 1);
    if (warp == 0) tc::tmem_alloc(&tb, 512);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = tb;
    // (2) A operand into TMEM columns [256, 320): thread = row (lane 32*warp + lane)
    {
        uint32_t v[64];
        for (int k = 0; k < 64; k++) v[k] = __float_as_uint(g[(32 * warp + lane) * 64 + k]);
        tc::tmem_st16(tm + ((uint32_t)(32 * warp) << 16) + 256, v);
        tc::tmem_st16(tm + ((uint32_t)(32 * warp) << 16) + 272, v + 16);
        tc::tmem_st16(tm + ((uint32_t)(32 * warp) << 16) + 288, v + 32);
        tc::tmem_st16(tm + ((uint32_t)(32 * warp) << 16) + 304, v + 48);
        tc::tmem_st_wait();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (t == 0) {
        for (int s = 0; s < KR / 8; s++) {
            const uint64_t ad = tc::mnmajor_b32_desc(tc::smem_u32(as), s, KR, (uint32_t)sbo);
            const uint64_t bd = tc::mnmajor_b32_desc(tc::smem_u32(bs), s, KR, (uint32_t)sbo);
            tc::mma_tf32(tm, ad, bd, tc::idesc_tf32_major(MN, MN, true, true), s > 0);
        }
        for (int s = 0; s < 8; s++) {
            const uint64_t bd = tc::kmajor_sw128_desc(tc::smem_u32(ts), s, 64);
            tc::mma_tf32_ts(tm + 128, tm + 256 + 8 * s, bd, tc::idesc_tf32(128, 64), s > 0);
        }
        tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    for (int cb = 0; cb < 128; cb += 32) {
        float v[32];
        tc::tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + cb, v);
        for (int j = 0; j < 32; j++) d1[(32 * warp + lane) * MN + cb + j] = v[j];
    }
    for (int cb = 0; cb < 64; cb += 32) {
        float v[32];
        tc::tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + 128 + cb, v);
        for (int j = 0; j < 32; j++) d2[(32 * warp + lane) * 64 + cb + j] = v[j];
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free(tm, 512);
}

int main() {
    const int nA = KR * MN;
    float *ha = (float *)malloc(nA * 4), *hb = (float *)malloc(nA * 4);
    float *hg = (float *)malloc(128 * 64 * 4), *ht = (float *)malloc(64 * 64 * 4);
    float *o1 = (float *)malloc(MN * MN * 4), *o2 = (float *)malloc(128 * 64 * 4);
    srand(2);
    for (int i = 0; i < nA; i++) { ha[i] = (float)(rand() % 9 - 4); hb[i] = (float)(rand() % 7 - 3); }
    for (int i = 0; i < 128 * 64; i++) hg[i] = (float)(rand() % 9 - 4);
    for (int i = 0; i < 64 * 64; i++) ht[i] = (float)(rand() % 5 - 2);
    float *da, *db, *dg, *dt, *dd1, *dd2;
    cudaMalloc(&da, nA * 4); cudaMalloc(&db, nA * 4); cudaMalloc(&dg, 128 * 64 * 4); cudaMalloc(&dt, 64 * 64 * 4);
    cudaMalloc(&dd1, MN * MN * 4); cudaMalloc(&dd2, 128 * 64 * 4);
    cudaMemcpy(da, ha, nA * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb, nA * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dg, hg, 128 * 64 * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, ht, 64 * 64 * 4, cudaMemcpyHostToDevice);
    const size_t smem = (2 * nA + 64 * 64) * 4;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int fails = 0;
    const int sbos[3] = {512, 1024, 128};
    for (int v = 0; v < 3; v++) {
        cudaMemset(dd1, 0xff, MN * MN * 4);
        cudaMemset(dd2, 0xff, 128 * 64 * 4);
        probe<<<1, 128, smem>>>(da, db, dg, dt, dd1, dd2, sbos[v]);
        cudaError_t e = cudaDeviceSynchronize();
        printf("sbo %d: %s\n", sbos[v], cudaGetErrorString(e));
        if (e != cudaSuccess) return 2;
        cudaMemcpy(o1, dd1, MN * MN * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(o2, dd2, 128 * 64 * 4, cudaMemcpyDeviceToHost);
        int b1 = 0, b2 = 0;
        for (int i = 0; i < MN; i++)
            for (int j = 0; j < MN; j++) {
                double s = 0;
                for (int r = 0; r < KR; r++) s += (double)ha[r * MN + i] * hb[r * MN + j];
                if (o1[i * MN + j] != (float)s) { if (b1 < 3) printf("  D1[%d][%d] %g vs %g\n", i, j, o1[i * MN + j], s); b1++; }
            }
        for (int r = 0; r < 128; r++)
            for (int n = 0; n < 64; n++) {
                double s = 0;
                for (int k = 0; k < 64; k++) s += (double)hg[r * 64 + k] * ht[k * 64 + n];
                if (o2[r * 64 + n] != (float)s) { if (b2 < 3) printf("  D2[%d][%d] %g vs %g\n", r, n, o2[r * 64 + n], s); b2++; }
            }
        printf("sbo %d: MN-major BASE32B mismatches %d / %d; TMEM-A mismatches %d / %d\n", sbos[v], b1, MN * MN, b2,
               128 * 64);
        fails += (b1 != 0) + (b2 != 0);
    }
    return fails ? 1 : 0;
}
