// Probe: where does a cta_group::1 M=64 tcgen05 accumulator live in TMEM?
// A[64 x 8] = row index r in column 0 (others 0); B[N=64 x 8]: B(n,0)=1.
// D[r][n] = r.  Dump all 128 lanes x 64 columns.
#include "../../paper_2212_04540_b200/csrc/kgq_tc.cuh"
#include <cstdio>
using namespace kgq;
__global__ void probe(float *out) {
    constexpr int M = 64, N = 64, K = 8;
    __shared__ __align__(128) float a[M * K];
    __shared__ __align__(128) float b[N * K];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tb;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < M * K; i += 128) a[i] = 0.f;
    for (int i = t; i < N * K; i += 128) b[i] = 0.f;
    __syncthreads();
    if (t < M) a[tc::tile_off(t, 0, M) / 4] = (float)(t + 1);
    if (t < N) b[tc::tile_off(t, 0, N) / 4] = 1.0f;
    if (t == 0) tc::mbar_init(&mbar, 1);
    if (warp == 0) tc::tmem_alloc(&tb, 64);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    tc::fence_proxy_async();
    __syncthreads();
    if (t == 0) {
        tc::fence_after();
        constexpr uint32_t LBO_A = (M / 8) * 128, LBO_B = (N / 8) * 128;
        tc::mma_tf32(tb, tc::smem_desc(tc::smem_u32(a), LBO_A, 128), tc::smem_desc(tc::smem_u32(b), LBO_B, 128),
                     tc::idesc_tf32(M, N), 0);
        tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    for (int cb = 0; cb < 64; cb += 32) {
        float v[32];
        tc::tmem_ld32(tb + ((uint32_t)(32 * warp) << 16) + cb, v);
        for (int j = 0; j < 32; j++) out[(32 * warp + lane) * 64 + cb + j] = v[j];
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free(tb, 64);
}
int main() {
    float *d, h[128 * 64];
    cudaMalloc(&d, sizeof(h));
    cudaMemset(d, 0, sizeof(h));
    probe<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("err %s\n", cudaGetErrorString(e));
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int l = 0; l < 128; l++) {
        printf("lane %3d:", l);
        for (int c = 0; c < 64; c += 8) printf(" %5.0f", h[l * 64 + c]);
        printf("\n");
    }
}
