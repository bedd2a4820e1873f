// Sweep of the L2-resident random-row gather (not product code): how fast can
// 159,251 x 64 fp32 rows (40.8 MB, L2-resident) be gathered 6.4M times, as a
// function of lanes per row (LPR, float4 per lane = 16 / LPR... ) and
// neighbours in flight per row group (U), at full occupancy.  Sums only.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int LPR, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) gather_sum(const int *__restrict__ indptr, const int *__restrict__ idx,
                                                        const float4 *__restrict__ x, int n_rows, float *__restrict__ out) {
    constexpr int RPW = 32 / LPR, F = 16 / LPR;     // float4 per lane per row
    const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * RPW; base < n_rows; base += nw * RPW) {
        const int64_t row = base + grp;
        float4 a[F];
#pragma unroll
        for (int f = 0; f < F; f++) a[f] = make_float4(0, 0, 0, 0);
        if (row < n_rows) {
            const int beg = indptr[row], end = indptr[row + 1];
            for (int k = beg; k < end; k += U) {
                float4 xa[U][F];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int c = (k + u < end) ? __ldg(idx + k + u) : -1;
#pragma unroll
                    for (int f = 0; f < F; f++)
                        xa[u][f] = c >= 0 ? __ldg(x + (int64_t)c * 16 + gl + LPR * f) : make_float4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int f = 0; f < F; f++) {
                        a[f].x += xa[u][f].x; a[f].y += xa[u][f].y; a[f].z += xa[u][f].z; a[f].w += xa[u][f].w;
                    }
            }
        }
        float s = 0;
#pragma unroll
        for (int f = 0; f < F; f++) s += a[f].x + a[f].y + a[f].z + a[f].w;
        if (row < n_rows && gl == 0) out[row] = s;
    }
}

template <int LPR, int U, int MINB>
void run(const int *ip, const int *ix, const float *x, int n, float *out, int64_t nnz, int per_sm) {
    int grid = 148 * per_sm;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 5; w++) gather_sum<LPR, U, MINB><<<grid, 256>>>(ip, ix, (const float4 *)x, n, out);
    cudaEventRecord(a);
    const int reps = 50;
    for (int w = 0; w < reps; w++) gather_sum<LPR, U, MINB><<<grid, 256>>>(ip, ix, (const float4 *)x, n, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / reps;
    printf("LPR %2d U %d minb %d grid/sm %2d: %7.1f us  %7.1f GB/s  %s\n", LPR, U, MINB, per_sm, us,
           (double)nnz * 260 / us / 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int n = 159251, d = 64;
    const int64_t nnz = 6425569;
    std::mt19937_64 rng(1);
    std::vector<int> indptr(n + 1), idx(nnz);
    for (int r = 0; r <= n; r++) indptr[r] = (int)((nnz * (int64_t)r) / n);
    for (int64_t k = 0; k < nnz; k++) idx[k] = (int)(rng() % n);
    int *d_indptr, *d_idx; float *d_x, *d_out;
    cudaMalloc(&d_indptr, (n + 1) * sizeof(int)); cudaMalloc(&d_idx, nnz * sizeof(int));
    cudaMalloc(&d_x, (size_t)n * d * 4); cudaMalloc(&d_out, n * 4);
    cudaMemcpy(d_indptr, indptr.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemcpy(d_idx, idx.data(), nnz * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemset(d_x, 0, (size_t)n * d * 4);
    run<8, 4, 4>(d_indptr, d_idx, d_x, n, d_out, nnz, 4);
    run<8, 4, 4>(d_indptr, d_idx, d_x, n, d_out, nnz, 8);
    run<8, 2, 8>(d_indptr, d_idx, d_x, n, d_out, nnz, 8);
    run<8, 4, 6>(d_indptr, d_idx, d_x, n, d_out, nnz, 6);
    run<8, 8, 4>(d_indptr, d_idx, d_x, n, d_out, nnz, 4);
    run<16, 4, 6>(d_indptr, d_idx, d_x, n, d_out, nnz, 6);
    run<16, 8, 4>(d_indptr, d_idx, d_x, n, d_out, nnz, 4);
    run<16, 2, 8>(d_indptr, d_idx, d_x, n, d_out, nnz, 8);
    run<4, 2, 4>(d_indptr, d_idx, d_x, n, d_out, nnz, 4);
    run<4, 4, 3>(d_indptr, d_idx, d_x, n, d_out, nnz, 3);
}
