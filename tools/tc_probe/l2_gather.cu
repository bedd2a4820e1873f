// L2-resident random-row gather ceiling for the K4 SpMM roofline (not product
// code).  Table: 159,251 x 64 fp32 (40.8 MB, the Amazon embedding table);
// 6,425,569 random neighbour ids (the Amazon nnz), 40 per row on average.
// Each 8-lane group streams its row's neighbours exactly like K4's light path
// (two 128-bit loads per lane per neighbour, 4 neighbours in flight) but only
// sums them (no ordered chain, no scale): bytes gathered / time = the ceiling
// a gather-bound SpMM can reach on this box.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 4) gather_sum(const int *__restrict__ indptr, const int *__restrict__ idx,
                                                     const float4 *__restrict__ x, int n_rows, float *__restrict__ out) {
    const int lane = threadIdx.x & 31, gl = lane & 7, grp = lane >> 3;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 4; base < n_rows; base += nw * 4) {
        const int64_t row = base + grp;
        float4 a = make_float4(0, 0, 0, 0), b = a;
        if (row < n_rows) {
            const int beg = indptr[row], end = indptr[row + 1];
            for (int k = beg; k < end; k += 4) {
                float4 xa[4], xb[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int c = (k + u < end) ? __ldg(idx + k + u) : -1;
                    if (c >= 0) { xa[u] = __ldg(x + (int64_t)c * 16 + gl); xb[u] = __ldg(x + (int64_t)c * 16 + gl + 8); }
                    else { xa[u] = xb[u] = make_float4(0, 0, 0, 0); }
                }
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    a.x += xa[u].x; a.y += xa[u].y; a.z += xa[u].z; a.w += xa[u].w;
                    b.x += xb[u].x; b.y += xb[u].y; b.z += xb[u].z; b.w += xb[u].w;
                }
            }
        }
        float s = a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
        if (row < n_rows && gl == 0) out[row] = s;
    }
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
    int grid = 148 * 4;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 5; w++) gather_sum<<<grid, 256>>>(d_indptr, d_idx, (const float4 *)d_x, n, d_out);
    cudaEventRecord(a);
    const int reps = 50;
    for (int w = 0; w < reps; w++) gather_sum<<<grid, 256>>>(d_indptr, d_idx, (const float4 *)d_x, n, d_out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / reps;
    const double bytes = (double)nnz * (d * 4 + 4);
    printf("{\"probe\": \"l2_random_row_gather\", \"table_MB\": %.1f, \"nnz\": %lld, \"us\": %.1f, \"GBps\": %.1f, \"err\": \"%s\"}\n",
           n * d * 4 / 1e6, (long long)nnz, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
}
