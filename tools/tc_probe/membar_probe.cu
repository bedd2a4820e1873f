// Probe: does fence.proxy.async.shared::cta (SASS MEMBAR.ALL.CTA +
// FENCE.VIEW.ASYNC.S) wait for a global load still in flight?  Times the
// fence with and without an outstanding cold load (clock64, one warp).
#include <cstdio>
#include <cstdint>
__global__ void k(const float *in, float *out, long long *t, int mode) {
    __shared__ float s[64];
    long long t0 = clock64();
    float v = in[(size_t)threadIdx.x * 8192 + blockIdx.x * 977];     // cold, scattered
    s[threadIdx.x] = 1.f;
    long long t1 = clock64();
    if (mode == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (mode == 2) asm volatile("fence.acq_rel.cta;" ::: "memory");
    long long t2 = clock64();
    out[threadIdx.x + blockIdx.x * 32] = v + s[threadIdx.x ^ 1];
    long long t3 = clock64();
    if (threadIdx.x == 0) { t[blockIdx.x * 3] = t1 - t0; t[blockIdx.x * 3 + 1] = t2 - t1; t[blockIdx.x * 3 + 2] = t3 - t2; }
}
int main() {
    float *in, *out; long long *t, h[3];
    cudaMalloc(&in, (size_t)64 << 22); cudaMalloc(&out, 1 << 20); cudaMalloc(&t, 64);
    for (int mode = 0; mode < 3; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            k<<<1, 32>>>(in, out, t, mode);
            cudaMemcpy(h, t, 24, cudaMemcpyDeviceToHost);
        }
        printf("mode %d (%s): issue %lld  fence %lld  use %lld cycles\n", mode,
               mode == 0 ? "no fence" : mode == 1 ? "fence.proxy.async" : "fence.acq_rel.cta", h[0], h[1], h[2]);
    }
}
