// kgq_optim.cu -- fused Adam step (train.py:42-59) for sm_100a.
// One pass over (param, grad, m, v) with the reference's numpy float32 op
// order: every product, quotient, sqrt and sum is separately rounded, the
// Python scalars enter as float32 (NEP 50 weak scalars), and m/c1, v/c2 are
// true divisions -- bit-identical to the numpy update.
#include "kgq_common.cuh"

namespace kgq {

struct AdamScalars { float b1, omb1, b2, omb2, c1, c2, lr, eps; };

__device__ __forceinline__ void adam_elem(float &p, float g, float &m, float &v, const AdamScalars &a) {
    m = __fadd_rn(__fmul_rn(m, a.b1), __fmul_rn(a.omb1, g));
    v = __fadd_rn(__fmul_rn(v, a.b2), __fmul_rn(a.omb2, __fmul_rn(g, g)));
    const float mh = __fdiv_rn(m, a.c1);
    const float vh = __fdiv_rn(v, a.c2);
    p = __fsub_rn(p, __fdiv_rn(__fmul_rn(a.lr, mh), __fadd_rn(__fsqrt_rn(vh), a.eps)));
}

__global__ void __launch_bounds__(256)
adam_vec_kernel(float4 *__restrict__ p, const float4 *__restrict__ g, float4 *__restrict__ m,
                float4 *__restrict__ v, int64_t n4, AdamScalars a, const int64_t *__restrict__ status) {
    if (status && *(volatile const int64_t *)status) return;   // a step failed: no update
    // two float4 of each array per thread per iteration (8 loads in flight)
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + nthr < n4; i += 2 * nthr) {
        float4 pp[2], mm[2], vv[2], gg[2];
#pragma unroll
        for (int u = 0; u < 2; u++) {
            pp[u] = p[i + u * nthr];
            mm[u] = m[i + u * nthr];
            vv[u] = v[i + u * nthr];
            gg[u] = ldg_stream(g + i + u * nthr);
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
            adam_elem(pp[u].x, gg[u].x, mm[u].x, vv[u].x, a);
            adam_elem(pp[u].y, gg[u].y, mm[u].y, vv[u].y, a);
            adam_elem(pp[u].z, gg[u].z, mm[u].z, vv[u].z, a);
            adam_elem(pp[u].w, gg[u].w, mm[u].w, vv[u].w, a);
            p[i + u * nthr] = pp[u];
            m[i + u * nthr] = mm[u];
            v[i + u * nthr] = vv[u];
        }
    }
    if (i < n4) {
        float4 pp = p[i], mm = m[i], vv = v[i];
        const float4 gg = ldg_stream(g + i);
        adam_elem(pp.x, gg.x, mm.x, vv.x, a);
        adam_elem(pp.y, gg.y, mm.y, vv.y, a);
        adam_elem(pp.z, gg.z, mm.z, vv.z, a);
        adam_elem(pp.w, gg.w, mm.w, vv.w, a);
        p[i] = pp;
        m[i] = mm;
        v[i] = vv;
    }
}

// Graph-capturable variant: the bias corrections are read from a host-built
// table indexed on the device, c12[2i], c12[2i+1] = float32(1 - beta^t) for
// i = *step_ptr (the table's rows map i to the absolute step t; Python's float
// pow, exactly as the reference).
__global__ void __launch_bounds__(256)
adam_vec_dev_kernel(float4 *__restrict__ p, const float4 *__restrict__ g, float4 *__restrict__ m,
                    float4 *__restrict__ v, int64_t n4, AdamScalars a, const float *__restrict__ c12,
                    const int64_t *__restrict__ step_ptr, const int64_t *__restrict__ status) {
    if (status && *(volatile const int64_t *)status) return;
    const int64_t t = __ldg(step_ptr);
    a.c1 = __ldg(c12 + 2 * t);
    a.c2 = __ldg(c12 + 2 * t + 1);
    // two float4 of each array per thread per iteration (8 loads in flight)
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + nthr < n4; i += 2 * nthr) {
        float4 pp[2], mm[2], vv[2], gg[2];
#pragma unroll
        for (int u = 0; u < 2; u++) {
            pp[u] = p[i + u * nthr];
            mm[u] = m[i + u * nthr];
            vv[u] = v[i + u * nthr];
            gg[u] = ldg_stream(g + i + u * nthr);
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
            adam_elem(pp[u].x, gg[u].x, mm[u].x, vv[u].x, a);
            adam_elem(pp[u].y, gg[u].y, mm[u].y, vv[u].y, a);
            adam_elem(pp[u].z, gg[u].z, mm[u].z, vv[u].z, a);
            adam_elem(pp[u].w, gg[u].w, mm[u].w, vv[u].w, a);
            p[i + u * nthr] = pp[u];
            m[i + u * nthr] = mm[u];
            v[i + u * nthr] = vv[u];
        }
    }
    if (i < n4) {
        float4 pp = p[i], mm = m[i], vv = v[i];
        const float4 gg = ldg_stream(g + i);
        adam_elem(pp.x, gg.x, mm.x, vv.x, a);
        adam_elem(pp.y, gg.y, mm.y, vv.y, a);
        adam_elem(pp.z, gg.z, mm.z, vv.z, a);
        adam_elem(pp.w, gg.w, mm.w, vv.w, a);
        p[i] = pp;
        m[i] = mm;
        v[i] = vv;
    }
}

__global__ void adam_kernel(float *__restrict__ p, const float *__restrict__ g, float *__restrict__ m,
                            float *__restrict__ v, int64_t n, AdamScalars a,
                            const int64_t *__restrict__ status) {
    if (status && *(volatile const int64_t *)status) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float pp = p[i], mm = m[i], vv = v[i];
        adam_elem(pp, g[i], mm, vv, a);
        p[i] = pp;
        m[i] = mm;
        v[i] = vv;
    }
}

// ---------------------------------------------------------------------------
// Per-step health check (train.py:91-93 and tape.py:256-264 without a host
// sync): scan the loss and every gradient for non-finite values; the first
// failing tensor (in list order: loss, then gradients in parameter order) and
// the step are latched into status[0..1] once, and every later Adam update
// reads status[0] and skips.  status[2..3] are per-launch scratch (bit mask of
// failing tensors, finished-block counter) that the last block resets, so the
// launch can be replayed from a CUDA graph.
// ---------------------------------------------------------------------------
constexpr int kMaxCheck = 8;
struct CheckList { const float *p[kMaxCheck]; int64_t n[kMaxCheck]; };

__global__ void __launch_bounds__(256)
check_finite_kernel(CheckList L, int count, int code0, const int64_t *__restrict__ step_dev,
                    int64_t step_host, int64_t *__restrict__ status) {
    unsigned bad = 0;
    const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    for (int k = 0; k < count; k++) {
        const float *x = L.p[k];
        const int64_t n = L.n[k];
        bool any = false;
        if ((((uintptr_t)x) & 15u) == 0) {
            const int64_t n4 = n >> 2;
            const float4 *x4 = reinterpret_cast<const float4 *>(x);
            // x - x is NaN exactly for inf / NaN inputs; 8 independent loads in
            // flight per thread (one per iteration left the scan latency-bound)
            constexpr int U = 8;
            int64_t i = tid0;
            for (; i + (U - 1) * nthr < n4; i += U * nthr) {
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; u++) v[u] = ldg_stream(x4 + i + u * nthr);
#pragma unroll
                for (int u = 0; u < U; u++)
                    any |= !(__fsub_rn(v[u].x, v[u].x) == 0.0f) | !(__fsub_rn(v[u].y, v[u].y) == 0.0f) |
                           !(__fsub_rn(v[u].z, v[u].z) == 0.0f) | !(__fsub_rn(v[u].w, v[u].w) == 0.0f);
            }
            for (; i < n4; i += nthr) {
                const float4 v = ldg_stream(x4 + i);
                any |= !(__fsub_rn(v.x, v.x) == 0.0f) | !(__fsub_rn(v.y, v.y) == 0.0f) |
                       !(__fsub_rn(v.z, v.z) == 0.0f) | !(__fsub_rn(v.w, v.w) == 0.0f);
            }
            for (int64_t i = 4 * n4 + tid0; i < n; i += nthr) any |= !(__fsub_rn(x[i], x[i]) == 0.0f);
        } else {
            for (int64_t i = tid0; i < n; i += nthr) any |= !(__fsub_rn(x[i], x[i]) == 0.0f);
        }
        if (any) bad |= 1u << k;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    __shared__ unsigned s_bad;
    __shared__ bool s_last;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(&s_bad, bad);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_bad) atomicOr(reinterpret_cast<unsigned long long *>(status + 2), (unsigned long long)s_bad);
        __threadfence();
        const unsigned long long done = atomicAdd(reinterpret_cast<unsigned long long *>(status + 3), 1ull);
        s_last = done == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        const unsigned long long mask = *(volatile unsigned long long *)(status + 2);
        if (mask && status[0] == 0) {
            status[0] = code0 + __ffsll((long long)mask) - 1;
            status[1] = step_host + (step_dev ? *step_dev : 0);
        }
        status[2] = 0;
        status[3] = 0;
    }
}

}  // namespace kgq

using namespace kgq;

extern "C" int kgq_check_finite_f32(const float *const *tensors, const int64_t *sizes, int32_t count,
                                    int32_t code0, const int64_t *step_dev, int64_t step_host,
                                    int64_t *status, void *stream) {
    if (count < 1 || count > kMaxCheck || !tensors || !sizes || !status || code0 < 1)
        return KGQ_ERR_INVALID_ARG;
    CheckList L;
    int64_t total = 0;
    for (int k = 0; k < kMaxCheck; k++) {
        L.p[k] = k < count ? tensors[k] : nullptr;
        L.n[k] = k < count ? sizes[k] : 0;
        if (k < count && (L.n[k] < 0 || (L.n[k] > 0 && !L.p[k]))) return KGQ_ERR_INVALID_ARG;
        total += L.n[k];
    }
    int64_t blocks = (total / 4 + 255) / 256;
    if (blocks > (int64_t)kSMs * 4) blocks = (int64_t)kSMs * 4;
    if (blocks < 1) blocks = 1;
    check_finite_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(L, count, code0, step_dev, step_host,
                                                                     status);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_adam_step_f32(float *param, const float *grad, float *m, float *v, int64_t n,
                                 double lr, double beta1, double beta2, double eps, int64_t step,
                                 const int64_t *status, void *stream) {
    if (n < 0 || step < 1) return KGQ_ERR_INVALID_ARG;
    if (n == 0) return KGQ_OK;
    if (!param || !grad || !m || !v) return KGQ_ERR_INVALID_ARG;
    AdamScalars a;
    a.b1 = (float)beta1;
    a.omb1 = (float)(1.0 - beta1);
    a.b2 = (float)beta2;
    a.omb2 = (float)(1.0 - beta2);
    double p1 = 1.0, p2 = 1.0;            // beta ** t, as Python's float pow
    p1 = pow(beta1, (double)step);
    p2 = pow(beta2, (double)step);
    a.c1 = (float)(1.0 - p1);
    a.c2 = (float)(1.0 - p2);
    a.lr = (float)lr;
    a.eps = (float)eps;
    cudaStream_t s = (cudaStream_t)stream;
    const bool vec = (n & 3) == 0 &&
                     ((((uintptr_t)param) | ((uintptr_t)grad) | ((uintptr_t)m) | ((uintptr_t)v)) & 15u) == 0;
    if (vec) {
        const int64_t n4 = n / 4;
        int64_t blocks = (n4 + 255) / 256;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        adam_vec_kernel<<<(int)blocks, 256, 0, s>>>(reinterpret_cast<float4 *>(param),
                                                    reinterpret_cast<const float4 *>(grad),
                                                    reinterpret_cast<float4 *>(m),
                                                    reinterpret_cast<float4 *>(v), n4, a, status);
    } else {
        int64_t blocks = (n + 255) / 256;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        adam_kernel<<<(int)blocks, 256, 0, s>>>(param, grad, m, v, n, a, status);
    }
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_adam_step_dev_f32(float *param, const float *grad, float *m, float *v, int64_t n,
                                     double lr, double beta1, double beta2, double eps,
                                     const float *c12, const int64_t *step_ptr, const int64_t *status,
                                     void *stream) {
    if (n < 0 || !c12 || !step_ptr) return KGQ_ERR_INVALID_ARG;
    if (n == 0) return KGQ_OK;
    if (!param || !grad || !m || !v) return KGQ_ERR_INVALID_ARG;
    if ((n & 3) || ((((uintptr_t)param) | ((uintptr_t)grad) | ((uintptr_t)m) | ((uintptr_t)v)) & 15u))
        return KGQ_ERR_MISALIGNED;
    AdamScalars a;
    a.b1 = (float)beta1;
    a.omb1 = (float)(1.0 - beta1);
    a.b2 = (float)beta2;
    a.omb2 = (float)(1.0 - beta2);
    a.c1 = a.c2 = 1.0f;
    a.lr = (float)lr;
    a.eps = (float)eps;
    const int64_t n4 = n / 4;
    int64_t blocks = (n4 + 255) / 256;
    if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
    adam_vec_dev_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<float4 *>(param), reinterpret_cast<const float4 *>(grad),
        reinterpret_cast<float4 *>(m), reinterpret_cast<float4 *>(v), n4, a, c12, step_ptr, status);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

// A captured step's device counters advanced in one launch: *a += da,
// *b += db, *c += dc (step index, Adam step, tensor-id base; null = skip).
__global__ void counters_add_kernel(int64_t *a, int64_t da, int64_t *b, int64_t db, int64_t *c, int64_t dc) {
    if (threadIdx.x == 0) {
        if (a) *a += da;
        if (b) *b += db;
        if (c) *c += dc;
    }
}

extern "C" int kgq_counters_add(int64_t *a, int64_t da, int64_t *b, int64_t db, int64_t *c, int64_t dc,
                                void *stream) {
    counters_add_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(a, da, b, db, c, dc);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
