// kgq_bpr.cu -- the BPR + L2 head of a training step (tape.py:154-183 forward,
// tape.py:233-244 backward) as two kernels instead of ~30 framework launches.
//
// Forward (row CTAs + a 1-warp fold): margins[r] = sum_k u[r,k] * (p[r,k] - n[r,k]);
//   loss = mean_r logaddexp(0, -margins[r]) + (l2 * (|u|^2 + |p|^2 + |n|^2)) / B
// in fp32 with a fixed reduction tree (deterministic; the reference's numpy
// pairwise sums differ from any GPU order in the last bits -> tolerance).
// Backward (elementwise): with coef = sigmoid(-m)/B and reg = fp32(2*l2/B),
//   gu = g * (-coef * (ph - nh) + reg * uh)
//   gp = g * (-coef * uh + reg * ph)
//   gn = g * ( coef * uh + reg * nh)
// against the dequantized blocks, each product / sum rounded separately in
// the reference's evaluation order (no FMA contraction).
#include "kgq_common.cuh"

namespace kgq {


// Rows: 8 lanes per row (lane j sums features j, j+8, ...), 32 rows per
// 256-thread CTA, one CTA per 32 rows -> per-CTA partial sums of softplus and
// |.|^2 (fixed lane/warp tree); a 1-warp kernel then folds the partials in CTA
// order and forms the loss.  Deterministic, all row loads in flight at once.
constexpr int kBprRowsPerCta = 32;

__global__ void __launch_bounds__(256)
bpr_rows_kernel(const float *__restrict__ u, const float *__restrict__ p, const float *__restrict__ n,
                int64_t batch, int d, float *__restrict__ margins, float *__restrict__ part) {
    __shared__ float s_sp[8], s_rg[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane & 7, grp = lane >> 3;
    const int64_t r = (int64_t)blockIdx.x * kBprRowsPerCta + warp * 4 + grp;
    float m = 0.0f, q = 0.0f;
    if (r < batch) {
        for (int k = j; k < d; k += 8) {
            const float uv = __ldg(u + r * d + k), pv = __ldg(p + r * d + k), nv = __ldg(n + r * d + k);
            m = __fadd_rn(m, __fmul_rn(uv, __fsub_rn(pv, nv)));
            q = __fadd_rn(q, __fadd_rn(__fadd_rn(__fmul_rn(uv, uv), __fmul_rn(pv, pv)), __fmul_rn(nv, nv)));
        }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
        m = __fadd_rn(m, __shfl_xor_sync(0xffffffffu, m, o));
        q = __fadd_rn(q, __shfl_xor_sync(0xffffffffu, q, o));
    }
    float sp = 0.0f;
    if (j == 0 && r < batch) {
        margins[r] = m;
        // logaddexp(0, -m) = max(0, -m) + log1p(exp(-|m|))
        const float x = -m;
        sp = __fadd_rn(fmaxf(x, 0.0f), log1pf(expf(-fabsf(x))));
    } else {
        q = 0.0f;
    }
    sp = __fadd_rn(sp, __shfl_xor_sync(0xffffffffu, sp, 8));
    q = __fadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 8));
    sp = __fadd_rn(sp, __shfl_xor_sync(0xffffffffu, sp, 16));
    q = __fadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 16));
    if (lane == 0) {
        s_sp[warp] = sp;
        s_rg[warp] = q;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.0f, b2 = 0.0f;
        for (int w = 0; w < 8; w++) {
            a = __fadd_rn(a, s_sp[w]);
            b2 = __fadd_rn(b2, s_rg[w]);
        }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b2;
    }
}

__global__ void bpr_loss_kernel(const float *__restrict__ part, int nparts, int64_t batch, float l2,
                                float *__restrict__ loss) {
    const int lane = threadIdx.x;
    float a = 0.0f, b2 = 0.0f;
    for (int k = lane; k < nparts; k += 32) {       // lane-strided chains, then a fixed tree
        a = __fadd_rn(a, part[2 * k]);
        b2 = __fadd_rn(b2, part[2 * k + 1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
        b2 = __fadd_rn(b2, __shfl_xor_sync(0xffffffffu, b2, o));
    }
    if (lane == 0) {
        const float fb = (float)batch;
        const float data = __fdiv_rn(a, fb);
        const float reg = __fdiv_rn(__fmul_rn(l2, b2), fb);
        *loss = __fadd_rn(data, reg);
    }
}

__global__ void bpr_backward_kernel(const float *__restrict__ g, const float *__restrict__ margins,
                                    const float *__restrict__ uh, const float *__restrict__ ph,
                                    const float *__restrict__ nh, int64_t batch, int d, float reg,
                                    float *__restrict__ gu, float *__restrict__ gp, float *__restrict__ gn) {
    const int64_t total = batch * d;
    const float gg = __ldg(g);
    const float fb = (float)batch;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / d;
        const float m = __ldg(margins + r);
        const float sg = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(m)));      // sigmoid(-m)
        const float coef = __fdiv_rn(sg, fb);
        const float u = __ldg(uh + i), pv = __ldg(ph + i), nv = __ldg(nh + i);
        const float ru = __fmul_rn(reg, u);
        gu[i] = __fmul_rn(gg, __fadd_rn(__fmul_rn(-coef, __fsub_rn(pv, nv)), ru));
        gp[i] = __fmul_rn(gg, __fadd_rn(__fmul_rn(-coef, u), __fmul_rn(reg, pv)));
        gn[i] = __fmul_rn(gg, __fadd_rn(__fmul_rn(coef, u), __fmul_rn(reg, nv)));
    }
}

}  // namespace kgq

using namespace kgq;

extern "C" size_t kgq_bpr_forward_workspace_bytes(int64_t batch) {
    return (size_t)(2 * ((batch + kBprRowsPerCta - 1) / kBprRowsPerCta)) * sizeof(float);
}

extern "C" int kgq_bpr_forward_f32(const float *u, const float *p, const float *n, int64_t batch, int32_t d,
                                   float l2, float *margins, float *loss, void *workspace, size_t workspace_bytes,
                                   void *stream) {
    if (batch < 1 || d < 1 || !u || !p || !n || !margins || !loss) return KGQ_ERR_INVALID_ARG;
    if (!workspace || workspace_bytes < kgq_bpr_forward_workspace_bytes(batch)) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t blocks = (batch + kBprRowsPerCta - 1) / kBprRowsPerCta;
    if (blocks > 0x7fffffff) return KGQ_ERR_INVALID_ARG;
    float *part = reinterpret_cast<float *>(workspace);
    bpr_rows_kernel<<<(int)blocks, 256, 0, s>>>(u, p, n, batch, d, margins, part);
    bpr_loss_kernel<<<1, 32, 0, s>>>(part, (int)blocks, batch, l2, loss);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_bpr_backward_f32(const float *g, const float *margins, const float *uh, const float *ph,
                                    const float *nh, int64_t batch, int32_t d, float reg, float *gu,
                                    float *gp, float *gn, void *stream) {
    if (batch < 1 || d < 1 || !g || !margins || !uh || !ph || !nh || !gu || !gp || !gn)
        return KGQ_ERR_INVALID_ARG;
    const int64_t total = batch * d;
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)kSMs * 8) blocks = (int64_t)kSMs * 8;
    bpr_backward_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(g, margins, uh, ph, nh, batch, d, reg,
                                                                      gu, gp, gn);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
