// kgq_elementwise.cu -- ReLU + 1-bit mask (K5, tensorops.py:84-92 / tape.py:122-126)
// and its backward g * mask (tape.py:224-225) for sm_100a.
#include "kgq_common.cuh"

namespace kgq {

// spread the 8 bits of b so that bit k lands at bit 4k
__device__ __forceinline__ uint32_t spread4(uint32_t b) {
    b &= 0xFFu;
    b = (b | (b << 12)) & 0x000F000Fu;
    b = (b | (b << 6)) & 0x03030303u;
    b = (b | (b << 3)) & 0x11111111u;
    return b;
}

// relu + LSB-first flat bit mask.  A warp handles 128 elements per step:
// lane l loads float4 l; ballot e collects bit (4l+e); lanes 0..3 assemble
// the four 32-bit mask words.
__global__ void __launch_bounds__(256)
relu_mask_kernel(const float *__restrict__ x, int64_t n128, float *__restrict__ out,
                 uint32_t *__restrict__ mask) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < n128; c += nw) {
        const float4 v = ldg_stream(reinterpret_cast<const float4 *>(x) + c * 32 + lane);
        const uint32_t b0 = __ballot_sync(0xffffffffu, v.x > 0.0f);
        const uint32_t b1 = __ballot_sync(0xffffffffu, v.y > 0.0f);
        const uint32_t b2 = __ballot_sync(0xffffffffu, v.z > 0.0f);
        const uint32_t b3 = __ballot_sync(0xffffffffu, v.w > 0.0f);
        const float4 o = make_float4(relu_np(v.x), relu_np(v.y), relu_np(v.z), relu_np(v.w));
        stg_stream(reinterpret_cast<float4 *>(out) + c * 32 + lane, o);
        if (lane < 4) {
            const int sh = 8 * lane;
            const uint32_t w = spread4(b0 >> sh) | (spread4(b1 >> sh) << 1) |
                               (spread4(b2 >> sh) << 2) | (spread4(b3 >> sh) << 3);
            mask[c * 4 + lane] = w;
        }
    }
}

// tail / unaligned: thread per mask byte
__global__ void relu_mask_bytes_kernel(const float *__restrict__ x, int64_t start, int64_t n,
                                       float *__restrict__ out, uint8_t *__restrict__ mask) {
    const int64_t nb = (n - start + 7) / 8;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint32_t byte = 0;
        for (int t = 0; t < 8; t++) {
            const int64_t i = start + 8 * b + t;
            if (i >= n) break;
            const float v = x[i];
            out[i] = relu_np(v);
            byte |= (v > 0.0f ? 1u : 0u) << t;
        }
        mask[start / 8 + b] = (uint8_t)byte;
    }
}

// ReLU backward: out = g * float(mask bit) (tape.py:224-225: g * mask.to_bool())
__global__ void mask_apply_kernel(const float *__restrict__ g, const uint8_t *__restrict__ mask,
                                  int64_t n, float *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t bit = (mask[i >> 3] >> (i & 7)) & 1u;
        out[i] = __fmul_rn(g[i], bit ? 1.0f : 0.0f);
    }
}

__global__ void mask_apply_vec_kernel(const float4 *__restrict__ g, const uint8_t *__restrict__ mask,
                                      int64_t n4, float4 *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t m = (mask[i >> 1] >> (4 * (i & 1))) & 0xFu;
        const float4 v = ldg_stream(g + i);
        stg_stream(out + i, make_float4(__fmul_rn(v.x, (m & 1u) ? 1.0f : 0.0f),
                                        __fmul_rn(v.y, (m & 2u) ? 1.0f : 0.0f),
                                        __fmul_rn(v.z, (m & 4u) ? 1.0f : 0.0f),
                                        __fmul_rn(v.w, (m & 8u) ? 1.0f : 0.0f)));
    }
}

}  // namespace kgq

using namespace kgq;

extern "C" int kgq_relu_mask_f32(const float *x, int64_t n, float *out, uint8_t *mask, void *stream) {
    if (n < 0) return KGQ_ERR_INVALID_ARG;
    if (n == 0) return KGQ_OK;
    if (!x || !out || !mask) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    int64_t n128 = 0;
    if ((((uintptr_t)x | (uintptr_t)out) & 15u) == 0 && ((uintptr_t)mask & 3u) == 0) n128 = n / 128;
    if (n128) {
        int64_t blocks = (n128 + 7) / 8;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        relu_mask_kernel<<<(int)blocks, 256, 0, s>>>(x, n128, out, reinterpret_cast<uint32_t *>(mask));
    }
    const int64_t start = n128 * 128;
    if (start < n) {
        const int64_t nb = (n - start + 7) / 8;
        int64_t blocks = (nb + 255) / 256;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        relu_mask_bytes_kernel<<<(int)blocks, 256, 0, s>>>(x, start, n, out, mask);
    }
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_mask_apply_f32(const float *g, const uint8_t *mask, int64_t n, float *out,
                                  void *stream) {
    if (n < 0) return KGQ_ERR_INVALID_ARG;
    if (n == 0) return KGQ_OK;
    if (!g || !mask || !out) return KGQ_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if ((n & 3) == 0 && (((uintptr_t)g | (uintptr_t)out) & 15u) == 0) {
        const int64_t n4 = n / 4;
        int64_t blocks = (n4 + 255) / 256;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        mask_apply_vec_kernel<<<(int)blocks, 256, 0, s>>>(reinterpret_cast<const float4 *>(g), mask, n4,
                                                          reinterpret_cast<float4 *>(out));
    } else {
        int64_t blocks = (n + 255) / 256;
        if (blocks > (int64_t)kSMs * 16) blocks = (int64_t)kSMs * 16;
        mask_apply_kernel<<<(int)blocks, 256, 0, s>>>(g, mask, n, out);
    }
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}


// ---------------------------------------------------------------------------
// Deterministic scatter-add of several gathers' gradients into one source
// (tape.py:229-232 + the routing order of tape.py:204-209): list i is
// np.add.at(zeros, idx_i, g_i) -- duplicates accumulated sequentially in
// occurrence order, starting from +0 -- and the lists are combined as
// ((s_0 + s_1) + s_2) ... with absent rows contributing +0, exactly the
// reference's dense sums.  The caller sorts positions by (row, position)
// (positions are list-major), so one warp walks each row's occurrences in
// order; rows that occur in no list are left untouched (the caller zeroes).
// ---------------------------------------------------------------------------
constexpr int kMaxScatterLists = 8;
struct ListEnds { int64_t e[kMaxScatterLists]; };

__global__ void __launch_bounds__(256)
scatter_rows_multi_kernel(const int64_t *__restrict__ order, const int32_t *__restrict__ idx, int64_t m,
                          ListEnds list_end, int n_lists, const float *__restrict__ g,
                          int d, float *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= m) return;
    const int64_t pos0 = __ldg(order + i);
    const int32_t row = __ldg(idx + pos0);
    if (row < 0) return;                                             // not owned here: skipped
    if (i > 0 && __ldg(idx + __ldg(order + i - 1)) == row) return;   // not the first occurrence
    for (int f0 = 0; f0 < d; f0 += 32) {
        const int f = f0 + lane;
        float total = 0.0f, acc = 0.0f;
        int li = 0;                                   // next list to fold into total
        for (int64_t j = i; j < m; j++) {
            const int64_t pos = __ldg(order + j);
            if (__ldg(idx + pos) != row) break;
            int l = 0;
            while (l + 1 < n_lists && pos >= list_end.e[l]) l++;
            for (; li < l; li++) {                    // finish list li (complete or absent)
                total = li == 0 ? acc : __fadd_rn(total, acc);
                acc = 0.0f;
            }
            if (f < d) acc = __fadd_rn(acc, __ldg(g + pos * d + f));
        }
        for (; li < n_lists; li++) {
            total = li == 0 ? acc : __fadd_rn(total, acc);
            acc = 0.0f;
        }
        if (f < d) out[(int64_t)row * d + f] = total;
    }
}

// Sort-free variant (order == NULL, m <= 16384): warp w takes position w;
// it proceeds only if no earlier position holds the same row (a 32-wide
// ballot scan), then walks the later positions in order, so each row is
// still folded in position order by exactly one warp.  O(m^2 / 32) compares,
// all L1/L2-resident for a training batch (m = 3B).
__global__ void __launch_bounds__(256)
scatter_rows_multi_nosort_kernel(const int32_t *__restrict__ idx, int64_t m, ListEnds list_end, int n_lists,
                                 const float *__restrict__ g, int d, float *__restrict__ out,
                                 int32_t *__restrict__ rowmap = nullptr) {
    constexpr int NF = 4;                           // features per lane: d <= 128
    extern __shared__ int32_t sidx[];               // the whole id list (m <= 16384), staged once per CTA
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) sidx[k] = __ldg(idx + k);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= m) return;
    const int32_t row = sidx[i];
    if (row < 0) return;                            // not owned here: skipped
    // one pass over the lists, 4 chunks of 32 ids per step (independent
    // loads in flight): an earlier occurrence owns the row -> exit; later
    // ones are folded in position order, all features at once
    float total[NF], acc[NF];
#pragma unroll
    for (int k = 0; k < NF; k++) total[k] = acc[k] = 0.0f;
    int li = 0;
    for (int64_t j0 = 0; j0 < m; j0 += 128) {
        uint32_t hit[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int64_t j = j0 + 32 * u + lane;
            hit[u] = __ballot_sync(0xffffffffu, j < m && sidx[j] == row);
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            uint32_t hits = hit[u];
            const int64_t base = j0 + 32 * u;
            if (base + 32 <= i) {
                if (hits) return;                   // an earlier position holds the row
                continue;
            }
            if (base < i) {                         // chunk containing i
                if (hits & ((1u << (int)(i - base)) - 1u)) return;
                hits &= ~((1u << (int)(i - base)) - 1u);
            }
            while (hits) {
                // up to 4 occurrences: their rows are loaded together (independent
                // loads in flight), then folded strictly in position order
                int64_t ps[4];
                int cnt = 0;
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    if (hits) {
                        ps[t] = base + (__ffs(hits) - 1);
                        hits &= hits - 1;
                        cnt = t + 1;
                    } else {
                        ps[t] = ps[0];
                    }
                }
                float v[4][NF];
#pragma unroll
                for (int t = 0; t < 4; t++)
#pragma unroll
                    for (int k = 0; k < NF; k++) {
                        const int f = lane + 32 * k;
                        v[t][k] = (t < cnt && f < d) ? __ldg(g + ps[t] * d + f) : 0.0f;
                    }
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    if (t < cnt) {
                        int l = 0;
                        while (l + 1 < n_lists && ps[t] >= list_end.e[l]) l++;
                        for (; li < l; li++) {
#pragma unroll
                            for (int k = 0; k < NF; k++) {
                                total[k] = li == 0 ? acc[k] : __fadd_rn(total[k], acc[k]);
                                acc[k] = 0.0f;
                            }
                        }
#pragma unroll
                        for (int k = 0; k < NF; k++)
                            if (lane + 32 * k < d) acc[k] = __fadd_rn(acc[k], v[t][k]);
                    }
                }
            }
        }
    }
    for (; li < n_lists; li++) {
#pragma unroll
        for (int k = 0; k < NF; k++) {
            total[k] = li == 0 ? acc[k] : __fadd_rn(total[k], acc[k]);
            acc[k] = 0.0f;
        }
    }
    // dense: out[row]; compact (rowmap != null): out[i] and rowmap[row] = i
    float *orow = rowmap ? out + i * d : out + (int64_t)row * d;
    if (rowmap && lane == 0) rowmap[row] = (int32_t)i;
#pragma unroll
    for (int k = 0; k < NF; k++) {
        const int f = lane + 32 * k;
        if (f < d) orow[f] = total[k];
    }
}

// Compact form of kgq_scatter_rows_multi_f32 (sort-free kernel only): the
// summed row of each distinct id goes to rows[i], i = its first position in
// the concatenated lists, and rowmap[id] = i (rowmap pre-filled with -1 by
// the caller: the rows never touched stay -1, i.e. zero gradient).
extern "C" int kgq_scatter_rows_multi_sparse_f32(const int32_t *idx, int64_t m, const int64_t *list_end,
                                                 int32_t n_lists, const float *g, int32_t d, float *rows,
                                                 int32_t *rowmap, void *stream) {
    if (m < 0 || d < 1 || d > 128 || m > 16384 || n_lists < 1 || n_lists > kMaxScatterLists || !list_end)
        return KGQ_ERR_INVALID_ARG;
    if (m == 0) return KGQ_OK;
    if (!idx || !g || !rows || !rowmap) return KGQ_ERR_INVALID_ARG;
    ListEnds ends;
    for (int i = 0; i < kMaxScatterLists; i++) ends.e[i] = i < n_lists ? list_end[i] : m;
    const int64_t blocks = (m * 32 + 255) / 256;
    const size_t smem = (size_t)m * sizeof(int32_t);
    if (smem > 48 * 1024) {
        static bool attr = false;
        if (!attr) {
            cudaError_t e = cudaFuncSetAttribute(scatter_rows_multi_nosort_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
            if (e != cudaSuccess) return kgq_set_cuda_error(e);
            attr = true;
        }
    }
    scatter_rows_multi_nosort_kernel<<<(int)blocks, 256, smem, (cudaStream_t)stream>>>(idx, m, ends, n_lists, g, d,
                                                                                     rows, rowmap);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_scatter_rows_multi_f32(const int64_t *order, const int32_t *idx, int64_t m,
                                          const int64_t *list_end, int32_t n_lists, const float *g,
                                          int32_t d, float *out, void *stream) {
    if (m < 0 || d < 1 || n_lists < 1 || n_lists > kMaxScatterLists || !list_end) return KGQ_ERR_INVALID_ARG;
    if (m == 0) return KGQ_OK;
    if (!idx || !g || !out) return KGQ_ERR_INVALID_ARG;
    ListEnds ends;                                  // host array -> kernel parameter (graph-capturable)
    for (int i = 0; i < kMaxScatterLists; i++) ends.e[i] = i < n_lists ? list_end[i] : m;
    const int64_t blocks = (m * 32 + 255) / 256;
    if (!order) {
        if (m > 16384 || d > 128) return KGQ_ERR_INVALID_ARG;  // quadratic in m; <= 4 features per lane
        const size_t smem = (size_t)m * sizeof(int32_t);
        if (smem > 48 * 1024) {
            static bool attr = false;
            if (!attr) {
                cudaError_t e = cudaFuncSetAttribute(scatter_rows_multi_nosort_kernel,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
                if (e != cudaSuccess) return kgq_set_cuda_error(e);
                attr = true;
            }
        }
        scatter_rows_multi_nosort_kernel<<<(int)blocks, 256, smem, (cudaStream_t)stream>>>(idx, m, ends, n_lists,
                                                                                         g, d, out);
        KGQ_LAUNCH_CHECK();
        return KGQ_OK;
    }
    scatter_rows_multi_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(order, idx, m, ends, n_lists,
                                                                           g, d, out);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

// ---------------------------------------------------------------------------
// Gather of a lazily-summed readout (tape.LazySumWire): out[i] =
// ((t_0[idx[i]] + t_1[idx[i]]) + ...) in the terms' order -- the rows of
// the materialized sum, bit for bit, in one launch instead of one gather per
// term plus the adds.
// ---------------------------------------------------------------------------
constexpr int kMaxSumTerms = 8;
struct SumTerms { const float *t[kMaxSumTerms]; };

// base (optional, n_idx x d, may alias out): a running sum of earlier terms'
// gathered rows, added first -- ((base + t_0[idx]) + t_1[idx]) + ... -- so a
// readout can be accumulated term by term as each layer output dies.
__global__ void gather_rows_sum_kernel(const float *base, SumTerms terms, int n_terms,
                                       const int64_t *__restrict__ idx, int64_t n_idx, int d, float *out) {
    const int64_t total = n_idx * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / d;
        const int f = (int)(e - i * d);
        const int64_t r = __ldg(idx + i);
        float acc = base ? base[e] : __ldg(terms.t[0] + r * d + f);
        for (int k = base ? 0 : 1; k < n_terms; k++) acc = __fadd_rn(acc, __ldg(terms.t[k] + r * d + f));
        out[e] = acc;
    }
}

static int launch_gather_rows_sum(const float *base, const float *const *terms, int32_t n_terms, const int64_t *idx,
                                  int64_t n_idx, int32_t d, float *out, void *stream) {
    if (n_terms < 1 || n_terms > kMaxSumTerms || n_idx < 0 || d < 1 || !terms) return KGQ_ERR_INVALID_ARG;
    if (n_idx == 0) return KGQ_OK;
    if (!idx || !out) return KGQ_ERR_INVALID_ARG;
    SumTerms t;                                     // host array of device pointers -> kernel parameter
    for (int k = 0; k < kMaxSumTerms; k++) t.t[k] = k < n_terms ? terms[k] : nullptr;
    for (int k = 0; k < n_terms; k++) if (!t.t[k]) return KGQ_ERR_INVALID_ARG;
    const int64_t total = n_idx * d;
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)kSMs * 8) blocks = (int64_t)kSMs * 8;
    gather_rows_sum_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(base, t, n_terms, idx, n_idx, d, out);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_gather_rows_sum_f32(const float *const *terms, int32_t n_terms, const int64_t *idx,
                                       int64_t n_idx, int32_t d, float *out, void *stream) {
    return launch_gather_rows_sum(nullptr, terms, n_terms, idx, n_idx, d, out, stream);
}

extern "C" int kgq_gather_rows_acc_f32(const float *base, const float *const *terms, int32_t n_terms,
                                       const int64_t *idx, int64_t n_idx, int32_t d, float *out, void *stream) {
    if (!base) return KGQ_ERR_INVALID_ARG;
    return launch_gather_rows_sum(base, terms, n_terms, idx, n_idx, d, out, stream);
}

// The BPR batch's three gather index lists from one [B][3] (user, pos item,
// neg item) int32 batch: node ids users / num_users + pos / num_users + neg,
// as int32 (the gather contexts, tape.py:143-152) and int64 (the gathers).
__global__ void batch_indices_kernel(const int32_t *__restrict__ batch, int64_t B, int64_t num_users,
                                     int32_t *__restrict__ idx32, int64_t *__restrict__ idx64) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * B; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t list = i / B, r = i % B;
        const int64_t v = (int64_t)__ldg(batch + 3 * r + list) + (list ? num_users : 0);
        idx32[i] = (int32_t)v;
        idx64[i] = v;
    }
}

extern "C" int kgq_batch_indices(const int32_t *batch, int64_t B, int64_t num_users, int32_t *idx32,
                                 int64_t *idx64, void *stream) {
    if (B < 0 || num_users < 0) return KGQ_ERR_INVALID_ARG;
    if (B == 0) return KGQ_OK;
    if (!batch || !idx32 || !idx64) return KGQ_ERR_INVALID_ARG;
    const int64_t n = 3 * B, blocks = (n + 255) / 256 < 4 * kSMs ? (n + 255) / 256 : 4 * kSMs;
    batch_indices_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(batch, B, num_users, idx32, idx64);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
