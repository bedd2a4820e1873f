// kgq_topk.cu -- per-row Top-K of the evaluation score block (train.py:121-150:
// ``np.argsort(-s, kind="stable")[:k]`` after the train positives are set to
// -inf), replacing a full sort of every user's item scores.
//
// Order: descending score, ties by ascending item index (the stable argsort of
// -s), -0.0 == +0.0, -inf after every finite score, NaN after -inf (numpy
// sorts NaN last).  One 64-bit key per item carries the whole order:
//   hi = order-preserving bits of the score (NaN -> 0), lo = ~index,
// so "larger key" == "ranks earlier" and all keys of a row are distinct.
//
// One warp per row: lane l scans items l, l+32, ... keeping its own best KM
// keys in registers (sorted, fully unrolled insertion; an item only enters
// when it beats both the lane's KM-th key and the warp-wide threshold), then
// k rounds of a warp argmax over the lane heads pop the row's top-k in order.  The score block is read
// once, coalesced; nothing is written but k indices per row.
#include "kgq_common.cuh"

namespace kgq {

__device__ __forceinline__ uint64_t rank_key(float s, uint32_t idx) {
    uint32_t b = __float_as_uint(s);
    if (b == 0x80000000u) b = 0u;                              // -0.0 ranks as +0.0
    uint32_t o = (b & 0x80000000u) ? ~b : (b | 0x80000000u);   // monotone in s
    if (s != s) o = 0u;                                        // NaN: last
    return ((uint64_t)o << 32) | (uint64_t)(0xFFFFFFFFu - idx);
}

template <int KM>
__global__ void __launch_bounds__(256)
topk_rows_kernel(const float *__restrict__ scores, int64_t n_rows, int64_t n_cols, int64_t ld, int k,
                 int32_t *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= n_rows) return;
    const float *s = scores + row * ld;
    uint64_t L[KM];                     // descending; 0 = empty (below every real key)
#pragma unroll
    for (int j = 0; j < KM; j++) L[j] = 0ull;
    // thr = max over lanes of their KM-th best: that lane holds KM keys >= thr,
    // so no key below it can reach the row's top KM >= k (warp-shared pruning)
    uint64_t thr = 0ull;
    auto insert = [&](uint64_t x) {
        if (x <= thr || x <= L[KM - 1]) return;
#pragma unroll
        for (int j = KM - 1; j > 0; j--) {
            if (x > L[j - 1]) L[j] = L[j - 1];
            else if (x > L[j]) L[j] = x;
        }
        if (x > L[0]) L[0] = x;
    };
    int64_t c = lane;
    for (; c + 96 < n_cols; c += 128) {             // 4 loads in flight per lane
        const float v0 = __ldg(s + c), v1 = __ldg(s + c + 32), v2 = __ldg(s + c + 64), v3 = __ldg(s + c + 96);
        insert(rank_key(v0, (uint32_t)c));
        insert(rank_key(v1, (uint32_t)(c + 32)));
        insert(rank_key(v2, (uint32_t)(c + 64)));
        insert(rank_key(v3, (uint32_t)(c + 96)));
        uint64_t t = L[KM - 1];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t other = __shfl_xor_sync(0xffffffffu, t, o);
            t = other > t ? other : t;
        }
        thr = t;
    }
    for (; c < n_cols; c += 32) insert(rank_key(__ldg(s + c), (uint32_t)c));
    // k rounds: warp max over the lane heads; the winning lane pops its head
    for (int r = 0; r < k; r++) {
        uint64_t best = L[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t other = __shfl_xor_sync(0xffffffffu, best, o);
            best = other > best ? other : best;
        }
        if (lane == 0) out[row * k + r] = best ? (int32_t)(0xFFFFFFFFu - (uint32_t)best) : -1;
        if (best != 0ull && L[0] == best) {          // keys are distinct: exactly one lane
#pragma unroll
            for (int j = 0; j < KM - 1; j++) L[j] = L[j + 1];
            L[KM - 1] = 0ull;
        }
    }
}

}  // namespace kgq

using namespace kgq;

extern "C" int kgq_topk_rows_f32(const float *scores, int64_t n_rows, int64_t n_cols, int64_t ld, int32_t k,
                                 int32_t *out_idx, void *stream) {
    if (n_rows < 0 || n_cols < 0 || k < 1 || k > 64 || ld < n_cols || n_cols >= 0xFFFFFFFFll)
        return KGQ_ERR_INVALID_ARG;
    if (n_rows == 0) return KGQ_OK;
    if (!scores || !out_idx) return KGQ_ERR_INVALID_ARG;
    const int64_t blocks = (n_rows + 7) / 8;
    if (blocks > 0x7fffffff) return KGQ_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (k <= 16) topk_rows_kernel<16><<<(int)blocks, 256, 0, st>>>(scores, n_rows, n_cols, ld, k, out_idx);
    else if (k <= 32) topk_rows_kernel<32><<<(int)blocks, 256, 0, st>>>(scores, n_rows, n_cols, ld, k, out_idx);
    else topk_rows_kernel<64><<<(int)blocks, 256, 0, st>>>(scores, n_rows, n_cols, ld, k, out_idx);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
