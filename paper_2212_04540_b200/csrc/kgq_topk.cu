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
// One warp per row streams the row as float4 (scalar head/tail around the
// 16-byte boundaries) and keeps the row's exact running top-k as a sorted list
// distributed over the lanes (entry i in lane i % 32).  A key enters only if
// it beats entry k-1 (a ballot per loaded element; after the first few passes
// almost nothing does), by one ballot-count + shuffle-up.  The score block is
// read once, coalesced; nothing is written but k indices per row.
#include "kgq_common.cuh"

namespace kgq {

__device__ __forceinline__ uint64_t rank_key(float s, uint32_t idx) {
    uint32_t b = __float_as_uint(s);
    if (b == 0x80000000u) b = 0u;                              // -0.0 ranks as +0.0
    uint32_t o = (b & 0x80000000u) ? ~b : (b | 0x80000000u);   // monotone in s
    if (s != s) o = 0u;                                        // NaN: last
    return ((uint64_t)o << 32) | (uint64_t)(0xFFFFFFFFu - idx);
}

// The row's running top-k, distributed over the warp: entry i lives in lane
// i % 32 of register i / 32 (NR registers, k <= 32 * NR), descending; 0 = empty.
template <int NR>
struct WarpList {
    uint64_t e[NR];
    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int r = 0; r < NR; r++) e[r] = 0ull;
    }
    // entry j (warp-uniform j), broadcast to every lane
    __device__ __forceinline__ uint64_t at(int j) const {
        uint64_t v = e[0];
#pragma unroll
        for (int r = 1; r < NR; r++)
            if ((j >> 5) == r) v = e[r];
        return __shfl_sync(0xffffffffu, v, j & 31);
    }
    // insert a key larger than entry k-1 (warp-uniform x; keys are distinct)
    __device__ __forceinline__ void insert(uint64_t x, int lane) {
        int pos = 0;
#pragma unroll
        for (int r = 0; r < NR; r++) pos += __popc(__ballot_sync(0xffffffffu, e[r] > x));
        uint64_t carry = 0ull;                       // entry 32r - 1 of the old list
#pragma unroll
        for (int r = 0; r < NR; r++) {
            const uint64_t up = __shfl_up_sync(0xffffffffu, e[r], 1);
            const uint64_t last = __shfl_sync(0xffffffffu, e[r], 31);
            const int j = 32 * r + lane;
            const uint64_t shifted = lane == 0 ? carry : up;
            e[r] = j < pos ? e[r] : (j == pos ? x : shifted);
            carry = last;
        }
    }
};

template <int NR>
__global__ void __launch_bounds__(256)
topk_rows_kernel(const float *__restrict__ scores, int64_t n_rows, int64_t n_cols, int64_t ld, int k,
                 int32_t *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= n_rows) return;                       // warp-uniform
    const float *s = scores + row * ld;
    WarpList<NR> L;
    L.clear();
    uint64_t thr = 0ull;                             // entry k-1: the bar a key must clear
    // one candidate key per lane: every lane whose key clears the bar joins,
    // in lane order, re-checked against the bar as it rises
    auto offer = [&](uint64_t key, bool valid) {
        uint32_t m = __ballot_sync(0xffffffffu, valid && key > thr);
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const uint64_t x = __shfl_sync(0xffffffffu, key, src);
            if (x > thr) {
                L.insert(x, lane);
                thr = L.at(k - 1);
            }
        }
    };
    // head: scalar items up to the first 16-byte boundary of the row
    const int64_t h0 = (int64_t)((4u - (((uintptr_t)s >> 2) & 3u)) & 3u);
    const int64_t head = h0 < n_cols ? h0 : n_cols;
    offer(lane < head ? rank_key(__ldg(s + lane), (uint32_t)lane) : 0ull, lane < head);
    // body: float4 per lane, two per pass (256 items per warp per pass), the
    // next pass's two loaded before this one is ranked; warp-uniform trips
    const float4 *s4 = reinterpret_cast<const float4 *>(s + head);
    const int64_t n4 = (n_cols - head) >> 2;
    const float4 none = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 na = lane < n4 ? __ldg(s4 + lane) : none;
    float4 nb = lane + 32 < n4 ? __ldg(s4 + lane + 32) : none;
    for (int64_t base = 0; base < n4; base += 64) {
        const int64_t fa = base + lane, fb = fa + 32;
        const float4 a = na, b = nb;
        na = fa + 64 < n4 ? __ldg(s4 + fa + 64) : none;
        nb = fb + 64 < n4 ? __ldg(s4 + fb + 64) : none;
        const uint32_t ia = (uint32_t)(head + 4 * fa), ib = (uint32_t)(head + 4 * fb);
        const bool va = fa < n4, vb = fb < n4;
        offer(rank_key(a.x, ia), va);
        offer(rank_key(a.y, ia + 1), va);
        offer(rank_key(a.z, ia + 2), va);
        offer(rank_key(a.w, ia + 3), va);
        offer(rank_key(b.x, ib), vb);
        offer(rank_key(b.y, ib + 1), vb);
        offer(rank_key(b.z, ib + 2), vb);
        offer(rank_key(b.w, ib + 3), vb);
    }
    // tail: the last (n_cols - head) % 4 items
    const int64_t t0 = head + 4 * n4;
    const bool vt = lane < n_cols - t0;
    offer(vt ? rank_key(__ldg(s + t0 + lane), (uint32_t)(t0 + lane)) : 0ull, vt);
    // entries 0..k-1 are the answer, best first
#pragma unroll
    for (int r = 0; r < NR; r++) {
        const int j = 32 * r + lane;
        if (j < k) out[row * k + j] = L.e[r] ? (int32_t)(0xFFFFFFFFu - (uint32_t)L.e[r]) : -1;
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
    if (k <= 32) topk_rows_kernel<1><<<(int)blocks, 256, 0, st>>>(scores, n_rows, n_cols, ld, k, out_idx);
    else topk_rows_kernel<2><<<(int)blocks, 256, 0, st>>>(scores, n_rows, n_cols, ld, k, out_idx);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}
