// kgq_eval.cu -- K12: fused evaluation scoring + Top-K (train.py:121-160:
// scores = readout[u] @ item_emb^T; s[train positives] = -inf;
// np.argsort(-s, kind="stable")[:k]) with no score matrix in HBM.
//
// One CTA per block of 128 test users (M = 128), walking all items in tiles
// of 128 (N = 128), warp-specialized:
//   warp 0  TMA producer: item tiles of the pre-split item embeddings (3xTF32
//           hi and lo, [items][d] fp32, 128-row x 32-column SWIZZLE_128B boxes)
//           into a 2-stage ring;
//   warp 1  MMA issuer: scores tile = U . I^T as 3 passes (lo.hi, hi.lo,
//           hi.hi) of d/8 kind::tf32 MMAs, M = 128, N = 128, into one of two
//           TMEM accumulators (128 columns each);
//   warps 2-5  ranking, thread = user (its TMEM lane): each tile's 128 scores
//           come out of TMEM 32 at a time; a score is looked at closely only if
//           it is >= the score at the end of the user's running list (or the
//           list is not full yet): then the user's train positives (sorted;
//           one forward-moving cursor) decide whether it is -inf, and its
//           64-bit rank key (kgq_topk.cu: order-preserving score bits with
//           -0 == +0 and NaN last, then ~index) is inserted into the list held
//           in registers (KM keys, descending; keys are distinct, so the order
//           is numpy's stable one).
// The user rows are staged (split hi/lo) by the ranking warps at the start.
// 3xTF32 with fp32 accumulation: fp32-level scores (the reference's float32
// matmul ranks ties of equal fp32 scores by index; integer-valued embeddings
// give exact scores, tests/golden/eval.npz).
#include "kgq_tma.cuh"

namespace kgq {

constexpr int kEvM = 128, kEvN = 128, kEvStages = 2;
constexpr int kEvThreads = 192;

template <int D>
struct EvSmem {
    static constexpr uint32_t A = kEvM * D * 4;                    // user rows hi or lo
    static constexpr uint32_t BT = kEvN * D * 4;                   // item tile hi or lo
    static constexpr uint32_t STAGE = 2 * BT;
    static constexpr uint32_t SC = kEvM * 36 * 4;                 // per-user score spill (36-float rows)
    static constexpr uint32_t BAR = 2 * A + kEvStages * STAGE + SC;
    static constexpr size_t bytes = (size_t)BAR + 256 + 1024;
};

__device__ __forceinline__ uint64_t ev_key(float s, uint32_t idx) {
    uint32_t b = __float_as_uint(s);
    if (b == 0x80000000u) b = 0u;                              // -0.0 ranks as +0.0
    uint32_t o = (b & 0x80000000u) ? ~b : (b | 0x80000000u);   // monotone in s
    if (s != s) o = 0u;                                        // NaN: last
    return ((uint64_t)o << 32) | (uint64_t)(0xFFFFFFFFu - idx);
}
// score of a key's high word (empty / NaN -> NaN)
__device__ __forceinline__ float ev_key_score(uint64_t key) {
    const uint32_t o = (uint32_t)(key >> 32);
    if (o == 0u) return __uint_as_float(0x7FC00000u);
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

template <int D, int KM>
__global__ void __launch_bounds__(kEvThreads, 1)
score_topk_kernel(const __grid_constant__ CUtensorMap tm_ihi, const __grid_constant__ CUtensorMap tm_ilo,
                  const float *__restrict__ readout, const int64_t *__restrict__ users, int64_t n_users,
                  int64_t n_items, const int32_t *__restrict__ train_items,
                  const int64_t *__restrict__ train_start, const int64_t *__restrict__ train_end,
                  int32_t k, int32_t *__restrict__ out) {
    using S = EvSmem<D>;
    extern __shared__ uint8_t ev_raw[];
    uint8_t *sm = ev_raw + ((1024u - (tc::smem_u32(ev_raw) & 1023u)) & 1023u);
    float *ahi = reinterpret_cast<float *>(sm), *alo = reinterpret_cast<float *>(sm + S::A);
    uint8_t *stage0 = sm + 2 * S::A;
    float *spill = reinterpret_cast<float *>(sm + 2 * S::A + kEvStages * S::STAGE);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S::BAR);
    uint64_t *bfull = bar, *bempty = bar + kEvStages, *dfull = bar + 2 * kEvStages, *dempty = bar + 2 * kEvStages + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 2 * kEvStages + 4);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int64_t u0 = (int64_t)blockIdx.x * kEvM;
    const int n_tiles = (int)((n_items + kEvN - 1) / kEvN);

    if (t == 0) {
        for (int i = 0; i < kEvStages; i++) { tc::mbar_init(bfull + i, 1); tc::mbar_init(bempty + i, 1); }
        for (int i = 0; i < 2; i++) { tc::mbar_init(dfull + i, 1); tc::mbar_init(dempty + i, 128); }
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 256);
    // user rows, split hi/lo, K-major SWIZZLE_128B (thread = row: conflict-free 16-B stores)
    if (warp >= 2) {
        const int r = 32 * (warp & 3) + lane;
        const int64_t ur = u0 + r;
        const float4 *src = ur < n_users ? reinterpret_cast<const float4 *>(readout + __ldg(users + ur) * D) : nullptr;
#pragma unroll
        for (int c4 = 0; c4 < D / 4; c4++) {
            const float4 v = src ? __ldg(src + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
            float4 h, l;
            tc::split_tf32_fast(v.x, h.x, l.x);
            tc::split_tf32_fast(v.y, h.y, l.y);
            tc::split_tf32_fast(v.z, h.z, l.z);
            tc::split_tf32_fast(v.w, h.w, l.w);
            const uint32_t o = tc::sw128_off(r, 4 * c4, kEvM) / 4;
            *reinterpret_cast<float4 *>(ahi + o) = h;
            *reinterpret_cast<float4 *>(alo + o) = l;
        }
    }
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------
        if (lane == 0) {
            for (int it = 0; it < n_tiles; it++) {
                const int s = it % kEvStages;
                if (it >= kEvStages) tc::mbar_wait_sleep(bempty + s, (uint32_t)((it / kEvStages - 1) & 1));
                uint8_t *st = stage0 + s * S::STAGE;
                tma::expect_tx(bfull + s, S::STAGE);
#pragma unroll
                for (int cb = 0; cb < D / 32; cb++) {
                    tma::load_2d(st + cb * (kEvN * 128), &tm_ihi, 32 * cb, it * kEvN, bfull + s);
                    tma::load_2d(st + S::BT + cb * (kEvN * 128), &tm_ilo, 32 * cb, it * kEvN, bfull + s);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------ MMA issuer ------------------------------
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_tf32(kEvM, kEvN);
            const uint32_t ah = tc::smem_u32(ahi), al = tc::smem_u32(alo);
            for (int it = 0; it < n_tiles; it++) {
                const int s = it % kEvStages, b = it & 1;
                tc::mbar_wait_sleep(bfull + s, (uint32_t)((it / kEvStages) & 1));
                if (it >= 2) tc::mbar_wait_sleep(dempty + b, (uint32_t)(((it >> 1) - 1) & 1));
                tc::fence_after();
                const uint32_t bh = tc::smem_u32(stage0 + s * S::STAGE), bl = bh + S::BT;
                const uint32_t dd = tmem + 128u * b;
#pragma unroll
                for (int p = 0; p < 3; p++) {          // lo.hi, hi.lo, hi.hi
                    const uint32_t sa = p == 0 ? al : ah, sb = p == 1 ? bl : bh;
#pragma unroll
                    for (int ks = 0; ks < D / 8; ks++)
                        tc::mma_tf32(dd, tc::kmajor_sw128_desc(sa, ks, kEvM), tc::kmajor_sw128_desc(sb, ks, kEvN),
                                     idesc, (p | ks) != 0);
                }
                tc::commit(bempty + s);
                tc::commit(dfull + b);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------ ranking ------------------------------
        const int q = warp & 3;
        const int r = 32 * q + lane;
        const int64_t ur = u0 + r;
        const bool live = ur < n_users;
        int64_t tp = live ? __ldg(train_start + ur) : 0, te = live ? __ldg(train_end + ur) : 0;
        int32_t tnext = tp < te ? __ldg(train_items + tp) : 0x7FFFFFFF;
        uint64_t e[KM];
#pragma unroll
        for (int i = 0; i < KM; i++) e[i] = 0ull;
        float bar_f = 0.0f;
        bool open = true;                         // list not full: every item is looked at
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        for (int it = 0; it < n_tiles; it++) {
            const int b = it & 1;
            tc::mbar_wait(dfull + b, (uint32_t)((it >> 1) & 1));
            tc::fence_after();
#pragma unroll 1
            for (int ch = 0; ch < kEvN / 32; ch++) {
                float v[32];
                tc::tmem_ld32(tmem + lane_addr + 128u * b + 32u * ch, v);
                if (ch == kEvN / 32 - 1) {
                    tc::fence_before();
                    tc::mbar_arrive(dempty + b);
                }
                const int64_t base = (int64_t)it * kEvN + 32 * ch;
                // candidates: scores >= the list's last (a superset: the bar only rises)
                uint32_t cand = 0u;
#pragma unroll
                for (int j = 0; j < 32; j++) cand |= (open || v[j] >= bar_f) ? (1u << j) : 0u;
                const int64_t left = n_items - base;
                if (left < 32) cand &= left > 0 ? (1u << left) - 1u : 0u;
                if (live && cand) {
                    // one copy of the insertion code: the chunk goes through shared memory
                    float *sp = spill + r * 36;
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<float4 *>(sp + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                    while (cand) {
                        const int j = __ffs(cand) - 1;
                        cand &= cand - 1u;
                        float s = sp[j];
                        if (!(open || s >= bar_f)) continue;
                        const int32_t item = (int32_t)(base + j);
                        while (tnext < item) { ++tp; tnext = tp < te ? __ldg(train_items + tp) : 0x7FFFFFFF; }
                        if (tnext == item) s = -INFINITY;                   // train positive
                        const uint64_t x = ev_key(s, (uint32_t)item);
                        if (x > e[KM - 1]) {
#pragma unroll
                            for (int i = KM - 1; i > 0; i--) e[i] = e[i - 1] > x ? (e[i] > x ? e[i] : x) : e[i - 1];
                            e[0] = e[0] > x ? e[0] : x;
                            open = e[KM - 1] == 0ull;
                            bar_f = ev_key_score(e[KM - 1]);
                            if (bar_f != bar_f) open = true;      // NaN / empty tail: keep looking
                        }
                    }
                }
            }
        }
        if (live) {
            int32_t *o = out + ur * k;
#pragma unroll
            for (int i = 0; i < KM; i++)
                if (i < k) o[i] = e[i] ? (int32_t)(0xFFFFFFFFu - (uint32_t)(e[i] & 0xFFFFFFFFu)) : -1;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_free(tmem, 256);
}

// hi / lo = the 3xTF32 split of x (the item embeddings, once per evaluation)
__global__ void split_tf32_kernel(const float *__restrict__ x, int64_t n, float *__restrict__ hi,
                                  float *__restrict__ lo) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        tc::split_tf32_fast(__ldg(x + i), hi[i], lo[i]);
}

}  // namespace kgq

using namespace kgq;

extern "C" size_t kgq_score_topk_workspace_bytes(int64_t n_items, int32_t d) {
    return (size_t)2 * (size_t)n_items * (size_t)d * sizeof(float) + 256;
}

template <int D, int KM>
static int launch_score_topk(const CUtensorMap &th, const CUtensorMap &tl, const float *readout,
                             const int64_t *users, int64_t n_users, int64_t n_items, const int32_t *train_items,
                             const int64_t *train_start, const int64_t *train_end, int32_t k, int32_t *out,
                             cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(score_topk_kernel<D, KM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)EvSmem<D>::bytes);
        if (e != cudaSuccess) return kgq_set_cuda_error(e);
        attr = true;
    }
    const int64_t blocks = (n_users + kEvM - 1) / kEvM;
    score_topk_kernel<D, KM><<<(unsigned)blocks, kEvThreads, EvSmem<D>::bytes, s>>>(
        th, tl, readout, users, n_users, n_items, train_items, train_start, train_end, k, out);
    KGQ_LAUNCH_CHECK();
    return KGQ_OK;
}

extern "C" int kgq_score_topk_f32(const float *readout, const int64_t *users, int64_t n_users,
                                  const float *item_emb, int64_t n_items, int32_t d,
                                  const int32_t *train_items, const int64_t *train_start,
                                  const int64_t *train_end, int32_t k, int32_t *out,
                                  void *workspace, size_t workspace_bytes, void *stream) {
    if (n_users < 0 || n_items < 0 || k < 1 || k > 32) return KGQ_ERR_INVALID_ARG;
    if (d != 32 && d != 64) return KGQ_ERR_INVALID_ARG;
    if (n_users == 0) return KGQ_OK;
    if (!readout || !users || !item_emb || !train_items || !train_start || !train_end || !out || !workspace)
        return KGQ_ERR_INVALID_ARG;
    if (n_items < 1 || n_items > 0x7FFFFFFFll) return KGQ_ERR_INVALID_ARG;
    if (workspace_bytes < kgq_score_topk_workspace_bytes(n_items, d)) return KGQ_ERR_INVALID_ARG;
    if (((uintptr_t)readout | (uintptr_t)item_emb | (uintptr_t)workspace) & 15u) return KGQ_ERR_MISALIGNED;
    cudaStream_t s = (cudaStream_t)stream;
    float *hi = reinterpret_cast<float *>(workspace), *lo = hi + n_items * d;
    const int64_t n = n_items * d;
    split_tf32_kernel<<<(unsigned)((n + 255) / 256 < 4 * kSMs ? (n + 255) / 256 : 4 * kSMs), 256, 0, s>>>(
        item_emb, n, hi, lo);
    KGQ_LAUNCH_CHECK();
    CUtensorMap th, tl;
    if (!tma::make_rowmajor_f32(&th, hi, (uint64_t)n_items, (uint64_t)d, kEvN) ||
        !tma::make_rowmajor_f32(&tl, lo, (uint64_t)n_items, (uint64_t)d, kEvN))
        return KGQ_ERR_CUDA;
#define KGQ_EV(DD, KK) launch_score_topk<DD, KK>(th, tl, readout, users, n_users, n_items, train_items, \
                                                  train_start, train_end, k, out, s)
    if (d == 64) {
        if (k <= 8) return KGQ_EV(64, 8);
        if (k <= 16) return KGQ_EV(64, 16);
        if (k <= 24) return KGQ_EV(64, 24);
        return KGQ_EV(64, 32);
    }
    if (k <= 8) return KGQ_EV(32, 8);
    if (k <= 16) return KGQ_EV(32, 16);
    if (k <= 24) return KGQ_EV(32, 24);
    return KGQ_EV(32, 32);
#undef KGQ_EV
}
