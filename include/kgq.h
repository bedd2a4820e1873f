/*
 * kgq.h -- C ABI of libkgq (sm_100a), the B200 activation-compression hot path.
 *
 * Every entry point takes plain device pointers, element counts and a CUDA
 * stream (as void*, i.e. a cudaStream_t / CUstream; NULL = legacy default
 * stream).  The caller allocates every buffer: the device entry points never
 * allocate device memory, synchronise the stream, or throw, and keep no state
 * between calls beyond once-per-process kernel setup (dynamic shared-memory
 * opt-ins; the KGQ_BWD_TC A/B switch, read at first use).  They are
 * stream-ordered and CUDA-graph capturable.  The host-buffer entry points
 * (kgq_*_host_f32) block like the numpy calls they replace and create a
 * workspace and streams themselves when the caller passes none.  Return
 * value is a kgq_status (0 = OK).
 *
 * The reference (kgact, pure numpy) has no FFI; each entry point below names
 * the reference function whose semantics it replaces.  The Python host layer
 * (paper_2212_04540_b200/) binds these through ctypes and
 * maps status codes back to the reference's exception classes.
 *
 * Data layout ("group" = one quantization unit = one row of the (-1, G) view
 * of a row-major fp32 tensor; G = cols reproduces the reference's per-row
 * quantizer, quantize.py:184-186):
 *   codes   : uint8  [n_groups][ceil(G*bits/8)]  LSB-first, groups byte aligned
 *             (pack_codes, quantize.py:213-233)
 *   ranges  : fp32   [n_groups]   R = max - min   (quantize.py:185)
 *   offsets : fp32   [n_groups]   Z = min         (quantize.py:184)
 */
#ifndef KGQ_H_
#define KGQ_H_

#include <stddef.h>
#include <stdint.h>

#ifndef KGQ_API
#define KGQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum kgq_status {
    KGQ_OK = 0,
    KGQ_ERR_INVALID_ARG = 1,      /* -> ValueError                     */
    KGQ_ERR_UNSUPPORTED_BITS = 2, /* -> ValueError / EncodingError     */
    KGQ_ERR_CUDA = 3,             /* -> RuntimeError (kgq_last_cuda_error) */
    KGQ_ERR_MISALIGNED = 4,       /* -> ValueError                     */
    KGQ_ERR_SHAPE = 5             /* -> ShapeMismatchError             */
};

/* Rounding modes (QuantConfig.rounding, quantize.py:25-26, :48-49). */
enum kgq_rounding {
    KGQ_ROUND_NEAREST = 0,    /* np.rint, round-half-even (quantize.py:129-130)           */
    KGQ_ROUND_SR_FAST = 1,    /* stochastic, Philox4x32-7 16-bit uniforms     */
    KGQ_ROUND_SR_COMPAT = 2,  /* stochastic, numpy Philox4x64-10 stream (quantize.py:61-102) */
    KGQ_ROUND_SR_NOISE = 3    /* stochastic, caller-supplied float64 uniforms (test seam)  */
};

KGQ_API int kgq_version(void);
KGQ_API const char *kgq_status_string(int status);
/* cudaError_t of the last KGQ_ERR_CUDA returned on this thread. */
KGQ_API int kgq_last_cuda_error(void);

/* quantize_tensor(x, QuantConfig(bits, rounding), RandomStream(seed), tensor_id)
 * quantize.py:177-196 (+ _scale_rows :116-125, _round_block :128-132,
 * pack_codes :213-233, RandomStream :61-102).
 * bits in {1,2,4,8}; noise (n_groups*group float64) only for KGQ_ROUND_SR_NOISE.
 * group_offset: global index of group 0 (row-partitioned tensors key their
 * noise by global row, so any partitioning gives byte-identical codes).
 * tid_base (optional device pointer): the key's tensor id is
 * tensor_id + *tid_base, read on the device -- a captured CUDA graph advances
 * the base between replays so every replay draws fresh noise.             */
KGQ_API int kgq_quantize_f32(const float *x, int64_t n_groups, int32_t group, int32_t bits,
                     int32_t rounding, uint64_t seed, uint64_t tensor_id,
                     const uint64_t *tid_base, int64_t group_offset, const double *noise, uint8_t *codes, float *ranges, float *offsets,
                     void *stream);

/* dequantize_tensor(q, float32), quantize.py:199-210 (+ unpack_codes :236-247). */
KGQ_API int kgq_dequantize_f32(const uint8_t *codes, const float *ranges, const float *offsets,
                       int64_t n_groups, int32_t group, int32_t bits, float *out,
                       void *stream);

/* Host-buffer forms of the two calls above: the reference's own calling
 * convention (numpy arrays in, numpy arrays out; quantize.py:177-210).  The
 * tensor streams through the device in chunks of groups on n_streams CUDA
 * streams (H2D, kernel and D2H of different chunks overlap); the call blocks
 * until the host outputs are written.  Bytes are identical to the device
 * call for any chunking (noise keyed by global group index).
 *   workspace: device memory of kgq_host_workspace_bytes(chunk, ...) bytes,
 *              or NULL (allocated and freed inside the call).
 *   streams:   n_streams caller streams, or NULL (3 created inside the call).
 *   stream:    the work is ordered after this stream's pending work.
 * KGQ_ROUND_SR_NOISE is device-only (returns KGQ_ERR_INVALID_ARG). */
KGQ_API size_t kgq_host_workspace_bytes(int64_t chunk_groups, int32_t group, int32_t bits,
                                        int32_t n_streams);
KGQ_API int kgq_quantize_host_f32(const float *x, int64_t n_groups, int32_t group, int32_t bits,
                                  int32_t rounding, uint64_t seed, uint64_t tensor_id,
                                  int64_t group_offset, uint8_t *codes, float *ranges,
                                  float *offsets, void *workspace, size_t workspace_bytes,
                                  void *const *streams, int32_t n_streams, void *stream);
KGQ_API int kgq_dequantize_host_f32(const uint8_t *codes, const float *ranges, const float *offsets,
                                    int64_t n_groups, int32_t group, int32_t bits, float *out,
                                    void *workspace, size_t workspace_bytes,
                                    void *const *streams, int32_t n_streams, void *stream);

/* Export the exact SR noise a quantize call consumes (exported-noise parity route).
 * fast:   u16 per element, uniform = u16 / 65536.
 * compat: (raw >> 11) per element, uniform = value * 2^-53
 *         (== RandomStream(seed).matrix_uniforms(tid, n_groups, group)). */
KGQ_API int kgq_fast_noise_u16(uint64_t seed, uint64_t tensor_id, int64_t group_offset,
                       int64_t n_groups, int32_t group, uint16_t *out, void *stream);
KGQ_API int kgq_compat_noise_raw53(uint64_t seed, uint64_t tensor_id, int64_t group_offset,
                           int64_t n_groups, int32_t group, uint64_t *out, void *stream);

/* pack_codes / unpack_codes, quantize.py:213-247 (rows byte-aligned, LSB-first).
 * pack: codes uint8 [rows][cols] -> packed [rows][ceil(cols*bits/8)]; a code
 * >= 2^bits sets *overflow (device int32, caller-zeroed) -> EncodingError. */
KGQ_API int kgq_pack_codes(const uint8_t *codes, int64_t rows, int32_t cols, int32_t bits,
                   uint8_t *packed, int32_t *overflow, void *stream);
KGQ_API int kgq_unpack_codes(const uint8_t *packed, int64_t rows, int32_t cols, int32_t bits,
                     uint8_t *codes, void *stream);

/* spmm(A, X) with A in CSR (int32 indptr/indices, fp32 values), X [n_cols][d]
 * row-major: out[i] = sum_{jj in row i, ascending} vals[jj] * X[indices[jj]],
 * accumulated in column order with separate mul and add (tensorops.py:37-50,
 * bit-identical to scipy csr_matvecs).  For the symmetric A_hat this is also
 * spmm_t (tape.py:217-218).  Row i of the output uses indptr[i]..indptr[i+1]
 * as given, so a row-partitioned CSR (global column ids) works unchanged.
 * row_order (optional, n_rows int32): the order rows are scheduled in, by
 * decreasing degree; its first n_heavy rows (long rows) each get a whole CTA
 * (features split across threads, neighbours streamed through shared memory),
 * the rest are processed d/8 lanes per row.  Neither changes the result.    */
KGQ_API int kgq_spmm_csr_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                     int64_t n_rows, const int32_t *row_order, int64_t n_heavy,
                     const float *x, int32_t d, float *out, void *stream);

/* relu + BitMask.from_bool, tensorops.py:84-92 / tape.py:122-126:
 * out = max(x, 0), mask bit i = x[i] > 0, LSB-first flat, ceil(n/8) bytes.  */
KGQ_API int kgq_relu_mask_f32(const float *x, int64_t n, float *out, uint8_t *mask, void *stream);

/* ReLU backward, tape.py:224-225: out = g * mask (mask as above). */
KGQ_API int kgq_mask_apply_f32(const float *g, const uint8_t *mask, int64_t n, float *out,
                       void *stream);

/* Fused decompressor -> weight gradient, tape.py:220-222:
 *   dtheta (+)= dequantize(codes, ranges, offsets)^T @ g
 * codes are per-row groups (group == d), g is [rows][d] fp32, dtheta [d][d].
 * The dequantized activation is never written to memory.  workspace must
 * hold kgq_dequant_gemm_workspace_bytes(rows, d) bytes.  accumulate != 0
 * adds into dtheta.  Deterministic (fixed reduction order). */
KGQ_API size_t kgq_dequant_gemm_workspace_bytes(int64_t rows, int32_t d);
KGQ_API int kgq_dequant_gemm_tn_f32(const uint8_t *codes, const float *ranges, const float *offsets,
                            int64_t rows, int32_t d, int32_t bits, const float *g,
                            float *dtheta, void *workspace, size_t workspace_bytes,
                            int32_t accumulate, void *stream);

/* Adam step, train.py:42-59, fused into one pass with the reference's numpy
 * float32 op order (scalars rounded to float32, true divisions, separate
 * roundings) -- bit-identical to the numpy update.  step >= 1 is the
 * post-increment step count t.  status (nullable, device int64[4] of
 * kgq_check_finite_f32): when status[0] != 0 the update is skipped, so a
 * failed step leaves parameters and moments as they were (train.py:91-93
 * raises before adam_step). */
KGQ_API int kgq_adam_step_f32(float *param, const float *grad, float *m, float *v, int64_t n,
                      double lr, double beta1, double beta2, double eps, int64_t step,
                      const int64_t *status, void *stream);

/* Same update for CUDA-graph replay: i = *step_ptr (device int64) indexes a
 * host-built float32 table c12[2i], c12[2i+1] = 1 - beta1^t, 1 - beta2^t of
 * the steps t the replays run.  n % 4 == 0 and 16-byte alignment. */
KGQ_API int kgq_adam_step_dev_f32(float *param, const float *grad, float *m, float *v, int64_t n,
                          double lr, double beta1, double beta2, double eps,
                          const float *c12, const int64_t *step_ptr, const int64_t *status,
                          void *stream);

/* Per-step health check replacing the reference's host checks
 * (train.py:91-92 non-finite loss -> FloatingPointError; tape.py:256-264
 * non-finite gradient -> ValueError) without a host sync.  tensors[k] (device
 * fp32, sizes[k] elements, k < count <= 8; host arrays read at launch) are
 * scanned; if any holds inf/NaN and status[0] == 0, status[0] = code0 + the
 * first failing k and status[1] = step_host + (*step_dev if step_dev).  The
 * latch is sticky; status[2..3] are scratch the launch resets itself
 * (CUDA-graph replayable).  status: device int64[4], zeroed by the caller. */
KGQ_API int kgq_check_finite_f32(const float *const *tensors, const int64_t *sizes, int32_t count,
                         int32_t code0, const int64_t *step_dev, int64_t step_host,
                         int64_t *status, void *stream);

/* out[rows][d] = a[rows][d] . theta (transpose_theta = 0) or . theta^T (1) on
 * the tcgen05 tensor cores (kind::tf32, 3xTF32 split: fp32-level accuracy),
 * accumulator in TMEM.  d in {32, 64}; other d -> KGQ_ERR_INVALID_ARG (the
 * host falls back to cuBLAS).  The d x d layer GEMM of tape.py:223. */
KGQ_API int kgq_rowmm_f32(const float *a, int64_t rows, int32_t d, const float *theta,
                  int32_t transpose_theta, float *out, void *stream);

/* Fused KGNN layer backward (tape.py:217-225), d in {32, 64, 128}:
 *   g_j = (g_read + g_e) * mask;  dh = g_j . theta^T;  dtheta (+)= Hhat^T . g_j
 * with Hhat = dequantize(codes, ranges, offsets) never materialized.  g_read
 * or g_e may be NULL (not both).  workspace: kgq_layer_backward_workspace_bytes.
 * d = 64 runs on tcgen05 (3xTF32 MMAs, TMEM accumulators; KGQ_BWD_TC=0 selects
 * the FFMA kernel), d = 32 / 128 on FFMA; dtheta is reduced in a fixed order.
 * Other d -> KGQ_ERR_INVALID_ARG (the host falls back to the unfused ops). */
KGQ_API size_t kgq_layer_backward_workspace_bytes(int64_t rows, int32_t d);
KGQ_API int kgq_layer_backward_f32(const float *g_read, const float *g_e, const uint8_t *mask,
                           const uint8_t *codes, const float *ranges, const float *offsets,
                           int64_t rows, int32_t d, int32_t bits, const float *theta, float *dh,
                           float *dtheta, void *workspace, size_t workspace_bytes,
                           int32_t accumulate, void *stream);

/* Fused KGNN layer forward (model.py:81-85 + tape.py:101-126), one pass:
 *   H = spmm(A, E); ctx = quantize(H) (group = d); J = H @ theta;
 *   E_next = relu(J); mask = J > 0.
 * H and J are never written to memory.  h_out (optional, may be NULL) receives
 * H for debugging/parity.  d in {32, 64, 128}. */
KGQ_API int kgq_layer_forward_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                          int64_t n_rows, const int32_t *row_order, int64_t n_heavy,
                          const float *e, int32_t d, const float *theta,
                          int32_t bits, int32_t rounding, uint64_t seed, uint64_t tensor_id,
                          const uint64_t *tid_base, int64_t row_offset, uint8_t *codes, float *ranges, float *offsets, float *e_next,
                          uint8_t *mask, float *h_out, void *stream);

/* Split layer forward, part 2: the epilogue of kgq_layer_forward_f32 on an H
 * already produced by kgq_spmm_csr_f32 (rows in natural order):
 *   ctx = quantize(H) (group = d); J = H @ theta; E_next = relu(J); mask.
 * Bit-identical to the fused kernel (same lanes, noise calls, FFMA order);
 * spmm + epilogue keeps the gather kernel at full occupancy, which is faster
 * when H is L2-resident.  d in {32, 64, 128}.  For bits != 32, e_next may
 * equal h (E' written over H in place: every tile's H rows are read before
 * its E' rows are stored); for bits == 32 H is the context and must stay. */
KGQ_API int kgq_layer_epilogue_f32(const float *h, int64_t n_rows, int32_t d, const float *theta,
                           int32_t bits, int32_t rounding, uint64_t seed, uint64_t tensor_id,
                           const uint64_t *tid_base, int64_t row_offset, uint8_t *codes,
                           float *ranges, float *offsets, float *e_next, uint8_t *mask, void *stream);

/* BPR + L2 head forward (tape.py:154-170): margins[r] = sum_k u*(p-n);
 * loss[0] = mean logaddexp(0, -margins) + (l2 * (|u|^2+|p|^2+|n|^2)) / batch,
 * fixed reduction order (deterministic).  u, p, n: batch x d fp32 row-major.
 * workspace: kgq_bpr_forward_workspace_bytes(batch) of device memory. */
KGQ_API size_t kgq_bpr_forward_workspace_bytes(int64_t batch);
KGQ_API int kgq_bpr_forward_f32(const float *u, const float *p, const float *n, int64_t batch, int32_t d,
                        float l2, float *margins, float *loss, void *workspace, size_t workspace_bytes,
                        void *stream);

/* BPR head backward (tape.py:233-244) against the dequantized blocks:
 * coef = sigmoid(-m)/batch; gu = g*(-coef*(ph-nh) + reg*uh); gp = g*(-coef*uh
 * + reg*ph); gn = g*(coef*uh + reg*nh); g is a device scalar, reg = fp32(2*l2/batch). */
KGQ_API int kgq_bpr_backward_f32(const float *g, const float *margins, const float *uh, const float *ph,
                         const float *nh, int64_t batch, int32_t d, float reg, float *gu,
                         float *gp, float *gn, void *stream);

/* Deterministic scatter-add of n_lists gathers' gradients into one source
 * (tape.py:229-232 with the routing order of tape.py:204-209): rows of
 * out get ((s_0 + s_1) + ...) where s_i = np.add.at over list i (occurrence
 * order, from +0).  idx/g hold the lists back to back (list i ends at
 * list_end[i]: a HOST int64 array, n_lists <= 8, passed by value to the
 * kernel so the call is graph-capturable); order = positions sorted by
 * (idx, position), device int64, or NULL for the sort-free kernel (m <= 16384;
 * a warp per first occurrence); rows in no list are not written (zero first);
 * negative indices are skipped (rows owned by another rank). */
KGQ_API int kgq_scatter_rows_multi_f32(const int64_t *order, const int32_t *idx, int64_t m,
                               const int64_t *list_end, int32_t n_lists, const float *g,
                               int32_t d, float *out, void *stream);

/* Rows idx of a sum of n_terms (<= 8) row-major n x d tensors, summed in
 * order ((t_0 + t_1) + ...): the gather of the KGNN sum readout (model.py:86-88
 * + tape.py:143-152) without materializing the sum.  terms: HOST array of
 * device pointers (passed by value, graph-capturable); idx: device int64. */
KGQ_API int kgq_gather_rows_sum_f32(const float *const *terms, int32_t n_terms, const int64_t *idx,
                            int64_t n_idx, int32_t d, float *out, void *stream);

/* The same gather added onto a running sum: out = ((base + t_0[idx]) +
 * t_1[idx]) + ... with base an n_idx x d row block (may alias out): the sum
 * readout accumulated term by term as each layer output dies
 * (model.forward_all(readout_rows=...)), bit-identical to gathering the sum. */
KGQ_API int kgq_gather_rows_acc_f32(const float *base, const float *const *terms, int32_t n_terms,
                            const int64_t *idx, int64_t n_idx, int32_t d, float *out, void *stream);

/* One source-block phase of the pipelined SpMM (the partitioned step's
 * exchange overlap, parallel.partitioned_step overlap=True): for the n_slots
 * rows row_order[0..n_slots) (the first n_heavy get a CTA each), continue the
 * running sums in out[row] (zeroed before the first phase) over the row's
 * nonzeros [seg_beg[row], seg_end[row]) in ascending order, each step
 * acc = acc + a*x as kgq_spmm_csr_f32 does; running the source blocks of the
 * columns in ascending order therefore leaves exactly kgq_spmm_csr_f32's
 * result.  d in {32, 64, 128}; x, out 16-byte aligned. */
KGQ_API int kgq_spmm_csr_seg_f32(const int32_t *indptr, const int32_t *indices, const float *vals,
                                 int64_t n_slots, const int32_t *row_order, int64_t n_heavy,
                                 const int32_t *seg_beg, const int32_t *seg_end, const float *x, int32_t d,
                                 float *out, void *stream);

/* Compact scatter (kgq_scatter_rows_multi_f32 without the sort, m <= 16384,
 * d <= 128): the summed gradient of each distinct id to rows[i] (i = its first
 * position in the concatenated lists) and rowmap[id] = i; rowmap is
 * pre-filled with -1 by the caller (untouched ids: zero gradient). */
KGQ_API int kgq_scatter_rows_multi_sparse_f32(const int32_t *idx, int64_t m, const int64_t *list_end,
                                              int32_t n_lists, const float *g, int32_t d, float *rows,
                                              int32_t *rowmap, void *stream);

/* kgq_layer_backward_f32 with g_read in that compact form (row r: gr_rows[gr_map[r]]
 * if gr_map[r] >= 0, else +0), so the readout gradient of a batch is never
 * densified.  d = 64 only (else KGQ_ERR_INVALID_ARG). */
KGQ_API int kgq_layer_backward_rows_f32(const int32_t *gr_map, const float *gr_rows, const float *g_e,
                                        const uint8_t *mask, const uint8_t *codes, const float *ranges,
                                        const float *offsets, int64_t rows, int32_t d, int32_t bits,
                                        const float *theta, float *dh, float *dtheta, void *workspace,
                                        size_t workspace_bytes, int32_t accumulate, void *stream);

/* Device counters of a captured training step advanced in one launch:
 * *a += da, *b += db, *c += dc (null pointers skipped). */
KGQ_API int kgq_counters_add(int64_t *a, int64_t da, int64_t *b, int64_t db, int64_t *c, int64_t dc,
                             void *stream);

/* The BPR batch's gather index lists (train.py:80-85): from a row-major
 * [B][3] int32 (user, positive item, negative item) batch, the node ids
 * users | num_users + pos | num_users + neg as int32 and int64 [3][B]. */
KGQ_API int kgq_batch_indices(const int32_t *batch, int64_t B, int64_t num_users, int32_t *idx32,
                              int64_t *idx64, void *stream);

/* Per-row Top-K of an evaluation score block (replaces train.py:141-143:
 * s[train positives] = -inf; np.argsort(-s, kind="stable")[:k]): for each of
 * n_rows rows (row stride ld floats) the indices of the k best of n_cols
 * scores, best first; descending score, ties by ascending index, -0.0 == +0.0,
 * -inf after every finite score, NaN last; -1 past n_cols.  1 <= k <= 64;
 * out_idx: n_rows x k int32.  Reads the block once, no workspace. */
KGQ_API int kgq_topk_rows_f32(const float *scores, int64_t n_rows, int64_t n_cols, int64_t ld, int32_t k,
                      int32_t *out_idx, void *stream);

/* Fused evaluation scoring + Top-K (K12; replaces train.py:121-160's score
 * block + per-user argsort): for each of n_users rows users[i] of readout
 * (n x d fp32, row-major), the k best items of readout[users[i]] . item_emb^T
 * (item_emb: n_items x d fp32) after setting the user's train positives
 * train_items[train_start[i] .. train_end[i]) (sorted ascending) to -inf,
 * best first, in kgq_topk_rows_f32's order (descending score, ties by
 * ascending index, -0.0 == +0.0, -inf then NaN last); -1 past n_items.
 * Scores are 3xTF32 tensor-core dot products (fp32-level); no score matrix is
 * written.  d in {32, 64}, 1 <= k <= 32 (others: KGQ_ERR_INVALID_ARG, the host
 * uses scores + kgq_topk_rows_f32).  workspace >= kgq_score_topk_workspace_bytes
 * (the split item embeddings), 16-byte aligned.  out: n_users x k int32. */
KGQ_API size_t kgq_score_topk_workspace_bytes(int64_t n_items, int32_t d);
KGQ_API int kgq_score_topk_f32(const float *readout, const int64_t *users, int64_t n_users,
                               const float *item_emb, int64_t n_items, int32_t d,
                               const int32_t *train_items, const int64_t *train_start,
                               const int64_t *train_end, int32_t k, int32_t *out,
                               void *workspace, size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* KGQ_H_ */
