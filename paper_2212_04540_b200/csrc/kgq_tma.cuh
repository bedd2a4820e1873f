// kgq_tma.cuh -- TMA (cp.async.bulk.tensor) helpers: host-side tensor-map
// encoding through the driver entry point (no -lcuda link), device-side 2-D
// tile loads / stores signalled through mbarriers.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include "kgq_tc.cuh"

namespace kgq {
namespace tma {

// Row-major fp32 [rows][cols] in global memory, boxes of box_rows x 32 columns
// (128 B inner extent) landing in shared memory with the SWIZZLE_128B pattern:
// row r's 16-byte chunk c at chunk c ^ (r & 7) of its 128-byte row (box base
// 1024-B aligned).  Rows past `rows` read as zeros.  Returns false on failure.
inline bool make_rowmajor_f32(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t cols,
                              uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * sizeof(float)};
    const cuuint32_t box[2] = {32, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// byte offset of (row r, column c) inside a 32-column SWIZZLE_128B box
__host__ __device__ constexpr uint32_t box_off(int r, int c) {
    return (uint32_t)(r * 128 + ((((c & 31) >> 2) ^ (r & 7)) << 4) + (c & 3) * 4);
}

__device__ __forceinline__ void expect_tx(uint64_t *mbar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
                 :: "r"(tc::smem_u32(mbar)), "r"(bytes) : "memory");
}
// box (c0 = first column, c1 = first row) -> shared memory, completion on mbar
__device__ __forceinline__ void load_2d(void *dst, const CUtensorMap *m, int c0, int c1, uint64_t *mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        :: "r"(tc::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1),
           "r"(tc::smem_u32(mbar)) : "memory");
}
// shared memory box -> global (rows past the tensor end are clipped)
__device__ __forceinline__ void store_2d(const CUtensorMap *m, const void *src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
                 :: "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(tc::smem_u32(src)) : "memory");
}
__device__ __forceinline__ void store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N committed store groups still read shared memory
template <int N>
__device__ __forceinline__ void store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void store_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(threads) : "memory");
}

}  // namespace tma
}  // namespace kgq
