// kgq_host.cu -- host-buffer entry points: the reference's numpy-in/numpy-out
// calling convention (quantize.py:177-210 take and return host arrays) on the
// device kernels.  The tensor is streamed through the GPU in group chunks on
// several CUDA streams, so the H2D copy of chunk c+1, the kernel of chunk c
// and the D2H copy of chunk c-1 overlap (PCIe is full duplex).  The noise is
// keyed by the global group index, so the bytes do not depend on the chunking.
//
// Blocking like the numpy calls they replace: the outputs are in host memory
// when the call returns.  Pinned host buffers give the overlap; pageable ones
// work but copy synchronously.
#include "kgq_common.cuh"

namespace {

constexpr int kMaxSlots = 8;
constexpr int64_t kDefaultChunkElems = 16ll << 20;   // 64 MB of fp32 per slot

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

inline int64_t group_bytes(int32_t group, int32_t bits) {
    return ((int64_t)group * bits + 7) / 8;
}

// Bytes of one slot holding chunk_groups groups: fp32 data, codes, ranges, offsets.
inline size_t slot_bytes(int64_t chunk_groups, int32_t group, int32_t bits) {
    return align256((size_t)chunk_groups * group * sizeof(float)) +
           align256((size_t)chunk_groups * group_bytes(group, bits)) +
           2 * align256((size_t)chunk_groups * sizeof(float));
}

struct Slot {
    float *data;
    uint8_t *codes;
    float *ranges, *offsets;
};

inline Slot carve(void *base, int64_t chunk_groups, int32_t group, int32_t bits) {
    uint8_t *p = reinterpret_cast<uint8_t *>(base);
    Slot s;
    s.data = reinterpret_cast<float *>(p);
    p += align256((size_t)chunk_groups * group * sizeof(float));
    s.codes = p;
    p += align256((size_t)chunk_groups * group_bytes(group, bits));
    s.ranges = reinterpret_cast<float *>(p);
    p += align256((size_t)chunk_groups * sizeof(float));
    s.offsets = reinterpret_cast<float *>(p);
    return s;
}

// Streams + workspace for one call: caller-provided or created here.
struct Pipeline {
    cudaStream_t st[kMaxSlots] = {};
    int n = 0;
    bool own_streams = false, own_ws = false;
    void *ws = nullptr;
    int64_t chunk_groups = 0;
    cudaEvent_t start = nullptr;

    int setup(int64_t n_groups, int32_t group, int32_t bits, void *workspace, size_t ws_bytes,
              void *const *streams, int32_t n_streams, void *order_stream) {
        cudaError_t e;
        if (streams && n_streams > 0) {
            n = n_streams < kMaxSlots ? n_streams : kMaxSlots;
            for (int i = 0; i < n; i++) st[i] = (cudaStream_t)streams[i];
        } else {
            n = 3;
            own_streams = true;
            for (int i = 0; i < n; i++) {
                if ((e = cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking)) != cudaSuccess) {
                    n = i;
                    return kgq_set_cuda_error(e);
                }
            }
        }
        const size_t per_group = (size_t)group * sizeof(float) + group_bytes(group, bits) + 2 * sizeof(float);
        if (workspace) {
            // largest multiple-of-8 chunk whose n slots fit the workspace
            // (start from the unaligned bound, step down past the padding)
            int64_t cg = (int64_t)(ws_bytes / (size_t)n / per_group);
            cg = cg / 8 * 8;
            while (cg > 0 && (size_t)n * slot_bytes(cg, group, bits) > ws_bytes) cg -= 8;
            if (cg <= 0) return KGQ_ERR_INVALID_ARG;
            chunk_groups = cg;
            ws = workspace;
        } else {
            int64_t cg = kDefaultChunkElems / group;
            cg = cg < 8 ? 8 : cg / 8 * 8;
            const int64_t need = (n_groups + 7) / 8 * 8;
            chunk_groups = cg < need ? cg : need;
            if ((e = cudaMalloc(&ws, (size_t)n * slot_bytes(chunk_groups, group, bits))) != cudaSuccess)
                return kgq_set_cuda_error(e);
            own_ws = true;
        }
        // order after the caller's stream (the workspace may come from a
        // stream-ordered allocator whose previous user is still pending)
        if ((e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming)) != cudaSuccess)
            return kgq_set_cuda_error(e);
        if ((e = cudaEventRecord(start, (cudaStream_t)order_stream)) != cudaSuccess) return kgq_set_cuda_error(e);
        for (int i = 0; i < n; i++)
            if ((e = cudaStreamWaitEvent(st[i], start, 0)) != cudaSuccess) return kgq_set_cuda_error(e);
        return KGQ_OK;
    }

    Slot slot(int c, int32_t group, int32_t bits) const {
        return carve(reinterpret_cast<uint8_t *>(ws) + (size_t)(c % n) * slot_bytes(chunk_groups, group, bits),
                     chunk_groups, group, bits);
    }

    // Wait for every stream; release what this call created.  Returns the
    // first error seen (status of the pipeline or of the teardown).
    int finish(int status) {
        for (int i = 0; i < n; i++) {
            cudaError_t e = cudaStreamSynchronize(st[i]);
            if (e != cudaSuccess && status == KGQ_OK) status = kgq_set_cuda_error(e);
        }
        if (start) cudaEventDestroy(start);
        if (own_ws && ws) cudaFree(ws);
        if (own_streams)
            for (int i = 0; i < n; i++) cudaStreamDestroy(st[i]);
        return status;
    }
};

}  // namespace

extern "C" size_t kgq_host_workspace_bytes(int64_t chunk_groups, int32_t group, int32_t bits,
                                           int32_t n_streams) {
    if (chunk_groups < 1 || group < 1 || n_streams < 1) return 0;
    const int n = n_streams < kMaxSlots ? n_streams : kMaxSlots;
    const int64_t cg = (chunk_groups + 7) / 8 * 8;
    return (size_t)n * slot_bytes(cg, group, bits);
}

extern "C" int kgq_quantize_host_f32(const float *x, int64_t n_groups, int32_t group, int32_t bits,
                                     int32_t rounding, uint64_t seed, uint64_t tensor_id,
                                     int64_t group_offset, uint8_t *codes, float *ranges,
                                     float *offsets, void *workspace, size_t workspace_bytes,
                                     void *const *streams, int32_t n_streams, void *stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (group < 1 || n_groups < 0 || group_offset < 0) return KGQ_ERR_INVALID_ARG;
    if (rounding == KGQ_ROUND_SR_NOISE) return KGQ_ERR_INVALID_ARG;   // device-only parity seam
    if (n_groups == 0) return KGQ_OK;
    if (!x || !codes || !ranges || !offsets) return KGQ_ERR_INVALID_ARG;
    Pipeline pl;
    int st = pl.setup(n_groups, group, bits, workspace, workspace_bytes, streams, n_streams, stream);
    if (st != KGQ_OK) return pl.finish(st);
    const int64_t GB = group_bytes(group, bits);
    int c = 0;
    for (int64_t g0 = 0; g0 < n_groups && st == KGQ_OK; g0 += pl.chunk_groups, c++) {
        const int64_t ng = n_groups - g0 < pl.chunk_groups ? n_groups - g0 : pl.chunk_groups;
        const Slot sl = pl.slot(c, group, bits);
        cudaStream_t s = pl.st[c % pl.n];
        cudaError_t e = cudaMemcpyAsync(sl.data, x + g0 * group, (size_t)ng * group * sizeof(float),
                                        cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) { st = kgq_set_cuda_error(e); break; }
        st = kgq_quantize_f32(sl.data, ng, group, bits, rounding, seed, tensor_id, nullptr,
                              group_offset + g0, nullptr, sl.codes, sl.ranges, sl.offsets, s);
        if (st != KGQ_OK) break;
        if ((e = cudaMemcpyAsync(codes + g0 * GB, sl.codes, (size_t)ng * GB, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(ranges + g0, sl.ranges, (size_t)ng * sizeof(float), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(offsets + g0, sl.offsets, (size_t)ng * sizeof(float), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
            st = kgq_set_cuda_error(e);
    }
    return pl.finish(st);
}

extern "C" int kgq_dequantize_host_f32(const uint8_t *codes, const float *ranges, const float *offsets,
                                       int64_t n_groups, int32_t group, int32_t bits, float *out,
                                       void *workspace, size_t workspace_bytes,
                                       void *const *streams, int32_t n_streams, void *stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return KGQ_ERR_UNSUPPORTED_BITS;
    if (group < 1 || n_groups < 0) return KGQ_ERR_INVALID_ARG;
    if (n_groups == 0) return KGQ_OK;
    if (!codes || !ranges || !offsets || !out) return KGQ_ERR_INVALID_ARG;
    Pipeline pl;
    int st = pl.setup(n_groups, group, bits, workspace, workspace_bytes, streams, n_streams, stream);
    if (st != KGQ_OK) return pl.finish(st);
    const int64_t GB = group_bytes(group, bits);
    int c = 0;
    for (int64_t g0 = 0; g0 < n_groups && st == KGQ_OK; g0 += pl.chunk_groups, c++) {
        const int64_t ng = n_groups - g0 < pl.chunk_groups ? n_groups - g0 : pl.chunk_groups;
        const Slot sl = pl.slot(c, group, bits);
        cudaStream_t s = pl.st[c % pl.n];
        cudaError_t e;
        if ((e = cudaMemcpyAsync(sl.codes, codes + g0 * GB, (size_t)ng * GB, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(sl.ranges, ranges + g0, (size_t)ng * sizeof(float), cudaMemcpyHostToDevice, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(sl.offsets, offsets + g0, (size_t)ng * sizeof(float), cudaMemcpyHostToDevice, s)) != cudaSuccess) {
            st = kgq_set_cuda_error(e);
            break;
        }
        st = kgq_dequantize_f32(sl.codes, sl.ranges, sl.offsets, ng, group, bits, sl.data, s);
        if (st != KGQ_OK) break;
        if ((e = cudaMemcpyAsync(out + g0 * group, sl.data, (size_t)ng * group * sizeof(float),
                                 cudaMemcpyDeviceToHost, s)) != cudaSuccess)
            st = kgq_set_cuda_error(e);
    }
    return pl.finish(st);
}
