// kgq_capi.cu -- status plumbing for the libkgq C ABI (include/kgq.h).
#include "kgq_common.cuh"

static thread_local int g_last_cuda_error = 0;

int kgq_set_cuda_error(cudaError_t e) {
    g_last_cuda_error = (int)e;
    return KGQ_ERR_CUDA;
}

extern "C" int kgq_version(void) { return 1; }

extern "C" int kgq_last_cuda_error(void) { return g_last_cuda_error; }

extern "C" const char *kgq_status_string(int status) {
    switch (status) {
        case KGQ_OK: return "ok";
        case KGQ_ERR_INVALID_ARG: return "invalid argument";
        case KGQ_ERR_UNSUPPORTED_BITS: return "unsupported bit width (expected 1, 2, 4 or 8)";
        case KGQ_ERR_CUDA: return cudaGetErrorString((cudaError_t)g_last_cuda_error);
        case KGQ_ERR_MISALIGNED: return "misaligned buffer";
        case KGQ_ERR_SHAPE: return "shape mismatch";
    }
    return "unknown status";
}
