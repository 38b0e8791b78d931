// zc_write.cu -- micro: device -> host writes by SM stores into page-locked host memory
// (zero-copy under UVA) instead of the copy engines (tools/micro/d2h_interference.py).
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_zc_copy(const int4 *__restrict__ src, int4 *dst, int64_t n16) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

extern "C" int zc_copy(void *dst_host, const void *src_dev, int64_t bytes, int ctas, void *stream) {
    k_zc_copy<<<ctas, 256, 0, (cudaStream_t)stream>>>((const int4 *)src_dev, (int4 *)dst_host, bytes / 16);
    return (int)cudaGetLastError();
}
