#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
__global__ void k(long long *p) { if (threadIdx.x == 0) p[0] += 1; }
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    long long *d, *h; cudaMalloc(&d, 64); cudaHostAlloc((void**)&h, 64, 0);
    for (int mode = 0; mode < 3; mode++) {
        for (int it = 0; it < 2; it++) {
            const int N = 2000;
            auto t0 = std::chrono::high_resolution_clock::now();
            for (int i = 0; i < N; i++) {
                k<<<1, 32, 0, s>>>(d);
                if (mode >= 1) cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, s);
                if (mode == 2) cudaStreamSynchronize(s);
            }
            cudaStreamSynchronize(s);
            auto t1 = std::chrono::high_resolution_clock::now();
            printf("mode %d (%s): %.2f us/iter\n", mode, mode == 0 ? "launch only" : mode == 1 ? "launch+d2h" : "launch+d2h+sync",
                   std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
        }
    }
    // spin vs blocking sync flags
    return 0;
}
