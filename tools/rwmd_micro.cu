// rwmd_micro.cu -- which FP32 instruction mix feeds the RWMD all-pairs min
// fastest on sm_100a?  Same tiling as k_rwmd_f32 (R sources per thread in
// registers, targets broadcast from shared memory), four inner loops:
//   V0 direct scalar : FADD FADD FMUL FFMA FMNMX          per evaluation
//   V1 direct packed : FADD2 FADD2 FMUL2 FFMA2 + FMNMX3   per 2 evaluations
//   V2 expand scalar : FFMA FFMA FMNMX                    per evaluation
//   V3 expand packed : FFMA2 FFMA2 + FMNMX3               per 2 evaluations
//   V4 expand packed, source pairs: the target broadcast as the scalar operand,
//      two sources per FFMA2 (FFMA2 FFMA2 per 2 evaluations, FMNMX3 per 2 targets)
//   V5 = V3 with 16 sources per thread
// (expand: min_t |t|^2 - 2 q.t, |q|^2 added after the min).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rwmd_micro tools/rwmd_micro.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int BLOCK = 256;
constexpr int TILE = 2048;
template <int V>
struct RofV {
    static constexpr int R = V == 5 ? 16 : 8;
};

__device__ __forceinline__ float min3(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

template <int V>
__global__ void __launch_bounds__(BLOCK) k(const float2 *q, int nq, const float2 *t, int nt, int chunk,
                                           unsigned *out) {
    // V0/V2 layout: float4 = (x_j, y_j, x_j+1, y_j+1) [V2: x' , y', |t|^2 ...]
    // V1/V3 layout: x pair, y pair, (V3) t2 pair
    __shared__ float4 s4[TILE / 2];
    __shared__ float2 s2[TILE / 2];
    constexpr int R = RofV<V>::R;
    const int q0 = blockIdx.x * (BLOCK * R) + threadIdx.x;
    float qx[R], qy[R], m[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
        int i = q0 + r * BLOCK;
        float2 p = i < nq ? q[i] : make_float2(0.f, 0.f);
        if (V >= 2) {
            qx[r] = -2.f * p.x;
            qy[r] = -2.f * p.y;
        } else {
            qx[r] = p.x;
            qy[r] = p.y;
        }
        m[r] = INFINITY;
    }
    const int tb0 = blockIdx.y * chunk, te = min(nt, tb0 + chunk);
    for (int tb = tb0; tb < te; tb += TILE) {
        const int cnt = min(TILE, te - tb);
        __syncthreads();
        for (int j = threadIdx.x; j < TILE / 2; j += BLOCK) {
            float2 a = 2 * j < cnt ? t[tb + 2 * j] : make_float2(1e18f, 1e18f);
            float2 b = 2 * j + 1 < cnt ? t[tb + 2 * j + 1] : make_float2(1e18f, 1e18f);
            if (V == 0)
                s4[j] = make_float4(a.x, a.y, b.x, b.y);
            else if (V == 1)
                s4[j] = make_float4(a.x, b.x, a.y, b.y);
            else if (V == 2)
                s4[j] = make_float4(a.x, a.y, a.x * a.x + a.y * a.y, 0.f), s2[j] = make_float2(b.x, b.y);
            else if (V == 4)
                s4[j] = make_float4(a.x, a.y, b.x, b.y),
                s2[j] = make_float2(a.x * a.x + a.y * a.y, b.x * b.x + b.y * b.y);
            else {
                s4[j] = make_float4(a.x, b.x, a.y, b.y);
                s2[j] = make_float2(a.x * a.x + a.y * a.y, b.x * b.x + b.y * b.y);
            }
        }
        __syncthreads();
        const int pairs = (cnt + 1) >> 1;
#pragma unroll 2
        for (int j = 0; j < pairs; j++) {
            const float4 v = s4[j];
            if (V == 0) {
#pragma unroll
                for (int r = 0; r < R; r++) {
                    float dx = qx[r] - v.x, dy = qy[r] - v.y;
                    float d = fmaf(dy, dy, dx * dx);
                    float ex = qx[r] - v.z, ey = qy[r] - v.w;
                    float e = fmaf(ey, ey, ex * ex);
                    m[r] = min3(m[r], d, e);
                }
            } else if (V == 1) {
                const float2 tx = make_float2(v.x, v.y), ty = make_float2(v.z, v.w);
#pragma unroll
                for (int r = 0; r < R; r++) {
                    float2 dx = __fadd2_rn(make_float2(qx[r], qx[r]), make_float2(-tx.x, -tx.y));
                    float2 dy = __fadd2_rn(make_float2(qy[r], qy[r]), make_float2(-ty.x, -ty.y));
                    float2 d = __ffma2_rn(dy, dy, __fmul2_rn(dx, dx));
                    m[r] = min3(m[r], d.x, d.y);
                }
            } else if (V == 2) {
                const float2 w = s2[j];
                const float w2 = w.x * w.x + w.y * w.y;
#pragma unroll
                for (int r = 0; r < R; r++) {
                    float d = fmaf(qy[r], v.y, fmaf(qx[r], v.x, v.z));
                    float e = fmaf(qy[r], w.y, fmaf(qx[r], w.x, w2));
                    m[r] = min3(m[r], d, e);
                }
            } else if (V == 4) {
                const float2 tt = s2[j];
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    const float2 qx2 = make_float2(qx[r], qx[r + 1]), qy2 = make_float2(qy[r], qy[r + 1]);
                    float2 d0 = __ffma2_rn(make_float2(v.y, v.y), qy2,
                                           __ffma2_rn(make_float2(v.x, v.x), qx2, make_float2(tt.x, tt.x)));
                    float2 d1 = __ffma2_rn(make_float2(v.w, v.w), qy2,
                                           __ffma2_rn(make_float2(v.z, v.z), qx2, make_float2(tt.y, tt.y)));
                    m[r] = min3(m[r], d0.x, d1.x);
                    m[r + 1] = min3(m[r + 1], d0.y, d1.y);
                }
            } else {
                const float2 tx = make_float2(v.x, v.y), ty = make_float2(v.z, v.w), tt = s2[j];
#pragma unroll
                for (int r = 0; r < R; r++) {
                    float2 d = __ffma2_rn(make_float2(qy[r], qy[r]), ty,
                                          __ffma2_rn(make_float2(qx[r], qx[r]), tx, tt));
                    m[r] = min3(m[r], d.x, d.y);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
        int i = q0 + r * BLOCK;
        if (i < nq) atomicMin(&out[i], __float_as_uint(m[r] + 4.0f));
    }
}

template <int V>
float run(const float2 *q, int nq, const float2 *t, int nt, unsigned *out, int sms) {
    constexpr int R = RofV<V>::R;
    const int gx = (nq + BLOCK * R - 1) / (BLOCK * R);
    int gy = (16 * sms + gx - 1) / gx;
    int chunk = (nt + gy - 1) / gy;
    chunk = (chunk + 1) & ~1;
    gy = (nt + chunk - 1) / chunk;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<V><<<dim3(gx, gy), BLOCK>>>(q, nq, t, nt, chunk, out);
    cudaEventRecord(a);
    const int reps = 5;
    for (int i = 0; i < reps; i++) k<V><<<dim3(gx, gy), BLOCK>>>(q, nq, t, nt, chunk, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 100000;
    std::vector<float2> h(2 * n);
    srand(1);
    for (auto &p : h) p = make_float2(rand() / (float)RAND_MAX - 0.5f, rand() / (float)RAND_MAX - 0.5f);
    float2 *d;
    unsigned *o;
    cudaMalloc(&d, sizeof(float2) * 2 * n);
    cudaMalloc(&o, sizeof(unsigned) * n);
    cudaMemcpy(d, h.data(), sizeof(float2) * 2 * n, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double evals = (double)n * n;
    const double peak = sms * 128.0 * 2 * clk * 1e3;  // FP32 FLOP/s at the max clock
    const char *names[] = {"V0 direct scalar", "V1 direct packed", "V2 expand scalar", "V3 expand packed",
                           "V4 expand packed, source pairs", "V5 expand packed, R=16"};
    float ms[6] = {run<0>(d, n, d + n, n, o, sms), run<1>(d, n, d + n, n, o, sms),
                   run<2>(d, n, d + n, n, o, sms), run<3>(d, n, d + n, n, o, sms),
                   run<4>(d, n, d + n, n, o, sms), run<5>(d, n, d + n, n, o, sms)};
    printf("{\"n\": %d, \"sms\": %d, \"clock_khz\": %d, \"variants\": [", n, sms, clk);
    for (int v = 0; v < 6; v++)
        printf("%s{\"name\": \"%s\", \"ms\": %.4f, \"Geval_per_s\": %.1f, \"tflops_5flop\": %.2f, "
               "\"frac_nominal_fp32\": %.3f}",
               v ? ", " : "", names[v], ms[v], evals / ms[v] / 1e6, 5 * evals / ms[v] / 1e9,
               5 * evals / (ms[v] * 1e-3) / peak);
    printf("], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
