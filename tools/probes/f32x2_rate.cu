// Probe: issue rate of packed f32x2 FMA/ADD/MUL (FFMA2/FADD2/FMUL2, sm_100a) against scalar
// FFMA/FADD/FMUL with register operands. 16 independent f32 chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f32x2_rate f32x2_rate.cu && ./f32x2_rate
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }

template <int OP>
__global__ void scalar_k(float* out, float b, float c, int iters) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    float bb = b + threadIdx.x * 1e-7f, cc = c - threadIdx.x * 1e-7f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(bb), "f"(cc));
            if (OP == 1) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(bb));
            if (OP == 2) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(bb));
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
__global__ void packed_k(float* out, float b, float c, int iters) {
    u64 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = pk(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
    u64 bb = pk(b + threadIdx.x * 1e-7f, b), cc = pk(c - threadIdx.x * 1e-7f, c);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(bb), "l"(cc));
            if (OP == 1) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(bb));
            if (OP == 2) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(bb));
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); s += x + y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: 8 scalar FFMA + 4 FADD2 per step (does the packed add co-issue with FMA work?)
__global__ void mixed_k(float* out, float b, float c, int iters) {
    float a[8]; u64 p[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = pk(threadIdx.x * 1e-3f + i, 1.f);
    float bb = b + threadIdx.x * 1e-7f, cc = c; u64 b2 = pk(bb, b);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[2*i]) : "f"(bb), "f"(cc));
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(b2));
            asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[2*i+1]) : "f"(bb), "f"(cc));
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(p[i])); s += x + y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
float timeit(K k, float* out, int blocks, int threads, int iters) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<blocks, threads>>>(out, 1.0000001f, 1e-7f, iters);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, 1.0000001f, 1e-7f, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 5;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 512, blocks = sms * 4, iters = 4096;
    float* out; cudaMalloc(&out, (size_t)blocks * threads * 4);
    const double lanes_ops = (double)blocks * threads * iters * 16;  // f32 operations per launch
    const char* names[3] = {"fma", "add", "mul"};
    for (int op = 0; op < 3; ++op) {
        float ms_s = op == 0 ? timeit(scalar_k<0>, out, blocks, threads, iters) : op == 1 ? timeit(scalar_k<1>, out, blocks, threads, iters) : timeit(scalar_k<2>, out, blocks, threads, iters);
        float ms_p = op == 0 ? timeit(packed_k<0>, out, blocks, threads, iters) : op == 1 ? timeit(packed_k<1>, out, blocks, threads, iters) : timeit(packed_k<2>, out, blocks, threads, iters);
        printf("%s: scalar %.3f ms (%.1f G f32 op/s, %.1f G warp-inst/s)  f32x2 %.3f ms (%.1f G f32 op/s, %.1f G warp-inst/s)\n",
               names[op], ms_s, lanes_ops / ms_s / 1e6, lanes_ops / 32 / ms_s / 1e6,
               ms_p, lanes_ops / ms_p / 1e6, lanes_ops / 64 / ms_p / 1e6);
    }
    float ms_m = timeit(mixed_k, out, blocks, threads, iters);
    // per step: 8 FFMA + 4 FADD2 = 16 f32 ops, 12 warp instructions
    printf("mixed 8 FFMA + 4 FADD2: %.3f ms (%.1f G f32 op/s, %.1f G warp-inst/s)\n", ms_m,
           lanes_ops / ms_m / 1e6, (double)blocks * threads * iters * 12 / 32 / ms_m / 1e6);
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
