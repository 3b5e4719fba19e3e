// Probe for the round-2 spatial design: how fast an
// 8-CTA cluster can corner-turn a 512 x 257 c64 frame held in distributed shared memory.
// Each CTA holds 64 rows x 256 c64 (128 KiB) of a frame; for the column phase every CTA reads
// its 32 columns x 512 rows from all 8 CTAs (ld.shared::cluster, 16-byte loads). Reported:
// aggregate DSMEM read bandwidth over the whole GPU and time per 1024 frames.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 dsmem_probe.cu -o dsmem_probe
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

constexpr int kCluster = 8;
constexpr int kRows = 64;      // rows per CTA
constexpr int kCols = 256;     // c64 columns per row (257th handled apart in the real kernel)
constexpr int kThreads = 1024;

__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads)
corner_turn_probe(int frames, float4* sink) {
    extern __shared__ float4 tile[];   // kRows x kCols c64 = kRows x kCols/2 float4
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    for (int i = threadIdx.x; i < kRows * kCols / 2; i += kThreads)
        tile[i] = make_float4(rank, i, 0.f, 1.f);
    float4 acc = make_float4(0, 0, 0, 0);
    const int nclusters = gridDim.x / kCluster;
    const int cid = blockIdx.x / kCluster;
    for (int f = cid; f < frames; f += nclusters) {
        cluster.sync();   // row phase of frame f done in every CTA
        // column phase: this CTA owns columns [32 rank, 32 rank + 32): 16 float4 per row,
        // 512 rows spread over the 8 source CTAs
        // 32 loads per thread, issued 8 at a time (independent) to keep several in flight
        constexpr int kPer = kCluster * kRows * 16 / kThreads;
#pragma unroll
        for (int u = 0; u < kPer; u += 8) {
            float4 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = threadIdx.x + (u + k) * kThreads;
                const int src = i / (kRows * 16), rem = i % (kRows * 16);
                const int row = rem / 16, c4 = rem % 16;
                const float4* remote = cluster.map_shared_rank(tile, src);
                v[k] = remote[row * (kCols / 2) + rank * 16 + c4];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w;
            }
        }
    }
    cluster.sync();
    if (acc.x == -1.f) sink[blockIdx.x * kThreads + threadIdx.x] = acc;   // keep the loads
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = size_t(kRows) * kCols * 8;
    cudaFuncSetAttribute(corner_turn_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int blocks = (sms / kCluster) * kCluster;
    float4* sink;
    cudaMalloc(&sink, size_t(blocks) * kThreads * sizeof(float4));
    const int frames = 1024;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        corner_turn_probe<<<blocks, kThreads, smem>>>(frames, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = double(frames) * 512 * kCols * 8;   // every c64 of the frame read once
        std::printf("{\"clusters\": %d, \"frames\": %d, \"ms\": %.4f, \"dsmem_GBps\": %.1f, \"err\": \"%s\"}\n",
                    blocks / kCluster, frames, ms, bytes / (ms * 1e-3) / 1e9,
                    cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
