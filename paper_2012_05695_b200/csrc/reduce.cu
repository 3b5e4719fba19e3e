// Small device reductions used around the hot path:
//   reduce_stats  : finite / max / min over the result map, so `ResultArchive::validate`
//                   (`archive.cpp:44-58`) costs one HBM read instead of a host scan;
//   radial_means  : the azimuthal ring average (`analysis.cpp:61-97`) as a deterministic
//                   segmented sum over bin-sorted wave vectors (no float atomics: every
//                   (lag, bin) sum is reduced by one warp in a fixed order).
#include <cfloat>
#include <cmath>
#include <map>
#include <mutex>

#include "engine.hpp"

namespace ddm::b200 {

namespace {

template <typename T>
__global__ void stats_kernel(const T* __restrict__ d, int64_t n, double* __restrict__ part) {
    double mx = -DBL_MAX, mn = DBL_MAX, bad = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)d[i];
        if (!isfinite(v)) bad = 1.0;
        else {
            mx = fmax(mx, v);
            mn = fmin(mn, v);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        bad = fmax(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    }
    __shared__ double s[3][32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { s[0][w] = mx; s[1][w] = mn; s[2][w] = bad; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            mx = fmax(mx, s[0][i]);
            mn = fmin(mn, s[1][i]);
            bad = fmax(bad, s[2][i]);
        }
        part[3 * blockIdx.x] = mx;
        part[3 * blockIdx.x + 1] = mn;
        part[3 * blockIdx.x + 2] = bad;
    }
}

// one warp per (lag, bin): sum of values at order[offsets[b] .. offsets[b+1])
__global__ void radial_kernel(const double* __restrict__ values, int64_t n_lags, int64_t plane,
                              const int64_t* __restrict__ order, const int64_t* __restrict__ off,
                              int64_t nbins, double* __restrict__ means) {
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= n_lags * nbins) return;
    const int64_t li = wid / nbins, b = wid - li * nbins;
    const double* row = values + li * plane;
    const int64_t lo = off[b], hi = off[b + 1];
    double acc = 0.0;
    for (int64_t j = lo + lane; j < hi; j += 32) acc += row[order[j]];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) means[wid] = hi > lo ? acc / (double)(hi - lo) : 0.0;
}

// one warp per (lag, bin): the bin's sum over this slice's columns order[off[b] .. off[b+1])
template <typename T>
__global__ void ring_sums_kernel(const T* __restrict__ values, int64_t n_lags, int64_t stride,
                                 const int64_t* __restrict__ order, const int64_t* __restrict__ off,
                                 int64_t nbins, double* __restrict__ sums) {
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= n_lags * nbins) return;
    const int64_t li = wid / nbins, b = wid - li * nbins;
    const T* row = values + li * stride;
    double acc = 0.0;
    for (int64_t j = off[b] + lane; j < off[b + 1]; j += 32) acc += (double)row[order[j]];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sums[wid] = acc;
}

}  // namespace

template <typename T>
static void reduce_stats_t(const T* d, int64_t n, cudaStream_t stream, bool* finite, double* max_v,
                           double* min_v) {
    constexpr int blocks = 296, threads = 256;
    // per-device partials and their pinned host copy, allocated once: a cudaMallocAsync /
    // pageable copy per call cost ~0.4 ms next to sub-millisecond runs
    struct Slot {
        double* dev = nullptr;
        double* host = nullptr;
    };
    static std::mutex mu;
    static std::map<int, Slot> slots;
    int device = 0;
    check(cudaGetDevice(&device), "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    Slot& sl = slots[device];
    if (!sl.dev) {
        check(cudaMalloc(reinterpret_cast<void**>(&sl.dev), sizeof(double) * 3 * blocks), "cudaMalloc");
        check(cudaMallocHost(reinterpret_cast<void**>(&sl.host), sizeof(double) * 3 * blocks),
              "cudaMallocHost");
    }
    stats_kernel<T><<<blocks, threads, 0, stream>>>(d, n, sl.dev);
    check(cudaGetLastError(), "stats kernel");
    check(cudaMemcpyAsync(sl.host, sl.dev, sizeof(double) * 3 * blocks, cudaMemcpyDeviceToHost, stream),
          "stats copy");
    check(cudaStreamSynchronize(stream), "sync");
    const double* host = sl.host;
    double mx = -DBL_MAX, mn = DBL_MAX, bad = 0.0;
    for (int i = 0; i < blocks; ++i) {
        mx = std::fmax(mx, host[3 * i]);
        mn = std::fmin(mn, host[3 * i + 1]);
        bad = std::fmax(bad, host[3 * i + 2]);
    }
    *finite = bad == 0.0;
    *max_v = n > 0 ? mx : 0.0;
    *min_v = n > 0 ? mn : 0.0;
}

void reduce_stats(const double* d, int64_t n, cudaStream_t stream, bool* finite, double* max_v,
                  double* min_v) {
    reduce_stats_t(d, n, stream, finite, max_v, min_v);
}
void reduce_stats(const float* d, int64_t n, cudaStream_t stream, bool* finite, double* max_v,
                  double* min_v) {
    reduce_stats_t(d, n, stream, finite, max_v, min_v);
}

void ring_sums(const void* d_values, bool f64, int64_t n_lags, int64_t stride, const int64_t* d_order,
               const int64_t* d_offsets, int64_t nbins, double* d_sums, cudaStream_t stream) {
    const int64_t warps = n_lags * nbins;
    const int threads = 256;
    const int64_t blocks = (warps * 32 + threads - 1) / threads;
    if (blocks == 0) return;
    if (f64)
        ring_sums_kernel<double><<<(unsigned)blocks, threads, 0, stream>>>(
            static_cast<const double*>(d_values), n_lags, stride, d_order, d_offsets, nbins, d_sums);
    else
        ring_sums_kernel<float><<<(unsigned)blocks, threads, 0, stream>>>(
            static_cast<const float*>(d_values), n_lags, stride, d_order, d_offsets, nbins, d_sums);
    check(cudaGetLastError(), "ring sums kernel");
}

void radial_means(const double* d_values, int64_t n_lags, int64_t plane, const int64_t* d_order,
                  const int64_t* d_offsets, int64_t nbins, double* d_means, cudaStream_t stream) {
    const int64_t warps = n_lags * nbins;
    const int threads = 256;
    const int64_t blocks = (warps * 32 + threads - 1) / threads;
    if (blocks == 0) return;
    radial_kernel<<<(unsigned)blocks, threads, 0, stream>>>(d_values, n_lags, plane, d_order,
                                                            d_offsets, nbins, d_means);
    check(cudaGetLastError(), "radial kernel");
}

}  // namespace ddm::b200
