// WITHOUT_FT on the device (sm_100a): the reference's O(N * lags) spectral-difference
// algorithm (`pairwise.cpp:11-72`, `run_without_ft` `scheduler.cpp:182-286`), also used for
// `Algorithm::Direct` (`pairwise.cpp:74-116`) on f64 spectra, which Eq. 1 equals by linearity
// of the spatial transform.
//
// Per wave vector q and requested lag m > 0:
//     d(q, m) = 1/(N - m) * sum_{n=m}^{N-1} |(double)S_{n-m} - (double)S_n|^2
// with the reference's arithmetic: the difference in f64 of the working-precision spectra,
// re*re + im*im without contraction, accumulated in f64 in ascending n. Every (q, m) sum has
// the reference's order, so the maps match it to the last bits of the final division.
//
// Layout: one CTA per wave vector. Its sequence (wave-vector-major spectra, layout T = 1) is
// widened to f64 in shared memory once; each warp takes 32 consecutive requested lags, lane
// l owns lag m_l and walks n upward, reading S_n (a broadcast) and S_{n - m_l}.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace ddmk {

namespace {

constexpr int kPairThreads = 256;

template <typename S>
__global__ void __launch_bounds__(kPairThreads)
pairwise_kernel(const cpx<S>* __restrict__ spec, int N, int64_t nq, const int* __restrict__ lags,
                int n_lags, double* __restrict__ out, int64_t out_stride,
                const int64_t* __restrict__ dest_of_slot) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* s = reinterpret_cast<double2*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
        __syncthreads();
        const cpx<S>* src = spec + q * (int64_t)N;
        for (int n = threadIdx.x; n < N; n += blockDim.x) s[n] = make_double2((double)src[n].x, (double)src[n].y);
        __syncthreads();
        const int64_t dst = dest_of_slot ? dest_of_slot[q] : q;
        for (int l0 = warp * 32; l0 < n_lags; l0 += nwarps * 32) {
            const int li = l0 + lane;
            const int m = li < n_lags ? lags[li] : N;   // lanes past the list idle
            const int m_first = __shfl_sync(0xffffffffu, m, 0);   // lags ascend
            double acc = 0.0;
            for (int n = m_first; n < N; ++n) {
                if (n >= m) {
                    const double2 a = s[n - m], b = s[n];
                    const double re = __dsub_rn(a.x, b.x), im = __dsub_rn(a.y, b.y);
                    acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
                }
            }
            if (li < n_lags) out[(int64_t)li * out_stride + dst] = m == 0 ? 0.0 : acc * (1.0 / (double)(N - m));
        }
    }
}

// Contiguous lag range: lane l of a group owns lags L = base + kLpl l + k (k < kLpl) and walks
// its own n = L - k + t. The S_{n - L} operand is then s[t - k], the same for every lane:
// one broadcast load per step feeds a kLpl-deep register ring, and the per-lane operand S_n
// is one load shared by the lane's kLpl sums. Every (q, L) sum still runs over ascending n
// with the reference's arithmetic (bit-identical to pairwise_kernel); shared traffic per
// pair drops ~kLpl x, so the loop is FP64-bound. Lag groups of 32 kLpl are dealt to warps
// in (g, G - 1 - g) pairs, which balances the N - L trip counts.
constexpr int kLpl = 4;
constexpr int kConsecThreads = 128;

__device__ __forceinline__ int pad_idx(int i) { return i + i / kLpl; }   // breaks the kLpl stride

__device__ __forceinline__ double pair_norm(double2 a, double2 b) {
    const double re = __dsub_rn(a.x, b.x), im = __dsub_rn(a.y, b.y);
    return __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
}

template <typename S>
__global__ void __launch_bounds__(kConsecThreads)
pairwise_consec_kernel(const cpx<S>* __restrict__ spec, int N, int64_t nq, int lag0, int n_lags,
                       double* __restrict__ out, int64_t out_stride,
                       const int64_t* __restrict__ dest_of_slot) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* s = reinterpret_cast<double2*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    constexpr int kGroup = 32 * kLpl;
    const int groups = (n_lags + kGroup - 1) / kGroup;
    const int pairs = (groups + 1) / 2;
    for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
        __syncthreads();
        const cpx<S>* src = spec + q * (int64_t)N;
        for (int n = threadIdx.x; n < N; n += blockDim.x)
            s[pad_idx(n)] = make_double2((double)src[n].x, (double)src[n].y);
        __syncthreads();
        const int64_t dst = dest_of_slot ? dest_of_slot[q] : q;
        for (int p = warp; p < pairs; p += nwarps) {
#pragma unroll 1
            for (int side = 0; side < 2; ++side) {
                const int g = side == 0 ? p : groups - 1 - p;
                if (side == 1 && g == p) break;
                const int base = lag0 + g * kGroup + kLpl * lane;   // this lane's first lag
                double acc[kLpl];
#pragma unroll
                for (int k = 0; k < kLpl; ++k) acc[k] = 0.0;
                double2 ring[kLpl];
                // n = base + t; lag base + k is summed from t = k on
#pragma unroll
                for (int j = 0; j < kLpl; ++j) {
                    const int n = base + j;
                    if (n < N) {
                        ring[j] = s[pad_idx(j)];
                        const double2 b = s[pad_idx(n)];
#pragma unroll
                        for (int k = 0; k <= j; ++k) acc[k] = __dadd_rn(acc[k], pair_norm(ring[j - k], b));
                    }
                }
                for (int t0 = kLpl; base + t0 < N; t0 += kLpl) {
#pragma unroll
                    for (int j = 0; j < kLpl; ++j) {
                        const int t = t0 + j, n = base + t;
                        if (n < N) {
                            ring[j] = s[pad_idx(t)];
                            const double2 b = s[pad_idx(n)];
#pragma unroll
                            for (int k = 0; k < kLpl; ++k)
                                acc[k] = __dadd_rn(acc[k], pair_norm(ring[(j - k + kLpl) % kLpl], b));
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < kLpl; ++k) {
                    const int m = base + k, li = m - lag0;
                    if (li < n_lags && m < N)
                        out[(int64_t)li * out_stride + dst] = m == 0 ? 0.0 : acc[k] * (1.0 / (double)(N - m));
                }
            }
        }
    }
}

}  // namespace

template <typename S>
cudaError_t launch_pairwise(const void* spec, int N, int64_t nq, const int* lags, int n_lags,
                            double* out, int64_t out_stride, const int64_t* dest_of_slot,
                            int num_sms, cudaStream_t stream, int lag0) {
    static const bool generic = std::getenv("DDM_PAIRWISE_GENERIC") != nullptr;   // A/B
    // a contiguous range of at least one full lag group (32 lanes x kLpl lags): shorter ranges
    // leave most lanes idle and stay on the one-lane-per-lag kernel
    // The window buffer needs (N + N/kLpl + 1) values: past 227 KiB (N >= 11623) the
    // one-lane-per-lag kernel serves the range too (it needs N values, up to N = 14528).
    const size_t consec_smem = (size_t)(N + N / kLpl + 1) * sizeof(double2);
    if (lag0 >= 0 && !generic && n_lags >= 32 * kLpl && consec_smem <= 227 * 1024) {
        const size_t smem = consec_smem;
        auto k = pairwise_consec_kernel<S>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        // one warp per (g, G-1-g) group pair, at most kConsecThreads / 32 per CTA
        const int pairs = ((n_lags + 32 * kLpl - 1) / (32 * kLpl) + 1) / 2;
        const int threads = 32 * std::min(kConsecThreads / 32, std::max(1, pairs));
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem);
        const int64_t grid = std::min<int64_t>(nq, (int64_t)std::max(1, occ) * num_sms * 4);
        if (grid == 0) return cudaSuccess;
        k<<<(unsigned)grid, threads, smem, stream>>>(static_cast<const cpx<S>*>(spec), N, nq, lag0, n_lags,
                                                     out, out_stride, dest_of_slot);
        return cudaGetLastError();
    }
    const size_t smem = (size_t)N * sizeof(double2);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    auto k = pairwise_kernel<S>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kPairThreads, smem);
    const int64_t grid = std::min<int64_t>(nq, (int64_t)std::max(1, occ) * num_sms * 4);
    if (grid == 0) return cudaSuccess;
    k<<<(unsigned)grid, kPairThreads, smem, stream>>>(static_cast<const cpx<S>*>(spec), N, nq, lags,
                                                       n_lags, out, out_stride, dest_of_slot);
    return cudaGetLastError();
}

namespace {

// frame-major spectra [N][plane] -> wave-vector-major sequences [count][N] of the retained
// positions flat[k] (SpectrumStack -> the pairwise kernel's layout); 32 x 8 tiles through
// shared memory so both sides are coalesced
template <typename S>
__global__ void gather_sequences_kernel(const cpx<S>* __restrict__ frames, int N, int64_t plane,
                                        const int64_t* __restrict__ flat, int64_t count,
                                        cpx<S>* __restrict__ seq) {
    __shared__ cpx<S> tile[32][33];
    const int64_t k0 = (int64_t)blockIdx.x * 32;
    const int n0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int j = ty; j < 32; j += 8) {
        const int n = n0 + j;
        const int64_t k = k0 + tx;
        if (n < N && k < count) tile[j][tx] = frames[(int64_t)n * plane + flat[k]];
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
        const int64_t k = k0 + j;
        const int n = n0 + tx;
        if (n < N && k < count) seq[k * N + n] = tile[tx][j];
    }
}

}  // namespace

template <typename S>
cudaError_t launch_gather_sequences(const void* frames, int N, int64_t plane, const int64_t* flat,
                                    int64_t count, void* seq, cudaStream_t stream) {
    if (count == 0 || N == 0) return cudaSuccess;
    dim3 grid((unsigned)((count + 31) / 32), (unsigned)((N + 31) / 32));
    gather_sequences_kernel<S><<<grid, dim3(32, 8), 0, stream>>>(
        static_cast<const cpx<S>*>(frames), N, plane, flat, count, static_cast<cpx<S>*>(seq));
    return cudaGetLastError();
}

template cudaError_t launch_gather_sequences<float>(const void*, int, int64_t, const int64_t*, int64_t,
                                                    void*, cudaStream_t);
template cudaError_t launch_gather_sequences<double>(const void*, int, int64_t, const int64_t*, int64_t,
                                                     void*, cudaStream_t);

template cudaError_t launch_pairwise<float>(const void*, int, int64_t, const int*, int, double*,
                                            int64_t, const int64_t*, int, cudaStream_t, int);
template cudaError_t launch_pairwise<double>(const void*, int, int64_t, const int*, int, double*,
                                             int64_t, const int64_t*, int, cudaStream_t, int);

}  // namespace ddmk
