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

}  // namespace

template <typename S>
cudaError_t launch_pairwise(const void* spec, int N, int64_t nq, const int* lags, int n_lags,
                            double* out, int64_t out_stride, const int64_t* dest_of_slot,
                            int num_sms, cudaStream_t stream) {
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

template cudaError_t launch_pairwise<float>(const void*, int, int64_t, const int*, int, double*,
                                            int64_t, const int64_t*, int, cudaStream_t);
template cudaError_t launch_pairwise<double>(const void*, int, int64_t, const int*, int, double*,
                                             int64_t, const int64_t*, int, cudaStream_t);

}  // namespace ddmk
