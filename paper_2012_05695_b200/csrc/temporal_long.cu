// Long-sequence temporal dispatch (sm_100a): padded length N2 = 1024 R (R = 4: N in
// (1024, 2048], the 1024^2 x 2048 case; R = 8: N in (2048, 4096], the 2048^2 x 4096 case).
// The engine itself is temporal_long2.cu (two warp groups per CTA, one wave vector each). In
// map mode it writes a q-major block out_q[q - q0][m] (contiguous, coalesced), which
// transpose_lags_kernel turns into the reference's lag-major planes (`result_map.hpp:12-32`);
// ring mode adds d into per-item sums like the warp engine.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "temporal_common.cuh"
#include "warp_fft.cuh"

namespace ddmk {

namespace {

using namespace tc;

// out_q [q][N] f32 (q in [q0, q1)) -> out[li * out_stride + dest(q)], 32 x 32 tiles (any
// lag list, cutoff destinations, partial tiles)
template <typename OutT>
__global__ void transpose_lags_kernel(const float* __restrict__ out_q, int N, int64_t q0, int64_t nq,
                                      const int* __restrict__ lag_index, OutT* __restrict__ out,
                                      int64_t out_stride, const int64_t* __restrict__ dest_of_slot) {
    __shared__ float tile[32][33];
    const int64_t qb = blockIdx.x * 32;
    const int mb = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        const int64_t qq = qb + k;
        const int m = mb + tx;
        tile[k][tx] = (qq < nq && m < N) ? out_q[qq * N + m] : 0.f;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int m = mb + k;
        const int64_t qq = qb + tx;
        if (m >= N || qq >= nq) continue;
        const int li = lag_index ? lag_index[m] : m;
        if (li < 0) continue;
        const int64_t dst = dest_of_slot ? dest_of_slot[q0 + qq] : q0 + qq;
        out[(int64_t)li * out_stride + dst] = (OutT)tile[tx][k];
    }
}

// The common case (every lag, identity destinations, whole 64 x 64 tiles): 16-byte loads
// along m from the q-major block, 16-byte stores of 4 consecutive wave vectors per lag row
// (a 64-wave-vector row run is 256 B f32 / 512 B f64: whole sectors), streaming hints (the
// staging block is read once; the map is not re-read here)
template <typename OutT>
__global__ void __launch_bounds__(256)
transpose_lags64_kernel(const float* __restrict__ out_q, int N, int64_t q0, OutT* __restrict__ out,
                        int64_t out_stride) {
    __shared__ float tile[64][65];   // [q][m]
    const int64_t qb = (int64_t)blockIdx.x * 64;
    const int mb = blockIdx.y * 64;
    const int t = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int e = t + 256 * i;             // 1024 float4: 64 q rows x 16 float4 along m
        const int qq = e >> 4, m4 = (e & 15) * 4;
        const float4 v = __ldcs(reinterpret_cast<const float4*>(out_q + (qb + qq) * N + mb + m4));
        tile[qq][m4] = v.x;
        tile[qq][m4 + 1] = v.y;
        tile[qq][m4 + 2] = v.z;
        tile[qq][m4 + 3] = v.w;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int e = t + 256 * i;             // 64 m rows x 16 groups of 4 q
        const int mm = e >> 4, q4 = (e & 15) * 4;
        OutT* dst = out + (int64_t)(mb + mm) * out_stride + q0 + qb + q4;
        if constexpr (sizeof(OutT) == 4) {
            __stcs(reinterpret_cast<float4*>(dst),
                   make_float4(tile[q4][mm], tile[q4 + 1][mm], tile[q4 + 2][mm], tile[q4 + 3][mm]));
        } else {
            __stcs(reinterpret_cast<double2*>(dst), make_double2(tile[q4][mm], tile[q4 + 1][mm]));
            __stcs(reinterpret_cast<double2*>(dst) + 1, make_double2(tile[q4 + 2][mm], tile[q4 + 3][mm]));
        }
    }
}

}  // namespace

cudaError_t launch_long2(const TemporalArgs& a, int64_t q0, int64_t q1, float* out_q, int num_sms,
                         cudaStream_t stream);

bool temporal_long_supported(int N, int N2, int scalar_bytes) {
    return scalar_bytes == 4 && (N2 == 4096 || N2 == 8192) && N > N2 / 4 && N <= N2 / 2 && N % 2 == 0;
}

int64_t temporal_long_chunk(int N) {
    // q-major staging block of the map mode: ~1 GiB of f32 (DDM_LONG_CHUNK_MB overrides)
    static const char* env = std::getenv("DDM_LONG_CHUNK_MB");
    const int64_t bytes = env ? (int64_t)std::max(1, std::atoi(env)) << 20 : (int64_t)1 << 30;
    return std::max<int64_t>(1, bytes / 4 / N);
}

cudaError_t launch_temporal_long(const TemporalArgs& a, int num_sms, void* out_q,
                                 cudaStream_t stream) {
    if (reinterpret_cast<uintptr_t>(a.spec) % 16 != 0) return cudaErrorMisalignedAddress;
    if (!temporal_warp_segments_ok(a.segs, a.N)) return cudaErrorInvalidValue;
    auto launch = [&](int64_t q0, int64_t q1) {
        return launch_long2(a, q0, q1, static_cast<float*>(out_q), num_sms, stream);
    };
    if (a.ring.nitems > 0) return launch(0, 0);
    const int64_t nq = a.layout.g_count, chunk = temporal_long_chunk(a.N);
    for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
        const int64_t q1 = std::min(nq, q0 + chunk);
        cudaError_t e = launch(q0, q1);
        if (e != cudaSuccess) return e;
        const int64_t nq64 = (!a.lag_index && !a.dest_of_slot && a.N % 64 == 0 &&
                              (q0 % 4) == 0 && a.out_stride % 4 == 0 &&
                              reinterpret_cast<uintptr_t>(a.out) % 16 == 0)
                                 ? (q1 - q0) / 64 * 64 : 0;
        if (nq64 > 0) {
            dim3 g64((unsigned)(nq64 / 64), (unsigned)(a.N / 64));
            if (a.out_f64)
                transpose_lags64_kernel<double><<<g64, 256, 0, stream>>>(
                    static_cast<const float*>(out_q), a.N, q0, static_cast<double*>(a.out), a.out_stride);
            else
                transpose_lags64_kernel<float><<<g64, 256, 0, stream>>>(
                    static_cast<const float*>(out_q), a.N, q0, static_cast<float*>(a.out), a.out_stride);
        }
        // the rest (tail wave vectors, lag lists, cutoff destinations): 32 x 32 tiles
        const int64_t r0 = q0 + nq64;
        if (r0 == q1) {
            e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            continue;
        }
        dim3 grid((unsigned)((q1 - r0 + 31) / 32), (unsigned)((a.N + 31) / 32));
        const float* rq = static_cast<const float*>(out_q) + nq64 * (int64_t)a.N;
        if (a.out_f64)
            transpose_lags_kernel<double><<<grid, dim3(32, 8), 0, stream>>>(
                rq, a.N, r0, q1 - r0, a.lag_index, static_cast<double*>(a.out), a.out_stride,
                a.dest_of_slot);
        else
            transpose_lags_kernel<float><<<grid, dim3(32, 8), 0, stream>>>(
                rq, a.N, r0, q1 - r0, a.lag_index, static_cast<float*>(a.out), a.out_stride,
                a.dest_of_slot);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace ddmk
