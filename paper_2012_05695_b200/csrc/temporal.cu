// Step 2 of the WITH_FT pipeline on B200: one fused kernel per tile of T wave vectors that
// replaces `SequenceEngine<S>::with_ft` (`temporal.cpp:77-112`) for every sequence of a
// group, plus the lag selection / d(0)=0 (`scheduler.cpp:155-161`) and the partial/merge
// scatter (`scheduler.cpp:531-540`).  Per sequence s_n, n < N:
//   mu   = sum s_n / N                         in complex f64      (`temporal.cpp:82-87`)
//   t_n  = s_n - (S)mu                         in S                (`temporal.cpp:89-92`)
//   C[m] = sum_{n<m} |t_n|^2                   f64 prefix sums ->  d_a (`temporal.cpp:19-42`)
//   X    = FFT_{N2}(t zero-padded), sign -1    in S                (`temporal.cpp:56-59`)
//   P    = |X|^2                               in S                (`temporal.cpp:60-64`)
//   corr = Re IFFT_{N2}(P)[m] / N2, m < N                          (`temporal.cpp:65-73`)
//   d(m) = d_a(m) - 2 corr(m) / (N - m), d(0) = 0                  (`temporal.cpp:114-129`)
// P is real, so the inverse runs at half length: u[j] = P[2j] + i P[2j+1] through an N2/2
// complex transform, then the standard real-input unfold. Every sequence is transformed on
// its own, so results never depend on which wave vectors share a tile (cutoff and group
// boundaries are bitwise invisible, as in the reference).
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace ddmk {

namespace {

// NT threads per CTA: 256, or 512 for long f64 transforms (T * N2 <= 8192 with one radix-16
// butterfly per thread; more warps to hide the f64 shared-memory passes' latency)
template <typename S, typename OutT, int N2, int NT>
__global__ void __launch_bounds__(NT, 1) temporal_kernel(const cpx<S>* __restrict__ spec, int N, SpecLayout lay,
                                const cpx<S>* __restrict__ tw,
                                const cpx<S>* __restrict__ tw_half,
                                const int* __restrict__ lag_index, OutT* __restrict__ out,
                                int64_t out_stride, const int64_t* __restrict__ dest_of_slot,
                                double* __restrict__ corr_out, double* __restrict__ mean_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int T = lay.T;
    // E: T transform buffers of N2; C: T prefix arrays of N+1 (f64)
    cpx<S>* E = reinterpret_cast<cpx<S>*>(smem_raw);
    double* C = reinterpret_cast<double*>(smem_raw + (size_t)T * N2 * sizeof(cpx<S>));
    double* mu = C + (size_t)T * (N + 1);  // T complex means (re, im)

    const int64_t tile = blockIdx.x;
    const int64_t s0 = tile * T;
    const int nvalid = (int)(lay.g_count - s0 < T ? lay.g_count - s0 : T);
    const cpx<S>* src = spec + tile * (int64_t)N * T;

    // 1. tile block [N][T] -> E[j][n] (coalesced: j fastest), zero padding beyond N; q-major
    //    spectra: T contiguous sequences (coalesced along n), zeros past the group's end
    if (lay.qmajor) {
        const cpx<S>* qsrc = spec + s0 * (int64_t)N;
        for (int idx = threadIdx.x; idx < N * T; idx += blockDim.x) {
            const int j = idx / N, n = idx - j * N;
            E[(size_t)j * N2 + n] = j < nvalid ? qsrc[idx] : cpx<S>{S(0), S(0)};
        }
    } else {
        for (int idx = threadIdx.x; idx < N * T; idx += blockDim.x) {
            const int n = idx / T, j = idx - n * T;
            E[(size_t)j * N2 + n] = src[idx];
        }
    }
    for (int idx = threadIdx.x; idx < T * (N2 - N); idx += blockDim.x) {
        const int j = idx / (N2 - N), n = N + idx - j * (N2 - N);
        E[(size_t)j * N2 + n] = {S(0), S(0)};
    }
    __syncthreads();

    // 2. per-sequence mean (f64), shift (S), f64 prefix sums of |t|^2 : one warp per sequence
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (int j = warp; j < T; j += nwarps) {
        cpx<S>* e = E + (size_t)j * N2;
        double sx = 0.0, sy = 0.0;
        for (int n = lane; n < N; n += 32) {
            sx += (double)e[n].x;
            sy += (double)e[n].y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
            sy += __shfl_xor_sync(0xffffffffu, sy, o);
        }
        const double mx = sx / N, my = sy / N;
        const S ox = (S)mx, oy = (S)my;
        double* c = C + (size_t)j * (N + 1);
        if (lane == 0) {
            c[0] = 0.0;
            mu[2 * j] = mx;
            mu[2 * j + 1] = my;
        }
        double carry = 0.0;
        for (int n0 = 0; n0 < N; n0 += 32) {
            const int n = n0 + lane;
            double p = 0.0;
            if (n < N) {
                cpx<S> t = e[n];
                t.x = t.x - ox;
                t.y = t.y - oy;
                e[n] = t;
                p = (double)t.x * (double)t.x + (double)t.y * (double)t.y;
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double v = __shfl_up_sync(0xffffffffu, p, o);
                if (lane >= o) p += v;
            }
            if (n < N) c[n + 1] = carry + p;
            carry += __shfl_sync(0xffffffffu, p, 31);
        }
    }
    __syncthreads();

    // 3. forward transforms of all T sequences
    constexpr int kB16 = ((N2 > 8192 ? 4 : 2) * 256 / NT) > 0 ? ((N2 > 8192 ? 4 : 2) * 256 / NT) : 1;
    smem_fft_ct<N2, 1, -1, kB16>(E, N2, T, tw);

    // 4. power spectrum folded for a half-length inverse: u[j] = P[2j] + i P[2j+1], P = |X|^2
    //    (read everything first, then overwrite the first half of each buffer in place)
    {
        constexpr int H2 = N2 / 2;
        constexpr int MAXU = (N2 > 8192 ? 8192 : 4096) / NT + 1;  // items per thread bound
        cpx<S> u[MAXU];
#pragma unroll
        for (int it = 0; it < MAXU; ++it) {
            const int idx = threadIdx.x + it * blockDim.x;
            if (idx < T * H2) {
                const int j = idx / H2, k = idx - j * H2;
                const cpx<S> a = E[(size_t)j * N2 + 2 * k];
                const cpx<S> b = E[(size_t)j * N2 + 2 * k + 1];
                u[it] = {a.x * a.x + a.y * a.y, b.x * b.x + b.y * b.y};
            }
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < MAXU; ++it) {
            const int idx = threadIdx.x + it * blockDim.x;
            if (idx < T * H2) {
                const int j = idx / H2, k = idx - j * H2;
                E[(size_t)j * N2 + k] = u[it];
            }
        }
        __syncthreads();
    }

    // 5. backward transforms of length N2/2 (sign +1)
    if constexpr (N2 >= 2) smem_fft_ct<N2 / 2, 1, +1, kB16>(E, N2, T, tw_half);

    // 6. real-input unfold: R(m) = E(m) + e^{+2 pi i m / N2} O(m) with
    //    E = (U[m] + conj U[N2/2 - m]) / 2, O = (U[m] - conj U[N2/2 - m]) / (2i);
    //    corr(m) = Re R(m) / N2; combine; lag scatter (j fastest: a tile's outputs of one
    //    lag are adjacent in memory).
    const double inv_n2 = 1.0 / (double)N2;
    constexpr int H2 = N2 / 2;
    for (int idx = threadIdx.x; idx < N * T; idx += blockDim.x) {
        const int m = idx / T, j = idx - m * T;
        if (j >= nvalid) continue;
        const int li = lag_index ? lag_index[m] : m;
        if (li < 0 && !corr_out) continue;
        const cpx<S>* U = E + (size_t)j * N2;
        const cpx<S> A = U[m];
        const cpx<S> Bc = U[m == 0 ? 0 : H2 - m];
        const S h = S(0.5);
        const S ex = (A.x + Bc.x) * h;              // Re E
        const S ox = (A.y + Bc.y) * h;              // O = (A - conj B) / (2i)
        const S oy = -(A.x - Bc.x) * h;
        const cpx<S> w = tw[m];                      // exp(-2 pi i m / N2)
        const S re = ex + (w.x * ox + w.y * oy);     // Re(conj(w) * O)
        const double corr = (double)re * inv_n2;
        const double* c = C + (size_t)j * (N + 1);
        const double ramp = (double)(N - m);
        const double d_a = (c[N - m] + (c[N] - c[m])) / ramp;
        const double d = d_a - 2.0 * corr / ramp;
        const int64_t s = s0 + j;
        if (corr_out) corr_out[s * N + m] = corr;
        if (li >= 0) {
            const int64_t dest = dest_of_slot ? dest_of_slot[s] : s;
            out[(int64_t)li * out_stride + dest] = (OutT)(m == 0 ? 0.0 : d);
        }
    }
    if (mean_out && threadIdx.x < nvalid) {
        mean_out[2 * (s0 + threadIdx.x)] = mu[2 * threadIdx.x];
        mean_out[2 * (s0 + threadIdx.x) + 1] = mu[2 * threadIdx.x + 1];
    }
}

}  // namespace

size_t temporal_smem_bytes(int N, int N2, int T, int scalar_bytes) {
    return (size_t)T * N2 * 2 * scalar_bytes + (size_t)T * (N + 1) * 8 + (size_t)T * 16;
}

int temporal_threads(int N2, int T, int scalar_bytes) {
    static const bool t256 = std::getenv("DDM_GENERIC_T256") != nullptr;
    return (!t256 && scalar_bytes == 8 && N2 >= 4096 && (size_t)T * N2 <= 8192) ? 512 : 256;
}

// Sequences per tile. Capacity: 256 threads x 2 radix-16 butterflies -> T * N2 <= 8192
// (N2 = 16384 runs alone with 4 butterflies per thread). Prefer the largest T <= 8 whose
// shared memory lets two CTAs share an SM (<= 113 KB) if that keeps T >= 4, otherwise the
// largest T that fits one CTA. DDM_B200_TILE overrides (experiments).
namespace {

// recv [source s][q][n_s] -> spec tile-major [(q / T) * N + n][q % T]; one thread per output
// element, consecutive threads walk q % T then n so stores are contiguous.
template <typename S>
__global__ void repack_segments_kernel(const cpx<S>* __restrict__ recv, int64_t q_count,
                                       const __grid_constant__ SegTable segs, int N, int T,
                                       cpx<S>* __restrict__ spec) {
    const int64_t tiles = (q_count + T - 1) / T;
    const int64_t total = tiles * N * T;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tile = i / ((int64_t)N * T);
        const int r = (int)(i - tile * N * T);
        const int n = r / T, j = r - n * T;
        const int64_t q = tile * T + j;
        cpx<S> v = {S(0), S(0)};
        if (q < q_count) {
            int s = 0;
            while (s + 1 < segs.count && n >= segs.off[s + 1]) ++s;
            v = recv[segs.base[s] + q * segs.n[s] + (n - segs.off[s])];
        }
        spec[i] = v;
    }
}

}  // namespace

template <typename S>
cudaError_t launch_repack_segments(const void* recv, int64_t q_count, const SegTable& segs, int N,
                                   int T, void* spec, cudaStream_t stream) {
    const int64_t total = (q_count + T - 1) / T * N * T;
    const int blocks = (int)std::min<int64_t>(148 * 8, (total + 255) / 256);
    if (blocks == 0) return cudaSuccess;
    repack_segments_kernel<S><<<blocks, 256, 0, stream>>>(static_cast<const cpx<S>*>(recv), q_count,
                                                          segs, N, T, static_cast<cpx<S>*>(spec));
    return cudaGetLastError();
}

template cudaError_t launch_repack_segments<float>(const void*, int64_t, const SegTable&, int, int,
                                                   void*, cudaStream_t);
template cudaError_t launch_repack_segments<double>(const void*, int64_t, const SegTable&, int, int,
                                                    void*, cudaStream_t);

int temporal_tile(int N, int N2, int scalar_bytes) {
    auto ok = [&](int T, size_t cap) {
        const bool cap_bfly = (N2 > 8192) ? (T == 1) : (T * N2 <= 8192);
        return cap_bfly && temporal_smem_bytes(N, N2, T, scalar_bytes) <= cap;
    };
    if (const char* env = std::getenv("DDM_B200_TILE")) {
        const int t = std::atoi(env);
        if (t >= 1 && t <= 16 && ok(t, 227 * 1024)) return t;
    }
    for (int T = 8; T >= 4; T >>= 1)
        if (ok(T, 113 * 1024)) return T;
    for (int T = 8; T >= 1; T >>= 1)
        if (ok(T, 220 * 1024)) return T;
    return 0;
}

namespace {

template <typename S, typename OutT, int N2>
void launch_t(const TemporalArgs& a, cudaStream_t stream) {
    const int T = a.layout.T;
    const size_t smem = temporal_smem_bytes(a.N, N2, T, sizeof(S));
    const int threads = temporal_threads(N2, T, sizeof(S));
    auto k = threads == 512 ? temporal_kernel<S, OutT, N2, 512> : temporal_kernel<S, OutT, N2, 256>;
    // a failed attribute stays the last error (the caller's cudaGetLastError reports it):
    // no launch that would fail later with an unrelated message
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return;
    k<<<(unsigned)a.layout.tiles(), threads, smem, stream>>>(
        static_cast<const cpx<S>*>(a.spec), a.N, a.layout, static_cast<const cpx<S>*>(a.tw.ptr),
        static_cast<const cpx<S>*>(a.tw_half.ptr),
        a.lag_index, static_cast<OutT*>(a.out), a.out_stride, a.dest_of_slot, a.corr_out,
        a.mean_out);
}

template <typename S, typename OutT>
cudaError_t dispatch_t(const TemporalArgs& a, cudaStream_t stream) {
    switch (a.N2) {
#define DDMK_T_CASE(LEN) \
    case LEN: launch_t<S, OutT, LEN>(a, stream); break;
        DDMK_T_CASE(2) DDMK_T_CASE(4) DDMK_T_CASE(8) DDMK_T_CASE(16) DDMK_T_CASE(32)
        DDMK_T_CASE(64) DDMK_T_CASE(128) DDMK_T_CASE(256) DDMK_T_CASE(512) DDMK_T_CASE(1024)
        DDMK_T_CASE(2048) DDMK_T_CASE(4096) DDMK_T_CASE(8192) DDMK_T_CASE(16384)
#undef DDMK_T_CASE
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace

template <typename S>
cudaError_t launch_temporal(const TemporalArgs& a, cudaStream_t stream) {
    if (a.layout.tiles() == 0) return cudaSuccess;
    return a.out_f64 ? dispatch_t<S, double>(a, stream) : dispatch_t<S, float>(a, stream);
}

template cudaError_t launch_temporal<float>(const TemporalArgs&, cudaStream_t);
template cudaError_t launch_temporal<double>(const TemporalArgs&, cudaStream_t);

}  // namespace ddmk
