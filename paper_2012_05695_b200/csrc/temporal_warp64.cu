// Temporal engine for f64, the reference's default precision (`scheduler.hpp:80`): one warp per
// wave vector, padded length N2 = 2048 (N in (512, 1024], even), register-resident FFT_1024s in
// double. Same algorithm as the f32 warp engine (temporal_warp.cu; `SequenceEngine<double>::
// with_ft`, `temporal.cpp:77-129`), everything in f64 as the reference computes it there:
//   mean (f64) and shift                                         `temporal.cpp:82-92`
//   X(2k) = FFT_1024(t)(k), X(2k+1) = FFT_1024(t W_2048^n)(k)     (zero-padded FFT_2048)
//   u(k) = |X(2k)|^2 + i |X(2k+1)|^2, U = IFFT_1024(u), real-input unfold (`:56-73`)
//   S(m) = sum_{n >= m} (p_n + p_{N-1-n}) = (N - m) d_a(m)         (`:19-42`, suffix form)
//   d(m) = (S(m) - 2 Re r(m) / N2) / (N - m), d(0) = 0             (`:114-129`, `scheduler.cpp:157`)
// A complex<double> sequence of 1,024 values is 128 registers per lane, so nothing else stays
// in registers across the transforms: the sequence is read from global memory (q-major spectra,
// L2-prefetched one tile ahead) once per use, |X(2k)|^2 waits in shared memory during the odd
// transform, and 2 Re r(m), |t|^2, S(m) and d(m) share a per-warp f64 buffer. The CTA's warps
// store consecutive wave vectors per lag row (48-byte runs of the f64 map).
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "temporal_common.cuh"
#include "warp_fft.cuh"

namespace ddmk {

namespace {

constexpr int kL = 1024;
constexpr int kN2 = 2048;
constexpr int kP = 33;                 // exchange pitch in complex doubles (16-byte rows)
constexpr int kXD = 32 * kP;
constexpr int kPadD = kL + kL / 32;    // padded f64 slots

__device__ __forceinline__ int padded(int n) { return n + (n >> 5); }

struct Warp64 {
    cpx<double> x[kXD];    // FFT exchange; |t|^2 at padded(n) after the transforms
    double w[kPadD];       // |X(2k)|^2 at padded(k); then 2 Re r(m), S-combined d(m) at padded(m)
};

// Length-1024 transform in double (lane a holds x[a + 32 b]; on return lane c holds
// X[c + 32 d]): DFT_32 over b, exchange, DFT_32 over a with the four-step twiddles of row c of
// twt fused into its first butterflies (even W_1024^{a c}; odd W_2048^{a (2c+1)} with the input's
// W_64^{b} factor fused into the first DFT_32)
template <int SIGN, bool ODD>
__device__ __forceinline__ void fft1024d(cpx<double> (&v)[32], cpx<double>* x, int lane,
                                         const cpx<double>* __restrict__ twt) {
    if constexpr (ODD)
        dft32_fused<SIGN, double, true>(v, [](int b) { return ct_w<SIGN, double>(b, 64); });
    else
        RegDft<32, SIGN, double>::run(v);
#pragma unroll
    for (int c = 0; c < 32; ++c) x[c * kP + lane] = v[c];
    __syncwarp();
#pragma unroll
    for (int a = 0; a < 32; ++a) v[a] = x[lane * kP + a];
    __syncwarp();
    const cpx<double>* tw = twt + lane * kP;
    auto twf = [tw](int a) {
        cpx<double> w = tw[a];
        if (SIGN > 0) w.y = -w.y;
        return w;
    };
    dft32_fused<SIGN, double, true>(v, twf);
}

template <bool FULL, int kWarps>
__global__ void __launch_bounds__(32 * kWarps, 1)
temporal_warp64_kernel(const cpx<double>* __restrict__ spec, int N_rt, int64_t nq,
                       const int* __restrict__ lag_index, double* __restrict__ out, int64_t out_stride,
                       const int64_t* __restrict__ dest_of_slot) {
    const int N = FULL ? kL : N_rt;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Warp64* ws = reinterpret_cast<Warp64*>(smem_raw);
    cpx<double>* tw_even = reinterpret_cast<cpx<double>*>(ws + kWarps);   // [a][c] W_1024^{a c}
    cpx<double>* tw_odd = tw_even + kXD;                                    // [c][a] W_2048^{a(2c+1)}
    double* rcp = reinterpret_cast<double*>(tw_odd + kXD);                  // 1 / (N - m) at padded(m)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Warp64& my = ws[warp];
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
        const int a = i >> 5, c = i & 31;
        double sn, cs;
        sincospi(-2.0 * (double)(a * c) / 1024, &sn, &cs);
        tw_even[a * kP + c] = {cs, sn};
        sincospi(-2.0 * (double)(a * (2 * c + 1)) / 2048, &sn, &cs);
        tw_odd[c * kP + a] = {cs, sn};
    }
    for (int m = threadIdx.x; m < N; m += blockDim.x) rcp[padded(m)] = 1.0 / (double)(N - m);
    cpx<double> base_unf;   // W_N2^{-lane}
    sincospi(2.0 * (double)lane / kN2, &base_unf.y, &base_unf.x);
    const double inv_n = 1.0 / (double)N;
    constexpr double inv_n2 = 1.0 / (double)kN2;
    const bool vec_store = ((uintptr_t)out & 15) == 0 && (out_stride % 2) == 0;
    __syncthreads();

    const int64_t ntiles = (nq + kWarps - 1) / kWarps;
    auto load = [&](const cpx<double>* t, bool live, cpx<double> (&v)[32]) {
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            const int n = lane + 32 * b;
            v[b] = (live && n < N) ? t[n] : cpx<double>{0.0, 0.0};
        }
    };

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t q = tile * kWarps + warp;
        const bool live = q < nq;
        const cpx<double>* t = spec + (live ? q : 0) * (int64_t)N;
        {   // the next tile's sequence into L2 (three reads per sequence hit L2)
            const int64_t qn = q + (int64_t)gridDim.x * kWarps;
            if (lane == 0 && qn < nq) tc::l2_prefetch(spec + qn * (int64_t)N, (uint32_t)N * 16u);
        }
        // mean (f64, `temporal.cpp:82-85`) and shift
        cpx<double> v[32];
        load(t, live, v);
        double mx = 0.0, my_ = 0.0;
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            mx += v[b].x;
            my_ += v[b].y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx += __shfl_xor_sync(0xffffffffu, mx, o);
            my_ += __shfl_xor_sync(0xffffffffu, my_, o);
        }
        mx *= inv_n;
        my_ *= inv_n;
        auto shift = [&](cpx<double> (&v)[32]) {
#pragma unroll
            for (int b = 0; b < 32; ++b)
                if (lane + 32 * b < N) {
                    v[b].x -= mx;
                    v[b].y -= my_;
                }
        };
        shift(v);
        // the previous tile's d(m) sit in every warp's buffer until the CTA has stored them
        __syncthreads();

        // even outputs: FFT_1024(t); |X(2k)|^2 to the warp buffer (this lane's own slots)
        fft1024d<-1, false>(v, my.x, lane, tw_even);
#pragma unroll
        for (int d = 0; d < 32; ++d) my.w[padded(lane + 32 * d)] = v[d].x * v[d].x + v[d].y * v[d].y;
        // odd outputs: FFT_1024(t W_2048^n)
        load(t, live, v);
        shift(v);
        fft1024d<-1, true>(v, my.x, lane, tw_odd);
#pragma unroll
        for (int d = 0; d < 32; ++d)
            v[d] = {my.w[padded(lane + 32 * d)], v[d].x * v[d].x + v[d].y * v[d].y};
        // half-length inverse; real-input unfold: 2 Re r(m) for m = lane + 32 d
        fft1024d<+1, false>(v, my.x, lane, tw_even);
        {
            const int src = (32 - lane) & 31;
            // opaque per-sequence copy of the lane base: stops the compiler from hoisting the 32
            // products base * W_N2^{32 d} (128 registers) out of the tile loop
            cpx<double> bu;
            asm volatile("mov.b64 %0, %1;" : "=d"(bu.x) : "d"(base_unf.x));
            asm volatile("mov.b64 %0, %1;" : "=d"(bu.y) : "d"(base_unf.y));
            // two lags per step: 2 Re r(m) = S1 + P, 2 Re r(L - m) = S1 - P (temporal_warp.cu)
#pragma unroll
            for (int d = 0; d < 16; ++d) {
                const int m = lane + 32 * d;
                cpx<double> B;
                B.x = __shfl_sync(0xffffffffu, v[31 - d].x, src);
                B.y = __shfl_sync(0xffffffffu, v[31 - d].y, src);
                if (lane == 0) B = v[(32 - d) & 31];
                const cpx<double> A = v[d];
                const cpx<double> w = cmul(bu, ct_w<+1, double>(32 * d, kN2));
                const double S1 = A.x + B.x;
                const double P = w.x * (A.y + B.y) + w.y * (A.x - B.x);
                my.w[padded(m)] = S1 + P;
                if (kL - m < kL) my.w[padded(kL - m)] = S1 - P;
            }
            if (lane == 0) {   // lag 512, its own mirror
                const cpx<double> A = v[16];
                const cpx<double> w = ct_w<+1, double>(512, kN2);
                my.w[padded(512)] = (A.x + A.x) + w.x * (A.y + A.y);
            }
        }
        // |t|^2 (f64, `temporal.cpp:25-30`) of the shifted sequence into the exchange area
        load(t, live, v);
        shift(v);
        double* pw = reinterpret_cast<double*>(my.x);
#pragma unroll
        for (int b = 0; b < 32; ++b) pw[padded(lane + 32 * b)] = v[b].x * v[b].x + v[b].y * v[b].y;
        __syncwarp();
        // S(m) on m = 32 lane + j: in-lane suffix sums, lane totals suffix-summed by shuffles;
        // combine with 2 Re r(m) and 1 / (N - m), d(0) = 0; d(m) replaces 2 Re r(m)
        {
            double qv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = 32 * lane + j;
                qv[j] = (n < N) ? pw[padded(n)] + pw[padded(N - 1 - n)] : 0.0;
            }
            double r = 0.0;
#pragma unroll
            for (int j = 31; j >= 0; --j) {
                r += qv[j];
                qv[j] = r;
            }
            double incl = r;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double tt = __shfl_down_sync(0xffffffffu, incl, o);
                if (lane + o < 32) incl += tt;
            }
            const double base = incl - r;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int m = 32 * lane + j;
                if (m < N) {
                    const double re2 = my.w[padded(m)];
                    const double val = (qv[j] + base - re2 * inv_n2) * rcp[padded(m)];
                    my.w[padded(m)] = (m == 0) ? 0.0 : val;
                }
            }
        }

        // tile store: lag rows of kWarps consecutive wave vectors
        __syncthreads();
        auto dval = [&](int j, int m) -> double { return ws[j].w[padded(m)]; };
        const int64_t q0 = tile * kWarps;
        if (!lag_index && !dest_of_slot && q0 + kWarps <= nq && vec_store) {
            constexpr int TPR = kWarps / 2;   // threads per row, one double2 each
            const int k = threadIdx.x % TPR;
            const int rows = blockDim.x / TPR;
            double* pdst = out + (int64_t)(threadIdx.x / TPR) * out_stride + q0 + 2 * k;
            const int64_t pstep = (int64_t)rows * out_stride;
            for (int m = threadIdx.x / TPR; m < N; m += rows, pdst += pstep)
                *reinterpret_cast<double2*>(pdst) = make_double2(dval(2 * k, m), dval(2 * k + 1, m));
        } else {
            for (int idx = threadIdx.x; idx < N * kWarps; idx += blockDim.x) {
                const int m = idx / kWarps, j = idx - m * kWarps;
                if (q0 + j >= nq) continue;
                const int li = lag_index ? lag_index[m] : m;
                if (li < 0) continue;
                const int64_t dst = dest_of_slot ? dest_of_slot[q0 + j] : q0 + j;
                out[(int64_t)li * out_stride + dst] = dval(j, m);
            }
        }
    }
}

constexpr int kW64 = 6;

}  // namespace

bool temporal_warp64_supported(int N, int N2) {
    return N2 == kN2 && N > kL / 2 && N <= kL;
}

cudaError_t launch_temporal_warp64(const TemporalArgs& a, int num_sms, cudaStream_t stream) {
    if (!a.out_f64 || a.corr_out || a.mean_out || a.ring.nitems > 0 || a.segs.count != 0 ||
        !temporal_warp64_supported(a.N, a.N2))
        return cudaErrorInvalidValue;
    const size_t smem = sizeof(Warp64) * kW64 + 2 * kXD * sizeof(cpx<double>) + kPadD * sizeof(double);
    const int64_t work = (a.layout.g_count + kW64 - 1) / kW64;
    const int grid = (int)std::min<int64_t>(work, (int64_t)num_sms);
    if (grid == 0) return cudaSuccess;
    auto k = a.N == kL ? temporal_warp64_kernel<true, kW64> : temporal_warp64_kernel<false, kW64>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 32 * kW64, smem, stream>>>(static_cast<const cpx<double>*>(a.spec), a.N, a.layout.g_count,
                                         a.lag_index, static_cast<double*>(a.out), a.out_stride,
                                         a.dest_of_slot);
    return cudaGetLastError();
}

}  // namespace ddmk
