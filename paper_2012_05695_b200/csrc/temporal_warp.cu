// Temporal engine v2: one warp per wave vector, register-resident FFTs (sm_100a).
//
// Same arithmetic contract as temporal.cu (`SequenceEngine<S>::with_ft`, `temporal.cpp:77-129`)
// for the sizes that dominate the benchmarks: f32, padded length N2 = 2048 (N in [513, 1024];
// the 512x512x1024 headline and the 500x500x1000 case), input laid out wave-vector major
// (spec[q * N + n]).  Per sequence, with L = N2/2 = 1024 = 32 lanes x 32 registers:
//   mean (f64) and shift (f32)                                   `temporal.cpp:82-92`
//   d_a(m) = sum_{n >= m} (p_n + p_{N-1-n}) / (N - m), p = |t|^2 in f64  (`:19-42`, suffix form)
//   X(2k)   = FFT_L(t)(k),  X(2k+1) = FFT_L(t * W_N2^n)(k)       (zero-padded FFT_N2, `:56-59`)
//   u(k)    = |X(2k)|^2 + i |X(2k+1)|^2                          (P = |X|^2 in f32, `:60-64`)
//   U       = IFFT_L(u);  corr(m) = Re[E(m) + W_N2^{-m} O(m)] / N2  (real-input unfold, `:65-73`)
//   d(m)    = d_a(m) - 2 corr(m) / (N - m), d(0) = 0             (`:114-129`, `scheduler.cpp:157`)
// Each FFT_L is the four-step of warp_fft.cuh: one shared-memory exchange, no block barrier.
// A CTA is 8 warps = a tile of 8 consecutive wave vectors, persistent over tiles; every warp
// prefetches its next sequence with cp.async while it computes the current one, and the
// 8 results are transposed through shared memory so each lag row is stored as 32 B.
#include <cuda_pipeline_primitives.h>

#include <algorithm>

#include "kernels.cuh"
#include "warp_fft.cuh"

namespace ddmk {

namespace {

constexpr int kL = 1024;              // half padded length
constexpr int kN2 = 2048;
constexpr int kWarps = 8;             // wave vectors per tile
constexpr int kPad = kL + kL / 32;    // padded complex slots per buffer (index n + n/32)

__device__ __forceinline__ int padded(int n) { return n + (n >> 5); }

struct WarpSmem {
    cpx<float> stage[2][kPad];   // input double buffer; the current one doubles as FFT scratch
    double d[kPad];              // d_a(m), then the output value of lag m
    double pad_[4];              // sizeof = 32 mod 128 B: the tile store reads 8 regions at once
};
static_assert(sizeof(WarpSmem) % 128 == 32, "region stride must stagger banks");

template <typename OutT, bool FULL>
__global__ void __launch_bounds__(32 * kWarps, 1)
temporal_warp_kernel(const cpx<float>* __restrict__ spec, int N_rt, int64_t nq,
                     const int* __restrict__ lag_index, OutT* __restrict__ out,
                     int64_t out_stride, const int64_t* __restrict__ dest_of_slot,
                     double* __restrict__ corr_out, double* __restrict__ mean_out) {
    // FULL: N == L, every bound below folds at compile time
    const int N = FULL ? kL : N_rt;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem* ws = reinterpret_cast<WarpSmem*>(smem_raw);
    cpx<float>* tb_fwd = reinterpret_cast<cpx<float>*>(ws + kWarps);  // W_N2^{32 b}, b < 32
    cpx<float>* tb_unf = tb_fwd + 32;                                   // W_N2^{-b},   b < 32
    double* rcp = reinterpret_cast<double*>(tb_unf + 32);               // 1 / (N - m) at padded(m)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& my = ws[warp];

    for (int m = threadIdx.x; m < N; m += blockDim.x) rcp[padded(m)] = 1.0 / (double)(N - m);
    const double inv_n = 1.0 / (double)N;
    if (threadIdx.x < 32) {
        double s, c;
        sincospi(-2.0 * (double)(32 * threadIdx.x) / kN2, &s, &c);
        tb_fwd[threadIdx.x] = {(float)c, (float)s};
        sincospi(2.0 * (double)threadIdx.x / kN2, &s, &c);
        tb_unf[threadIdx.x] = {(float)c, (float)s};
    }
    // per-lane constants: four-step twiddles W_L^{lane c}, W_N2^{lane}, W_N2^{-32 lane}
    LaneTw<32, float> tw;
    tw.init(lane, kL);
    cpx<float> base_fwd, base_unf;
    {
        double s, c;
        sincospi(-2.0 * (double)lane / kN2, &s, &c);
        base_fwd = {(float)c, (float)s};
        sincospi(2.0 * (double)(32 * lane) / kN2, &s, &c);
        base_unf = {(float)c, (float)s};
    }
    __syncthreads();

    const int64_t ntiles = (nq + kWarps - 1) / kWarps;
    // cp.async of one sequence into a padded stage buffer; lanes beyond N are zero-filled
    auto prefetch = [&](int64_t tile, int buf) {
        const int64_t q = tile * kWarps + warp;
        const bool live = tile < ntiles && q < nq;
        const cpx<float>* src = spec + (live ? q : 0) * (int64_t)N;
#pragma unroll 4
        for (int b = 0; b < 32; ++b) {
            const int n = lane + 32 * b;
            const bool ok = live && n < N;
            __pipeline_memcpy_async(&my.stage[buf][padded(n)], ok ? src + n : src, 8, ok ? 0 : 8);
        }
        __pipeline_commit();
    };

    int buf = 0;
    prefetch(blockIdx.x, 0);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
        prefetch(tile + gridDim.x, buf ^ 1);
        __pipeline_wait_prior(1);
        __syncwarp();
        const int64_t q = tile * kWarps + warp;
        const bool live = q < nq;
        cpx<float>* st = my.stage[buf];

        // ---- mean (f64) and shifted sequence in registers: lane a holds t[a + 32 b]
        cpx<float> t[32];
        double sx = 0.0, sy = 0.0;
        {
            double ax[4] = {0, 0, 0, 0}, ay[4] = {0, 0, 0, 0};
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                t[b] = st[padded(lane + 32 * b)];
                ax[b & 3] += (double)t[b].x;
                ay[b & 3] += (double)t[b].y;
            }
            sx = (ax[0] + ax[1]) + (ax[2] + ax[3]);
            sy = (ay[0] + ay[1]) + (ay[2] + ay[3]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
            sy += __shfl_xor_sync(0xffffffffu, sy, o);
        }
        const double mx = sx * inv_n, my_ = sy * inv_n;
        const float ox = (float)mx, oy = (float)my_;
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            if (lane + 32 * b < N) {
                t[b].x -= ox;
                t[b].y -= oy;
            }
        }

        // ---- S(m) = sum_{n >= m} (p_n + p_{N-1-n}) = (N - m) d_a(m), p = |t|^2 in f64:
        //      p goes to D in the strided order, is read back per lane as 32 consecutive n
        //      (plus the mirrored n), suffix-summed in lane and across lanes, and S(m) is
        //      left in D for the epilogue; lane a owns m = 32 a + b
        {
#pragma unroll
            for (int b = 0; b < 32; ++b)
                my.d[padded(lane + 32 * b)] = (double)t[b].x * t[b].x + (double)t[b].y * t[b].y;
            __syncwarp();
            double qv[32];
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                const int n = 32 * lane + b;
                double v = 0.0;
                if (n < N) v = my.d[padded(n)] + my.d[padded(N - 1 - n)];
                qv[b] = v;
            }
            __syncwarp();
            // in-lane suffix sums as 4 independent chains of 8, then chain offsets
            double part[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                double r = 0.0;
#pragma unroll
                for (int b = 8 * c + 7; b >= 8 * c; --b) {
                    r += qv[b];
                    qv[b] = r;
                }
                part[c] = r;
            }
            const double tot = (part[0] + part[1]) + (part[2] + part[3]);
            // exclusive suffix over lanes: sum of totals of lanes > lane
            double incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double v = __shfl_down_sync(0xffffffffu, incl, o);
                if (lane + o < 32) incl += v;
            }
            const double base = incl - tot;
            const double off[4] = {base + part[1] + part[2] + part[3], base + part[2] + part[3],
                                   base + part[3], base};
#pragma unroll
            for (int b = 0; b < 32; ++b) my.d[padded(32 * lane + b)] = qv[b] + off[b >> 3];
        }
        __syncwarp();  // stage is about to become FFT scratch

        // ---- forward: even outputs FFT_L(t), odd outputs FFT_L(t * W_N2^n)
        float pe[32];
        {
            cpx<float> u[32];
#pragma unroll
            for (int b = 0; b < 32; ++b) u[b] = t[b];
            group_fft<32, 32, -1, float>(u, st, lane, tw);
#pragma unroll
            for (int d = 0; d < 32; ++d) pe[d] = u[d].x * u[d].x + u[d].y * u[d].y;
        }
        cpx<float> z[32];
#pragma unroll
        for (int b = 0; b < 32; ++b) z[b] = cmul(t[b], cmul(base_fwd, tb_fwd[b]));
        group_fft<32, 32, -1, float>(z, st, lane, tw);
#pragma unroll
        for (int d = 0; d < 32; ++d) z[d] = {pe[d], z[d].x * z[d].x + z[d].y * z[d].y};

        // ---- half-length inverse, then U to shared memory (natural order, padded)
        group_fft<32, 32, +1, float>(z, st, lane, tw);
#pragma unroll
        for (int d = 0; d < 32; ++d) st[padded(lane + 32 * d)] = z[d];
        __syncwarp();

        // ---- unfold + combine; lane a owns m = 32 a + b
        //      d(m) = (S(m) - 2 corr(m)) / (N - m), corr = Re R(m) / N2, d(0) = 0
        const double two_over_n2 = 2.0 / (double)kN2;
        const float h = 0.5f;
#pragma unroll 8
        for (int b = 0; b < 32; ++b) {
            const int m = 32 * lane + b;
            if (m < N) {
                const cpx<float> A = st[padded(m)];
                const cpx<float> Bc = st[padded(m == 0 ? 0 : kL - m)];
                const float ex = (A.x + Bc.x) * h;
                const float ox2 = (A.y + Bc.y) * h;
                const float oy2 = -(A.x - Bc.x) * h;
                const cpx<float> w = cmul(base_unf, tb_unf[b]);  // exp(+2 pi i m / N2)
                const float re = ex + (w.x * ox2 - w.y * oy2);
                const double dval = (my.d[padded(m)] - (double)re * two_over_n2) * rcp[padded(m)];
                my.d[padded(m)] = (m == 0) ? 0.0 : dval;
                if (corr_out && live) corr_out[q * N + m] = (double)re * (0.5 * two_over_n2);
            }
        }
        if (mean_out && live && lane == 0) {
            mean_out[2 * q] = mx;
            mean_out[2 * q + 1] = my_;
        }

        // ---- tile store: lag rows of 8 consecutive wave vectors
        __syncthreads();
        const int64_t q0 = tile * kWarps;
        if (!lag_index && !dest_of_slot && q0 + kWarps <= nq) {
            // every lag, identity destinations: one thread per lag row, 8 values per store
            for (int m = threadIdx.x; m < N; m += blockDim.x) {
                OutT v[kWarps];
#pragma unroll
                for (int j = 0; j < kWarps; ++j) v[j] = (OutT)ws[j].d[padded(m)];
                OutT* dst = out + (int64_t)m * out_stride + q0;
                if constexpr (sizeof(OutT) == 4) {
                    if (((uintptr_t)dst & 15) == 0) {
                        reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
                        reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
                        continue;
                    }
                }
#pragma unroll
                for (int j = 0; j < kWarps; ++j) dst[j] = v[j];
            }
        } else {
            for (int idx = threadIdx.x; idx < N * kWarps; idx += blockDim.x) {
                const int m = idx >> 3, j = idx & 7;
                if (q0 + j >= nq) continue;
                const int li = lag_index ? lag_index[m] : m;
                if (li < 0) continue;
                const int64_t dst = dest_of_slot ? dest_of_slot[q0 + j] : q0 + j;
                out[(int64_t)li * out_stride + dst] = (OutT)ws[j].d[padded(m)];
            }
        }
        __syncthreads();
    }
    __pipeline_wait_prior(0);
}

}  // namespace

bool temporal_warp_supported(int N, int N2, int scalar_bytes) {
    return scalar_bytes == 4 && N2 == kN2 && N > kL / 2 && N <= kL;
}

size_t temporal_warp_smem() {
    return sizeof(WarpSmem) * kWarps + 64 * sizeof(cpx<float>) + kPad * sizeof(double);
}

cudaError_t launch_temporal_warp(const TemporalArgs& a, int num_sms, cudaStream_t stream) {
    const size_t smem = temporal_warp_smem();
    const int64_t tiles = (a.layout.g_count + kWarps - 1) / kWarps;
    const int grid = (int)std::min<int64_t>(tiles, (int64_t)num_sms);
    if (grid == 0) return cudaSuccess;
    const cpx<float>* spec = static_cast<const cpx<float>*>(a.spec);
    const bool full = a.N == kL;
    if (a.out_f64) {
        auto k = full ? temporal_warp_kernel<double, true> : temporal_warp_kernel<double, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, 32 * kWarps, smem, stream>>>(spec, a.N, a.layout.g_count, a.lag_index,
                                               static_cast<double*>(a.out), a.out_stride,
                                               a.dest_of_slot, a.corr_out, a.mean_out);
    } else {
        auto k = full ? temporal_warp_kernel<float, true> : temporal_warp_kernel<float, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, 32 * kWarps, smem, stream>>>(spec, a.N, a.layout.g_count, a.lag_index,
                                               static_cast<float*>(a.out), a.out_stride,
                                               a.dest_of_slot, a.corr_out, a.mean_out);
    }
    return cudaGetLastError();
}

}  // namespace ddmk
