// Temporal engine v2: one warp per wave vector, register-resident FFTs (sm_100a).
//
// Same arithmetic contract as temporal.cu (`SequenceEngine<S>::with_ft`, `temporal.cpp:77-129`)
// for the sizes that dominate the benchmarks: f32, padded length N2 = 2048 (N in [513, 1024];
// the 512x512x1024 headline and the 500x500x1000 case), input laid out wave-vector major
// (spec[q * N + n]).  Per sequence, with L = N2/2 = 1024 = 32 lanes x 32 registers:
//   mean and shift (f32)                                         `temporal.cpp:82-92`
//   d_a(m) = sum_{n >= m} (p_n + p_{N-1-n}) / (N - m), p = |t|^2 in f64  (`:19-42`, suffix form)
//   X(2k)   = FFT_L(t)(k),  X(2k+1) = FFT_L(t * W_N2^n)(k)       (zero-padded FFT_N2, `:56-59`)
//   u(k)    = |X(2k)|^2 + i |X(2k+1)|^2                          (P = |X|^2 in f32, `:60-64`)
//   U       = IFFT_L(u);  corr(m) = Re[E(m) + W_N2^{-m} O(m)] / N2  (real-input unfold, `:65-73`)
//   d(m)    = (S(m) - 2 corr(m)) / (N - m), d(0) = 0             (`:114-129`, `scheduler.cpp:157`)
// The time mean only conditions the subtraction (d is offset invariant, `temporal.hpp:258-262`),
// so it is formed with a pairwise f32 sum; everything the reference keeps in f64 (power,
// averages term, combination) stays f64.
//
// Data movement per sequence: one TMA bulk copy (cp.async.bulk, 8 KB) into the warp's stage
// buffer, issued one tile ahead; three four-step FFTs (warp_fft.cuh, one shared-memory
// exchange each, the stage buffer doubles as scratch); the unfold reads U(L-m) from the
// mirrored lane with shuffles; d(m) goes to the warp's D array and a CTA of 8 warps stores
// 8 consecutive wave vectors per lag row.
#include <algorithm>

#include "kernels.cuh"
#include "warp_fft.cuh"

namespace ddmk {

namespace {

constexpr int kL = 1024;              // half padded length
constexpr int kN2 = 2048;
constexpr int kWarps = 8;             // wave vectors per tile
constexpr int kPad = kL + kL / 32;    // slots per buffer (FFT scratch pitch 33 x 32)

__device__ __forceinline__ int padded(int n) { return n + (n >> 5); }

struct WarpSmem {
    cpx<float> stage[2][kPad];   // input double buffer (dense [0, L)), then FFT scratch
    double d[kPad];              // S(m) at padded(m), then the output value of lag m
    unsigned long long bar[2];   // mbarriers of the two stage buffers
    double pad_[2];              // sizeof = 32 mod 128 B: the tile store reads 8 regions at once
};
static_assert(sizeof(WarpSmem) % 128 == 32, "region stride must stagger banks");

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}

// lane 0: expect `bytes` on `bar` and start the bulk copy global -> shared
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          unsigned long long* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

template <typename OutT, bool FULL>
__global__ void __launch_bounds__(32 * kWarps, 1)
temporal_warp_kernel(const cpx<float>* __restrict__ spec, int N_rt, int64_t nq,
                     const int* __restrict__ lag_index, OutT* __restrict__ out,
                     int64_t out_stride, const int64_t* __restrict__ dest_of_slot,
                     double* __restrict__ corr_out, double* __restrict__ mean_out) {
    // FULL: N == L, every bound below folds at compile time
    const int N = FULL ? kL : N_rt;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WarpSmem* ws = reinterpret_cast<WarpSmem*>(smem_raw);
    cpx<float>* tb_fwd = reinterpret_cast<cpx<float>*>(ws + kWarps);  // W_N2^{32 b}, b < 32

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& my = ws[warp];

    if (threadIdx.x < 32) {
        double s, c;
        sincospi(-2.0 * (double)(32 * threadIdx.x) / kN2, &s, &c);
        tb_fwd[threadIdx.x] = {(float)c, (float)s};
    }
    if (lane == 0) {
        mbar_init(&my.bar[0]);
        mbar_init(&my.bar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // per-lane constants: four-step twiddles W_L^{lane c}, W_N2^{lane}, W_N2^{-lane}
    LaneTw<32, float> tw;
    tw.init(lane, kL);
    cpx<float> base_fwd, base_unf;
    {
        double s, c;
        sincospi(-2.0 * (double)lane / kN2, &s, &c);
        base_fwd = {(float)c, (float)s};
        base_unf = {(float)c, (float)-s};
    }
    const float inv_nf = 1.0f / (float)N;
    __syncthreads();

    const int64_t ntiles = (nq + kWarps - 1) / kWarps;
    const uint32_t bytes = (uint32_t)N * 8u;
    auto prefetch = [&](int64_t tile, int buf) {
        const int64_t q = tile * kWarps + warp;
        if (lane == 0 && tile < ntiles && q < nq)
            bulk_load(my.stage[buf], spec + q * (int64_t)N, bytes, &my.bar[buf]);
    };

    int buf = 0;
    uint32_t phase[2] = {0u, 0u};
    prefetch(blockIdx.x, 0);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
        prefetch(tile + gridDim.x, buf ^ 1);
        const int64_t q = tile * kWarps + warp;
        const bool live = q < nq;
        cpx<float>* st = my.stage[buf];
        if (live) {
            mbar_wait(&my.bar[buf], phase[buf]);
            phase[buf] ^= 1u;
        }

        // ---- load (lane a holds s[a + 32 b]), mean by a pairwise f32 sum, shift
        cpx<float> t[32];
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            const int n = lane + 32 * b;
            t[b] = (live && n < N) ? st[n] : cpx<float>{0.f, 0.f};
        }
        float mx, my_;
        {
            float ax[16], ay[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                ax[i] = t[i].x + t[i + 16].x;
                ay[i] = t[i].y + t[i + 16].y;
            }
#pragma unroll
            for (int w = 8; w > 0; w >>= 1)
#pragma unroll
                for (int i = 0; i < w; ++i) {
                    ax[i] += ax[i + w];
                    ay[i] += ay[i + w];
                }
            mx = ax[0];
            my_ = ay[0];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mx += __shfl_xor_sync(0xffffffffu, mx, o);
                my_ += __shfl_xor_sync(0xffffffffu, my_, o);
            }
            mx *= inv_nf;
            my_ *= inv_nf;
        }
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            if (lane + 32 * b < N) {
                t[b].x -= mx;
                t[b].y -= my_;
            }
        }

        // ---- S(m) = sum_{n >= m} (p_n + p_{N-1-n}) = (N - m) d_a(m), p = |t|^2 in f64:
        //      p goes to D in the strided order, is read back per lane as 32 consecutive n
        //      (plus the mirrored n), suffix-summed in lane and across lanes; S(m) stays in D
        {
#pragma unroll
            for (int b = 0; b < 32; ++b)
                my.d[padded(lane + 32 * b)] = (double)t[b].x * t[b].x + (double)t[b].y * t[b].y;
            __syncwarp();
            double qv[32];
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                const int n = 32 * lane + b;
                qv[b] = (n < N) ? my.d[padded(n)] + my.d[padded(N - 1 - n)] : 0.0;
            }
            __syncwarp();
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

        // ---- half-length inverse: lane c holds U[c + 32 d] in z[d]
        group_fft<32, 32, +1, float>(z, st, lane, tw);

        // ---- unfold + combine on the lane's own m = c + 32 d; U[L - m] sits in lane
        //      (32 - c) mod 32, register 31 - d (lane 0: its own register (32 - d) mod 32)
        //      2 Re R(m) = (A.x + B.x) + w.x (A.y + B.y) + w.y (A.x - B.x), w = W_N2^{-m}
        const int src = (32 - lane) & 31;
        const double inv_n2 = 1.0 / (double)kN2;
#pragma unroll
        for (int d = 0; d < 32; ++d) {
            const int m = lane + 32 * d;
            cpx<float> Bc;
            Bc.x = __shfl_sync(0xffffffffu, z[31 - d].x, src);
            Bc.y = __shfl_sync(0xffffffffu, z[31 - d].y, src);
            if (lane == 0) Bc = z[(32 - d) & 31];
            const cpx<float> A = z[d];
            const cpx<float> w = cmul(base_unf, ct_w<+1, float>(32 * d, kN2));  // exp(+2 pi i m / N2)
            const float re2 = (A.x + Bc.x) + (w.x * (A.y + Bc.y) + w.y * (A.x - Bc.x));
            if (m < N) {
                const double corr2 = (double)re2 * inv_n2;  // 2 corr(m)
                const double val = (my.d[padded(m)] - corr2) * __drcp_rn((double)(N - m));
                my.d[padded(m)] = (m == 0) ? 0.0 : val;
                if (corr_out && live) corr_out[q * N + m] = 0.5 * corr2;
            }
        }
        if (mean_out && live && lane == 0) {
            mean_out[2 * q] = (double)mx;
            mean_out[2 * q + 1] = (double)my_;
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
}

}  // namespace

bool temporal_warp_supported(int N, int N2, int scalar_bytes) {
    // bulk copies need 16-byte sizes: even N
    return scalar_bytes == 4 && N2 == kN2 && N > kL / 2 && N <= kL && N % 2 == 0;
}

size_t temporal_warp_smem() { return sizeof(WarpSmem) * kWarps + 32 * sizeof(cpx<float>); }

cudaError_t launch_temporal_warp(const TemporalArgs& a, int num_sms, cudaStream_t stream) {
    const size_t smem = temporal_warp_smem();
    const int64_t tiles = (a.layout.g_count + kWarps - 1) / kWarps;
    const int grid = (int)std::min<int64_t>(tiles, (int64_t)num_sms);
    if (grid == 0) return cudaSuccess;
    if (reinterpret_cast<uintptr_t>(a.spec) % 16 != 0) return cudaErrorMisalignedAddress;
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
