// Temporal engine for long sequences (sm_100a): one CTA of R warps per wave vector,
// padded length N2 = 1024 R (R = 4: N in (1024, 2048], the 1024^2 x 2048 case; R = 8:
// N in (2048, 4096], the 2048^2 x 4096 case). Same arithmetic contract as temporal_warp.cu
// (`SequenceEngine<S>::with_ft`, `temporal.cpp:77-129`), f32 transforms, f64-free except for
// the suffix-sum carries.
//
// With H = R/2, n = n' + 1024 j (j < H) and k = R k' + r:
//   forward  X(R k' + r) = FFT_1024( W_N2^{n' r} sum_j t[n' + 1024 j] W_R^{j r} )(k')  warp r
//   power    P_r(k') = |X(R k' + r)|^2                                           (f32, smem)
//   inverse  u[j] = P[2j] + i P[2j+1] (the real-input half-length trick), j = H j' + s:
//            E_s = IFFT_1024(P_{2s} + i P_{2s+1}),                               warps s < H
//            U(m' + 1024 p) = sum_s E_s(m') e^{2 pi i s m' / L} e^{2 pi i s p / H}  (L = N2/2)
//   unfold   2 Re R(m) from U(m), U(L - m) exactly as the warp engine            all warps
//   S(m)     suffix sums of |t|^2 (warps >= H, while warps < H run the inverse)
//   d(m)     = (S(m) - 2 Re R(m) / N2) / (N - m), d(0) = 0
// Output: map mode writes a q-major block out_q[q - q0][m] (contiguous, coalesced; the host
// turns it lag-major with transpose_lags_kernel), ring mode adds d into per-item sums like
// the warp engine. The sequence arrives by TMA bulk copy (segmented for the sharded corner
// turn), the next one is in flight while the current one is transformed.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "temporal_common.cuh"
#include "warp_fft.cuh"

namespace ddmk {

namespace {

using namespace tc;

constexpr int kF = 1024;
constexpr int kFPad = kXS;                 // exchange buffer per warp (pitch kXP)

__device__ __forceinline__ int pad32(int n) { return n + (n >> 5); }

template <int R>
struct LongGeom {
    static constexpr int N2 = kF * R, L = N2 / 2, NMAX = L, T = 32 * R, H = R / 2;
    // shared-memory carve-up (bytes)
    static constexpr size_t stage = (size_t)NMAX * 8;
    static constexpr size_t pu = (size_t)L * 8;               // P (f32 R x 1024), then U (cpx L)
    static constexpr size_t pw = (size_t)(NMAX + NMAX / 32) * 4;
    static constexpr size_t scratch = (size_t)R * kFPad * 8;
    static constexpr size_t acc = pw;
    static constexpr size_t tw_even = (size_t)kXS * 8;
    static constexpr size_t tw_pre = (size_t)R * 32 * 8;
    static constexpr size_t comb_d = (size_t)H * 32 * 8;
    static constexpr size_t red = 64 * 8;
    static constexpr size_t total(bool ring) {
        return stage + pu + pw + scratch + (ring ? acc : 0) + tw_even + tw_pre + comb_d + red + 16;
    }
};

// FULL: N == N2 / 2, every bound folds at compile time
template <int R, bool kRing, bool FULL>
__global__ void __launch_bounds__(32 * R, (R == 4 ? 2 : 1))
temporal_long_kernel(const cpx<float>* __restrict__ spec, const __grid_constant__ SegTable segs,
                     int N_rt, int64_t q0, int64_t q1, float* __restrict__ out_q,
                     const __grid_constant__ RingArgs ring) {
    using G = LongGeom<R>;
    const int N = FULL ? G::NMAX : N_rt;
    constexpr int T = G::T, H = G::H;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* p = smem;
    cpx<float>* stage = reinterpret_cast<cpx<float>*>(p); p += G::stage;
    float* pf = reinterpret_cast<float*>(p);                 // P_r[k'] at pf[r * 1024 + k']
    cpx<float>* ubuf = reinterpret_cast<cpx<float>*>(p); p += G::pu;
    float* pw = reinterpret_cast<float*>(p); p += G::pw;    // |t|^2 by n, then S(m) (pad32)
    cpx<float>* scratch = reinterpret_cast<cpx<float>*>(p); p += G::scratch;
    float* acc = reinterpret_cast<float*>(p); if (kRing) p += G::acc;
    cpx<float>* tw_even = reinterpret_cast<cpx<float>*>(p); p += G::tw_even;
    cpx<float>* tw_pre = reinterpret_cast<cpx<float>*>(p); p += G::tw_pre;   // [r][b] W_N2^{32 b r}
    cpx<float>* comb_d = reinterpret_cast<cpx<float>*>(p); p += G::comb_d;   // [s][d] e^{+2pi i 32 s d / L}
    double* red = reinterpret_cast<double*>(p); p += G::red;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(p);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    cpx<float>* my_scratch = scratch + warp * kFPad;

    fill_fft1024_tables(tw_even, nullptr, tid, T);
    for (int i = tid; i < R * 32; i += T) {
        const int r = i >> 5, b = i & 31;
        double sn, cs;
        sincospi(-2.0 * (double)(32 * b * r) / G::N2, &sn, &cs);
        tw_pre[i] = {(float)cs, (float)sn};
        if (r < H) {
            sincospi(2.0 * (double)(32 * r * b) / G::L, &sn, &cs);
            comb_d[i] = {(float)cs, (float)sn};
        }
    }
    if (tid == 0) {
        mbar_init(bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // per-thread constants
    cpx<float> tw_lane, comb_lane, unf_base, wj[H];
    {
        double sn, cs;
        sincospi(-2.0 * (double)(lane * warp) / G::N2, &sn, &cs);
        tw_lane = {(float)cs, (float)sn};
        sincospi(2.0 * (double)(warp * lane) / G::L, &sn, &cs);   // used by warps < H
        comb_lane = {(float)cs, (float)sn};
        sincospi(2.0 * (double)tid / G::N2, &sn, &cs);
        unf_base = {(float)cs, (float)sn};
#pragma unroll
        for (int j = 0; j < H; ++j) {
            sincospi(-2.0 * (double)((j * warp) % R) / R, &sn, &cs);
            wj[j] = {(float)cs, (float)sn};
        }
    }
    if (kRing)
        for (int m = tid; m < G::NMAX + G::NMAX / 32; m += T) acc[m] = 0.f;
    __syncthreads();

    // ---- work list: map mode q = q0 + blockIdx.x + k grid; ring mode: slots of the items
    //      blockIdx.x + k grid in order
    int64_t cur_item = blockIdx.x, cur_i = -1;   // ring cursor
    auto ring_first = [&](int64_t it, int64_t& item, int64_t& i) {
        for (item = it; item < ring.nitems; item += gridDim.x) {
            if (ring.item_off[item] < ring.item_off[item + 1]) {
                i = ring.item_off[item];
                return;
            }
        }
        i = -1;
    };
    const uint32_t bytes = (uint32_t)N * 8u;
    auto prefetch = [&](int64_t q) {
        if (q < 0) return;
        if (segs.count == 0) {
            bulk_load(stage, spec + q * (int64_t)N, bytes, bar);
        } else {
            fence_expect(bar, bytes);
            for (int s = 0; s < segs.count; ++s)
                bulk_copy(stage + segs.off[s], spec + segs.base[s] + q * (int64_t)segs.n[s],
                          (uint32_t)segs.n[s] * 8u, bar);
        }
    };

    int64_t q;                     // current sequence
    int64_t nq_item = 0, nq_i = 0;   // ring: the next sequence's cursor
    if (kRing) {
        ring_first(blockIdx.x, cur_item, cur_i);
        q = cur_i >= 0 ? ring.order[cur_i] : -1;
    } else {
        q = q0 + blockIdx.x < q1 ? q0 + blockIdx.x : -1;
    }
    if (tid == 0) prefetch(q);
    uint32_t phase = 0u;
    const float inv_nf = 1.0f / (float)N;
    constexpr float inv_n2 = 1.0f / (float)G::N2;

    while (q >= 0) {
        // next sequence of this CTA (uniform)
        int64_t qn;
        if (kRing) {
            nq_item = cur_item;
            nq_i = cur_i + 1;
            if (nq_i >= ring.item_off[cur_item + 1]) ring_first(cur_item + gridDim.x, nq_item, nq_i);
            qn = nq_i >= 0 ? ring.order[nq_i] : -1;
        } else {
            qn = q + gridDim.x < q1 ? q + gridDim.x : -1;
        }
        mbar_wait(bar, phase);
        phase ^= 1u;

        // ---- mean (f32, fixed order: thread strides, warp tree, warps in order)
        {
            float sx = 0.f, sy = 0.f;
            for (int n = tid; n < N; n += T) {
                sx += stage[n].x;
                sy += stage[n].y;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sx += __shfl_xor_sync(0xffffffffu, sx, o);
                sy += __shfl_xor_sync(0xffffffffu, sy, o);
            }
            if (lane == 0) {
                red[2 * warp] = sx;
                red[2 * warp + 1] = sy;
            }
        }
        __syncthreads();  // (A)
        float mx = 0.f, my = 0.f;
#pragma unroll
        for (int w = 0; w < R; ++w) {
            mx += (float)red[2 * w];
            my += (float)red[2 * w + 1];
        }
        mx *= inv_nf;
        my *= inv_nf;

        // ---- forward input of warp r: y[n'] = W_N2^{n' r} sum_j t[n' + 1024 j] W_R^{j r};
        //      warp r < H also keeps |t|^2 of its chunk j = r for the averages term
        cpx<float> v[32];
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            const int n1 = lane + 32 * b;
            cpx<float> a = {0.f, 0.f};
#pragma unroll
            for (int j = 0; j < H; ++j) {
                const int n = n1 + kF * j;
                if (FULL || n < N) {
                    const cpx<float> t = {stage[n].x - mx, stage[n].y - my};
                    a = (j == 0) ? t : cadd(a, cmul(t, wj[j]));
                }
            }
            v[b] = cmul(cmul(a, tw_lane), tw_pre[warp * 32 + b]);
        }
        if (warp < H) {
            // |t|^2 of chunk j = warp for the averages term (one warp-uniform branch)
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                const int n = lane + 32 * b + kF * warp;
                if (FULL || n < N) {
                    const float tx = stage[n].x - mx, ty = stage[n].y - my;
                    pw[pad32(n)] = tx * tx + ty * ty;
                }
            }
        }
        __syncthreads();  // (B) the stage is free
        if (tid == 0) prefetch(qn);

        fft1024<-1, false>(v, my_scratch, lane, tw_even);
#pragma unroll
        for (int d = 0; d < 32; ++d) pf[warp * kF + lane + 32 * d] = v[d].x * v[d].x + v[d].y * v[d].y;
        __syncthreads();  // (C) P and |t|^2 complete

        if (warp < H) {
            // ---- inverse quarter/half: E_s = IFFT_1024(P_{2s} + i P_{2s+1}), twisted by
            //      e^{2 pi i s m' / L}, parked in the warp's scratch as [m']
            const int s = warp;
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                const int j = lane + 32 * b;
                v[b] = {pf[(2 * s) * kF + j], pf[(2 * s + 1) * kF + j]};
            }
            fft1024<+1, false>(v, my_scratch, lane, tw_even);
#pragma unroll
            for (int d = 0; d < 32; ++d)
                my_scratch[lane + 32 * d] = cmul(v[d], cmul(comb_lane, comb_d[s * 32 + d]));
        } else {
            // ---- S(m) = sum_{n >= m} (p_n + p_{N-1-n}): thread u of the TS = 32 H threads
            //      scans n = 32 u + j in f32, thread totals are suffix-summed in f64
            const int u = tid - 32 * H;
            float qv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = 32 * u + j;
                qv[j] = (n < N) ? pw[pad32(n)] + pw[pad32(N - 1 - n)] : 0.f;
            }
            float r = 0.f;
#pragma unroll
            for (int j = 31; j >= 0; --j) {
                r += qv[j];
                qv[j] = r;
            }
            double incl = (double)r;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_down_sync(0xffffffffu, incl, o);
                if (lane + o < 32) incl += t;
            }
            // warp totals (lane 0 holds the inclusive suffix of its warp = the warp total)
            if (lane == 0) red[2 * R + (warp - H)] = incl;
            asm volatile("bar.sync 1, %0;" ::"r"(32 * H) : "memory");
            double later = 0.0;
            for (int w = warp - H + 1; w < H; ++w) later += red[2 * R + w];
            const float base = (float)(incl - (double)r + later);
#pragma unroll
            for (int j = 0; j < 32; ++j) pw[pad32(32 * u + j)] = qv[j] + base;
        }
        __syncthreads();  // (D) E'_s and S(m) complete

        // ---- U(m' + 1024 p) = sum_s E'_s(m') e^{2 pi i s p / H}
#pragma unroll
        for (int i = 0; i < kF / T; ++i) {
            const int m1 = tid + T * i;
            cpx<float> e[H];
#pragma unroll
            for (int s = 0; s < H; ++s) e[s] = scratch[s * kFPad + m1];
            if constexpr (H == 2) {
                ubuf[m1] = cadd(e[0], e[1]);
                ubuf[m1 + kF] = csub(e[0], e[1]);
            } else {
                dft4<+1>(e[0], e[1], e[2], e[3]);
#pragma unroll
                for (int pp = 0; pp < H; ++pp) ubuf[m1 + kF * pp] = e[pp];
            }
        }
        __syncthreads();  // (E) U complete

        // ---- unfold + combine: 2 Re R(m) = (A.x + B.x) + w.x (A.y + B.y) + w.y (A.x - B.x)
        //      with A = U(m), B = U(L - m), w = e^{2 pi i m / N2}; m = tid + T i
#pragma unroll
        for (int i = 0; i < G::NMAX / T; ++i) {
            const int m = tid + T * i;
            if (m < N) {
                const cpx<float> A = ubuf[m];
                const cpx<float> B = ubuf[(G::L - m) & (G::L - 1)];
                const cpx<float> w = cmul(unf_base, ct_w<+1, float>(i, 32));
                const float re2 = (A.x + B.x) + (w.x * (A.y + B.y) + w.y * (A.x - B.x));
                float val = fmaf(-re2, inv_n2, pw[pad32(m)]) * __frcp_rn((float)(N - m));
                if (m == 0) val = 0.f;
                if constexpr (kRing) acc[pad32(m)] += val;
                else out_q[(q - q0) * (int64_t)N + m] = val;
            }
        }
        if constexpr (kRing) {
            // item done: its per-lag sums leave (each thread owns the same m every sequence)
            if (nq_item != cur_item || qn < 0) {
                double* dst = ring.partial + cur_item * (int64_t)N;
#pragma unroll
                for (int i = 0; i < G::NMAX / T; ++i) {
                    const int m = tid + T * i;
                    if (m < N) {
                        dst[m] = (double)acc[pad32(m)];
                        acc[pad32(m)] = 0.f;
                    }
                }
            }
            cur_item = nq_item;
            cur_i = nq_i;
        }
        __syncthreads();  // (F) pw / U free for the next sequence
        q = qn;
    }
}

template <int R>
cudaError_t launch_long(const TemporalArgs& a, int64_t q0, int64_t q1, float* out_q, int num_sms,
                        cudaStream_t stream) {
    using G = LongGeom<R>;
    const bool ring = a.ring.nitems > 0;
    const size_t smem = G::total(ring);
    const int per_sm = R == 4 ? 2 : 1;
    const int64_t work = ring ? a.ring.nitems : q1 - q0;
    const int grid = (int)std::min<int64_t>(work, (int64_t)num_sms * per_sm);
    if (grid <= 0) return cudaSuccess;
    const bool full = a.N == G::NMAX;
    auto k = ring ? (full ? temporal_long_kernel<R, true, true> : temporal_long_kernel<R, true, false>)
                  : (full ? temporal_long_kernel<R, false, true> : temporal_long_kernel<R, false, false>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, G::T, smem, stream>>>(static_cast<const cpx<float>*>(a.spec), a.segs, a.N, q0, q1, out_q,
                                    a.ring);
    return cudaGetLastError();
}

// out_q [q][N] f32 (q in [q0, q1)) -> out[li * out_stride + dest(q)], 32 x 32 tiles
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

}  // namespace

cudaError_t launch_long2(const TemporalArgs& a, int64_t q0, int64_t q1, float* out_q, int num_sms,
                         cudaStream_t stream);

bool temporal_long_supported(int N, int N2, int scalar_bytes) {
    return scalar_bytes == 4 && (N2 == 4096 || N2 == 8192) && N > N2 / 4 && N <= N2 / 2 && N % 2 == 0;
}

int64_t temporal_long_chunk(int N) {
    // q-major staging block of the map mode: ~1 GiB of f32
    return std::max<int64_t>(1, (int64_t)(1u << 28) / N);
}

cudaError_t launch_temporal_long(const TemporalArgs& a, int num_sms, void* out_q,
                                 cudaStream_t stream) {
    if (reinterpret_cast<uintptr_t>(a.spec) % 16 != 0) return cudaErrorMisalignedAddress;
    if (!temporal_warp_segments_ok(a.segs, a.N)) return cudaErrorInvalidValue;
    const int R = a.N2 / kF;
    // the balanced two-group engine (temporal_long2.cu) unless DDM_LONG_V1 asks for this one
    static const bool v1 = std::getenv("DDM_LONG_V1") != nullptr;
    auto launch = [&](int64_t q0, int64_t q1) {
        if (!v1) return launch_long2(a, q0, q1, static_cast<float*>(out_q), num_sms, stream);
        return R == 4 ? launch_long<4>(a, q0, q1, static_cast<float*>(out_q), num_sms, stream)
                      : launch_long<8>(a, q0, q1, static_cast<float*>(out_q), num_sms, stream);
    };
    if (a.ring.nitems > 0) return launch(0, 0);
    const int64_t nq = a.layout.g_count, chunk = temporal_long_chunk(a.N);
    for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
        const int64_t q1 = std::min(nq, q0 + chunk);
        cudaError_t e = launch(q0, q1);
        if (e != cudaSuccess) return e;
        dim3 grid((unsigned)((q1 - q0 + 31) / 32), (unsigned)((a.N + 31) / 32));
        if (a.out_f64)
            transpose_lags_kernel<double><<<grid, dim3(32, 8), 0, stream>>>(
                static_cast<const float*>(out_q), a.N, q0, q1 - q0, a.lag_index,
                static_cast<double*>(a.out), a.out_stride, a.dest_of_slot);
        else
            transpose_lags_kernel<float><<<grid, dim3(32, 8), 0, stream>>>(
                static_cast<const float*>(out_q), a.N, q0, q1 - q0, a.lag_index,
                static_cast<float*>(a.out), a.out_stride, a.dest_of_slot);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace ddmk
