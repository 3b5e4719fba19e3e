// The warp temporal engine K3 (`temporal_warp_kernel`) and its launcher, shared by
// temporal_warp.cu (map mode and the SequenceEngine diagnostics, scalar f32 codelets) and
// temporal_warp_ring.cu (fused ring average, packed f32x2 codelets): the including
// translation unit chooses DDM_F32X2 before including it. See temporal_warp.cu for the
// algorithm.
#pragma once

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "temporal_common.cuh"
#include "warp_fft.cuh"

namespace ddmk {

namespace {

using namespace tc;

constexpr bool kBackoff = true;       // sleep between polls of the sequence copy
constexpr int kL = 1024;              // half padded length
constexpr int kN2 = 2048;
constexpr int kPad = kL + kL / 32;    // slots per buffer (FFT scratch pitch 33 x 32)

__device__ __forceinline__ int padded(int n) { return n + (n >> 5); }

// Per-warp shared memory (16.5 KB):
//   stage   : TMA target of the sequence (dense [0, N) complex), read by the even and odd
//             transforms and the averages term
//   scratch : exchange buffer of the three FFTs; then, as f32 at padded(n): |t|^2, S(m) in
//             place, d(m) in place (the tile store's source in map mode)
struct WarpSmem {
    cpx<float> stage[kL];
    cpx<float> scratch[kXS];     // FFT exchange (pitch kXP)
    unsigned long long bar;
    unsigned long long pad_;
};

// kDiag: the batched SequenceEngine API's extra outputs (corr, mean); compiled out of the
// run path so none of its predicated f64 work is issued there.
// kRing: fused azimuthal average (RingArgs) instead of the map.
template <typename OutT, bool FULL, bool kDiag, bool kRing, int kWarps>
__global__ void __launch_bounds__(32 * kWarps, 1)
temporal_warp_kernel(const cpx<float>* __restrict__ spec, const __grid_constant__ SegTable segs, int N_rt, int64_t nq,
                     const int* __restrict__ lag_index, OutT* __restrict__ out,
                     int64_t out_stride, const int64_t* __restrict__ dest_of_slot,
                     double* __restrict__ corr_out, double* __restrict__ mean_out,
                     const __grid_constant__ RingArgs ring) {
    // FULL: N == L, every bound below folds at compile time
    const int N = FULL ? kL : N_rt;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WarpSmem* ws = reinterpret_cast<WarpSmem*>(smem_raw);
    cpx<float>* tw_even = reinterpret_cast<cpx<float>*>(ws + kWarps);  // [a][c] W_1024^{a c}
    cpx<float>* tw_odd = tw_even + kXS;                                  // [c][a] W_2048^{a (2c+1)}
    float* rcp = reinterpret_cast<float*>(tw_odd + kXS);                 // 1 / (N - m)
    float* acc_base = rcp + kL;                                          // kRing: [warp][kPad]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& my = ws[warp];

    for (int m = threadIdx.x; m < N; m += blockDim.x) rcp[m] = (float)(1.0 / (double)(N - m));
    if (lane == 0) {
        mbar_init(&my.bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fill_fft1024_tables(tw_even, tw_odd, threadIdx.x, blockDim.x);
    cpx<float> base_unf;  // W_N2^{-lane}
    {
        double sn, cs;
        sincospi(2.0 * (double)lane / kN2, &sn, &cs);
        base_unf = {(float)cs, (float)sn};
    }
    const float inv_nf = 1.0f / (float)N;
    // 16-byte vector stores of whole tiles: aligned base and row stride (f32 map, or the f64
    // map of the reference's ResultMap)
    const bool vec_store = ((uintptr_t)out & 15) == 0 && (out_stride % (16 / (int)sizeof(OutT))) == 0;
    __syncthreads();

    const int64_t ntiles = (nq + kWarps - 1) / kWarps;
    const uint32_t bytes = (uint32_t)N * 8u;
    auto prefetch_q = [&](int64_t q) {   // q < 0: nothing to fetch
        if (lane == 0 && q >= 0) {
            if (segs.count == 0) {
                bulk_load(my.stage, spec + q * (int64_t)N, bytes, &my.bar);
            } else {
                // sharded corner turn: one bulk copy per source segment, one transaction count
                fence_expect(&my.bar, bytes);
                for (int s = 0; s < segs.count; ++s)
                    bulk_copy(my.stage + segs.off[s], spec + segs.base[s] + q * (int64_t)segs.n[s],
                              (uint32_t)segs.n[s] * 8u, &my.bar);
            }
        }
    };

    // L2 prefetch of a sequence whose bulk copy is issued one sequence later
    auto prefetch_l2 = [&](int64_t q) {
        if (lane == 0 && q >= 0) {
            if (segs.count == 0) {
                l2_prefetch(spec + q * (int64_t)N, bytes);
            } else {
                for (int s = 0; s < segs.count; ++s)
                    l2_prefetch(spec + segs.base[s] + q * (int64_t)segs.n[s], (uint32_t)segs.n[s] * 8u);
            }
        }
    };

    auto tile_q = [&](int64_t tile) -> int64_t {
        const int64_t q = tile * kWarps + warp;
        return (tile < ntiles && q < nq) ? q : -1;
    };

    uint32_t phase = 0u;
    float* sw = reinterpret_cast<float*>(my.scratch);   // the exchange buffer as f32 work space
    // One sequence: wait for its copy, transform, call after_stage() once the stage has been
    // read for the last time (to start the next copy), emit(m, d(m)) for every m < N.
    auto process = [&](int64_t q, bool live, auto&& after_stage, auto&& emit) {
        if (live) {
            if (kBackoff) mbar_wait_backoff(&my.bar, phase);
            else mbar_wait(&my.bar, phase);
            phase ^= 1u;
        }

        // ---- load (lane a holds s[a + 32 b]), mean by a pairwise f32 sum, shift
        cpx<float> v[32];
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            const int n = lane + 32 * b;
            v[b] = (live && n < N) ? my.stage[n] : cpx<float>{0.f, 0.f};
        }
        float mx, my_;
        {
            cpx<float> acc[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] = cadd(v[i], v[i + 16]);
#pragma unroll
            for (int w = 8; w > 0; w >>= 1)
#pragma unroll
                for (int i = 0; i < w; ++i) acc[i] = cadd(acc[i], acc[i + w]);
            mx = acc[0].x;
            my_ = acc[0].y;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mx += __shfl_xor_sync(0xffffffffu, mx, o);
                my_ += __shfl_xor_sync(0xffffffffu, my_, o);
            }
            mx *= inv_nf;
            my_ *= inv_nf;
        }
        // shift in registers; the odd transform re-reads the raw sequence and shifts it again
        // (writing the shifted sequence back cost 64 shared-memory wavefronts per sequence,
        // K3's busiest unit: 0.887 vs 0.880 ms measured, profiles/r02z_f32x2_ab.txt)
#pragma unroll
        for (int b = 0; b < 32; ++b)
            if (lane + 32 * b < N) v[b] = csub(v[b], cpx<float>{mx, my_});

        // map mode: the previous tile's d values sit in every warp's exchange buffer until
        // the CTA has stored them; the store overlaps this sequence's copy wait and mean
        if constexpr (!kRing) __syncthreads();

        // ---- even outputs of the zero-padded FFT_2048: FFT_1024(t); P in f32 (`temporal.cpp:60-64`),
        //      kept in registers while the odd half is transformed
        float pe[32];
        fft1024<-1, false>(v, my.scratch, lane, tw_even);
#pragma unroll
        for (int d = 0; d < 32; ++d) pe[d] = v[d].x * v[d].x + v[d].y * v[d].y;

        // ---- odd outputs: t again from the stage (shifted again); its last read, so |t|^2 (f32, of the
        //      shifted sequence) replaces it there for the averages term
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            const int n = lane + 32 * b;
            v[b] = (n < N) ? csub(my.stage[n], cpx<float>{mx, my_}) : cpx<float>{0.f, 0.f};
        }
        __syncwarp();
        float* pw = reinterpret_cast<float*>(my.stage);   // |t|^2 at padded(n)
#pragma unroll
        for (int b = 0; b < 32; ++b) pw[padded(lane + 32 * b)] = v[b].x * v[b].x + v[b].y * v[b].y;
        fft1024<-1, true>(v, my.scratch, lane, tw_odd);
#pragma unroll
        for (int d = 0; d < 32; ++d) v[d] = {pe[d], v[d].x * v[d].x + v[d].y * v[d].y};

        // ---- half-length inverse: lane c holds U[c + 32 d] in v[d]
        fft1024<+1, false>(v, my.scratch, lane, tw_even);

        // ---- S(m) = sum_{n >= m} (p_n + p_{N-1-n}) = (N - m) d_a(m)  (`temporal.cpp:19-42`):
        //      lane a scans n = 32 a + j in f32, lane totals are suffix-summed in f64
        float* sarea = sw;  // S(m) replaces |t|^2
        {
            float qv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = 32 * lane + j;
                qv[j] = (n < N) ? pw[padded(n)] + pw[padded(N - 1 - n)] : 0.f;
            }
            // the stage has been read for the last time: start the next sequence's copy
            __syncwarp();
            after_stage();
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
            const float base = (float)(incl - (double)r);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 32; ++j) sarea[padded(32 * lane + j)] = qv[j] + base;
            __syncwarp();
        }

        // ---- unfold + combine, two lags per step: for m = c + 32 d (d < 16), U[L - m] sits in
        //      lane (32 - c) mod 32, register 31 - d (lane 0: its own register (32 - d) mod 32), and
        //      with S1 = A.x + B.x, P = w.x (A.y + B.y) + w.y (A.x - B.x), w = W_N2^{-m}:
        //      2 Re R(m) = S1 + P and 2 Re R(L - m) = S1 - P (w(L - m) = -conj w(m), A and B
        //      swap). L - m = (32 - c) + 32 (31 - d) is the mirrored lane's upper half (lane 0:
        //      its own, lag 512 separately), so every lag is produced once; S(m) and 1/(N - m)
        //      come from shared memory. d(m) = (S(m) - 2 corr(m)) / (N - m), 2 corr = 2 Re R / N2.
        const int src = (32 - lane) & 31;
        // opaque per-sequence copy of the lane base: stops the compiler from hoisting the 16
        // products base * W_N2^{-32 d} out of the sequence loop
        cpx<float> bu;
        asm volatile("mov.b32 %0, %1;" : "=f"(bu.x) : "f"(base_unf.x));
        asm volatile("mov.b32 %0, %1;" : "=f"(bu.y) : "f"(base_unf.y));
        constexpr float inv_n2 = 1.0f / (float)kN2;
        auto finish = [&](int m, float re2) {
            if (m < N) {
                const float val = fmaf(-re2, inv_n2, sarea[padded(m)]) * rcp[m];
                emit(m, (m == 0) ? 0.f : val);
                if constexpr (kDiag)
                    if (corr_out && live) corr_out[q * N + m] = 0.5 * (double)re2 / (double)kN2;
            }
        };
#pragma unroll
        for (int d = 0; d < 16; ++d) {
            const int m = lane + 32 * d;
            cpx<float> Bc;
            Bc.x = __shfl_sync(0xffffffffu, v[31 - d].x, src);
            Bc.y = __shfl_sync(0xffffffffu, v[31 - d].y, src);
            if (lane == 0) Bc = v[(32 - d) & 31];
            const cpx<float> A = v[d];
            const cpx<float> w = cmul(bu, ct_w<+1, float>(32 * d, kN2));  // exp(+2 pi i m / N2)
            const float S1 = A.x + Bc.x;
            const float P = w.x * (A.y + Bc.y) + w.y * (A.x - Bc.x);
            finish(m, S1 + P);
            finish(kL - m, S1 - P);   // kL - m = kL (d = 0, lane 0) is never < N
        }
        if (lane == 0) {   // lag 512 = L / 2, its own mirror: U[512] in register 16
            const cpx<float> A = v[16];
            const cpx<float> w = ct_w<+1, float>(512, kN2);
            finish(512, (A.x + A.x) + (w.x * (A.y + A.y)));
        }
        if (kDiag && mean_out && live && lane == 0) {
            mean_out[2 * q] = (double)mx;
            mean_out[2 * q + 1] = (double)my_;
        }
    };

    if constexpr (kRing) {
        // ---- fused azimuthal average: work items are ring pieces; warp w owns slots
        //      w, w + kWarps, ... of an item, warps are combined in order in f64
        float* acc = acc_base + warp * kPad;
        auto first_from = [&](int64_t it) -> int64_t {   // this warp's first slot at item >= it
            for (; it < ring.nitems; it += gridDim.x) {
                const int64_t i = ring.item_off[it] + warp;
                if (i < ring.item_off[it + 1]) return i;
            }
            return -1;
        };
        int64_t pi = first_from(blockIdx.x);   // the next slot this warp fetches
        prefetch_q(pi >= 0 ? ring.order[pi] : -1);
        for (int64_t it = blockIdx.x; it < ring.nitems; it += gridDim.x) {
            const int64_t beg = ring.item_off[it], end = ring.item_off[it + 1];
#pragma unroll
            for (int d = 0; d < 32; ++d) acc[padded(lane + 32 * d)] = 0.f;
            for (int64_t i = beg + warp; i < end; i += kWarps) {
                pi = (i + kWarps < end) ? i + kWarps : first_from(it + gridDim.x);
                prefetch_l2(pi >= 0 ? ring.order[pi] : -1);
                process(ring.order[i], true, [&] { prefetch_q(pi >= 0 ? ring.order[pi] : -1); },
                        [&](int m, float val) { acc[padded(m)] += val; });
            }
            __syncthreads();
            double* dst = ring.partial + it * (int64_t)N;
            for (int m = threadIdx.x; m < N; m += blockDim.x) {
                double sum = 0.0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) sum += (double)acc_base[w * kPad + padded(m)];
                dst[m] = sum;
            }
            __syncthreads();
        }
        return;
    }

    prefetch_q(tile_q(blockIdx.x));
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t q = tile * kWarps + warp;
        const bool live = q < nq;
        prefetch_l2(tile_q(tile + gridDim.x));
        process(q, live, [&] { prefetch_q(tile_q(tile + gridDim.x)); },
                [&](int m, float val) { sw[padded(m)] = val; });   // S(m) was read into sv

        // ---- tile store: lag rows of kWarps consecutive wave vectors
        __syncthreads();
        auto dval = [&](int j, int m) -> float {
            return reinterpret_cast<const float*>(ws[j].scratch)[padded(m)];
        };
        const int64_t q0 = tile * kWarps;
        // the thread index re-read per tile: keeps the compiler from hoisting the store
        // addressing (64-bit row offsets and strides) out of the tile loop, where it would
        // hold registers through the transforms
        unsigned tid;
        asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
        if (!lag_index && !dest_of_slot && q0 + kWarps <= nq) {
            OutT* dst = out + (int64_t)tid * out_stride + q0;
            const int64_t step = (int64_t)blockDim.x * out_stride;
            if (vec_store) {
                // TPR threads cover one lag row's run of kWarps values (48 B f32 / 96 B f64 at
                // 12 warps), each storing VPT consecutive wave vectors as one 16-byte vector:
                // a store instruction writes whole rows instead of one value per row
                constexpr int VPT = 16 / (int)sizeof(OutT);
                constexpr int TPR = kWarps / VPT;
                static_assert(kWarps % VPT == 0, "whole 16-byte vectors per row");
                const int k = tid % TPR;
                const int rows = blockDim.x / TPR;
                OutT* pdst = out + (int64_t)(tid / TPR) * out_stride + q0 + VPT * k;
                const int64_t pstep = (int64_t)rows * out_stride;
#pragma unroll 4
                for (int m = tid / TPR; m < N; m += rows, pdst += pstep) {
                    if constexpr (VPT == 4) {
                        float4 v4;
                        v4.x = dval(4 * k + 0, m);
                        v4.y = dval(4 * k + 1, m);
                        v4.z = dval(4 * k + 2, m);
                        v4.w = dval(4 * k + 3, m);
                        *reinterpret_cast<float4*>(pdst) = v4;
                    } else {
                        double2 v2;
                        v2.x = (double)dval(2 * k, m);
                        v2.y = (double)dval(2 * k + 1, m);
                        *reinterpret_cast<double2*>(pdst) = v2;
                    }
                }
            } else {
                for (int m = tid; m < N; m += blockDim.x, dst += step) {
#pragma unroll
                    for (int j = 0; j < kWarps; ++j)
                        dst[j] = (OutT)dval(j, m);
                }
            }
        } else {
            for (int idx = tid; idx < N * kWarps; idx += blockDim.x) {
                const int m = idx / kWarps, j = idx - m * kWarps;
                if (q0 + j >= nq) continue;
                const int li = lag_index ? lag_index[m] : m;
                if (li < 0) continue;
                const int64_t dst = dest_of_slot ? dest_of_slot[q0 + j] : q0 + j;
                out[(int64_t)li * out_stride + dst] = (OutT)dval(j, m);
            }
        }
        // no barrier here: the next sequence's copy wait and mean run while the stores drain;
        // the exchange buffers are rewritten only after the barrier inside process()
    }
}


// Warps (wave vectors) per CTA, one CTA per SM: 12 in map mode (168 registers without
// spills, the unfold twiddles are not hoisted; 218 KB of shared memory), 8 in ring mode (its
// per-warp ring accumulators need 4 KB more per warp).
#ifndef DDM_K3_WARPS
#define DDM_K3_WARPS 12
#endif
constexpr int kTW = DDM_K3_WARPS;
constexpr int kTWRing = 8;

template <typename OutT, bool kDiag, bool kRing>
cudaError_t launch_w(const TemporalArgs& a, int num_sms, cudaStream_t stream) {
    constexpr int W = kRing ? kTWRing : kTW;
    const size_t smem = sizeof(WarpSmem) * W + 2 * kXS * sizeof(cpx<float>) + kL * sizeof(float) +
                        (kRing ? (size_t)W * kPad * sizeof(float) : 0);
    const int64_t work = kRing ? a.ring.nitems : (a.layout.g_count + W - 1) / W;
    const int grid = (int)std::min<int64_t>(work, (int64_t)num_sms);
    if (grid == 0) return cudaSuccess;
    const cpx<float>* spec = static_cast<const cpx<float>*>(a.spec);
    auto k = a.N == kL ? temporal_warp_kernel<OutT, true, kDiag, kRing, W>
                       : temporal_warp_kernel<OutT, false, kDiag, kRing, W>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 32 * W, smem, stream>>>(spec, a.segs, a.N, a.layout.g_count, a.lag_index,
                                      static_cast<OutT*>(a.out), a.out_stride, a.dest_of_slot,
                                      a.corr_out, a.mean_out, a.ring);
    return cudaGetLastError();
}

}  // namespace
}  // namespace ddmk
