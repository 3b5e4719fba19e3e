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
// Working precision: the FFTs, P = |X|^2 and |t|^2 are f32 as in the reference's f32
// engine (`temporal.cpp:56-64` computes in S); the mean is a pairwise f32 sum (it only
// conditions the subtraction: d is offset invariant, `temporal.hpp:258-262`); S(m) is summed
// in f32 within each lane's run of 32 terms with the 32 lane totals carried in f64; the
// combination is one f32 FMA. The reference keeps power, d_a and the combination in f64
// (`temporal.cpp:24-41,114-129`); here their f32 rounding (~1e-7 relative) stays below the
// f32 transform error both engines share, measured at every BASELINE shape against the
// reference's own f32 maps (relative L2 1.5e-6 at C2, tests/test_gpu_shapes.py up to C4).
//
// Why one CTA-wide barrier per tile (all 12 warps in phase): splitting the CTA into three
// 4-warp groups on named barriers (measured, r02i) cost 7%: the groups' 16-byte row pieces
// were written at different times, so L2 evicted half-written sectors (ECC read-modify-write:
// +376 MB DRAM reads, +318 MB writes per launch), and warps running different parts of the
// 117 KB unrolled kernel raised instruction-fetch stalls from 0.17 to 0.46 per issue.
//
// Data movement per sequence: one TMA bulk copy (cp.async.bulk, 8 KB) into the warp's stage.
// The first pass shifts the sequence in registers; the odd transform re-reads and re-shifts
// it and leaves |t|^2 in its place for the averages term; once that has been read the next sequence's copy
// is issued, so it lands during the S(m) scan, the unfold and the tile store (an L2 prefetch
// of the same bytes goes out one sequence earlier). Three four-step FFTs (warp_fft.cuh, one
// shared-memory exchange each); the exchange buffer then holds S(m) and d(m); the
// unfold reads U(L-m) from the mirrored lane with shuffles; a CTA of 12 warps stores 12
// consecutive wave vectors per lag row.
//
// Occupancy: 12 warps per SM at <= 168 registers (218 KB of shared memory). The per-lane
// unfold twiddles W_N2^{-(lane + 32 d)} are loop invariants the compiler would otherwise
// keep in 64 registers for the kernel's life; they are formed per sequence from an opaque
// copy of the lane base.
// K3 runs the packed f32x2 codelets (fft_core.cuh: FADD2/FMUL2/FFMA2, 20% fewer issued
// instructions). They first measured 1.8% slower (0.902 vs 0.886 ms at C2): the register
// pairs pushed K3 past its 168-register cap (12 warps per SM) and the spill reloads sat on the
// tile loop. With the tile store's addressing recomputed per tile (the thread index re-read
// in temporal_warp_kernel.cuh, so the 64-bit row offsets are not held through the
// transforms) only the copy phase bit spills and K3 runs 0.867 ms against 0.878 ms scalar
// (three interleaved A/B rounds, tools/gpu_ab3.sh, profiles/r02z_f32x2_ab.txt). The scalar
// codelets with that change measured 0.885 ms (the hoisted addressing suits them).
// Sums stay scalar (FADD; products packed), as in the row/column passes: 0.865 vs 0.867 ms.
// DDM_F32X2_TW=0 selects the scalar codelets for A/B builds. The ring mode (8 warps per SM)
// is in temporal_warp_ring.cu.
// The kernel template and its launcher live in temporal_warp_kernel.cuh.
#ifndef DDM_F32X2
#ifdef DDM_F32X2_TW
#define DDM_F32X2 DDM_F32X2_TW
#else
#define DDM_F32X2 1
#endif
#endif
#ifndef DDM_F32X2_ADD
#define DDM_F32X2_ADD 0
#endif
#include "temporal_warp_kernel.cuh"

namespace ddmk {

cudaError_t launch_temporal_warp_ring(const TemporalArgs& a, int num_sms, cudaStream_t stream);

bool temporal_warp_supported(int N, int N2, int scalar_bytes) {
    // bulk copies need 16-byte sizes: even N
    return scalar_bytes == 4 && N2 == kN2 && N > kL / 2 && N <= kL && N % 2 == 0;
}


size_t temporal_warp_smem() {
    return sizeof(WarpSmem) * kTW + 2 * kXS * sizeof(cpx<float>) + kL * sizeof(float);
}

bool temporal_warp_segments_ok(const SegTable& segs, int N) {
    if (segs.count < 0 || segs.count > SegTable::kMax) return false;
    int total = 0;
    for (int s = 0; s < segs.count; ++s) {
        // bulk copies: 16-byte sizes, 16-byte aligned source and stage addresses
        if (segs.n[s] < 1 || segs.n[s] % 2 || segs.off[s] != total || segs.base[s] % 2) return false;
        total += segs.n[s];
    }
    return segs.count == 0 || total == N;
}

cudaError_t launch_temporal_warp(const TemporalArgs& a, int num_sms, cudaStream_t stream) {
    if (reinterpret_cast<uintptr_t>(a.spec) % 16 != 0) return cudaErrorMisalignedAddress;
    if (!temporal_warp_segments_ok(a.segs, a.N)) return cudaErrorInvalidValue;
    if (a.ring.nitems > 0) return launch_temporal_warp_ring(a, num_sms, stream);
    if (a.corr_out || a.mean_out) {
        if (!a.out_f64) return cudaErrorInvalidValue;
        return launch_w<double, true, false>(a, num_sms, stream);
    }
    return a.out_f64 ? launch_w<double, false, false>(a, num_sms, stream)
                     : launch_w<float, false, false>(a, num_sms, stream);
}

namespace {

// one thread per (lag, ring): items of the ring added in order
__global__ void ring_means_kernel(const double* __restrict__ partial, int N,
                                  const int* __restrict__ lag_index,
                                  const int64_t* __restrict__ ring_item_off,
                                  const int64_t* __restrict__ ring_bin,
                                  const int64_t* __restrict__ ring_count, int64_t nrings,
                                  double* __restrict__ means, int64_t nbins) {
    const int64_t total = nrings * (int64_t)N;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = x / N;
        const int m = (int)(x - r * N);
        const int li = lag_index ? lag_index[m] : m;
        if (li < 0) continue;
        double sum = 0.0;
        for (int64_t it = ring_item_off[r]; it < ring_item_off[r + 1]; ++it) sum += partial[it * N + m];
        means[(int64_t)li * nbins + ring_bin[r]] = (m == 0) ? 0.0 : sum / (double)ring_count[r];
    }
}

}  // namespace

cudaError_t launch_ring_means(const double* partial, int N, const int* lag_index,
                              const int64_t* ring_item_off, const int64_t* ring_bin,
                              const int64_t* ring_count, int64_t nrings, double* means,
                              int64_t nbins, cudaStream_t stream) {
    const int64_t total = nrings * (int64_t)N;
    const int blocks = (int)std::min<int64_t>(148 * 8, (total + 255) / 256);
    if (blocks == 0) return cudaSuccess;
    ring_means_kernel<<<blocks, 256, 0, stream>>>(partial, N, lag_index, ring_item_off, ring_bin,
                                                  ring_count, nrings, means, nbins);
    return cudaGetLastError();
}

}  // namespace ddmk
