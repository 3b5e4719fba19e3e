// Launch interface of the DDM device kernels (spatial r2c + corner turn, temporal engine).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "fft_core.cuh"

namespace ddmk {

// Twiddle table tw[j] = exp(-2 pi i j / len), j < len, in the working precision.
struct TwTable {
    int len = 0;
    const void* ptr = nullptr;  // cpx<S>*
};

// Spectra layout on device ("tile-major corner turn"): the retained wave vectors of one
// group, slots s in [0, g_count), are cut into tiles of T consecutive slots and stored
//     spec[((s / T) * N + n) * T + (s % T)]        (complex, working precision)
// so one tile is a contiguous N x T block: the spatial kernel writes T-wide runs per
// frame, the temporal kernel streams a whole tile as one contiguous block.
struct SpecLayout {
    int T = 4;
    int64_t g_begin = 0;   // first retained index of the group
    int64_t g_count = 0;   // slots in the group
    // q-major spectra (spec[slot * N + n], what the register spatial kernels write) read by the
    // generic temporal engine T sequences per CTA (f64 on register-friendly frame sizes)
    bool qmajor = false;
    int64_t tiles() const { return (g_count + T - 1) / T; }
};

// Fused corner turn over NVLink: the column pass stores wave vector k of the
// shard's frames straight into the receive buffer of the rank that owns k,
//     base[d] + (k - q_begin[d]) * N + n     for q_begin[d] <= k < q_begin[d + 1]
// (base[d] = that rank's receive buffer + this rank's segment offset, a peer pointer).
struct PeerTable {
    static constexpr int kMax = 8;
    int ranks = 0;                     // 0 = local spectra (spec / layout)
    int64_t q_begin[kMax + 1] = {};
    void* base[kMax] = {};
};

struct SpatialArgs {
    const void* frames = nullptr;  // [N][H][W] pixels
    int pixel_bytes = 2;           // 2 u16, 1 u8, 4 f32, 8 f64 (real-valued frames)
    int W = 0, H = 0, N = 0;
    int frame0 = 0, nframes = 0;   // chunk of frames to transform
    void* mid = nullptr;           // [chunk frame][W/2+1][H] complex scratch
    void* spec = nullptr;
    SpecLayout layout;
    const int* slot_of_flat = nullptr;  // nullable: flat (row*(W/2+1)+col) -> retained index
    PeerTable peers;                    // register-resident kernels only
    TwTable tw_row, tw_post, tw_col;    // row (W/2 or W), post (W), column (H)
};

// Sequences assembled from frame segments (the sharded corner turn): sequence
// q of a group of q_count is the concatenation over s < count of
//     spec + base[s] + q * n[s]      (n[s] complex values each; base[s] = q_count * off[s])
// i.e. the receive buffer of the all-to-all, [source][q][frames of that source].
struct SegTable {
    static constexpr int kMax = 8;
    int count = 0;                     // 0 = one contiguous segment of N (layout T = 1)
    int n[kMax] = {};
    int off[kMax] = {};                // frame offset of segment s within the sequence
    int64_t base[kMax] = {};           // complex offset of segment s's [q][n[s]] block
};

// Fused azimuthal (q-ring) average (`analysis.cpp:61-97`) in the warp engine. The retained
// sequence slots, sorted by ring (bin) and ascending within a ring, are `order`; they are cut
// into work items of at most a few dozen slots that never straddle a ring:
// item i = order[item_off[i] .. item_off[i+1]). The temporal kernel writes, per item, the f64
// sum over its slots of d(q, m) for every m (partial[i][m]); ring_means_kernel then adds the
// items of each ring in order (deterministic) into means[li * nbins + bin] / count.
struct RingArgs {
    int64_t nitems = 0;                 // 0 = map mode
    const int64_t* order = nullptr;
    const int64_t* item_off = nullptr;  // nitems + 1
    double* partial = nullptr;          // [nitems][N]
};

struct TemporalArgs {
    const void* spec = nullptr;
    SegTable segs;                     // warp engine only (the generic engine repacks first)
    int N = 0, N2 = 0;
    SpecLayout layout;
    TwTable tw;                        // length N2
    TwTable tw_half;                   // length N2 / 2
    const int* lag_index = nullptr;    // [N] -> output lag slot or -1
    void* out = nullptr;               // out[li * out_stride + dest(s)]
    int out_f64 = 1;
    int64_t out_stride = 0;
    const int64_t* dest_of_slot = nullptr;  // nullable: slot -> destination column
    // optional diagnostics for the batched SequenceEngine API: corr in the shifted basis,
    // f64 [slot][N], and the per-slot mean (complex f64) used for the restore
    double* corr_out = nullptr;
    double* mean_out = nullptr;
    RingArgs ring;                     // warp engine only
};

template <typename S>
cudaError_t launch_spatial(const SpatialArgs& a, cudaStream_t stream);

template <typename S>
cudaError_t launch_temporal(const TemporalArgs& a, cudaStream_t stream);

// Ring means from the per-item partial sums: ring r = items [ring_item_off[r],
// ring_item_off[r+1]) with ring_count[r] slots, landing in bin ring_bin[r].
cudaError_t launch_ring_means(const double* partial, int N, const int* lag_index,
                              const int64_t* ring_item_off, const int64_t* ring_bin,
                              const int64_t* ring_count, int64_t nrings, double* means,
                              int64_t nbins, cudaStream_t stream);

// WITHOUT_FT (`pairwise.cpp:11-72`): spec wave-vector-major [q][N] in the working precision,
// lags ascending (n_lags entries, 0 allowed), out[li * out_stride + dest(q)] f64.
template <typename S>
// lag0 >= 0: the lags are the contiguous range [lag0, lag0 + n_lags) (the common "all lags"
// request), served by the register-windowed kernel; lag0 < 0: any ascending list
cudaError_t launch_pairwise(const void* spec, int N, int64_t nq, const int* lags, int n_lags,
                            double* out, int64_t out_stride, const int64_t* dest_of_slot,
                            int num_sms, cudaStream_t stream, int lag0 = -1);

// Synthetic frames (csrc/synth.cu): d_pos [frames][particles][2] particle positions ->
// d_out [frames][H][W] u16, the reference's `render_frame` arithmetic (`synth.cpp:42-79`).
cudaError_t launch_render_frames(const double* d_pos, int particles, int W, int H, int frames,
                                 double psf_sigma, double amplitude, double background,
                                 uint16_t* d_out, cudaStream_t stream);

// frame-major spectra [N][plane] -> wave-vector-major [count][N] at positions flat[k]
template <typename S>
cudaError_t launch_gather_sequences(const void* frames, int N, int64_t plane, const int64_t* flat,
                                    int64_t count, void* seq, cudaStream_t stream);

// Relaxation fits, one warp per ring (`analysis.cpp:108-224`): means [n_lags][nbins] f64;
// flag 0 ok, 1 degenerate, 2 no_converge, -1 not fitted.
cudaError_t launch_fit_rings(const double* means, const int64_t* lags, int n_lags,
                             const int64_t* counts, int64_t nbins, double dt, double* amp,
                             double* base, double* tau, double* resid, int* flag,
                             cudaStream_t stream);

// Segmented sequences (SegTable over q_count sequences) -> the engine's tile-major layout T.
template <typename S>
cudaError_t launch_repack_segments(const void* recv, int64_t q_count, const SegTable& segs, int N,
                                   int T, void* spec, cudaStream_t stream);

// Warp-per-sequence temporal engine (temporal_warp.cu): f32, N2 == 2048, wave-vector-major
// spectra (layout T = 1).
bool temporal_warp_supported(int N, int N2, int scalar_bytes);
size_t temporal_warp_smem();
bool temporal_warp_segments_ok(const SegTable& segs, int N);
cudaError_t launch_temporal_warp(const TemporalArgs& a, int num_sms, cudaStream_t stream);

// CTA-per-sequence temporal engine (temporal_long.cu): f32, N2 in {4096, 8192}, layout T = 1
// (or segments), map mode through a q-major staging block `out_q` of temporal_long_chunk(N)
// sequences x N f32, or ring mode (RingArgs).
bool temporal_long_supported(int N, int N2, int scalar_bytes);
int64_t temporal_long_chunk(int N);
cudaError_t launch_temporal_long(const TemporalArgs& a, int num_sms, void* out_q, cudaStream_t stream);

// Register-resident spatial kernels (spatial_warp.cu): f32, power-of-two W/2 and H in
// [16, 1024], u16/u8 frames, wave-vector-major output (layout T = 1).
bool spatial_warp_supported(int W, int H, int pixel_bytes, int scalar_bytes);
// f64 warp temporal engine (temporal_warp64.cu): N2 = 2048, q-major spectra, f64 map or
// partial, no ring / diagnostics / segments
bool temporal_warp64_supported(int N, int N2);
cudaError_t launch_temporal_warp64(const TemporalArgs& a, int num_sms, cudaStream_t stream);
// the same frame sizes with f64 arithmetic (launch_spatial_warp<double>; q-major output)
bool spatial_warp_f64_supported(int W, int H, int pixel_bytes);

// H = 2048 f32 column pass with two warps per column (spatial_warp.cu; DDM_COLS2_PAIR=0 off)
bool spatial_cols_pair();
// frames one column-pass CTA transforms together (the run length of its corner-turn stores)
int spatial_warp_col_frames(int H);
// parts: 1 = row pass (frames -> mid), 2 = column pass (mid -> spectra), 3 = both
template <typename S>
cudaError_t launch_spatial_warp(const SpatialArgs& a, cudaStream_t stream, int parts = 3);


// Shared memory / tile geometry chosen for the temporal kernel; the spectra layout T must
// match it. Returns 0 when the sequence length is beyond what one CTA can hold.
int temporal_tile(int N, int N2, int scalar_bytes);
size_t temporal_smem_bytes(int N, int N2, int T, int scalar_bytes);
int temporal_threads(int N2, int T, int scalar_bytes);

// One unnormalised complex transform of `len` points in place (fft1d.cu; sign -1 forward,
// +1 backward); scratch holds len complex, tw = exp(-2 pi i j / len) in the same precision.
cudaError_t launch_fft1d(void* data, void* scratch, int len, bool f64, int sign, const void* tw,
                         cudaStream_t stream);

}  // namespace ddmk
