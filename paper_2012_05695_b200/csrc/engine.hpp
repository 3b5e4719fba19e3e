// Device orchestration of the WITH_FT hot path on one B200 (internal C++ API; the public
// boundaries are include/ddm_b200.h (C-ABI) and include/ddm/*.hpp (reference-mirroring C++).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ddm::b200 {

// CUDA failure (status 4 at the C-ABI).
class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

void check(cudaError_t e, const char* what);

// Owning device allocation.
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    void* ensure(size_t bytes);  // grows, never shrinks; contents not preserved
    void* get() const { return ptr_; }
    size_t size() const { return bytes_; }
    void release();

private:
    void* ptr_ = nullptr;
    size_t bytes_ = 0;
};

// Seconds of device time per phase, measured with CUDA events on the engine stream.
struct PhaseTimes {
    double spatial_ms = 0.0;
    double temporal_ms = 0.0;
    int spatial_launches = 0;
    int temporal_launches = 0;
    double d2h_ms = 0.0;      // host_out mode: first map chunk copy start -> last copy end
};

struct RunSpec {
    int W = 0, H = 0, N = 0;
    bool f64 = false;                 // working precision of the transforms
    int pixel_bytes = 2;              // 2 = u16, 1 = u8
    const void* d_frames = nullptr;   // device [N][H][W]
    std::vector<int64_t> lags;        // sorted, unique, within [0, N)
    std::vector<int64_t> flat;        // retained flat indices (row*(W/2+1)+col), ascending
    bool identity = true;             // flat[k] == k for every k (no cutoff)
    std::vector<std::pair<int64_t, int64_t>> groups;  // [begin, end) over the retained list
    // Output. Full-map mode: out[li * out_stride + flat[k]] (out_stride = plane), the
    // caller zero-fills positions outside the cutoff. Partial mode: per group a lag-major
    // [L][g_count] block (the reference PartialResult layout) handed to on_partial.
    void* d_out = nullptr;
    bool out_f64 = true;
    int64_t out_stride = 0;
    bool partial_mode = false;
    std::function<void(size_t group, const void* d_partial, int64_t g_count)> on_partial;
    // End-to-end streaming (optional):
    //   frames_ready: (frames resident, event) pairs in ascending frame order, recorded on the
    //   caller's upload stream; the spatial pass waits for the event covering each chunk.
    //   host_out: page-locked host map (same layout as d_out): the temporal pass runs in
    //   wave-vector chunks and each chunk's columns of every lag row are copied out on the
    //   engine's D2H stream while the next chunk computes (single-group identity map, warp
    //   temporal engine); the copies complete by finish_host_out().
    std::vector<std::pair<int, cudaEvent_t>> frames_ready;
    void* host_out = nullptr;
};

// Ring geometry of a retained wave-vector set for the azimuthal average
// (`analysis.cpp:61-97`): bin = llround(|q|) per retained slot.
struct RingPlan {
    int64_t nbins = 0;
    std::vector<int64_t> counts;       // per bin (geometry only)
    std::vector<int64_t> bin_off;      // CSR by bin, nbins + 1
    std::vector<int64_t> by_bin;       // retained slots sorted by bin, ascending within a bin
    std::vector<int64_t> flat_by_bin;  // the same as flat plane positions
    // fused-kernel work items (ring pieces of <= kItem slots, in by_bin order) and rings
    std::vector<int64_t> item_off;       // nitems + 1, offsets into by_bin
    std::vector<int64_t> ring_item_off;  // nrings + 1, offsets into the items
    std::vector<int64_t> ring_bin, ring_count;
    static constexpr int64_t kItem = 64;
};
RingPlan make_ring_plan(const std::vector<int64_t>& flat, int W, int H);

class Engine {
public:
    explicit Engine(int device);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    int device() const { return device_; }
    cudaStream_t stream() const { return stream_; }

    // Runs every group of `spec` on the engine stream (asynchronous w.r.t. the host unless
    // on_partial needs the data). Returns the number of spatial passes (= frames x groups).
    uint64_t run(const RunSpec& spec, PhaseTimes* times = nullptr);

    // Pinned host frames -> frame buffer in `chunks` pieces on the engine's upload stream;
    // returns (frames resident, event) pairs for RunSpec::frames_ready (valid until the next
    // call). The copies are ordered after nothing else; the caller holds the engine lock.
    std::vector<std::pair<int, cudaEvent_t>> upload_frames_async(void* d_frames, const void* host,
                                                                  int N, size_t frame_bytes, int chunks);

    // Waits for the map copies a host_out run() queued (no-op otherwise); adds their span to
    // times->d2h_ms. Returns whether run() streamed the map out.
    bool finish_host_out(PhaseTimes* times);
    // duration of the last upload_frames_async (waits for it)
    double upload_ms();

    // Batched SequenceEngine::with_ft: q sequences of n complex values, q-major on device
    // (working precision). d_out [q][n] f64; optional d_a / corr [q][n] f64 restored to the
    // original basis like `temporal.cpp:96-110`.
    void sequences(const void* d_seq, int64_t q, int64_t n, bool f64, double* d_out,
                   double* d_a_out, double* corr_out);

    // Batched spatial transform only (`compute_spectra`): frames [N][H][W] (pixel_bytes 2 u16,
    // 1 u8, 4 f32, 8 f64) -> d_out [N][H][W/2+1] complex in the working precision.
    void spectra(const void* d_frames, int pixel_bytes, int W, int H, int N, bool f64,
                 void* d_out);

    // One unnormalised complex 1D transform of d_data (len complex, working precision) in
    // place on the engine stream, sign -1 forward / +1 backward (`ddm::TemporalTransform`).
    void transform1d(void* d_data, int len, bool f64, int sign);

    // Sharded WITH_FT, step 1 on one rank: the rank's frame shard
    // d_frames [n][H][W] -> d_spec [H*(W/2+1)][n] (every wave vector, q-major, working
    // precision). Consecutive wave-vector ranges of d_spec are the all-to-all send blocks.
    // With `peers` (ranks > 0) the column pass stores straight into the owners' receive
    // buffers (fused NVLink corner turn; register-resident spatial kernels only) and d_spec
    // is unused.
    void spatial_shard(const void* d_frames, int pixel_bytes, int W, int H, int n, bool f64,
                       void* d_spec, PhaseTimes* times = nullptr,
                       const ddmk::PeerTable* peers = nullptr);

    // Sharded WITH_FT, step 2 on one rank: q_count full sequences whose frames arrive as
    // segments ([source][q][n_s] receive buffer, seg_frames[s] = n_s, sum = N) -> lag-major
    // out[li * out_stride + q] for the requested lags (sorted, unique, within [0, N)).
    void temporal_segments(const void* d_recv, int64_t q_count, const std::vector<int>& seg_frames,
                           bool f64, const std::vector<int64_t>& lags, void* d_out,
                           int64_t out_stride, bool out_f64, PhaseTimes* times = nullptr);

    // WITH_FT + azimuthal average in one pass (single group): d_means [lags][nbins] f64 on
    // device. Register engines: the ring sums are fused into the temporal kernel and no map
    // is materialised (returns true); otherwise the map goes through a device f64 buffer and
    // the ring reduction (returns false).
    bool run_rings(const RunSpec& spec, const RingPlan& rings, double* d_means,
                   PhaseTimes* times = nullptr);  // rings: from ring_plan()

    // WITHOUT_FT (and Direct, given f64) over every retained wave vector: spatial pass into the
    // wave-vector-major layout, then the pairwise kernel writing the f64 lag-major map
    // (spec.d_out, spec.out_stride, identity or flat positions). Single group.
    void run_pairwise(const RunSpec& spec, PhaseTimes* times = nullptr);

    // Pinned host staging buffer `slot` (0 or 1) of at least `bytes`, kept across runs.
    void* pinned(int slot, size_t bytes);

    // Device staging buffer for frames owned by the engine.
    void* frame_buffer(size_t bytes) { return frames_.ensure(bytes); }
    void* scratch(size_t bytes) { return user_scratch_.ensure(bytes); }
    // Named, growable device buffers owned by the engine (result maps, staging, ...).
    void* buffer(const std::string& name, size_t bytes);

    // Last spatial-chunk / tile geometry (for reports).
    int last_tile() const { return last_T_; }
    // Kernels the last run() / run_rings() selected, e.g.
    // "spatial=rows2<256>+cols2<512> temporal=warp<1024>:map" (tests assert on it, so a shape
    // cannot silently fall back to the generic engines)
    const std::string& last_engines() const { return last_engines_; }
    int last_chunk_frames() const { return last_F_; }

    std::mutex& mutex() { return mu_; }

    static Engine& instance(int device);

private:
    // Spatial passes over all frames of `sa` (frame chunks sized for L2), into sa.spec with
    // layout sa.layout, ordered on stream_.
    void spatial_pass(ddmk::SpatialArgs sa, bool f64, bool warp_s, PhaseTimes* times);
    ddmk::SpatialArgs spatial_args(const void* d_frames, int pixel_bytes, int W, int H, int N,
                                   bool f64);
    const int* upload_lags(const std::vector<int64_t>& lags, int N);
    const void* twiddles(int len, bool f64);           // exp(-2 pi i j / len), j < len
    const void* post_twiddles(int W, bool f64);        // exp(-2 pi i k / W), k <= W/2

    int device_;
    int num_sms_ = 148;
    cudaStream_t stream_ = nullptr;
    cudaEvent_t ev_[4] = {};
    DeviceBuffer frames_, spec_, mid_, lagidx_, slotmap_, dest_, partial_, user_scratch_;
    DeviceBuffer seq_aux_;
    std::map<std::pair<int, int>, std::unique_ptr<DeviceBuffer>> tw_;
    std::map<std::pair<int, int>, std::unique_ptr<DeviceBuffer>> post_;
    std::map<std::string, std::unique_ptr<DeviceBuffer>> named_;
    int last_T_ = 0, last_F_ = 0;
    std::string last_engines_;
    std::vector<int> lag_cache_;               // lag slots last uploaded to lagidx_
    std::vector<cudaEvent_t> timing_events_;   // reusable phase-timing events
    std::vector<cudaEvent_t> chunk_events_;    // row/column pass ordering across streams
    cudaStream_t cols_stream_ = nullptr;       // column passes (overlapped spatial step)
    cudaStream_t d2h_stream_ = nullptr;        // map chunks out (RunSpec::host_out)
    bool d2h_pending_ = false;
    cudaStream_t h2d_stream_ = nullptr;        // frame chunks in (upload_frames_async)
    std::vector<cudaEvent_t> h2d_events_;      // per frame chunk, [chunks] order, [chunks+1] start
    int h2d_chunks_ = 0;
    std::vector<cudaEvent_t> d2h_events_;      // [0] first copy start, [1] last copy end, [2..] chunks
    // spatial passes: wait on stream `st` until frames [0, frame_end) are resident
    const std::vector<std::pair<int, cudaEvent_t>>* frames_ready_ = nullptr;
    void wait_frames(cudaStream_t st, int frame_end);
    void* pinned_[2] = {nullptr, nullptr};
    size_t pinned_bytes_[2] = {0, 0};
    std::mutex mu_;
    // last ring plan and its device copy (geometry only, reused across runs)
    struct RingCache {
        int W = 0, H = 0;
        std::vector<int64_t> flat;
        const RingPlan* plan = nullptr;
        std::unique_ptr<RingPlan> own;
        const int64_t *order = nullptr, *item_off = nullptr, *ring_item_off = nullptr,
                      *ring_bin = nullptr, *ring_count = nullptr, *flat_by_bin = nullptr,
                      *bin_off = nullptr;
    } ring_cache_;

public:
    // ring plan of (flat, W, H), built once and cached with its device arrays
    const RingPlan& ring_plan(const std::vector<int64_t>& flat, int W, int H);
};

// Hardware limits of the one-CTA temporal kernel (longest supported sequence).
int64_t max_frames(bool f64);
// true when an f32 WITH_FT run of N frames uses a register temporal engine (warp or long),
// which computes d(q, m) in f32: its map is exactly representable as f32
bool f32_register_temporal(int N);

// Device reduction over n doubles: all finite?, max, min (for ResultArchive::validate).
void reduce_stats(const double* d, int64_t n, cudaStream_t stream, bool* finite, double* max_v,
                  double* min_v);
void reduce_stats(const float* d, int64_t n, cudaStream_t stream, bool* finite, double* max_v,
                  double* min_v);

// Deterministic ring average on device (`analysis.cpp:61-97`): values [L][plane] f64 device,
// bins [plane] int32 (-1 = not retained), order/offsets = retained positions sorted by bin
// (CSR), means [L][nbins] f64 device.
// Per-(lag, ring) sums of one wave-vector slice's map [n_lags][stride] (f32 or f64, device),
// CSR over the slice's columns in ring order: the sharded ring average.
void ring_sums(const void* d_values, bool f64, int64_t n_lags, int64_t stride, const int64_t* d_order,
               const int64_t* d_offsets, int64_t nbins, double* d_sums, cudaStream_t stream);
void radial_means(const double* d_values, int64_t n_lags, int64_t plane, const int64_t* d_order,
                  const int64_t* d_offsets, int64_t nbins, double* d_means, cudaStream_t stream);

}  // namespace ddm::b200
