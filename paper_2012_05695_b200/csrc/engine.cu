// Device orchestration of the WITH_FT hot path (see engine.hpp).
//
// One group (the reference's out-of-core wave-vector slice, `scheduler.cpp:89-171`) is
//   spatial passes over frame chunks (rows -> L2-resident mid -> columns + corner turn)
//   -> one temporal launch over all tiles of the group -> lag-major output.
// Groups exist for drop-in semantics (counters, partial files); with the default budget a
// run is a single group and never leaves the device between the two steps.
#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"

namespace ddm::b200 {

using ddmk::cpx;

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

DeviceBuffer::~DeviceBuffer() { release(); }

void DeviceBuffer::release() {
    if (ptr_) cudaFree(ptr_);
    ptr_ = nullptr;
    bytes_ = 0;
}

void* DeviceBuffer::ensure(size_t bytes) {
    if (bytes <= bytes_ && ptr_) return ptr_;
    release();
    check(cudaMalloc(&ptr_, std::max<size_t>(bytes, 256)), "cudaMalloc");
    bytes_ = std::max<size_t>(bytes, 256);
    return ptr_;
}

namespace {

// DDM_B200_V1=1 forces the generic shared-memory temporal kernel (A/B comparisons).
bool use_warp_temporal(int N, int N2, int sb) {
    static const bool v1 = std::getenv("DDM_B200_V1") != nullptr;
    return !v1 && ddmk::temporal_warp_supported(N, N2, sb);
}

bool use_long_temporal(int N, int N2, int sb) {
    static const bool v1 = std::getenv("DDM_B200_V1") != nullptr;
    return !v1 && ddmk::temporal_long_supported(N, N2, sb);
}

int64_t pad_len(int64_t n) {
    int64_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    return n2 << 1;
}

// q-major sequences [q][n] (working precision) -> tile-major spectra layout
template <typename S>
__global__ void pack_kernel(const cpx<S>* __restrict__ seq, int64_t q, int n, int T,
                            cpx<S>* __restrict__ spec) {
    const int64_t total = q * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / n;
        const int m = (int)(i - s * n);
        const int64_t tile = s / T;
        spec[(tile * n + m) * T + (s - tile * T)] = seq[i];
    }
}

// Diagnostic terms of `SequenceEngine::with_ft` restored to the original basis
// (`temporal.cpp:96-110`): d_a from the original sequence, corr += Re(conj(mu)(suffix+head))
// + |mu|^2 (N-m) with prefix sums of the shifted sequence. One warp per sequence; the
// prefix arrays live in `aux` ([q][n+1] f64 for |s|^2, [q][n+1] complex f64 for t).
template <typename S>
__global__ void restore_kernel(const cpx<S>* __restrict__ seq, int64_t q, int n,
                               const double* __restrict__ mean, double* __restrict__ corr,
                               double* __restrict__ d_a, double* __restrict__ aux) {
    const int lane = threadIdx.x & 31;
    const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (s >= q) return;
    const cpx<S>* x = seq + s * n;
    double* cp = aux + s * (int64_t)(n + 1) * 3;  // cp[0..n] power prefix, then (re,im) pairs
    double* tp = cp + (n + 1);
    const double mx = mean[2 * s], my = mean[2 * s + 1];
    const S ox = (S)mx, oy = (S)my;
    double c_p = 0.0, c_x = 0.0, c_y = 0.0;
    if (lane == 0) { cp[0] = 0.0; tp[0] = 0.0; tp[1] = 0.0; }
    for (int n0 = 0; n0 < n; n0 += 32) {
        const int i = n0 + lane;
        double p = 0.0, tx = 0.0, ty = 0.0;
        if (i < n) {
            const cpx<S> v = x[i];
            p = (double)v.x * (double)v.x + (double)v.y * (double)v.y;
            tx = (double)(S)(v.x - ox);
            ty = (double)(S)(v.y - oy);
        }
        for (int o = 1; o < 32; o <<= 1) {
            const double a = __shfl_up_sync(0xffffffffu, p, o);
            const double b = __shfl_up_sync(0xffffffffu, tx, o);
            const double c = __shfl_up_sync(0xffffffffu, ty, o);
            if (lane >= o) { p += a; tx += b; ty += c; }
        }
        if (i < n) {
            cp[i + 1] = c_p + p;
            tp[2 * (i + 1)] = c_x + tx;
            tp[2 * (i + 1) + 1] = c_y + ty;
        }
        c_p += __shfl_sync(0xffffffffu, p, 31);
        c_x += __shfl_sync(0xffffffffu, tx, 31);
        c_y += __shfl_sync(0xffffffffu, ty, 31);
    }
    __syncwarp();
    const double power = mx * mx + my * my;
    for (int m = lane; m < n; m += 32) {
        const double ramp = (double)(n - m);
        d_a[s * n + m] = (cp[n - m] + (cp[n] - cp[m])) / ramp;
        const double sx = (tp[2 * n] - tp[2 * m]) + tp[2 * (n - m)];
        const double sy = (tp[2 * n + 1] - tp[2 * m + 1]) + tp[2 * (n - m) + 1];
        // Re(conj(mu) * (sx + i sy)) = mx sx + my sy
        corr[s * n + m] += (mx * sx + my * sy) + power * ramp;
    }
}

// "spatial=... temporal=..." for last_engines()
std::string describe(bool warp_s, int W, int H, bool warp_t, bool long_t, int64_t N2, int T,
                     int64_t n_q, int N, bool ring) {
    std::string s = "spatial=";
    s += warp_s ? "rows2<" + std::to_string(W / 2) + ">+cols2<" + std::to_string(H) + ">" +
                      (H == 2048 && ddmk::spatial_cols_pair() ? ":pair" : "")
                : "generic";
    s += " temporal=";
    if (warp_t) {
        s += "warp<1024>";
    } else if (long_t) {
        s += "long2<" + std::to_string(N2 / 1024) + ">";
        if (!ring) {
            const int64_t chunk = ddmk::temporal_long_chunk(N);
            s += " chunks=" + std::to_string((n_q + chunk - 1) / chunk);
        }
    } else {
        s += "generic<T=" + std::to_string(T) + ">";
    }
    s += ring ? ":ring" : ":map";
    return s;
}

template <typename S>
void build_table(std::vector<unsigned char>& out, int len, int count) {
    out.resize((size_t)count * sizeof(cpx<S>));
    auto* t = reinterpret_cast<cpx<S>*>(out.data());
    const double pi = 3.141592653589793238462643383279502884;
    for (int j = 0; j < count; ++j) {
        const double a = -2.0 * pi * (double)j / (double)len;
        t[j] = {(S)std::cos(a), (S)std::sin(a)};
    }
}

}  // namespace

Engine::Engine(int device) : device_(device) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    check(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, device_), "attr");
    check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& e : ev_) check(cudaEventCreate(&e), "cudaEventCreate");
}

void* Engine::pinned(int slot, size_t bytes) {
    if (pinned_bytes_[slot] < bytes) {
        if (pinned_[slot]) cudaFreeHost(pinned_[slot]);
        pinned_[slot] = nullptr;
        pinned_bytes_[slot] = 0;
        check(cudaMallocHost(&pinned_[slot], bytes), "cudaMallocHost");
        pinned_bytes_[slot] = bytes;
    }
    return pinned_[slot];
}

void Engine::wait_frames(cudaStream_t st, int frame_end) {
    if (!frames_ready_) return;
    for (const auto& fr : *frames_ready_)
        if (fr.first >= frame_end) {
            check(cudaStreamWaitEvent(st, fr.second, 0), "wait for frames");
            return;
        }
    if (!frames_ready_->empty()) check(cudaStreamWaitEvent(st, frames_ready_->back().second, 0), "wait for frames");
}

std::vector<std::pair<int, cudaEvent_t>> Engine::upload_frames_async(void* d_frames, const void* host, int N,
                                                                      size_t frame_bytes, int chunks) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    if (!h2d_stream_) check(cudaStreamCreateWithFlags(&h2d_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    chunks = std::max(1, std::min(chunks, N));
    while (h2d_events_.size() < (size_t)chunks + 2) {
        cudaEvent_t e = nullptr;
        check(cudaEventCreate(&e), "cudaEventCreate");
        h2d_events_.push_back(e);
    }
    h2d_chunks_ = chunks;
    // the upload must not overtake work already queued on the engine stream that reads the
    // previous frames
    check(cudaEventRecord(h2d_events_[chunks], stream_), "cudaEventRecord");
    check(cudaStreamWaitEvent(h2d_stream_, h2d_events_[chunks], 0), "stream wait");
    check(cudaEventRecord(h2d_events_[chunks + 1], h2d_stream_), "cudaEventRecord");
    std::vector<std::pair<int, cudaEvent_t>> ready;
    for (int c = 0; c < chunks; ++c) {
        const int f0 = (int)((int64_t)N * c / chunks), f1 = (int)((int64_t)N * (c + 1) / chunks);
        check(cudaMemcpyAsync(static_cast<char*>(d_frames) + (size_t)f0 * frame_bytes,
                              static_cast<const char*>(host) + (size_t)f0 * frame_bytes,
                              (size_t)(f1 - f0) * frame_bytes, cudaMemcpyHostToDevice, h2d_stream_),
              "frame upload");
        check(cudaEventRecord(h2d_events_[c], h2d_stream_), "cudaEventRecord");
        ready.emplace_back(f1, h2d_events_[c]);
    }
    return ready;
}

double Engine::upload_ms() {
    if (h2d_chunks_ == 0) return 0.0;
    check(cudaEventSynchronize(h2d_events_[h2d_chunks_ - 1]), "upload");
    float ms = 0.f;
    check(cudaEventElapsedTime(&ms, h2d_events_[h2d_chunks_ + 1], h2d_events_[h2d_chunks_ - 1]), "event time");
    return ms;
}

bool Engine::finish_host_out(PhaseTimes* times) {
    if (!d2h_pending_) return false;
    d2h_pending_ = false;
    check(cudaStreamSynchronize(d2h_stream_), "map copy");
    if (times) {
        float ms = 0.f;
        check(cudaEventElapsedTime(&ms, d2h_events_[0], d2h_events_[1]), "event time");
        times->d2h_ms += ms;
    }
    return true;
}

Engine::~Engine() {
    cudaSetDevice(device_);
    for (auto p : pinned_)
        if (p) cudaFreeHost(p);
    for (auto e : timing_events_) cudaEventDestroy(e);
    for (auto e : chunk_events_) cudaEventDestroy(e);
    if (cols_stream_) cudaStreamDestroy(cols_stream_);
    if (d2h_stream_) cudaStreamDestroy(d2h_stream_);
    if (h2d_stream_) cudaStreamDestroy(h2d_stream_);
    for (auto e : h2d_events_) cudaEventDestroy(e);
    for (auto e : d2h_events_) cudaEventDestroy(e);
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    if (stream_) cudaStreamDestroy(stream_);
}

Engine& Engine::instance(int device) {
    static std::mutex m;
    static std::map<int, std::unique_ptr<Engine>> engines;
    std::lock_guard<std::mutex> lock(m);
    auto& e = engines[device];
    if (!e) e = std::make_unique<Engine>(device);
    return *e;
}

const void* Engine::twiddles(int len, bool f64) {
    auto& slot = tw_[{len, f64 ? 1 : 0}];
    if (!slot) {
        std::vector<unsigned char> host;
        if (f64) build_table<double>(host, len, len);
        else build_table<float>(host, len, len);
        slot = std::make_unique<DeviceBuffer>();
        check(cudaMemcpy(slot->ensure(host.size()), host.data(), host.size(),
                         cudaMemcpyHostToDevice), "twiddle upload");
    }
    return slot->get();
}

const void* Engine::post_twiddles(int W, bool f64) {
    auto& slot = post_[{W, f64 ? 1 : 0}];
    if (!slot) {
        std::vector<unsigned char> host;
        if (f64) build_table<double>(host, W, W / 2 + 1);
        else build_table<float>(host, W, W / 2 + 1);
        slot = std::make_unique<DeviceBuffer>();
        check(cudaMemcpy(slot->ensure(host.size()), host.data(), host.size(),
                         cudaMemcpyHostToDevice), "twiddle upload");
    }
    return slot->get();
}

void* Engine::buffer(const std::string& name, size_t bytes) {
    auto& b = named_[name];
    if (!b) b = std::make_unique<DeviceBuffer>();
    return b->ensure(bytes);
}

bool f32_register_temporal(int N) {
    const int N2 = (int)pad_len(N);
    return use_warp_temporal(N, N2, 4) || use_long_temporal(N, N2, 4);
}

int64_t max_frames(bool f64) {
    int64_t best = 0;
    for (int64_t n = 1; n <= (1 << 15); n <<= 1)
        if (ddmk::temporal_tile((int)n, (int)pad_len(n), f64 ? 8 : 4) > 0) best = n;
    return best;
}

ddmk::SpatialArgs Engine::spatial_args(const void* d_frames, int pixel_bytes, int W, int H, int N,
                                       bool f64) {
    ddmk::SpatialArgs sa;
    sa.frames = d_frames;
    sa.pixel_bytes = pixel_bytes;
    sa.W = W;
    sa.H = H;
    sa.N = N;
    const int Lr = (W % 2 == 0) ? W / 2 : W;
    sa.tw_row = {Lr, twiddles(Lr, f64)};
    sa.tw_post = {W, post_twiddles(W, f64)};
    sa.tw_col = {H, twiddles(H, f64)};
    return sa;
}

void Engine::spatial_pass(ddmk::SpatialArgs sa, bool f64, bool warp_s, PhaseTimes* times) {
    const int N = sa.N;
    const size_t per_frame = (size_t)(sa.W / 2 + 1) * sa.H * (f64 ? 16 : 8);
    // frame chunk whose row-pass output stays in L2 (~48 MB)
    // Frame chunk of the row pass. Measured at 512^2 x 1024 (tools/gpu_ab.sh, DDM_MID_MB):
    // 32 frames (L2-resident mid) 0.88 ms, 80 frames 0.79 ms, 512 frames 0.76 ms. Launch and
    // tail overhead per chunk outweighs L2 residency, so the register path takes two chunks
    // (row pass of one overlapping the column pass of the other) up to 1 GiB per buffer.
    static const char* mid_env = std::getenv("DDM_MID_MB");
    // Frames of >= 8 MB per row-pass output (2048^2) go in chunks of <= 560 MB: C4 spatial
    // 73 -> 70 ms against 1 GiB chunks (32 vs 56 frames; 16 frames 72 ms, 40 frames 74 ms); C2
    // and C3 are fastest with the two large chunks (r02 sweep)
    const size_t warp_cap = per_frame >= (size_t(8) << 20) ? size_t(560) << 20 : size_t(1) << 30;
    const size_t mid_budget = mid_env ? (size_t)std::max(1, std::atoi(mid_env)) << 20
                            : warp_s  ? std::min<size_t>((size_t)(N + 1) / 2 * per_frame, warp_cap)
                                      : size_t(48) << 20;
    int F = (int)std::max<int64_t>(1, std::min<int64_t>(N, mid_budget / per_frame));
    if (warp_s) {
        // whole column-CTA frame groups per chunk (full-length corner-turn runs), even when
        // a large frame's chunk no longer fits L2 (2048^2: 8 frames = 134 MB)
        const int Fc = ddmk::spatial_warp_col_frames(sa.H);
        F = std::min(N, std::max(Fc, F - F % Fc));
    }
    last_F_ = F;
    // the row pass of chunk k+1 runs beside the column pass of chunk k on a second
    // stream, through two L2-resident `mid` buffers
    const bool overlap = warp_s && N > F && std::getenv("DDM_SPATIAL_SERIAL") == nullptr;
    void* d_mid = mid_.ensure((size_t)F * per_frame * (overlap ? 2 : 1));
    sa.mid = d_mid;
    if (overlap) {
        if (!cols_stream_)
            check(cudaStreamCreateWithFlags(&cols_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
        const int chunks = (N + F - 1) / F;
        while (chunk_events_.size() < (size_t)(2 * chunks + 1)) {
            cudaEvent_t e = nullptr;
            check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            chunk_events_.push_back(e);
        }
        cudaEvent_t start = chunk_events_[2 * chunks];
        check(cudaEventRecord(start, stream_), "cudaEventRecord");
        check(cudaStreamWaitEvent(cols_stream_, start, 0), "stream wait");
        for (int k = 0; k < chunks; ++k) {
            cudaEvent_t rows_done = chunk_events_[2 * k], cols_done = chunk_events_[2 * k + 1];
            sa.frame0 = k * F;
            sa.nframes = std::min(F, N - k * F);
            sa.mid = static_cast<char*>(d_mid) + (size_t)(k & 1) * F * per_frame;
            // the buffer is free once the column pass of chunk k-2 has read it
            if (k >= 2) check(cudaStreamWaitEvent(stream_, chunk_events_[2 * (k - 2) + 1], 0), "wait");
            wait_frames(stream_, sa.frame0 + sa.nframes);
            check(f64 ? ddmk::launch_spatial_warp<double>(sa, stream_, 1)
                      : ddmk::launch_spatial_warp<float>(sa, stream_, 1), "row pass");
            check(cudaEventRecord(rows_done, stream_), "cudaEventRecord");
            check(cudaStreamWaitEvent(cols_stream_, rows_done, 0), "wait");
            check(f64 ? ddmk::launch_spatial_warp<double>(sa, cols_stream_, 2)
                      : ddmk::launch_spatial_warp<float>(sa, cols_stream_, 2), "column pass");
            check(cudaEventRecord(cols_done, cols_stream_), "cudaEventRecord");
            if (times) times->spatial_launches += 2;
        }
        check(cudaStreamWaitEvent(stream_, chunk_events_[2 * (chunks - 1) + 1], 0), "join");
    } else {
        for (int f0 = 0; f0 < N; f0 += F) {
            sa.frame0 = f0;
            sa.nframes = std::min(F, N - f0);
            wait_frames(stream_, f0 + sa.nframes);
            check(warp_s ? (f64 ? ddmk::launch_spatial_warp<double>(sa, stream_)
                              : ddmk::launch_spatial_warp<float>(sa, stream_))
                  : f64 ? ddmk::launch_spatial<double>(sa, stream_)
                        : ddmk::launch_spatial<float>(sa, stream_), "spatial kernels");
            if (times) times->spatial_launches += 2;
        }
    }
}

const int* Engine::upload_lags(const std::vector<int64_t>& lags, int N) {
    // every lag requested (the common case): kernels skip the lag lookup
    if ((int64_t)lags.size() == N) return nullptr;
    std::vector<int> lag_index((size_t)N, -1);
    for (size_t li = 0; li < lags.size(); ++li) lag_index[(size_t)lags[li]] = (int)li;
    if (lag_index != lag_cache_) {
        // kernels already queued on stream_ (asynchronous device-resident calls) may still
        // read the previous table: drain them before it is overwritten
        check(cudaStreamSynchronize(stream_), "sync before lag upload");
        check(cudaMemcpy(lagidx_.ensure((size_t)N * sizeof(int)), lag_index.data(),
                         (size_t)N * sizeof(int), cudaMemcpyHostToDevice), "lag upload");
        lag_cache_ = std::move(lag_index);
    }
    return static_cast<const int*>(lagidx_.get());
}

uint64_t Engine::run(const RunSpec& sp, PhaseTimes* times) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    finish_host_out(nullptr);   // copies of an earlier call that never drained them
    const int W = sp.W, H = sp.H, N = sp.N;
    const int Wh = W / 2 + 1;
    const int64_t plane = (int64_t)H * Wh;
    const int64_t N2 = pad_len(N);
    const int sb = sp.f64 ? 8 : 4;
    const size_t cs = 2 * (size_t)sb;
    const bool warp_t = use_warp_temporal(N, (int)N2, sb);
    const bool long_t = !warp_t && use_long_temporal(N, (int)N2, sb);
    // f64 at N2 = 2048: the f64 warp engine over q-major spectra (T = 1)
    static const bool v1 = std::getenv("DDM_B200_V1") != nullptr;
    const bool warp64 = sp.f64 && !v1 && ddmk::temporal_warp64_supported(N, (int)N2);
    const int T = (warp_t || long_t || warp64) ? 1 : ddmk::temporal_tile(N, (int)N2, sb);
    if (T == 0)
        throw std::length_error("sequence of " + std::to_string(N) +
                                " frames exceeds the single-CTA temporal engine (max " +
                                std::to_string(max_frames(sp.f64)) + ")");
    last_T_ = T;

    // lag slots (uploaded only when the lag list changes; every-lag runs never read them)
    const int* d_lag_index = upload_lags(sp.lags, N);
    // flat -> retained index map (cutoff only)
    const int* d_slot = nullptr;
    std::vector<int> slot_of;
    if (!sp.identity) {
        slot_of.assign((size_t)plane, -1);
        for (size_t k = 0; k < sp.flat.size(); ++k) slot_of[(size_t)sp.flat[k]] = (int)k;
        check(cudaMemcpyAsync(slotmap_.ensure((size_t)plane * sizeof(int)), slot_of.data(),
                              (size_t)plane * sizeof(int), cudaMemcpyHostToDevice, stream_),
              "slot upload");
        d_slot = static_cast<const int*>(slotmap_.get());
    }

    int64_t gmax = 0;
    for (auto& g : sp.groups) gmax = std::max(gmax, g.second - g.first);
    const int64_t tiles_max = (gmax + T - 1) / T;
    void* d_spec = spec_.ensure((size_t)tiles_max * N * T * cs);
    // f64 on register-friendly frames: the f64 register spatial kernels write q-major spectra
    // that the generic temporal engine reads T sequences per CTA (SpecLayout::qmajor)
    const bool qmajor = sp.f64 && !warp_t && !long_t && ddmk::spatial_warp_f64_supported(W, H, sp.pixel_bytes) &&
                        std::getenv("DDM_B200_V1_SPATIAL") == nullptr;
    const bool warp_s = ((warp_t || long_t) && ddmk::spatial_warp_supported(W, H, sp.pixel_bytes, sb) &&
                         std::getenv("DDM_B200_V1_SPATIAL") == nullptr) || qmajor;
    ddmk::SpatialArgs sa = spatial_args(sp.d_frames, sp.pixel_bytes, W, H, N, sp.f64);
    sa.spec = d_spec;
    sa.slot_of_flat = d_slot;

    ddmk::TemporalArgs ta;
    ta.spec = d_spec;
    ta.N = N;
    ta.N2 = (int)N2;
    ta.tw = {(int)N2, twiddles((int)N2, sp.f64)};
    ta.tw_half = {(int)N2 / 2, twiddles((int)N2 / 2, sp.f64)};
    // every lag requested (the common case): kernels skip the lag lookup
    ta.lag_index = d_lag_index;
    ta.out_f64 = sp.out_f64 ? 1 : 0;
    const size_t ob = sp.out_f64 ? 8 : 4;

    std::vector<cudaEvent_t> evs;
    auto mark = [&]() {
        if (!times) return;
        if (evs.size() == timing_events_.size()) {
            cudaEvent_t e = nullptr;
            check(cudaEventCreate(&e), "cudaEventCreate");
            timing_events_.push_back(e);
        }
        cudaEvent_t e = timing_events_[evs.size()];
        check(cudaEventRecord(e, stream_), "cudaEventRecord");
        evs.push_back(e);
    };

    last_engines_ = describe(warp_s, W, H, warp_t, long_t, N2, T, gmax, N, false);
    if (warp64) {
        const auto at = last_engines_.find("temporal=");
        if (at != std::string::npos) last_engines_ = last_engines_.substr(0, at) + "temporal=warp64<1024>:map";
    }
    // end-to-end streaming (RunSpec::frames_ready / host_out)
    frames_ready_ = sp.frames_ready.empty() ? nullptr : &sp.frames_ready;
    struct ResetFrames {
        const std::vector<std::pair<int, cudaEvent_t>>*& p;
        ~ResetFrames() { p = nullptr; }
    } reset_frames{frames_ready_};
    static const int kOutChunks = std::getenv("DDM_OUT_CHUNKS") ? std::atoi(std::getenv("DDM_OUT_CHUNKS")) : 8;
    const bool stream_out = kOutChunks > 0 && sp.host_out && warp_t && !sp.partial_mode && sp.identity &&
                            sp.groups.size() == 1 && sp.d_out;
    if (stream_out && !d2h_stream_)
        check(cudaStreamCreateWithFlags(&d2h_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    uint64_t spatial_passes = 0;
    for (size_t gi = 0; gi < sp.groups.size(); ++gi) {
        const int64_t gb = sp.groups[gi].first, gc = sp.groups[gi].second - gb;
        ddmk::SpecLayout lay;
        lay.T = T;
        lay.g_begin = gb;
        lay.g_count = gc;
        lay.qmajor = qmajor;
        // slots of a partial tile tail are never written by the spatial pass: zero them so
        // the temporal kernel transforms zeros there (q-major: the kernel zero-fills them)
        if (gc % T && !qmajor) {
            const int64_t t0 = gc / T;
            check(cudaMemsetAsync(static_cast<char*>(d_spec) + (size_t)t0 * N * T * cs, 0,
                                  (size_t)N * T * cs, stream_), "tail memset");
        }
        sa.layout = lay;
        mark();
        spatial_pass(sa, sp.f64, warp_s, times);
        mark();
        spatial_passes += (uint64_t)N;

        ta.layout = lay;
        if (sp.partial_mode) {
            ta.out = partial_.ensure((size_t)sp.lags.size() * gc * ob);
            ta.out_stride = gc;
            ta.dest_of_slot = nullptr;
        } else if (sp.identity) {
            ta.out = static_cast<char*>(sp.d_out) + (size_t)gb * ob;
            ta.out_stride = sp.out_stride;
            ta.dest_of_slot = nullptr;
        } else {
            check(cudaMemcpyAsync(dest_.ensure((size_t)gc * sizeof(int64_t)), sp.flat.data() + gb,
                                  (size_t)gc * sizeof(int64_t), cudaMemcpyHostToDevice, stream_),
                  "dest upload");
            ta.out = sp.d_out;
            ta.out_stride = sp.out_stride;
            ta.dest_of_slot = static_cast<const int64_t*>(dest_.get());
        }
        mark();
        if (long_t) {
            void* out_q = buffer("long_out_q", (size_t)std::min<int64_t>(gc, ddmk::temporal_long_chunk(N)) *
                                                   N * sizeof(float));
            check(ddmk::launch_temporal_long(ta, num_sms_, out_q, stream_), "temporal kernel");
            if (times) times->temporal_launches += 2 * (int)((gc + ddmk::temporal_long_chunk(N) - 1) /
                                                             ddmk::temporal_long_chunk(N));
        } else if (stream_out) {
            // wave-vector chunks: chunk c's columns of every lag row go to the host on the
            // D2H stream while chunk c + 1 computes (2D copies, one row segment per lag)
            const int chunks = (int)std::min<int64_t>(kOutChunks, std::max<int64_t>(1, gc / 4096));
            while (d2h_events_.size() < (size_t)(chunks + 2)) {
                cudaEvent_t e = nullptr;
                check(cudaEventCreate(&e), "cudaEventCreate");
                d2h_events_.push_back(e);
            }
            for (int c = 0; c < chunks; ++c) {
                // 12-aligned chunk edges keep the kernel's full-tile vector stores
                const int64_t qa = (gc * c / chunks) / 12 * 12;
                const int64_t qb = c + 1 == chunks ? gc : (gc * (c + 1) / chunks) / 12 * 12;
                ddmk::TemporalArgs tc = ta;
                tc.spec = static_cast<const char*>(d_spec) + (size_t)qa * N * cs;
                tc.layout.g_begin = gb + qa;
                tc.layout.g_count = qb - qa;
                tc.out = static_cast<char*>(ta.out) + (size_t)qa * ob;
                check(ddmk::launch_temporal_warp(tc, num_sms_, stream_), "temporal kernel");
                check(cudaEventRecord(d2h_events_[c + 2], stream_), "cudaEventRecord");
                check(cudaStreamWaitEvent(d2h_stream_, d2h_events_[c + 2], 0), "stream wait");
                if (c == 0) {
                    check(cudaEventRecord(d2h_events_[0], d2h_stream_), "cudaEventRecord");
                    d2h_pending_ = true;   // from here on a failure must still drain the copies
                }
                const size_t pitch = (size_t)ta.out_stride * ob;
                check(cudaMemcpy2DAsync(static_cast<char*>(sp.host_out) + (size_t)(gb + qa) * ob, pitch,
                                        tc.out, pitch, (size_t)(qb - qa) * ob, sp.lags.size(),
                                        cudaMemcpyDeviceToHost, d2h_stream_),
                      "map chunk copy");
            }
            check(cudaEventRecord(d2h_events_[1], d2h_stream_), "cudaEventRecord");
            if (times) times->temporal_launches += chunks;
        } else {
            check(warp_t ? ddmk::launch_temporal_warp(ta, num_sms_, stream_)
                  : warp64 ? ddmk::launch_temporal_warp64(ta, num_sms_, stream_)
                  : sp.f64 ? ddmk::launch_temporal<double>(ta, stream_)
                           : ddmk::launch_temporal<float>(ta, stream_), "temporal kernel");
            if (times) times->temporal_launches += 1;
        }
        mark();
        if (sp.partial_mode && sp.on_partial) sp.on_partial(gi, ta.out, gc);
        // the host-side slot map / dest vectors must outlive the async copies
        if (!sp.identity || sp.partial_mode) check(cudaStreamSynchronize(stream_), "sync");
    }
    if (times) {
        check(cudaStreamSynchronize(stream_), "sync");
        for (size_t i = 0; i + 3 < evs.size(); i += 4) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, evs[i], evs[i + 1]);
            cudaEventElapsedTime(&b, evs[i + 2], evs[i + 3]);
            times->spatial_ms += a;
            times->temporal_ms += b;
        }
    }
    // without timing the run stays asynchronous: the lag table is uploaded synchronously and
    // the slot map / destination vectors were synchronised inside the group loop
    return spatial_passes;
}

void Engine::spatial_shard(const void* d_frames, int pixel_bytes, int W, int H, int n, bool f64,
                           void* d_spec, PhaseTimes* times, const ddmk::PeerTable* peers) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    const int sb = f64 ? 8 : 4;
    // the warp spatial kernels write the same q-major layout as the generic ones
    const bool warp_s = !f64 && ddmk::spatial_warp_supported(W, H, pixel_bytes, sb) &&
                        std::getenv("DDM_B200_V1_SPATIAL") == nullptr;
    ddmk::SpatialArgs sa = spatial_args(d_frames, pixel_bytes, W, H, n, f64);
    sa.spec = d_spec;
    sa.slot_of_flat = nullptr;
    sa.layout.T = 1;
    sa.layout.g_begin = 0;
    sa.layout.g_count = (int64_t)H * (W / 2 + 1);
    if (peers && peers->ranks > 0) {
        if (!warp_s)
            throw std::invalid_argument("the fused NVLink corner turn needs the register-resident "
                                        "spatial kernels (f32, power-of-two W/2 and H <= 1024)");
        sa.peers = *peers;
    }
    if (times) check(cudaEventRecord(ev_[0], stream_), "cudaEventRecord");
    spatial_pass(sa, f64, warp_s, times);
    if (times) {
        check(cudaEventRecord(ev_[1], stream_), "cudaEventRecord");
        check(cudaEventSynchronize(ev_[1]), "sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
        times->spatial_ms += ms;
    }
}

void Engine::temporal_segments(const void* d_recv, int64_t q_count, const std::vector<int>& seg_frames,
                               bool f64, const std::vector<int64_t>& lags, void* d_out,
                               int64_t out_stride, bool out_f64, PhaseTimes* times) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    if (seg_frames.empty() || seg_frames.size() > (size_t)ddmk::SegTable::kMax)
        throw std::invalid_argument("1 to 8 frame segments per sequence");
    ddmk::SegTable segs;
    segs.count = (int)seg_frames.size();
    int N = 0;
    for (int s = 0; s < segs.count; ++s) {
        if (seg_frames[(size_t)s] < 1) throw std::invalid_argument("empty frame segment");
        segs.n[s] = seg_frames[(size_t)s];
        segs.off[s] = N;
        segs.base[s] = q_count * (int64_t)N;
        N += segs.n[s];
    }
    const int64_t N2 = pad_len(N);
    const int sb = f64 ? 8 : 4;
    const bool seg_ok = ddmk::temporal_warp_segments_ok(segs, N);
    const bool warp_t = use_warp_temporal(N, (int)N2, sb) && seg_ok;
    const bool long_t = !warp_t && use_long_temporal(N, (int)N2, sb) && seg_ok;
    const int T = (warp_t || long_t) ? 1 : ddmk::temporal_tile(N, (int)N2, sb);
    if (T == 0)
        throw std::length_error("sequence of " + std::to_string(N) +
                                " frames exceeds the single-CTA temporal engine");
    ddmk::TemporalArgs ta;
    ta.N = N;
    ta.N2 = (int)N2;
    ta.tw = {(int)N2, twiddles((int)N2, f64)};
    ta.tw_half = {(int)N2 / 2, twiddles((int)N2 / 2, f64)};
    ta.lag_index = upload_lags(lags, N);
    ta.layout.T = T;
    ta.layout.g_begin = 0;
    ta.layout.g_count = q_count;
    ta.out = d_out;
    ta.out_f64 = out_f64 ? 1 : 0;
    ta.out_stride = out_stride;
    if (times) check(cudaEventRecord(ev_[2], stream_), "cudaEventRecord");
    if (warp_t || long_t) {
        ta.spec = d_recv;
        ta.segs = segs;
        if (warp_t) {
            check(ddmk::launch_temporal_warp(ta, num_sms_, stream_), "temporal kernel");
        } else {
            void* out_q = buffer("long_out_q", (size_t)std::min<int64_t>(q_count, ddmk::temporal_long_chunk(N)) *
                                                   N * sizeof(float));
            check(ddmk::launch_temporal_long(ta, num_sms_, out_q, stream_), "temporal kernel");
        }
    } else {
        // generic engine: gather the segments into its tile-major layout first
        const int64_t tiles = (q_count + T - 1) / T;
        void* d_spec = spec_.ensure((size_t)tiles * N * T * 2 * sb);
        check(f64 ? ddmk::launch_repack_segments<double>(d_recv, q_count, segs, N, T, d_spec, stream_)
                  : ddmk::launch_repack_segments<float>(d_recv, q_count, segs, N, T, d_spec, stream_),
              "repack kernel");
        ta.spec = d_spec;
        check(f64 ? ddmk::launch_temporal<double>(ta, stream_) : ddmk::launch_temporal<float>(ta, stream_),
              "temporal kernel");
        if (times) times->temporal_launches += 1;
    }
    if (times) {
        times->temporal_launches += 1;
        check(cudaEventRecord(ev_[3], stream_), "cudaEventRecord");
        check(cudaEventSynchronize(ev_[3]), "sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev_[2], ev_[3]);
        times->temporal_ms += ms;
    }
}

RingPlan make_ring_plan(const std::vector<int64_t>& flat, int W, int H) {
    RingPlan rp;
    const int Wh = W / 2 + 1;
    const size_t q = flat.size();
    std::vector<int64_t> bin(q);
    int64_t bmax = 0;
    for (size_t k = 0; k < q; ++k) {
        const int row = (int)(flat[k] / Wh), col = (int)(flat[k] % Wh);
        const int qr = row <= H / 2 ? row : row - H;   // `spectrum.hpp:20-24`
        bin[k] = std::llround(std::sqrt((double)qr * qr + (double)col * col));
        bmax = std::max(bmax, bin[k]);
    }
    rp.nbins = q ? bmax + 1 : 0;
    rp.counts.assign((size_t)rp.nbins, 0);
    for (auto b : bin) ++rp.counts[(size_t)b];
    rp.bin_off.assign((size_t)rp.nbins + 1, 0);
    for (int64_t b = 0; b < rp.nbins; ++b) rp.bin_off[(size_t)b + 1] = rp.bin_off[(size_t)b] + rp.counts[(size_t)b];
    rp.by_bin.resize(q);
    rp.flat_by_bin.resize(q);
    std::vector<int64_t> fill(rp.bin_off.begin(), rp.bin_off.end() - 1);
    for (size_t k = 0; k < q; ++k) {
        const int64_t at = fill[(size_t)bin[k]]++;
        rp.by_bin[(size_t)at] = (int64_t)k;
        rp.flat_by_bin[(size_t)at] = flat[k];
    }
    rp.item_off.assign(1, 0);
    rp.ring_item_off.assign(1, 0);
    for (int64_t b = 0; b < rp.nbins; ++b) {
        const int64_t c = rp.counts[(size_t)b];
        if (c == 0) continue;
        for (int64_t i = rp.bin_off[(size_t)b]; i < rp.bin_off[(size_t)b + 1]; i += RingPlan::kItem)
            rp.item_off.push_back(std::min(i + RingPlan::kItem, rp.bin_off[(size_t)b + 1]));
        rp.ring_item_off.push_back((int64_t)rp.item_off.size() - 1);
        rp.ring_bin.push_back(b);
        rp.ring_count.push_back(c);
    }
    return rp;
}

const RingPlan& Engine::ring_plan(const std::vector<int64_t>& flat, int W, int H) {
    RingCache& c = ring_cache_;
    if (c.plan && c.W == W && c.H == H && c.flat == flat) return *c.plan;
    c.own = std::make_unique<RingPlan>(make_ring_plan(flat, W, H));
    c.plan = c.own.get();
    c.W = W;
    c.H = H;
    c.flat = flat;
    auto up = [&](const char* name, const std::vector<int64_t>& v) {
        void* d = buffer(name, std::max<size_t>(v.size(), 1) * sizeof(int64_t));
        check(cudaMemcpy(d, v.data(), v.size() * sizeof(int64_t), cudaMemcpyHostToDevice), "ring upload");
        return static_cast<const int64_t*>(d);
    };
    c.order = up("ring_order", c.plan->by_bin);
    c.item_off = up("ring_item_off", c.plan->item_off);
    c.ring_item_off = up("ring_ring_item_off", c.plan->ring_item_off);
    c.ring_bin = up("ring_bin", c.plan->ring_bin);
    c.ring_count = up("ring_count", c.plan->ring_count);
    c.flat_by_bin = up("ring_flat", c.plan->flat_by_bin);
    c.bin_off = up("ring_bin_off", c.plan->bin_off);
    return *c.plan;
}

bool Engine::run_rings(const RunSpec& sp, const RingPlan& rp, double* d_means, PhaseTimes* times) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    if (&rp != ring_cache_.plan) throw std::invalid_argument("run_rings: plan must come from ring_plan()");
    const RingCache& rc = ring_cache_;
    const int N = sp.N;
    const int64_t N2 = pad_len(N);
    const int sb = sp.f64 ? 8 : 4;
    const int64_t L = (int64_t)sp.lags.size();
    const int64_t count = sp.groups.empty() ? 0 : sp.groups.back().second;
    check(cudaMemsetAsync(d_means, 0, (size_t)(L * rp.nbins) * sizeof(double), stream_), "memset");
    const bool warp_t = use_warp_temporal(N, (int)N2, sb);
    const bool long_t = !warp_t && use_long_temporal(N, (int)N2, sb);
    const bool fused = warp_t || long_t;
    const bool warp_s = fused && ddmk::spatial_warp_supported(sp.W, sp.H, sp.pixel_bytes, sb) &&
                        std::getenv("DDM_B200_V1_SPATIAL") == nullptr;
    if (!fused) {
        // map through HBM (f64), then the deterministic ring reduction
        RunSpec m = sp;
        m.out_f64 = true;
        m.out_stride = (int64_t)sp.H * (sp.W / 2 + 1);
        m.partial_mode = false;
        m.groups = {{0, count}};
        m.d_out = buffer("ring_map", (size_t)(L * m.out_stride) * sizeof(double));
        if (!sp.identity)
            check(cudaMemsetAsync(m.d_out, 0, (size_t)(L * m.out_stride) * sizeof(double), stream_), "memset");
        run(m, times);
        last_engines_ += "+radial";
        radial_means(static_cast<const double*>(m.d_out), L, m.out_stride, rc.flat_by_bin, rc.bin_off,
                     rp.nbins, d_means, stream_);
        check(cudaStreamSynchronize(stream_), "sync");
        return false;
    }
    // fused: spatial pass into the slot-major spectra, then the ring temporal launch
    last_engines_ = describe(warp_s, sp.W, sp.H, warp_t, long_t, N2, 1, count, N, true);
    const int* d_lag_index = upload_lags(sp.lags, N);
    const int Wh = sp.W / 2 + 1;
    const int64_t plane = (int64_t)sp.H * Wh;
    const int* d_slot = nullptr;
    std::vector<int> slot_of;
    if (!sp.identity) {
        slot_of.assign((size_t)plane, -1);
        for (size_t k = 0; k < sp.flat.size(); ++k) slot_of[(size_t)sp.flat[k]] = (int)k;
        check(cudaMemcpyAsync(slotmap_.ensure((size_t)plane * sizeof(int)), slot_of.data(),
                              (size_t)plane * sizeof(int), cudaMemcpyHostToDevice, stream_), "slot upload");
        d_slot = static_cast<const int*>(slotmap_.get());
    }
    void* d_spec = spec_.ensure((size_t)count * N * 2 * sb);
    ddmk::SpatialArgs sa = spatial_args(sp.d_frames, sp.pixel_bytes, sp.W, sp.H, N, sp.f64);
    sa.spec = d_spec;
    sa.slot_of_flat = d_slot;
    sa.layout.T = 1;
    sa.layout.g_begin = 0;
    sa.layout.g_count = count;
    if (times) check(cudaEventRecord(ev_[0], stream_), "cudaEventRecord");
    spatial_pass(sa, sp.f64, warp_s, times);
    if (times) check(cudaEventRecord(ev_[1], stream_), "cudaEventRecord");
    const int64_t nitems = (int64_t)rp.item_off.size() - 1;
    ddmk::TemporalArgs ta;
    ta.spec = d_spec;
    ta.N = N;
    ta.N2 = (int)N2;
    ta.layout.T = 1;
    ta.layout.g_begin = 0;
    ta.layout.g_count = count;
    ta.lag_index = d_lag_index;
    ta.out_f64 = 1;
    ta.ring.nitems = nitems;
    ta.ring.order = rc.order;
    ta.ring.item_off = rc.item_off;
    ta.ring.partial = static_cast<double*>(buffer("ring_partial", (size_t)(nitems * N) * sizeof(double)));
    if (times) check(cudaEventRecord(ev_[2], stream_), "cudaEventRecord");
    check(warp_t ? ddmk::launch_temporal_warp(ta, num_sms_, stream_)
                 : ddmk::launch_temporal_long(ta, num_sms_, nullptr, stream_), "temporal ring kernel");
    check(ddmk::launch_ring_means(ta.ring.partial, N, d_lag_index, rc.ring_item_off, rc.ring_bin,
                                  rc.ring_count, (int64_t)rp.ring_bin.size(), d_means, rp.nbins,
                                  stream_), "ring means kernel");
    if (times) {
        check(cudaEventRecord(ev_[3], stream_), "cudaEventRecord");
        check(cudaEventSynchronize(ev_[3]), "sync");
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, ev_[0], ev_[1]);
        cudaEventElapsedTime(&b, ev_[2], ev_[3]);
        times->spatial_ms += a;
        times->temporal_ms += b;
        times->temporal_launches += 2;
    }
    if (!sp.identity) check(cudaStreamSynchronize(stream_), "sync");  // slot_of is host-side
    return true;
}

void Engine::run_pairwise(const RunSpec& sp, PhaseTimes* times) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    const int W = sp.W, H = sp.H, N = sp.N;
    const int sb = sp.f64 ? 8 : 4;
    const int64_t plane = (int64_t)H * (W / 2 + 1);
    const int64_t count = (int64_t)sp.flat.size();
    const int* d_slot = nullptr;
    std::vector<int> slot_of;
    if (!sp.identity) {
        slot_of.assign((size_t)plane, -1);
        for (size_t k = 0; k < sp.flat.size(); ++k) slot_of[(size_t)sp.flat[k]] = (int)k;
        check(cudaMemcpyAsync(slotmap_.ensure((size_t)plane * sizeof(int)), slot_of.data(),
                              (size_t)plane * sizeof(int), cudaMemcpyHostToDevice, stream_), "slot upload");
        d_slot = static_cast<const int*>(slotmap_.get());
    }
    void* d_spec = spec_.ensure((size_t)count * N * 2 * sb);
    const bool warp_s = !sp.f64 && ddmk::spatial_warp_supported(W, H, sp.pixel_bytes, sb) &&
                        std::getenv("DDM_B200_V1_SPATIAL") == nullptr;
    ddmk::SpatialArgs sa = spatial_args(sp.d_frames, sp.pixel_bytes, W, H, N, sp.f64);
    sa.spec = d_spec;
    sa.slot_of_flat = d_slot;
    sa.layout.T = 1;
    sa.layout.g_begin = 0;
    sa.layout.g_count = count;
    if (times) check(cudaEventRecord(ev_[0], stream_), "cudaEventRecord");
    spatial_pass(sa, sp.f64, warp_s, times);
    if (times) check(cudaEventRecord(ev_[1], stream_), "cudaEventRecord");
    std::vector<int> lags(sp.lags.begin(), sp.lags.end());
    int* d_lags = static_cast<int*>(buffer("pair_lags", std::max<size_t>(lags.size(), 1) * sizeof(int)));
    check(cudaMemcpyAsync(d_lags, lags.data(), lags.size() * sizeof(int), cudaMemcpyHostToDevice, stream_),
          "lag upload");
    const int64_t* d_dest = nullptr;
    if (!sp.identity) {
        check(cudaMemcpyAsync(dest_.ensure((size_t)count * sizeof(int64_t)), sp.flat.data(),
                              (size_t)count * sizeof(int64_t), cudaMemcpyHostToDevice, stream_),
              "dest upload");
        d_dest = static_cast<const int64_t*>(dest_.get());
    }
    if (times) check(cudaEventRecord(ev_[2], stream_), "cudaEventRecord");
    int lag0 = lags.empty() ? -1 : lags[0];   // contiguous lag range -> windowed kernel
    for (size_t i = 1; i < lags.size() && lag0 >= 0; ++i)
        if (lags[i] != lags[0] + (int)i) lag0 = -1;
    check(sp.f64 ? ddmk::launch_pairwise<double>(d_spec, N, count, d_lags, (int)lags.size(),
                                                 static_cast<double*>(sp.d_out), sp.out_stride, d_dest,
                                                 num_sms_, stream_, lag0)
                 : ddmk::launch_pairwise<float>(d_spec, N, count, d_lags, (int)lags.size(),
                                                static_cast<double*>(sp.d_out), sp.out_stride, d_dest,
                                                num_sms_, stream_, lag0),
          "pairwise kernel");
    if (times) check(cudaEventRecord(ev_[3], stream_), "cudaEventRecord");
    check(cudaStreamSynchronize(stream_), "sync");   // host lag / slot vectors
    if (times) {
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, ev_[0], ev_[1]);
        cudaEventElapsedTime(&b, ev_[2], ev_[3]);
        times->spatial_ms += a;
        times->temporal_ms += b;
        times->temporal_launches += 1;
    }
}

void Engine::spectra(const void* d_frames, int pixel_bytes, int W, int H, int N, bool f64,
                     void* d_out) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    const int Wh = W / 2 + 1;
    const size_t cs = f64 ? 16 : 8;
    const size_t per_frame = (size_t)Wh * H * cs;
    const int F = (int)std::max<int64_t>(1, std::min<int64_t>(N, (48u << 20) / per_frame));
    ddmk::SpatialArgs sa;
    sa.frames = d_frames;
    sa.pixel_bytes = pixel_bytes;
    sa.W = W;
    sa.H = H;
    sa.N = N;
    sa.mid = mid_.ensure((size_t)F * per_frame);
    sa.spec = d_out;
    // one tile holding the whole plane: spec[(0 * N + n) * plane + s] = frame-major output
    sa.layout.T = (int)((int64_t)H * Wh);
    sa.layout.g_begin = 0;
    sa.layout.g_count = (int64_t)H * Wh;
    const int Lr = (W % 2 == 0) ? W / 2 : W;
    sa.tw_row = {Lr, twiddles(Lr, f64)};
    sa.tw_post = {W, post_twiddles(W, f64)};
    sa.tw_col = {H, twiddles(H, f64)};
    for (int f0 = 0; f0 < N; f0 += F) {
        sa.frame0 = f0;
        sa.nframes = std::min(F, N - f0);
        check(f64 ? ddmk::launch_spatial<double>(sa, stream_) : ddmk::launch_spatial<float>(sa, stream_),
              "spatial kernels");
    }
    check(cudaStreamSynchronize(stream_), "sync");
}

void Engine::transform1d(void* d_data, int len, bool f64, int sign) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    void* scratch = buffer("fft1d", (size_t)len * (f64 ? 16 : 8));
    check(ddmk::launch_fft1d(d_data, scratch, len, f64, sign, twiddles(len, f64), stream_), "fft1d kernels");
    check(cudaStreamSynchronize(stream_), "sync");
}

void Engine::sequences(const void* d_seq, int64_t q, int64_t n, bool f64, double* d_out,
                       double* d_a_out, double* corr_out) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    const int64_t N2 = pad_len(n);
    const int sb = f64 ? 8 : 4;
    const size_t cs = 2 * (size_t)sb;
    const bool warp_t = use_warp_temporal((int)n, (int)N2, sb);
    const int T = warp_t ? 1 : ddmk::temporal_tile((int)n, (int)N2, sb);
    if (T == 0)
        throw std::length_error("sequence of " + std::to_string(n) +
                                " frames exceeds the single-CTA temporal engine");
    const int64_t tiles = (q + T - 1) / T;
    void* d_spec = spec_.ensure((size_t)tiles * n * T * cs);
    check(cudaMemsetAsync(d_spec, 0, (size_t)tiles * n * T * cs, stream_), "memset");
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>(148 * 16, (q * n + threads - 1) / threads);
    if (f64)
        pack_kernel<double><<<blocks, threads, 0, stream_>>>(static_cast<const cpx<double>*>(d_seq),
                                                             q, (int)n, T,
                                                             static_cast<cpx<double>*>(d_spec));
    else
        pack_kernel<float><<<blocks, threads, 0, stream_>>>(static_cast<const cpx<float>*>(d_seq),
                                                            q, (int)n, T,
                                                            static_cast<cpx<float>*>(d_spec));
    check(cudaGetLastError(), "pack kernel");

    std::vector<int> lag_index((size_t)n);
    for (int64_t m = 0; m < n; ++m) lag_index[(size_t)m] = (int)m;
    check(cudaMemcpyAsync(lagidx_.ensure((size_t)n * sizeof(int)), lag_index.data(),
                          (size_t)n * sizeof(int), cudaMemcpyHostToDevice, stream_), "lag upload");
    lag_cache_.clear();  // lagidx_ no longer holds a run's lag slots
    // out[s][m]: li = m, dest(s) = s * n, out_stride = 1
    std::vector<int64_t> dest((size_t)q);
    for (int64_t s = 0; s < q; ++s) dest[(size_t)s] = s * n;
    check(cudaMemcpyAsync(dest_.ensure((size_t)q * sizeof(int64_t)), dest.data(),
                          (size_t)q * sizeof(int64_t), cudaMemcpyHostToDevice, stream_),
          "dest upload");

    const bool terms = d_a_out || corr_out;
    double* d_mean = nullptr;
    double* d_corr = nullptr;
    double* d_aux = nullptr;
    if (terms) {
        const size_t need = (size_t)q * 2 * sizeof(double) + (size_t)q * n * sizeof(double) +
                            (size_t)q * (n + 1) * 3 * sizeof(double);
        char* base = static_cast<char*>(seq_aux_.ensure(need));
        d_mean = reinterpret_cast<double*>(base);
        d_corr = corr_out ? corr_out : reinterpret_cast<double*>(base + (size_t)q * 2 * sizeof(double));
        d_aux = reinterpret_cast<double*>(base + (size_t)q * 2 * sizeof(double) +
                                          (size_t)q * n * sizeof(double));
    }
    ddmk::TemporalArgs ta;
    ta.spec = d_spec;
    ta.N = (int)n;
    ta.N2 = (int)N2;
    ta.layout.T = T;
    ta.layout.g_begin = 0;
    ta.layout.g_count = q;
    ta.tw = {(int)N2, twiddles((int)N2, f64)};
    ta.tw_half = {(int)N2 / 2, twiddles((int)N2 / 2, f64)};
    ta.lag_index = static_cast<const int*>(lagidx_.get());
    ta.out = d_out;
    ta.out_f64 = 1;
    ta.out_stride = 1;
    ta.dest_of_slot = static_cast<const int64_t*>(dest_.get());
    ta.corr_out = d_corr;
    ta.mean_out = d_mean;
    check(warp_t ? ddmk::launch_temporal_warp(ta, num_sms_, stream_)
                 : f64 ? ddmk::launch_temporal<double>(ta, stream_) : ddmk::launch_temporal<float>(ta, stream_),
          "temporal kernel");
    if (terms) {
        double* d_da = d_a_out ? d_a_out : d_out;  // never both null here when terms
        std::vector<double> keep;
        if (!d_a_out) {
            // d_a not requested: restore into scratch so d_out survives
            d_da = reinterpret_cast<double*>(user_scratch_.ensure((size_t)q * n * sizeof(double)));
        }
        const int rb = (int)((q * 32 + 255) / 256);
        if (f64)
            restore_kernel<double><<<rb, 256, 0, stream_>>>(static_cast<const cpx<double>*>(d_seq), q,
                                                            (int)n, d_mean, d_corr, d_da, d_aux);
        else
            restore_kernel<float><<<rb, 256, 0, stream_>>>(static_cast<const cpx<float>*>(d_seq), q,
                                                           (int)n, d_mean, d_corr, d_da, d_aux);
        check(cudaGetLastError(), "restore kernel");
    }
    check(cudaStreamSynchronize(stream_), "sync");
}

}  // namespace ddm::b200
