// Opaque staging session behind ddm_b200_create / stage_frames / run_with_ft (include/ddm_b200.h,
// SURVEY.md §8b "Required C-ABI"). The reference's seam is `ddm::run(FrameSource&, const
// RunConfig&)` (`proj/core/include/ddm/scheduler.hpp:106`), which re-reads and re-transforms
// the frames on every call; a session stages a stack into HBM once and runs the WITH_FT path
// over it for any number of (wave-vector list, lag list) requests, each with the contract of
// the reference's WithFt branch (`scheduler.cpp:413-483`): normalised lags, d(0) = 0, zeros
// outside the requested wave vectors, the lag-major f64 map, `validate()` floors, exact counters.
//
// Each session owns its own device Engine (buffers, streams) rather than the per-device one
// behind ddm_b200_run_*, so sessions on one GPU run concurrently; one session is used by one
// thread at a time (its calls are serialised by its own mutex).
#include "session.hpp"

#include "ddm/errors.hpp"
#include "ddm/scheduler.hpp"
#include "ddm/spectrum.hpp"
#include "ddm/temporal.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>

namespace ddm::detail {

Session::Session(int width, int height, int frames, int precision, int device)
    : W_(width), H_(height), N_(frames), f64_(precision != 0) {
    if (width < 1 || height < 1) throw InputError("frame dimensions must be positive");
    if (frames < 1) throw InputError("stack has no frames");
    if (precision != 0 && precision != 1) throw InputError("precision must be 0 (f32) or 1 (f64)");
    if (N_ > b200::max_frames(f64_))
        throw PlanError("sequence of " + std::to_string(N_) + " frames exceeds the device temporal "
                        "engine limit of " + std::to_string(b200::max_frames(f64_)));
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count)
        throw InputError("no such CUDA device: " + std::to_string(device));
    eng_ = std::make_unique<b200::Engine>(device);
    staged_.assign(std::size_t(N_), false);
}

Session::~Session() = default;

void Session::stage(const void* host, int pixel_bytes, int first, int count) {
    std::lock_guard<std::mutex> lock(mu_);
    if (!host) throw InputError("null frame buffer");
    if (first < 0 || count < 0 || first + count > N_)
        throw InputError("frames [" + std::to_string(first) + ", " + std::to_string(first + count) +
                         ") outside the session's " + std::to_string(N_) + " frames");
    if (pixel_bytes_ != 0 && pixel_bytes_ != pixel_bytes)
        throw InputError("a session's frames are either all u16 or all u8");
    const std::size_t frame_bytes = std::size_t(W_) * H_ * std::size_t(pixel_bytes);
    if (!d_frames_) d_frames_ = eng_->frame_buffer(frame_bytes * std::size_t(N_));
    pixel_bytes_ = pixel_bytes;
    if (count == 0) return;
    char* dst = static_cast<char*>(d_frames_) + frame_bytes * std::size_t(first);
    if (is_pinned(host)) {
        b200::check(cudaMemcpyAsync(dst, host, frame_bytes * std::size_t(count), cudaMemcpyHostToDevice,
                                    eng_->stream()), "frame upload");
        b200::check(cudaStreamSynchronize(eng_->stream()), "sync");
    } else {
        upload_pageable(*eng_, dst, host, frame_bytes * std::size_t(count), eng_->stream());
    }
    std::fill(staged_.begin() + first, staged_.begin() + first + count, true);
}

TimingBreakdown Session::run_with_ft(const std::int64_t* wv_flat, std::int64_t q_count,
                                     const std::int64_t* lags_in, std::int64_t n_lags, double* out,
                                     std::int64_t capacity, RunCounters* counters) {
    std::lock_guard<std::mutex> lock(mu_);
    const auto wall0 = std::chrono::steady_clock::now();
    if (!out) throw InputError("null output buffer");
    if (std::find(staged_.begin(), staged_.end(), false) != staged_.end())
        throw InputError("not every frame of the session has been staged");
    const std::int64_t plane = std::int64_t(H_) * half_cols(W_);
    const std::vector<std::int64_t> lags =
        (lags_in && n_lags > 0) ? normalize_lags(std::vector<std::int64_t>(lags_in, lags_in + n_lags), N_)
                                : all_lags(N_);
    if (lags.empty()) throw InputError("no lags");
    b200::RunSpec spec;
    spec.W = W_;
    spec.H = H_;
    spec.N = N_;
    spec.f64 = f64_;
    spec.pixel_bytes = pixel_bytes_;
    spec.d_frames = d_frames_;
    spec.lags = lags;
    if (wv_flat) {
        if (q_count < 1) throw InputError("wave-vector list is empty");
        spec.flat.assign(wv_flat, wv_flat + q_count);
        for (std::int64_t k = 0; k < q_count; ++k)
            if (spec.flat[std::size_t(k)] < 0 || spec.flat[std::size_t(k)] >= plane ||
                (k > 0 && spec.flat[std::size_t(k)] <= spec.flat[std::size_t(k - 1)]))
                throw InputError("wave-vector list must be ascending flat indices within the plane");
    } else {
        spec.flat.resize(std::size_t(plane));
        for (std::int64_t k = 0; k < plane; ++k) spec.flat[std::size_t(k)] = k;
    }
    const std::int64_t q = std::int64_t(spec.flat.size());
    spec.identity = q == plane;
    const std::int64_t total = plane * std::int64_t(lags.size());
    if (capacity < total) throw InputError("output capacity is smaller than lags x plane");
    spec.groups = {{0, q}};
    cudaStream_t st = eng_->stream();
    // DDM_D2H_WIDEN=1 (f32 sessions, register temporal engines): the map leaves the device as
    // f32 (half the PCIe bytes) and is widened on the host (exact)
    const bool widen = !f64_ && d2h_widen_enabled() && total >= (std::int64_t(1) << 22) &&
                       b200::f32_register_temporal(N_);
    const std::size_t eb = widen ? sizeof(float) : sizeof(double);
    void* d_map = eng_->buffer(widen ? "map32" : "map", std::size_t(total) * eb);
    if (!spec.identity) b200::check(cudaMemsetAsync(d_map, 0, std::size_t(total) * eb, st), "memset");
    spec.d_out = d_map;
    spec.out_f64 = !widen;
    spec.out_stride = plane;
    if (!widen && is_pinned(out)) spec.host_out = out;
    TimingBreakdown timing;
    b200::PhaseTimes times;
    struct DrainCopies {
        b200::Engine& e;
        ~DrainCopies() {
            try {
                e.finish_host_out(nullptr);
            } catch (...) {
            }
        }
    } drain{*eng_};
    eng_->run(spec, &times);
    bool finite = true;
    double peak = 0.0, lowest = 0.0;
    if (widen)
        b200::reduce_stats(static_cast<const float*>(d_map), total, st, &finite, &peak, &lowest);
    else
        b200::reduce_stats(static_cast<const double*>(d_map), total, st, &finite, &peak, &lowest);
    const bool streamed = eng_->finish_host_out(&times);
    if (!finite) throw InputError("result map contains non-finite values");
    const double eps = f64_ ? 1e-9 : 1e-4;
    if (lowest < -eps * std::max(peak, 1.0))
        throw InputError("result map contains negative values beyond tolerance");
    if (streamed) {
        timing.merge = times.d2h_ms * 1e-3;
    } else {
        const auto t0 = std::chrono::steady_clock::now();
        if (widen)
            download_widen(*eng_, out, static_cast<const float*>(d_map), std::size_t(total), st);
        else
            download_pageable(*eng_, out, d_map, std::size_t(total) * sizeof(double), st);
        timing.merge = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    timing.step1 = times.spatial_ms * 1e-3;
    timing.step2 = times.temporal_ms * 1e-3;
    if (counters) {
        counters->spatial_ffts = std::uint64_t(N_);
        counters->temporal_ffts = 2 * std::uint64_t(q);
        counters->pairs = 0;
    }
    timing.finish(std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count());
    last_engines_ = eng_->last_engines();
    return timing;
}

}  // namespace ddm::detail
