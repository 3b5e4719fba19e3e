// Staging session of the opaque-handle C-ABI (ddm_b200_create / _stage_frames /
// _run_with_ft / _destroy): one stack resident in HBM, its own device Engine.
#pragma once

#include "ddm/timing.hpp"
#include "run_internal.hpp"

#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace ddm::detail {

class Session {
public:
    Session(int width, int height, int frames, int precision, int device);
    ~Session();
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;

    // frames [first, first + count) from a frame-major host buffer (u16: pixel_bytes 2, u8: 1)
    void stage(const void* host, int pixel_bytes, int first, int count);
    // WITH_FT over the staged stack: wv_flat = NULL for every wave vector of the half plane,
    // else q_count ascending flat indices; lags = NULL for every lag. out: lag-major
    // [lags][H * (W/2+1)] f64, zeros outside the list.
    TimingBreakdown run_with_ft(const std::int64_t* wv_flat, std::int64_t q_count,
                                const std::int64_t* lags, std::int64_t n_lags, double* out,
                                std::int64_t capacity, RunCounters* counters);
    const std::string& last_engines() const { return last_engines_; }

private:
    int W_, H_, N_;
    bool f64_;
    int pixel_bytes_ = 0;
    std::unique_ptr<b200::Engine> eng_;
    void* d_frames_ = nullptr;
    std::vector<bool> staged_;
    std::mutex mu_;
    std::string last_engines_;
};

}  // namespace ddm::detail
