// Internal glue between the reference-mirroring C++ API and the device engine.
#pragma once

#include "../engine.hpp"
#include "ddm/archive.hpp"
#include "ddm/errors.hpp"
#include "ddm/frame_source.hpp"
#include "ddm/scheduler.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

namespace ddm::detail {

// Either a FrameSource (u16) or a raw u8 frame-major buffer.
struct Ingest {
    const FrameSource* source = nullptr;
    const std::uint8_t* u8 = nullptr;
    int width = 0, height = 0, frames = 0;
    double frame_interval = 1.0;
};

// ResultArchive::validate over n values (`archive.cpp:44-58`), same errors and precedence.
void validate_values(const double* values, std::size_t n, bool f32);
// write_partial with the payload from any host buffer (the run's own map when it is the
// whole partial), written by several threads
std::filesystem::path write_partial_payload(const PartialResult& header, const double* values,
                                            std::size_t count, const std::filesystem::path& out_dir);

ResultArchive run_core(const Ingest& in, const RunConfig& config, double* out,
                       std::int64_t capacity);

// fn(i) for i in [0, n) on up to 16 host threads; the first exception is rethrown
template <class Fn>
void parallel_for(std::size_t n, Fn&& fn) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const std::size_t nt = std::min<std::size_t>(n, hw);
    std::atomic<std::size_t> next{0};
    std::exception_ptr err;
    std::mutex mu;
    auto work = [&] {
        for (std::size_t i; (i = next.fetch_add(1)) < n;) {
            try {
                fn(i);
            } catch (...) {
                std::lock_guard<std::mutex> lock(mu);
                if (!err) err = std::current_exception();
                next.store(n);
            }
        }
    };
    std::vector<std::thread> pool;
    for (std::size_t t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    if (err) std::rethrow_exception(err);
}

// Host -> device copy of a large pageable buffer through the engine's two pinned slots:
// the pageable->pinned memcpy runs on the host pool while the previous slot's DMA is in
// flight (pageable cudaMemcpy goes through the driver's single bounce buffer). Caller holds
// the engine lock; the copy is complete on `stream` when this returns.
void upload_pageable(b200::Engine& eng, void* dst, const void* src, std::size_t bytes,
                     cudaStream_t stream);

// Device f32 -> host f64 (exact widening): chunks of the f32 map stream through the engine's
// two pinned slots while host threads widen the previous chunk into `out`, so PCIe carries
// 4 bytes per value instead of 8. Caller holds the engine lock.
void download_widen(b200::Engine& eng, double* out, const float* d, std::size_t n, cudaStream_t stream);

// DDM_TRACE=1: wall time of each host phase on stderr ("[tag] phase ms")
struct Trace {
    const char* tag;
    bool on = std::getenv("DDM_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit Trace(const char* t) : tag(t) {}
    void lap(const char* what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[%s] %-12s %9.3f ms\n", tag, what,
                     std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

// Device errors surface as ddm::DeviceError, allocation failures / kernel limits as
// ddm::PlanError (the reference's "budget cannot hold the job" class).
template <class Fn>
auto guard_device(Fn&& fn) -> decltype(fn()) {
    try {
        return fn();
    } catch (const b200::CudaError& e) {
        const std::string w = e.what();
        if (w.find("out of memory") != std::string::npos) throw PlanError(w);
        throw DeviceError(w);
    } catch (const std::length_error& e) {
        throw PlanError(e.what());
    }
}

}  // namespace ddm::detail
