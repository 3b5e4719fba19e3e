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
#include <type_traits>
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

// fn(i) for i in [0, n) on up to 16 host threads of a persistent pool (pool.cpp: workers are
// created once per process, so a call costs a wake-up, not thread creation); the first
// exception is rethrown. Calls from inside a pool task run inline.
void parallel_for_impl(std::size_t n, void (*call)(void*, std::size_t), void* ctx);

template <class Fn>
void parallel_for(std::size_t n, Fn&& fn) {
    using F = std::remove_reference_t<Fn>;
    parallel_for_impl(n, [](void* c, std::size_t i) { (*static_cast<F*>(c))(i); },
                      const_cast<void*>(static_cast<const void*>(&fn)));
}

// Host -> device copy of a large pageable buffer through the engine's two pinned slots:
// the pageable->pinned memcpy runs on the host pool while the previous slot's DMA is in
// flight (pageable cudaMemcpy goes through the driver's single bounce buffer). Caller holds
// the engine lock; the copy is complete on `stream` when this returns.
void upload_pageable(b200::Engine& eng, void* dst, const void* src, std::size_t bytes,
                     cudaStream_t stream);
// Device -> host copy into pageable memory through the two pinned slots (pinned or small
// destinations: one cudaMemcpy); complete when this returns
void download_pageable(b200::Engine& eng, void* dst, const void* src, std::size_t bytes,
                       cudaStream_t stream);
// page-locked (cudaMallocHost / registered) host memory: DMA reads it directly
bool is_pinned(const void* p);

// Device f32 -> host f64 (exact widening): chunks of the f32 map stream through the engine's
// two pinned slots while host threads widen the previous chunk into `out`, so PCIe carries
// 4 bytes per value instead of 8. Caller holds the engine lock.
void download_widen(b200::Engine& eng, double* out, const float* d, std::size_t n, cudaStream_t stream);
// f32 -> f64 with non-temporal stores (run.cpp)
void widen_stream(double* dst, const float* src, std::size_t n);
// DDM_D2H_WIDEN=1: f32 maps leave the device as f32 and are widened on the host
bool d2h_widen_enabled();

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
