// Internal glue between the reference-mirroring C++ API and the device engine.
#pragma once

#include "../engine.hpp"
#include "ddm/archive.hpp"
#include "ddm/errors.hpp"
#include "ddm/frame_source.hpp"
#include "ddm/scheduler.hpp"

#include <cstdint>
#include <new>
#include <string>

namespace ddm::detail {

// Either a FrameSource (u16) or a raw u8 frame-major buffer.
struct Ingest {
    const FrameSource* source = nullptr;
    const std::uint8_t* u8 = nullptr;
    int width = 0, height = 0, frames = 0;
    double frame_interval = 1.0;
};

ResultArchive run_core(const Ingest& in, const RunConfig& config, double* out,
                       std::int64_t capacity);

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
