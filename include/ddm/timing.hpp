// ddm-b200: phase timing and exact operation counters, same fields and semantics as the
// reference (`proj/core/include/ddm/timing.hpp:12-65`). On the GPU path step1 / step2 are
// device time of the spatial and temporal kernels; disk covers frame reads + host->device
// staging; merge covers device->host result transfer and partial-file I/O.
#ifndef DDM_B200_TIMING_HPP
#define DDM_B200_TIMING_HPP

#include <chrono>
#include <cstdint>

namespace ddm {

struct TimingBreakdown {
    double disk = 0.0;
    double step1 = 0.0;
    double step2 = 0.0;
    double merge = 0.0;
    double other = 0.0;
    double total = 0.0;

    double named_sum() const { return disk + step1 + step2 + merge; }
    void finish(double wall_total) {
        total = wall_total;
        const double rest = total - named_sum();
        other = rest > 0.0 ? rest : 0.0;
    }
};

/// spatial_ffts: 2D transforms executed (frames x groups); temporal_ffts: 1D transforms,
/// two per wave vector; pairs: WITHOUT_FT difference updates (always 0 on this path).
struct RunCounters {
    std::uint64_t spatial_ffts = 0;
    std::uint64_t temporal_ffts = 0;
    std::uint64_t pairs = 0;

    RunCounters& operator+=(const RunCounters& o) {
        spatial_ffts += o.spatial_ffts;
        temporal_ffts += o.temporal_ffts;
        pairs += o.pairs;
        return *this;
    }
};

class PhaseClock {
public:
    void start() { t0_ = std::chrono::steady_clock::now(); }
    void stop(double& acc) {
        acc += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
    }

private:
    std::chrono::steady_clock::time_point t0_{};
};

} // namespace ddm

#endif
