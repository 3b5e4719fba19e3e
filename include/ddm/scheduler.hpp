// ddm-b200: the drop-in entry point `ddm::run` (reference `proj/core/include/ddm/scheduler.hpp`).
// Algorithm::WithFt runs on the GPU: frames are staged to HBM once, each wave-vector group
// is one batched spatial pass + one fused temporal launch, results come back lag-major in
// f64. Group planning, counters, partial files, before_merge and validation keep the
// reference semantics. WithoutFt (the O(N * lags) spectral differences) and Direct (Eq. 1,
// always f64) run on the GPU too, through the pairwise kernel (csrc/pairwise.cu).
#ifndef DDM_B200_SCHEDULER_HPP
#define DDM_B200_SCHEDULER_HPP

#include "ddm/archive.hpp"
#include "ddm/frame_source.hpp"
#include "ddm/result_map.hpp"

#include <cstdint>
#include <filesystem>
#include <functional>
#include <optional>
#include <string>
#include <utility>
#include <vector>

namespace ddm {

enum class Algorithm { WithFt, WithoutFt, Direct };
enum class Precision { F32, F64 };

Algorithm parse_algorithm(const std::string& name);
Precision parse_precision(const std::string& name);
std::string to_string(Algorithm algorithm);
std::string to_string(Precision precision);

std::int64_t bytes_per_complex(Precision precision);
std::int64_t spectrum_bytes(std::int64_t width, std::int64_t height, Precision precision);

struct MemoryBudget {
    std::int64_t bytes = 0;
    Precision precision = Precision::F64;
    std::int64_t complex_size() const { return bytes_per_complex(precision); }
};

/// Contiguous wave-vector groups of at most K = floor(bytes / (N * bytes_per_complex)).
struct GroupPlan {
    std::int64_t capacity = 0;
    std::vector<std::pair<std::int64_t, std::int64_t>> groups;
    std::int64_t group_count() const { return std::int64_t(groups.size()); }
};

GroupPlan plan_with_ft(std::int64_t q_count, std::int64_t frames, const MemoryBudget& budget);

/// WITHOUT_FT lag passes: a pass holds capacity - 1 consecutive lags' spectra ring
/// (`plan_without_ft`, scheduler.cpp:386-411). On the device every pass shares one spatial
/// step; the plan fixes the reference's counters and PlanError semantics.
struct LagChunk {
    std::int64_t lo = 0, hi = 0;
    std::vector<std::int64_t> lags;
};
struct ChunkPlan {
    std::int64_t capacity = 0;
    std::vector<LagChunk> chunks;
    std::int64_t passes() const { return std::int64_t(chunks.size()); }
};
ChunkPlan plan_without_ft(std::int64_t frames, std::vector<std::int64_t> lags,
                          const MemoryBudget& budget, std::int64_t bytes_per_spectrum);

/// Sharded WITH_FT over `ranks` GPUs (b200 extension). Rank r transforms
/// frames [frame_begin[r], frame_begin[r+1]) in the spatial step and owns wave vectors
/// [q_begin[r], q_begin[r+1]) in the temporal step; the wave-vector slices are the
/// reference's GroupPlan with capacity ceil(Q / ranks) (plan_with_ft), so every rank's output
/// is one PartialResult. Frame shards are even-sized where N allows (bulk-copy alignment).
struct ShardPlan {
    int ranks = 1;
    std::int64_t frames = 0, q_count = 0;
    std::vector<std::int64_t> frame_begin;  // ranks + 1
    std::vector<std::int64_t> q_begin;      // ranks + 1
    std::int64_t frames_of(int r) const { return frame_begin[r + 1] - frame_begin[r]; }
    std::int64_t q_of(int r) const { return q_begin[r + 1] - q_begin[r]; }
};

ShardPlan plan_shards(std::int64_t q_count, std::int64_t frames, int ranks);

struct RunConfig {
    Algorithm algorithm = Algorithm::WithFt;
    Precision precision = Precision::F64;
    std::vector<std::int64_t> lags;  // empty = all lags 0..N-1
    std::optional<double> q_max;
    std::int64_t memory_bytes = 0;
    int workers = 2;                 // validated (>= 1); values never depend on it
    std::filesystem::path out_dir;   // non-empty: partials/ kept here
    std::function<void(const std::filesystem::path&)> before_merge;
    int device = 0;                  // CUDA device (b200 extension)
};

ResultArchive run(FrameSource& source, const RunConfig& config);

/// Run WITH_FT writing the lag-major f64 map straight into `out` (capacity values); the
/// archive's map.values stays empty. Used by the C-ABI to avoid a second copy.
ResultArchive run_into(FrameSource& source, const RunConfig& config, double* out,
                       std::int64_t capacity);

ResultMap merge_partials(const std::vector<std::filesystem::path>& files);

/// What `ddm analyze` writes (`tools/ddm_cli.cpp:206-240`), as a library call: run with the
/// workspace in `out_dir`, write_results (d_m<lag>.bin + index.json), the ring average
/// (radial.csv) and the ring fits (fits.csv). The CLI's own run.json echo is not written.
ResultArchive analyze(FrameSource& source, RunConfig config, const std::filesystem::path& out_dir);

struct CompareReport;
/// `ddm compare` as a library call: `config` with each algorithm in turn (analysis.hpp).
CompareReport compare(FrameSource& source, const RunConfig& config, Algorithm a, Algorithm b);

} // namespace ddm

#endif
