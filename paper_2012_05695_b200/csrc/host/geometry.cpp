// Host-side planning and geometry: wave-vector cutoff list (`spectrum.cpp:65-84`), lag lists
// (`result_map.cpp:22-57`), group planning (`scheduler.cpp:357-384`), enum names.
#include "ddm/errors.hpp"
#include "ddm/result_map.hpp"
#include "ddm/scheduler.hpp"
#include "ddm/spectrum.hpp"

#include <algorithm>
#include <cmath>

namespace ddm {

WaveVectorSet cutoff_set(int width, int height, std::optional<double> q_max) {
    if (width < 1 || height < 1) throw InputError("cutoff_set: dimensions must be positive");
    if (q_max && *q_max < 0.0) throw InputError("cutoff_set: q_max must be non-negative");
    WaveVectorSet set;
    set.width = width;
    set.height = height;
    set.q_max = q_max;
    const int hc = half_cols(width);
    set.indices.reserve(std::size_t(height) * hc);
    for (int r = 0; r < height; ++r)
        for (int c = 0; c < hc; ++c)
            if (!q_max || q_magnitude(r, c, height) <= *q_max) set.indices.push_back({r, c});
    return set;
}

std::int64_t ResultMap::lag_index(std::int64_t lag) const {
    const auto it = std::lower_bound(lags.begin(), lags.end(), lag);
    return (it == lags.end() || *it != lag) ? -1 : std::int64_t(it - lags.begin());
}

bool same_layout(const ResultMap& a, const ResultMap& b) {
    return a.width == b.width && a.height == b.height && a.lags == b.lags &&
           a.frame_interval == b.frame_interval;
}

double max_abs_difference(const ResultMap& a, const ResultMap& b) {
    if (!same_layout(a, b)) throw InputError("max_abs_difference: result layouts differ");
    double worst = 0.0;
    for (std::size_t i = 0; i < a.values.size(); ++i)
        worst = std::max(worst, std::abs(a.values[i] - b.values[i]));
    return worst;
}

std::vector<std::int64_t> normalize_lags(std::vector<std::int64_t> lags, std::int64_t frames) {
    std::sort(lags.begin(), lags.end());
    for (std::size_t i = 0; i < lags.size(); ++i) {
        if (lags[i] < 0 || lags[i] >= frames)
            throw InputError("lag " + std::to_string(lags[i]) + " outside [0, " +
                             std::to_string(frames - 1) + "]");
        if (i && lags[i] == lags[i - 1]) throw InputError("duplicate lag " + std::to_string(lags[i]));
    }
    return lags;
}

std::vector<std::int64_t> all_lags(std::int64_t frames) {
    std::vector<std::int64_t> v(std::size_t(std::max<std::int64_t>(frames, 0)));
    for (std::int64_t m = 0; m < frames; ++m) v[std::size_t(m)] = m;
    return v;
}

std::vector<std::int64_t> log_lags(std::int64_t frames) {
    std::vector<std::int64_t> v;
    for (std::int64_t m = 1; m < frames; m <<= 1) v.push_back(m);
    if (frames > 1 && (v.empty() || v.back() != frames - 1)) v.push_back(frames - 1);
    return v;
}

Algorithm parse_algorithm(const std::string& name) {
    if (name == "with_ft") return Algorithm::WithFt;
    if (name == "without_ft") return Algorithm::WithoutFt;
    if (name == "direct") return Algorithm::Direct;
    throw InputError("unknown algorithm '" + name + "'");
}

Precision parse_precision(const std::string& name) {
    if (name == "f32") return Precision::F32;
    if (name == "f64") return Precision::F64;
    throw InputError("unknown precision '" + name + "'");
}

std::string to_string(Algorithm a) {
    switch (a) {
    case Algorithm::WithFt: return "with_ft";
    case Algorithm::WithoutFt: return "without_ft";
    case Algorithm::Direct: return "direct";
    }
    return "?";
}

std::string to_string(Precision p) { return p == Precision::F32 ? "f32" : "f64"; }

std::int64_t bytes_per_complex(Precision p) { return p == Precision::F32 ? 8 : 16; }

std::int64_t spectrum_bytes(std::int64_t width, std::int64_t height, Precision p) {
    return height * (width / 2 + 1) * bytes_per_complex(p);
}

GroupPlan plan_with_ft(std::int64_t q_count, std::int64_t frames, const MemoryBudget& budget) {
    if (frames < 1) throw InputError("plan_with_ft: frame count must be at least 1");
    if (q_count < 1) throw InputError("plan_with_ft: empty wave-vector set");
    const std::int64_t per = frames * budget.complex_size();
    const std::int64_t cap = budget.bytes > 0 ? budget.bytes / per : 0;
    if (cap < 1)
        throw PlanError("memory budget " + std::to_string(budget.bytes) +
                        " bytes cannot hold one " + std::to_string(frames) + "-frame sequence (" +
                        std::to_string(per) + " bytes)");
    GroupPlan plan;
    plan.capacity = cap;
    for (std::int64_t b = 0; b < q_count; b += cap) plan.groups.emplace_back(b, std::min(b + cap, q_count));
    return plan;
}

ChunkPlan plan_without_ft(std::int64_t frames, std::vector<std::int64_t> lags,
                          const MemoryBudget& budget, std::int64_t bytes_per_spectrum) {
    // `scheduler.cpp:386-411`
    if (bytes_per_spectrum < 1) throw InputError("plan_without_ft: bad spectrum size");
    lags = normalize_lags(std::move(lags), frames);
    const std::int64_t capacity = budget.bytes > 0 ? budget.bytes / bytes_per_spectrum : 0;
    if (capacity < 2)
        throw PlanError("memory budget " + std::to_string(budget.bytes) + " bytes admits fewer than two " +
                        std::to_string(bytes_per_spectrum) + "-byte spectra");
    ChunkPlan plan;
    plan.capacity = capacity;
    const std::int64_t width = capacity - 1;  // lags per pass
    for (const std::int64_t lag : lags) {
        if (lag == 0) continue;  // zero by definition, never scheduled
        if (plan.chunks.empty() || lag > plan.chunks.back().lo + width - 1) plan.chunks.push_back({lag, lag, {}});
        plan.chunks.back().hi = lag;
        plan.chunks.back().lags.push_back(lag);
    }
    return plan;
}

}  // namespace ddm
