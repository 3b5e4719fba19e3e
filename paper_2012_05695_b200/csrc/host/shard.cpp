// Sharded WITH_FT plan: frames split across ranks for the spatial step,
// wave vectors split into the reference's contiguous group slices for the temporal step
// (`plan_with_ft`, `scheduler.cpp:365-384`: groups [b, min(b + K, Q)) of capacity K).
#include "ddm/errors.hpp"
#include "ddm/scheduler.hpp"

#include <algorithm>
#include <string>

namespace ddm {

ShardPlan plan_shards(std::int64_t q_count, std::int64_t frames, int ranks) {
    if (ranks < 1 || ranks > 8) throw InputError("ranks must be in [1, 8]");
    if (q_count < 1) throw InputError("need at least one wave vector");
    if (frames < ranks) throw InputError("need at least one frame per rank");
    ShardPlan p;
    p.ranks = ranks;
    p.frames = frames;
    p.q_count = q_count;
    p.frame_begin.assign(std::size_t(ranks) + 1, 0);
    p.q_begin.assign(std::size_t(ranks) + 1, 0);
    // frames: whole pairs per rank when there are enough (every segment then has an even
    // length, the temporal engine's bulk-copy granule), the odd frame of an odd N last
    const std::int64_t pairs = frames / 2;
    const bool paired = pairs >= ranks;
    const std::int64_t units = paired ? pairs : frames;
    for (int r = 0; r < ranks; ++r) {
        const std::int64_t u = units / ranks + (r < units % ranks ? 1 : 0);
        p.frame_begin[std::size_t(r) + 1] = p.frame_begin[std::size_t(r)] + (paired ? 2 * u : u);
    }
    p.frame_begin[std::size_t(ranks)] = frames;
    // wave vectors: GroupPlan with capacity K = ceil(Q / ranks)
    const std::int64_t K = (q_count + ranks - 1) / ranks;
    for (int r = 0; r <= ranks; ++r) p.q_begin[std::size_t(r)] = std::min<std::int64_t>(q_count, r * K);
    return p;
}

}  // namespace ddm
