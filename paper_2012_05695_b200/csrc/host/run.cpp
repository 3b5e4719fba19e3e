// ddm::run on the GPU (reference `proj/core/src/scheduler.cpp:413-483` + `run_with_ft`
// `:62-180` + `merge_partials` `:485-542`).
//
// What stays the reference's: validation and error taxonomy, lag normalisation, the
// wave-vector cutoff list, the budget floor and group plan from `memory_bytes`, the exact
// counters (spatial_ffts = N x groups, temporal_ffts = 2 Q), the partial-file workspace
// with `before_merge`, d(0) = 0, the lag-major f64 map and `validate()`.
// What changes: frames are staged to HBM once (a contiguous source is one DMA); each group
// is one batched spatial pass + one temporal launch on the device (engine.cu); without an
// out_dir / before_merge seam the map is written in place on the device and copied back
// once, instead of the partial write + re-read + scatter the reference always performs.
#include "ddm/errors.hpp"
#include "ddm/scheduler.hpp"
#include "ddm/spectrum.hpp"
#include "ddm/temporal.hpp"
#include "run_internal.hpp"

#include <algorithm>
#include <barrier>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <thread>

#include <emmintrin.h>
#include <sys/mman.h>
#include <unistd.h>

namespace fs = std::filesystem;

namespace ddm {

namespace {

struct TempWorkspace {
    fs::path path;
    bool active = false;
    ~TempWorkspace() {
        if (active) {
            std::error_code ec;
            fs::remove_all(path, ec);
        }
    }
};

fs::path make_temp_dir() {
    static std::atomic<std::uint64_t> counter{0};
    const auto base = fs::temp_directory_path();
    for (;;) {
        const auto p = base / ("ddm-b200-run-" + std::to_string(::getpid()) + "-" +
                               std::to_string(counter.fetch_add(1)));
        std::error_code ec;
        if (fs::create_directory(p, ec)) return p;
        if (ec) throw IoError("cannot create temp workspace " + p.string());
    }
}

// Frames -> device buffer of the engine. A contiguous u16/u8 source is one copy; otherwise
// frames are read through the FrameSource interface into pinned staging, double buffered.
// ready != nullptr: a page-locked contiguous stack is uploaded asynchronously in chunks
// (Engine::upload_frames_async) and *ready receives the per-chunk events for
// RunSpec::frames_ready; disk_s is then left to the caller (Engine::upload_ms).
const void* stage_frames(b200::Engine& eng, const detail::Ingest& in, double& disk_s,
                         std::vector<std::pair<int, cudaEvent_t>>* ready = nullptr) {
    const auto t0 = std::chrono::steady_clock::now();
    const std::size_t ppf = std::size_t(in.width) * in.height;
    const std::size_t pb = in.u8 ? 1 : 2;
    void* d = eng.frame_buffer(ppf * pb * std::size_t(in.frames));
    cudaStream_t st = eng.stream();
    if (in.u8 || (in.source && in.source->contiguous())) {
        const void* src = in.u8 ? static_cast<const void*>(in.u8)
                                : static_cast<const void*>(in.source->contiguous());
        const std::size_t bytes = ppf * pb * std::size_t(in.frames);
        if (ready && detail::is_pinned(src) && bytes >= (std::size_t(8) << 20)) {
            // four chunks: the first spatial chunk starts once its half of the stack is in
            *ready = eng.upload_frames_async(d, src, in.frames, ppf * pb, 4);
            return d;
        }
        if (detail::is_pinned(src)) {
            b200::check(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st), "frame upload");
            b200::check(cudaStreamSynchronize(st), "sync");
        } else {
            // pageable: the host pool copies through the engine's pinned slots (the driver's
            // own pageable path is one thread through one bounce buffer, ~10 GB/s)
            detail::upload_pageable(eng, d, src, bytes, st);
        }
    } else {
        // FrameSource::read_frame is thread-safe (`frame_source.hpp:16-17`): frames of a
        // 32 MiB chunk are read by a pool of threads into pinned staging, the chunk's DMA to
        // HBM runs while the next chunk is read (two pinned buffers, cached by the engine)
        const int chunk = int(std::max<std::size_t>(1, std::min<std::size_t>(
                                  std::size_t(in.frames), (32u << 20) / (ppf * 2))));
        std::uint16_t* pinned[2] = {
            static_cast<std::uint16_t*>(eng.pinned(0, ppf * 2 * std::size_t(chunk))),
            static_cast<std::uint16_t*>(eng.pinned(1, ppf * 2 * std::size_t(chunk)))};
        cudaEvent_t done[2];
        for (int i = 0; i < 2; ++i) b200::check(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
        struct Events {
            cudaEvent_t* e;
            ~Events() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); }
        } ev_guard{done};
        const int nthreads = int(std::max(1u, std::min(8u, std::thread::hardware_concurrency())));
        int slot = 0;
        bool used[2] = {false, false};
        for (int f0 = 0; f0 < in.frames; f0 += chunk) {
            const int nf = std::min(chunk, in.frames - f0);
            if (used[slot]) b200::check(cudaEventSynchronize(done[slot]), "sync");
            std::uint16_t* buf = pinned[slot];
            // raw stacks: each task is a contiguous run of frames read as one positioned read
            const auto* raw = dynamic_cast<const RawStackFileSource*>(in.source);
            static const bool per_frame = std::getenv("DDM_INGEST_PER_FRAME") != nullptr;
            const int run = (raw && !per_frame) ? std::max(1, (nf + nthreads - 1) / nthreads) : 1;
            try {
                detail::parallel_for(std::size_t((nf + run - 1) / run), [&](std::size_t t) {
                    const int i = int(t) * run, cnt = std::min(run, nf - i);
                    if (raw) raw->read_frames(f0 + i, cnt, buf + std::size_t(i) * ppf);
                    else
                        for (int k = 0; k < cnt; ++k)
                            in.source->read_frame(f0 + i + k, {buf + std::size_t(i + k) * ppf, ppf});
                });
            } catch (...) {
                cudaStreamSynchronize(st);
                throw;
            }
            b200::check(cudaMemcpyAsync(static_cast<std::uint16_t*>(d) + std::size_t(f0) * ppf, buf,
                                        ppf * 2 * nf, cudaMemcpyHostToDevice, st), "frame upload");
            b200::check(cudaEventRecord(done[slot], st), "cudaEventRecord");
            used[slot] = true;
            slot ^= 1;
        }
        b200::check(cudaStreamSynchronize(st), "sync");
    }
    disk_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return d;
}

}  // namespace

namespace detail {

// WITHOUT_FT (`scheduler.cpp:182-286`) and Direct (`:288-323`, always f64): one spatial step
// and the pairwise kernel straight into the lag-major map. The reference's pass plan fixes the
// counters (spatial_ffts = N x passes; pairs = sum over lags > 0 of N - m) and its PlanError.
ResultArchive run_pairwise_core(const Ingest& in, const RunConfig& config,
                                const std::vector<std::int64_t>& lags, const WaveVectorSet& wv,
                                ResultArchive& archive,
                                double* out, std::chrono::steady_clock::time_point wall0) {
    const int W = in.width, H = in.height, N = in.frames;
    const bool direct = config.algorithm == Algorithm::Direct;
    const bool f64 = direct || config.precision == Precision::F64;
    std::uint64_t pairs = 0;
    for (const auto m : lags)
        if (m > 0) pairs += std::uint64_t(N - m);
    std::uint64_t passes = 0;
    if (!direct) {
        const MemoryBudget budget{config.memory_bytes, config.precision};
        passes = plan_without_ft(N, lags, budget, spectrum_bytes(W, H, config.precision)).chunks.size();
    }
    if (std::int64_t(N) * 16 > 227 * 1024)
        throw PlanError("sequence of " + std::to_string(N) + " frames exceeds the device pairwise "
                        "engine limit of " + std::to_string(227 * 1024 / 16));
    const std::int64_t plane = archive.map.plane_size();
    const std::int64_t total = plane * std::int64_t(lags.size());

    TimingBreakdown timing;
    b200::Engine& eng = b200::Engine::instance(config.device);
    std::lock_guard<std::mutex> lock(eng.mutex());
    cudaStream_t st = eng.stream();
    Trace trace("pairwise");
    const void* d_frames = stage_frames(eng, in, timing.disk);
    trace.lap("stage");

    b200::RunSpec spec;
    spec.W = W;
    spec.H = H;
    spec.N = N;
    spec.f64 = f64;
    spec.pixel_bytes = in.u8 ? 1 : 2;
    spec.d_frames = d_frames;
    spec.lags = lags;
    spec.flat.resize(std::size_t(wv.count()));
    spec.identity = true;
    for (std::int64_t k = 0; k < wv.count(); ++k) {
        spec.flat[std::size_t(k)] = wv.flat(k);
        if (spec.flat[std::size_t(k)] != k) spec.identity = false;
    }
    spec.groups = {{0, wv.count()}};
    double* d_map = static_cast<double*>(eng.buffer("map", std::size_t(total) * sizeof(double)));
    if (!spec.identity)
        b200::check(cudaMemsetAsync(d_map, 0, std::size_t(total) * sizeof(double), st), "memset");
    spec.d_out = d_map;
    spec.out_f64 = true;
    spec.out_stride = plane;
    b200::PhaseTimes times;
    eng.run_pairwise(spec, &times);
    trace.lap("device run");
    bool finite = true;
    double peak = 0.0, lowest = 0.0;
    b200::reduce_stats(d_map, total, st, &finite, &peak, &lowest);
    trace.lap("stats");
    if (!finite) throw InputError("result map contains non-finite values");
    const double eps = f64 ? 1e-9 : 1e-4;
    if (lowest < -eps * std::max(peak, 1.0))
        throw InputError("result map contains negative values beyond tolerance");
    PhaseClock clock;
    clock.start();
    detail::download_pageable(eng, out, d_map, std::size_t(total) * sizeof(double), st);
    clock.stop(timing.merge);
    trace.lap("map d2h");
    timing.step1 = times.spatial_ms * 1e-3;
    timing.step2 = times.temporal_ms * 1e-3;
    archive.counters.spatial_ffts = direct ? pairs : std::uint64_t(N) * passes;
    archive.counters.pairs = pairs;
    timing.finish(std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count());
    archive.timing = timing;
    return archive;
}

ResultArchive run_core(const Ingest& in, const RunConfig& config, double* out,
                       std::int64_t capacity) {
    const auto wall0 = std::chrono::steady_clock::now();
    if (config.workers < 1) throw InputError("workers must be at least 1");
    if (in.frames < 1) throw InputError("stack has no frames");
    if (in.width < 1 || in.height < 1) throw InputError("frame dimensions must be positive");
    const int W = in.width, H = in.height, N = in.frames;
    const std::vector<std::int64_t> lags =
        config.lags.empty() ? all_lags(N) : normalize_lags(config.lags, N);
    if (lags.empty()) throw InputError("no lags");
    const WaveVectorSet wv = cutoff_set(W, H, config.q_max);
    if (wv.count() < 1) throw InputError("wave-vector cutoff retains nothing");

    ResultArchive archive;
    archive.frames = N;
    archive.algorithm = to_string(config.algorithm);
    archive.precision = config.algorithm == Algorithm::Direct ? "f64" : to_string(config.precision);
    archive.q_max = config.q_max;
    archive.workers = config.workers;
    archive.map.width = W;
    archive.map.height = H;
    archive.map.frame_interval = in.frame_interval;
    archive.map.lags = lags;
    const std::int64_t plane = archive.map.plane_size();
    const std::int64_t total = plane * std::int64_t(lags.size());
    if (capacity < total) throw InputError("output capacity is smaller than lags x plane");

    if (config.algorithm != Algorithm::WithFt)
        return run_pairwise_core(in, config, lags, wv, archive, out, wall0);

    // budget floor + group plan (`scheduler.cpp:73-84`, `:365-384`)
    const MemoryBudget budget{config.memory_bytes, config.precision};
    const std::int64_t floor_bytes =
        spectrum_bytes(W, H, config.precision) + pad_length(N) * budget.complex_size();
    if (budget.bytes < floor_bytes)
        throw PlanError("memory budget " + std::to_string(budget.bytes) +
                        " bytes is below the working minimum of " + std::to_string(floor_bytes) +
                        " bytes");
    const GroupPlan plan = plan_with_ft(wv.count(), N, budget);
    const bool f64 = config.precision == Precision::F64;
    if (N > b200::max_frames(f64))
        throw PlanError("sequence of " + std::to_string(N) + " frames exceeds the device temporal "
                        "engine limit of " + std::to_string(b200::max_frames(f64)) + " (" +
                        to_string(config.precision) + ")");

    TimingBreakdown timing;
    b200::Engine& eng = b200::Engine::instance(config.device);
    std::lock_guard<std::mutex> lock(eng.mutex());
    cudaStream_t st = eng.stream();

    Trace trace("run");
    const bool keep_partials_early = !config.out_dir.empty() || bool(config.before_merge);
    std::vector<std::pair<int, cudaEvent_t>> frames_ready;
    const void* d_frames = stage_frames(eng, in, timing.disk, keep_partials_early ? nullptr : &frames_ready);
    trace.lap("stage");

    b200::RunSpec spec;
    spec.W = W;
    spec.H = H;
    spec.N = N;
    spec.f64 = f64;
    spec.pixel_bytes = in.u8 ? 1 : 2;
    spec.d_frames = d_frames;
    spec.lags = lags;
    spec.identity = !config.q_max.has_value() || wv.count() == plane;
    spec.flat.resize(std::size_t(wv.count()));
    for (std::int64_t k = 0; k < wv.count(); ++k) spec.flat[std::size_t(k)] = wv.flat(k);
    if (spec.identity)
        for (std::int64_t k = 0; k < wv.count(); ++k)
            if (spec.flat[std::size_t(k)] != k) spec.identity = false;
    spec.groups = plan.groups;
    spec.out_f64 = true;
    spec.out_stride = plane;

    const bool keep_partials = !config.out_dir.empty() || bool(config.before_merge);
    TempWorkspace temp;
    fs::path workspace = config.out_dir;
    b200::PhaseTimes times;
    PhaseClock clock;

    if (keep_partials) {
        if (workspace.empty()) {
            workspace = make_temp_dir();
            temp.path = workspace;
            temp.active = true;
        } else {
            std::error_code ec;
            fs::create_directories(workspace, ec);
            if (ec) throw IoError("cannot create workspace " + workspace.string());
        }
        spec.partial_mode = true;
        // Without a before_merge hook nothing can touch the partials between their write and
        // the merge, so the map is assembled from the same host values the files are written
        // from (identical to re-reading them); with a hook the files are merged as written.
        const bool direct = !config.before_merge;
        const bool in_place = direct && spec.identity && plan.group_count() == 1;
        if (direct && !spec.identity) std::memset(out, 0, std::size_t(total) * sizeof(double));
        spec.on_partial = [&](std::size_t g, const void* d_partial, std::int64_t gc) {
            clock.start();
            PartialResult p;
            p.group = std::int64_t(g);
            p.wv_begin = plan.groups[g].first;
            p.wv_end = plan.groups[g].second;
            p.width = W;
            p.height = H;
            p.frames = N;
            p.frame_interval = in.frame_interval;
            p.q_max = config.q_max;
            p.lags = lags;
            const std::size_t cnt = lags.size() * std::size_t(gc);
            double* host = out;  // lag-major [lags][plane] is this partial's own layout
            if (!in_place) {
                p.values.resize(cnt);
                host = p.values.data();
            }
            b200::check(cudaMemcpyAsync(host, d_partial, cnt * sizeof(double), cudaMemcpyDeviceToHost, st),
                        "partial copy");
            b200::check(cudaStreamSynchronize(st), "sync");
            trace.lap("partial d2h");
            detail::write_partial_payload(p, host, cnt, workspace);
            trace.lap("partial file");
            if (direct && !in_place)
                for (std::size_t li = 0; li < lags.size(); ++li) {
                    double* dst = out + li * std::size_t(plane);
                    const double* src = host + li * std::size_t(gc);
                    for (std::int64_t j = 0; j < gc; ++j) dst[spec.flat[std::size_t(p.wv_begin + j)]] = src[j];
                }
            clock.stop(timing.merge);
        };
        eng.run(spec, &times);
        // stale partials of an earlier run in out_dir: merge from the files, as the reference
        // does (and fails as it does)
        const bool stale = direct && list_partials(workspace).size() != plan.groups.size();
        if (!direct || stale) {
            if (config.before_merge) config.before_merge(workspace);
            clock.start();
            const ResultMap merged = merge_partials(list_partials(workspace));
            trace.lap("merge");
            if (merged.lags != lags || std::int64_t(merged.values.size()) != total)
                throw InputError("merged partials do not match the run layout");
            std::memcpy(out, merged.values.data(), std::size_t(total) * sizeof(double));
            clock.stop(timing.merge);
        }
        // the reference's run() ends with archive.validate() whatever the merge path: a
        // before_merge hook may have edited a partial's payload
        detail::validate_values(out, std::size_t(total), !f64);
        archive.map.values.clear();
    } else {
        // DDM_D2H_WIDEN=1 (f32 runs): the map stays f32 on the device and is widened on the
        // host while it streams back (exact; half the PCIe bytes). Opt-in: on the measured
        // box 16 host threads widen at ~67 GB/s, about the PCIe rate, so the C2 e2e moved
        // 32.2 -> 31.5 ms in one A/B round and regressed in the other.
        const bool widen = !f64 && total >= (std::int64_t(1) << 22) && detail::d2h_widen_enabled() &&
                           b200::f32_register_temporal(N);
        const std::size_t eb = widen ? sizeof(float) : sizeof(double);
        void* d_map = eng.buffer(widen ? "map32" : "map", std::size_t(total) * eb);
        if (!spec.identity)
            b200::check(cudaMemsetAsync(d_map, 0, std::size_t(total) * eb, st), "memset");
        spec.d_out = d_map;
        spec.out_f64 = !widen;
        spec.frames_ready = frames_ready;
        // a page-locked destination: the map streams out chunk by chunk while the temporal
        // pass runs (Engine::run, RunSpec::host_out)
        if (!widen && detail::is_pinned(out)) spec.host_out = out;
        trace.lap("prepare");
        // map copies still in flight into `out` are drained on every exit path
        struct DrainCopies {
            b200::Engine& e;
            ~DrainCopies() {
                try {
                    e.finish_host_out(nullptr);
                } catch (...) {
                }
            }
        } drain_copies{eng};
        eng.run(spec, &times);
        if (!frames_ready.empty()) timing.disk += eng.upload_ms() * 1e-3;
        trace.lap("device run");
        // validate on the device (`archive.cpp:44-58`): before the copy, or beside the map
        // chunks still streaming out (their copies are drained before any error is thrown)
        bool finite = true;
        double peak = 0.0, lowest = 0.0;
        if (widen)
            b200::reduce_stats(static_cast<const float*>(d_map), total, st, &finite, &peak, &lowest);
        else
            b200::reduce_stats(static_cast<const double*>(d_map), total, st, &finite, &peak, &lowest);
        trace.lap("stats");
        const bool streamed = eng.finish_host_out(&times);
        if (!finite) throw InputError("result map contains non-finite values");
        const double eps = f64 ? 1e-9 : 1e-4;
        if (lowest < -eps * std::max(peak, 1.0))
            throw InputError("result map contains negative values beyond tolerance");
        if (streamed) {
            // the copies overlapped the temporal pass; merge = their span
            timing.merge += times.d2h_ms * 1e-3;
        } else {
            clock.start();
            if (widen)
                download_widen(eng, out, static_cast<const float*>(d_map), std::size_t(total), st);
            else
                detail::download_pageable(eng, out, d_map, std::size_t(total) * sizeof(double), st);
            clock.stop(timing.merge);
        }
        trace.lap("map d2h");
    }
    timing.step1 = times.spatial_ms * 1e-3;
    timing.step2 = times.temporal_ms * 1e-3;
    archive.counters.spatial_ffts = std::uint64_t(N) * std::uint64_t(plan.group_count());
    archive.counters.temporal_ffts = 2 * std::uint64_t(wv.count());
    timing.finish(std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count());
    archive.timing = timing;
    return archive;
}

// Bulk host copy with non-temporal 16-byte stores: the destination (a DMA bounce slot, or a
// map the caller reads later) is not re-read soon, and streaming stores skip the read-for-
// ownership a cached store does (2 instead of 3 bytes of memory traffic per byte copied)
void stream_copy(void* dst, const void* src, std::size_t n) {
    auto* d = static_cast<unsigned char*>(dst);
    const auto* s = static_cast<const unsigned char*>(src);
    const std::size_t head = std::min<std::size_t>(n, (16 - (reinterpret_cast<std::uintptr_t>(d) & 15)) & 15);
    std::memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    const std::size_t blocks = n / 64;
    for (std::size_t i = 0; i < blocks; ++i, d += 64, s += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
        const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(d), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), e);
    }
    std::memcpy(d, s, n - blocks * 64);
    _mm_sfence();
}

bool d2h_widen_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DDM_D2H_WIDEN");
        return e && e[0] == '1';
    }();
    return on;
}

// f32 -> f64 (exact) with non-temporal 16-byte stores: the map is written once and read by
// the caller later, so the stores skip the read-for-ownership of cached stores
void widen_stream(double* dst, const float* src, std::size_t n) {
    std::size_t k = 0;
    for (; k < n && (reinterpret_cast<std::uintptr_t>(dst + k) & 15) != 0; ++k) dst[k] = double(src[k]);
    for (; k + 4 <= n; k += 4) {
        const __m128 v = _mm_loadu_ps(src + k);
        _mm_stream_pd(dst + k, _mm_cvtps_pd(v));
        _mm_stream_pd(dst + k + 2, _mm_cvtps_pd(_mm_movehl_ps(v, v)));
    }
    for (; k < n; ++k) dst[k] = double(src[k]);
    _mm_sfence();
}

void upload_pageable(b200::Engine& eng, void* dst, const void* src, std::size_t bytes,
                     cudaStream_t stream) {
    // chunks of 1-32 MiB, at least four per copy so the pool's memcpy of one chunk runs
    // while the previous chunk's DMA is in flight; each chunk is copied in 16 pieces
    const std::size_t kChunk = std::clamp<std::size_t>(bytes / 4, std::size_t(1) << 20,
                                                       std::size_t(32) << 20);
    if (bytes < (std::size_t(1) << 20)) {
        b200::check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream), "upload");
        b200::check(cudaStreamSynchronize(stream), "sync");
        return;
    }
    const std::size_t kPiece = (kChunk + 15) / 16;
    cudaEvent_t done[2];
    for (auto& e : done) b200::check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    try {
        const char* s = static_cast<const char*>(src);
        char* d = static_cast<char*>(dst);
        for (std::size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
            const int slot = int(i & 1);
            const std::size_t n = std::min(kChunk, bytes - off);
            char* pin = static_cast<char*>(eng.pinned(slot, kChunk));
            if (i >= 2) b200::check(cudaEventSynchronize(done[slot]), "event sync");
            parallel_for((n + kPiece - 1) / kPiece, [&](std::size_t k) {
                const std::size_t o = k * kPiece;
                stream_copy(pin + o, s + off + o, std::min(kPiece, n - o));
            });
            b200::check(cudaMemcpyAsync(d + off, pin, n, cudaMemcpyHostToDevice, stream), "upload");
            b200::check(cudaEventRecord(done[slot], stream), "event");
        }
        b200::check(cudaStreamSynchronize(stream), "sync");
    } catch (...) {
        cudaStreamSynchronize(stream);
        for (auto e : done) cudaEventDestroy(e);
        throw;
    }
    for (auto e : done) cudaEventDestroy(e);
}

void download_pageable(b200::Engine& eng, void* dst, const void* src, std::size_t bytes,
                       cudaStream_t stream) {
    if (bytes < (std::size_t(1) << 20) || is_pinned(dst)) {
        b200::check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream), "download");
        b200::check(cudaStreamSynchronize(stream), "sync");
        return;
    }
    // a fresh destination (np.empty, a new std::vector) faults in on first touch: ask for
    // transparent huge pages over it first (512x fewer faults where THP is in madvise mode)
    if (bytes >= (std::size_t(8) << 20)) {
        constexpr std::uintptr_t kHuge = std::uintptr_t(2) << 20;
        const auto b = (reinterpret_cast<std::uintptr_t>(dst) + kHuge - 1) & ~(kHuge - 1);
        const auto e = (reinterpret_cast<std::uintptr_t>(dst) + bytes) & ~(kHuge - 1);
        if (e > b) ::madvise(reinterpret_cast<void*>(b), e - b, MADV_HUGEPAGE);
    }
    // DMA of chunk i+1 into one pinned slot while the pool copies chunk i out of the other
    const std::size_t kChunk = std::clamp<std::size_t>(bytes / 4, std::size_t(1) << 20,
                                                       std::size_t(32) << 20);
    const std::size_t kPiece = (kChunk + 15) / 16;
    const std::size_t chunks = (bytes + kChunk - 1) / kChunk;
    cudaEvent_t done[2];
    for (auto& e : done) b200::check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    char* pin[2] = {static_cast<char*>(eng.pinned(0, kChunk)), static_cast<char*>(eng.pinned(1, kChunk))};
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    auto issue = [&](std::size_t i) {
        const std::size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
        b200::check(cudaMemcpyAsync(pin[i & 1], s + off, n, cudaMemcpyDeviceToHost, stream), "download");
        b200::check(cudaEventRecord(done[i & 1], stream), "event");
    };
    try {
        issue(0);
        for (std::size_t i = 0; i < chunks; ++i) {
            if (i + 1 < chunks) issue(i + 1);
            b200::check(cudaEventSynchronize(done[i & 1]), "event sync");
            const std::size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
            const char* p = pin[i & 1];
            parallel_for((n + kPiece - 1) / kPiece, [&](std::size_t k) {
                const std::size_t o = k * kPiece;
                stream_copy(d + off + o, p + o, std::min(kPiece, n - o));
            });
            // slot i & 1 is reused by chunk i + 2, issued after this copy-out
        }
        b200::check(cudaStreamSynchronize(stream), "sync");
    } catch (...) {
        cudaStreamSynchronize(stream);
        for (auto e : done) cudaEventDestroy(e);
        throw;
    }
    for (auto e : done) cudaEventDestroy(e);
}

bool is_pinned(const void* p) {
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeHost;
}

void download_widen(b200::Engine& eng, double* out, const float* d, std::size_t n, cudaStream_t stream) {
    constexpr std::size_t kChunk = std::size_t(4) << 20;  // values (16 MiB of f32) per slot
    const std::size_t chunks = (n + kChunk - 1) / kChunk;
    if (chunks == 0) return;
    float* pin[2] = {static_cast<float*>(eng.pinned(0, kChunk * sizeof(float))),
                     static_cast<float*>(eng.pinned(1, kChunk * sizeof(float)))};
    cudaEvent_t ev[2];
    for (auto& e : ev) b200::check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cudaError_t err = cudaSuccess;
    auto issue = [&](std::size_t i) {
        const std::size_t off = i * kChunk, m = std::min(kChunk, n - off);
        if (err == cudaSuccess) err = cudaMemcpyAsync(pin[i & 1], d + off, m * sizeof(float), cudaMemcpyDeviceToHost, stream);
        if (err == cudaSuccess) err = cudaEventRecord(ev[i & 1], stream);
    };
    issue(0);
    if (chunks > 1) issue(1);
    const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::barrier sync(std::ptrdiff_t(T), [] () noexcept {});
    auto worker = [&](unsigned t) {
        for (std::size_t i = 0; i < chunks; ++i) {
            if (t == 0 && err == cudaSuccess) err = cudaEventSynchronize(ev[i & 1]);
            sync.arrive_and_wait();  // chunk i is in slot i & 1
            const std::size_t off = i * kChunk, m = std::min(kChunk, n - off);
            const std::size_t b = m * t / T, e = m * (t + 1) / T;
            widen_stream(out + off + b, pin[i & 1] + b, e - b);
            sync.arrive_and_wait();  // slot i & 1 is free again
            if (t == 0 && i + 2 < chunks) issue(i + 2);
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < T; ++t) pool.emplace_back(worker, t);
    worker(0);
    for (auto& th : pool) th.join();
    cudaStreamSynchronize(stream);
    for (auto e : ev) cudaEventDestroy(e);
    b200::check(err, "map download");
}

}  // namespace detail

ResultArchive run_into(FrameSource& source, const RunConfig& config, double* out,
                       std::int64_t capacity) {
    detail::Ingest in;
    in.source = &source;
    in.width = source.width();
    in.height = source.height();
    in.frames = source.frames();
    in.frame_interval = source.frame_interval();
    return detail::guard_device([&] { return detail::run_core(in, config, out, capacity); });
}

ResultArchive run(FrameSource& source, const RunConfig& config) {
    if (source.frames() < 1) throw InputError("stack has no frames");
    if (config.workers < 1) throw InputError("workers must be at least 1");
    const std::int64_t n_lags =
        config.lags.empty() ? source.frames() : std::int64_t(config.lags.size());
    detail::Trace trace("ddm::run");
    const std::size_t count =
        std::size_t(n_lags) * std::size_t(source.height()) * std::size_t(half_cols(source.width()));
    std::vector<double> values;
    values.reserve(count);
    // GB-sized maps: ask for transparent huge pages before the zero fill faults the range in
    // (4 KiB faults cost ~0.35 s per GiB; THP "madvise" mode is common)
    if (count * sizeof(double) >= (std::size_t(64) << 20)) {
        constexpr std::uintptr_t kHuge = std::uintptr_t(2) << 20;
        const auto b = (reinterpret_cast<std::uintptr_t>(values.data()) + kHuge - 1) & ~(kHuge - 1);
        const auto e = (reinterpret_cast<std::uintptr_t>(values.data() + count)) & ~(kHuge - 1);
        if (e > b) ::madvise(reinterpret_cast<void*>(b), e - b, MADV_HUGEPAGE);
    }
    values.resize(count);
    trace.lap("map alloc");
    ResultArchive a = run_into(source, config, values.data(), std::int64_t(values.size()));
    trace.lap("run_into");
    values.resize(std::size_t(a.map.plane_size()) * a.map.lags.size());
    a.map.values = std::move(values);
    return a;
}

ResultMap merge_partials(const std::vector<fs::path>& files) {
    if (files.empty()) throw InputError("no partial files to merge");
    std::vector<PartialResult> parts;
    parts.reserve(files.size());
    for (const auto& f : files) parts.push_back(read_partial(f));
    const PartialResult& first = parts.front();
    for (const auto& p : parts)
        if (p.width != first.width || p.height != first.height || p.frames != first.frames ||
            p.frame_interval != first.frame_interval || p.q_max != first.q_max || p.lags != first.lags)
            throw InputError("partial files disagree on geometry or lags");
    std::sort(parts.begin(), parts.end(),
              [](const PartialResult& a, const PartialResult& b) { return a.wv_begin < b.wv_begin; });
    const WaveVectorSet wv = cutoff_set(int(first.width), int(first.height), first.q_max);
    std::int64_t cursor = 0;
    for (const auto& p : parts) {
        if (p.wv_begin < cursor)
            throw InputError("partial files overlap at wave vector " + std::to_string(p.wv_begin));
        if (p.wv_begin > cursor)
            throw InputError("partial files leave a gap before wave vector " + std::to_string(p.wv_begin));
        cursor = p.wv_end;
    }
    if (cursor != wv.count())
        throw InputError("partial files cover " + std::to_string(cursor) + " of " +
                         std::to_string(wv.count()) + " wave vectors");
    ResultMap map;
    map.width = first.width;
    map.height = first.height;
    map.frame_interval = first.frame_interval;
    map.lags = first.lags;
    map.values.assign(std::size_t(map.plane_size()) * map.lags.size(), 0.0);
    for (const auto& p : parts) {
        const auto cnt = std::size_t(p.wv_count());
        for (std::size_t li = 0; li < p.lags.size(); ++li) {
            auto plane = map.lag_plane(std::int64_t(li));
            const double* src = p.values.data() + li * cnt;
            for (std::size_t j = 0; j < cnt; ++j)
                plane[std::size_t(wv.flat(p.wv_begin + std::int64_t(j)))] = src[j];
        }
    }
    return map;
}

}  // namespace ddm
