// extern "C" boundary (include/ddm_b200.h). Every entry point converts the library's
// exceptions into status codes + a thread-local message; nothing throws across it.
#include "ddm_b200.h"

#include "ddm/analysis.hpp"
#include "ddm/bench.hpp"
#include "ddm/errors.hpp"
#include "ddm/image_stack.hpp"
#include "ddm/scheduler.hpp"
#include "ddm/spectrum.hpp"
#include "ddm/synth.hpp"
#include "ddm/temporal.hpp"
#include "run_internal.hpp"
#include "session.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <new>
#include <optional>
#include <string>
#include <type_traits>

namespace {

thread_local std::string g_last_error;

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_last_error.clear();
        return DDM_B200_OK;
    } catch (const ddm::InputError& e) {
        g_last_error = e.what();
        return DDM_B200_E_INPUT;
    } catch (const ddm::PlanError& e) {
        g_last_error = e.what();
        return DDM_B200_E_PLAN;
    } catch (const ddm::IoError& e) {
        g_last_error = e.what();
        return DDM_B200_E_IO;
    } catch (const ddm::DeviceError& e) {
        g_last_error = e.what();
        return DDM_B200_E_CUDA;
    } catch (const ddm::b200::CudaError& e) {
        g_last_error = e.what();
        return DDM_B200_E_CUDA;
    } catch (const std::bad_alloc& e) {
        g_last_error = "out of host memory";
        return DDM_B200_E_PLAN;
    } catch (const std::length_error& e) {
        g_last_error = e.what();
        return DDM_B200_E_PLAN;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return DDM_B200_E_INTERNAL;
    } catch (...) {
        g_last_error = "unknown error";
        return DDM_B200_E_INTERNAL;
    }
}

ddm::RunConfig to_config(const ddm_b200_run_config* c) {
    if (!c) throw ddm::InputError("null run config");
    ddm::RunConfig r;
    r.algorithm = c->algorithm == 0 ? ddm::Algorithm::WithFt
                  : c->algorithm == 1 ? ddm::Algorithm::WithoutFt
                                      : ddm::Algorithm::Direct;
    r.precision = c->precision == 0 ? ddm::Precision::F32 : ddm::Precision::F64;
    if (c->lags && c->n_lags > 0) r.lags.assign(c->lags, c->lags + c->n_lags);
    if (c->has_q_max) r.q_max = c->q_max;
    r.memory_bytes = c->memory_bytes;
    r.workers = c->workers;
    if (c->out_dir && c->out_dir[0]) r.out_dir = c->out_dir;
    if (c->before_merge) {
        auto fn = c->before_merge;
        void* user = c->before_merge_user;
        r.before_merge = [fn, user](const std::filesystem::path& ws) { fn(ws.string().c_str(), user); };
    }
    r.device = c->device;
    return r;
}

void emit(const ddm::ResultArchive& a, int64_t* out_lags, int64_t* out_n_lags,
          ddm_b200_counters* counters, ddm_b200_timing* timing) {
    if (out_lags) std::copy(a.map.lags.begin(), a.map.lags.end(), out_lags);
    if (out_n_lags) *out_n_lags = int64_t(a.map.lags.size());
    if (counters) {
        counters->spatial_ffts = a.counters.spatial_ffts;
        counters->temporal_ffts = a.counters.temporal_ffts;
        counters->pairs = a.counters.pairs;
    }
    if (timing) {
        timing->disk = a.timing.disk;
        timing->step1 = a.timing.step1;
        timing->step2 = a.timing.step2;
        timing->merge = a.timing.merge;
        timing->other = a.timing.other;
        timing->total = a.timing.total;
    }
}

// Runs `fn` on the engine stream ordered after the caller's stream (cudaStream_t, may be
// NULL), and orders the caller's stream after it.
template <class Fn>
void on_engine_stream(ddm::b200::Engine& eng, void* stream, Fn&& fn) {
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaEvent_t ev;
    ddm::b200::check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    struct Destroy {
        cudaEvent_t e;
        ~Destroy() { cudaEventDestroy(e); }
    } guard{ev};
    ddm::b200::check(cudaEventRecord(ev, user), "event record");
    ddm::b200::check(cudaStreamWaitEvent(eng.stream(), ev, 0), "stream wait");
    fn();
    ddm::b200::check(cudaEventRecord(ev, eng.stream()), "event record");
    ddm::b200::check(cudaStreamWaitEvent(user, ev, 0), "stream wait");
}

}  // namespace

extern "C" {

const char* ddm_b200_last_error(void) { return g_last_error.c_str(); }

int ddm_b200_version(int* major, int* minor, int* patch) {
    if (major) *major = 0;
    if (minor) *minor = 1;
    if (patch) *patch = 0;
    return DDM_B200_OK;
}

int ddm_b200_device_count(int* count) {
    return guarded([&] {
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) n = 0;
        *count = n;
    });
}

int ddm_b200_last_engines(int device, char* buf, int64_t capacity) {
    return guarded([&] {
        if (!buf || capacity < 1) throw ddm::InputError("null or empty buffer");
        auto& eng = ddm::b200::Engine::instance(device);
        std::lock_guard<std::mutex> lock(eng.mutex());
        const std::string& s = eng.last_engines();
        const size_t n = std::min<size_t>(s.size(), (size_t)capacity - 1);
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    });
}

int64_t ddm_b200_pad_length(int64_t n) {
    if (n < 1) return -1;
    return ddm::pad_length(n);
}

int64_t ddm_b200_max_frames(int precision) { return ddm::b200::max_frames(precision != 0); }

int ddm_b200_plan_with_ft(int64_t q_count, int64_t frames, int64_t bytes, int precision,
                          int64_t* capacity, int64_t* groups) {
    return guarded([&] {
        const auto p = ddm::plan_with_ft(
            q_count, frames, {bytes, precision == 0 ? ddm::Precision::F32 : ddm::Precision::F64});
        *capacity = p.capacity;
        *groups = p.group_count();
    });
}

int ddm_b200_cutoff_set(int width, int height, int has_q_max, double q_max, int64_t* count,
                        int64_t* flat_out) {
    return guarded([&] {
        const auto s = ddm::cutoff_set(width, height,
                                       has_q_max ? std::optional<double>(q_max) : std::nullopt);
        *count = s.count();
        if (flat_out)
            for (int64_t k = 0; k < s.count(); ++k) flat_out[k] = s.flat(k);
    });
}

int ddm_b200_run_u16(const uint16_t* pixels, int width, int height, int frames,
                     double frame_interval, const ddm_b200_run_config* config, double* out_values,
                     int64_t out_capacity, int64_t* out_lags, int64_t* out_n_lags,
                     ddm_b200_counters* counters, ddm_b200_timing* timing) {
    return guarded([&] {
        if (!pixels || !out_values) throw ddm::InputError("null pixel or output buffer");
        ddm::ViewFrameSource src(pixels, width, height, frames, frame_interval);
        const auto a = ddm::run_into(src, to_config(config), out_values, out_capacity);
        emit(a, out_lags, out_n_lags, counters, timing);
    });
}

int ddm_b200_run_u8(const uint8_t* pixels, int width, int height, int frames, double frame_interval,
                    const ddm_b200_run_config* config, double* out_values, int64_t out_capacity,
                    int64_t* out_lags, int64_t* out_n_lags, ddm_b200_counters* counters,
                    ddm_b200_timing* timing) {
    return guarded([&] {
        if (!pixels || !out_values) throw ddm::InputError("null pixel or output buffer");
        ddm::detail::Ingest in;
        in.u8 = pixels;
        in.width = width;
        in.height = height;
        in.frames = frames;
        in.frame_interval = frame_interval;
        const auto cfg = to_config(config);
        const auto a = ddm::detail::guard_device(
            [&] { return ddm::detail::run_core(in, cfg, out_values, out_capacity); });
        emit(a, out_lags, out_n_lags, counters, timing);
    });
}

int ddm_b200_run_raw_stack(const char* path, const ddm_b200_run_config* config, double* out_values,
                           int64_t out_capacity, int64_t* out_lags, int64_t* out_n_lags,
                           ddm_b200_counters* counters, ddm_b200_timing* timing) {
    return guarded([&] {
        if (!path) throw ddm::InputError("null path");
        ddm::RawStackFileSource src(path);
        const auto a = ddm::run_into(src, to_config(config), out_values, out_capacity);
        emit(a, out_lags, out_n_lags, counters, timing);
    });
}

int ddm_b200_run_pgm_dir(const char* dir, const ddm_b200_run_config* config, double* out_values,
                         int64_t out_capacity, int64_t* out_lags, int64_t* out_n_lags,
                         ddm_b200_counters* counters, ddm_b200_timing* timing) {
    return guarded([&] {
        if (!dir) throw ddm::InputError("null path");
        ddm::PgmDirSource src(dir);
        const auto a = ddm::run_into(src, to_config(config), out_values, out_capacity);
        emit(a, out_lags, out_n_lags, counters, timing);
    });
}

int ddm_b200_analyze(const char* path, int format, const ddm_b200_run_config* config,
                     const char* out_dir, int64_t* out_n_lags, int64_t* fits_written,
                     ddm_b200_counters* counters, ddm_b200_timing* timing) {
    return guarded([&] {
        if (!path || !out_dir || !*out_dir) throw ddm::InputError("null path");
        // `ddm_cli.cpp:103-109`: auto = a directory is a PGM stack, anything else a raw stack
        const bool pgm = format == 1 || (format < 0 && std::filesystem::is_directory(path));
        const auto src = ddm::open_frame_source(path, pgm ? ddm::StackFormat::PgmDir
                                                          : ddm::StackFormat::RawStack);
        const auto a = ddm::analyze(*src, to_config(config), out_dir);
        if (fits_written) *fits_written = std::filesystem::exists(std::filesystem::path(out_dir) / "fits.csv");
        emit(a, nullptr, out_n_lags, counters, timing);
    });
}

int ddm_b200_bench_sweep(const int* frame_counts, int n_frame_counts, const int* sizes, int n_sizes,
                         const int* algorithms, int n_algorithms, const int* workers, int n_workers,
                         const int64_t* budgets, int n_budgets, int repetitions, int warmup,
                         const char* out_csv, int* crossover_sizes, int* crossover_n, int* n_crossover) {
    return guarded([&] {
        if (!out_csv || !*out_csv) throw ddm::InputError("null path");
        ddm::SweepSpec spec;
        auto take = [](const auto* p, int n) {
            using T = std::remove_cv_t<std::remove_pointer_t<decltype(p)>>;
            if (n < 0 || (n > 0 && !p)) throw ddm::InputError("sweep: bad axis");
            return std::vector<T>(p, p + n);
        };
        spec.frame_counts = take(frame_counts, n_frame_counts);
        spec.sizes = take(sizes, n_sizes);
        for (const int a : take(algorithms, n_algorithms))
            spec.algorithms.push_back(a == 0 ? ddm::Algorithm::WithFt
                                      : a == 1 ? ddm::Algorithm::WithoutFt : ddm::Algorithm::Direct);
        spec.worker_counts = take(workers, n_workers);
        spec.budgets = take(budgets, n_budgets);
        spec.repetitions = repetitions;
        spec.warmup = warmup;
        const auto table = ddm::sweep(spec, ddm::synthetic_stack_factory());
        const std::filesystem::path csv(out_csv);
        if (csv.has_parent_path()) std::filesystem::create_directories(csv.parent_path());
        ddm::write_bench_csv(table, csv);
        const auto xs = ddm::crossover(table);
        if (n_crossover) *n_crossover = int(xs.size());
        for (std::size_t i = 0; i < xs.size(); ++i) {
            if (crossover_sizes) crossover_sizes[i] = xs[i].size;
            if (crossover_n) crossover_n[i] = xs[i].n_star ? *xs[i].n_star : -1;
        }
    });
}

int ddm_b200_compare(const char* path, int format, const ddm_b200_run_config* config, int algorithm_a,
                     int algorithm_b, double* deviation, double* tolerance, int* pass,
                     ddm_b200_timing* timing_a, ddm_b200_timing* timing_b) {
    return guarded([&] {
        if (!path) throw ddm::InputError("null path");
        const bool pgm = format == 1 || (format < 0 && std::filesystem::is_directory(path));
        const auto src = ddm::open_frame_source(path, pgm ? ddm::StackFormat::PgmDir
                                                          : ddm::StackFormat::RawStack);
        auto alg = [](int a) {
            if (a < 0 || a > 2) throw ddm::InputError("unknown algorithm");
            return a == 0 ? ddm::Algorithm::WithFt : a == 1 ? ddm::Algorithm::WithoutFt : ddm::Algorithm::Direct;
        };
        const auto r = ddm::compare(*src, to_config(config), alg(algorithm_a), alg(algorithm_b));
        if (deviation) *deviation = r.deviation;
        if (tolerance) *tolerance = r.tolerance;
        if (pass) *pass = r.pass ? 1 : 0;
        ddm_b200_timing* t[2] = {timing_a, timing_b};
        for (int i = 0; i < 2; ++i)
            if (t[i]) {
                t[i]->disk = r.timing[i].disk;
                t[i]->step1 = r.timing[i].step1;
                t[i]->step2 = r.timing[i].step2;
                t[i]->merge = r.timing[i].merge;
                t[i]->other = r.timing[i].other;
                t[i]->total = r.timing[i].total;
            }
    });
}

int ddm_b200_synth(const char* out_dir, int64_t particles, double diffusion, double psf_sigma,
                   double amplitude, double background, int size, int frames, double frame_interval,
                   uint64_t seed) {
    return guarded([&] {
        if (!out_dir || !*out_dir) throw ddm::InputError("null path");
        ddm::SynthConfig c;
        c.particles = particles;
        c.diffusion = diffusion;
        c.psf_sigma = psf_sigma;
        c.amplitude = amplitude;
        c.background = background;
        c.width = c.height = size;
        c.frames = frames;
        c.frame_interval = frame_interval;
        c.seed = seed;
        const ddm::ImageStack st = ddm::generate(c);
        const std::filesystem::path out(out_dir);
        std::filesystem::create_directories(out);
        ddm::write_raw_stack(st, out / "stack.raw");
        ddm::write_synth_manifest(c, out / "synth.json");
    });
}

int ddm_b200_crossover(int64_t n_cells, const int* algorithm, const int* frames, const int* width,
                       const double* seconds_total, const int* failed, int* sizes_out, int* n_star_out,
                       int* n_out) {
    return guarded([&] {
        if (n_cells < 0 || (n_cells > 0 && (!algorithm || !frames || !width || !seconds_total)))
            throw ddm::InputError("null table");
        std::vector<ddm::BenchCell> table(static_cast<std::size_t>(n_cells));
        for (int64_t i = 0; i < n_cells; ++i) {
            auto& c = table[std::size_t(i)];
            c.algorithm = algorithm[i] == 0 ? "with_ft" : algorithm[i] == 1 ? "without_ft" : "direct";
            c.frames = frames[i];
            c.width = c.height = width[i];
            c.seconds_total = seconds_total[i];
            c.failed = failed && failed[i] != 0;
        }
        const auto xs = ddm::crossover(table);
        if (n_out) *n_out = int(xs.size());
        for (std::size_t i = 0; i < xs.size(); ++i) {
            if (sizes_out) sizes_out[i] = xs[i].size;
            if (n_star_out) n_star_out[i] = xs[i].n_star ? *xs[i].n_star : -1;
        }
    });
}

int ddm_b200_stack_dims(const char* path, int format, int* width, int* height, int* frames) {
    return guarded([&] {
        if (!path || !width || !height || !frames) throw ddm::InputError("null argument");
        const auto src = ddm::open_frame_source(path, format == 1 ? ddm::StackFormat::PgmDir
                                                                  : ddm::StackFormat::RawStack);
        *width = src->width();
        *height = src->height();
        *frames = src->frames();
    });
}

int ddm_b200_load_stack(const char* path, int format, uint16_t* out, int64_t capacity) {
    return guarded([&] {
        if (!path || !out) throw ddm::InputError("null argument");
        const auto st = ddm::load_stack(path, format == 1 ? ddm::StackFormat::PgmDir : ddm::StackFormat::RawStack);
        if (int64_t(st.pixels.size()) > capacity) throw ddm::InputError("output capacity too small");
        std::copy(st.pixels.begin(), st.pixels.end(), out);
    });
}

int ddm_b200_run_device(const void* d_frames, int pixel_bytes, int width, int height, int frames,
                        int precision, const int64_t* lags, int64_t n_lags, int has_q_max,
                        double q_max, void* d_out, int out_f64, int device, void* stream,
                        double* spatial_ms, double* temporal_ms, int* kernel_launches) {
    return guarded([&] {
        if (!d_frames || !d_out) throw ddm::InputError("null device buffer");
        if (pixel_bytes != 1 && pixel_bytes != 2) throw ddm::InputError("pixel_bytes must be 1 or 2");
        if (width < 1 || height < 1 || frames < 1) throw ddm::InputError("dimensions must be positive");
        const bool f64 = precision != 0;
        if (frames > ddm::b200::max_frames(f64))
            throw ddm::PlanError("sequence longer than the device temporal engine limit");
        std::vector<int64_t> lag_list = (lags && n_lags > 0)
                                            ? ddm::normalize_lags({lags, lags + n_lags}, frames)
                                            : ddm::all_lags(frames);
        const int64_t plane = int64_t(height) * (width / 2 + 1);
        ddm::WaveVectorSet wv;
        if (has_q_max) {
            wv = ddm::cutoff_set(width, height, std::optional<double>(q_max));
            if (wv.count() < 1) throw ddm::InputError("wave-vector cutoff retains nothing");
        }
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            cudaStream_t user = static_cast<cudaStream_t>(stream);
            cudaEvent_t ev;
            ddm::b200::check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
            ddm::b200::check(cudaEventRecord(ev, user), "event record");
            ddm::b200::check(cudaStreamWaitEvent(eng.stream(), ev, 0), "stream wait");
            ddm::b200::RunSpec sp;
            sp.W = width;
            sp.H = height;
            sp.N = frames;
            sp.f64 = f64;
            sp.pixel_bytes = pixel_bytes;
            sp.d_frames = d_frames;
            sp.lags = lag_list;
            // no cutoff: every wave vector, identity positions (no index list is built)
            sp.identity = true;
            int64_t count = plane;
            if (has_q_max) {
                count = wv.count();
                sp.flat.resize(size_t(count));
                for (int64_t k = 0; k < count; ++k) {
                    sp.flat[size_t(k)] = wv.flat(k);
                    if (sp.flat[size_t(k)] != k) sp.identity = false;
                }
            }
            sp.groups = {{0, count}};
            sp.d_out = d_out;
            sp.out_f64 = out_f64 != 0;
            sp.out_stride = plane;
            ddm::b200::PhaseTimes t;
            eng.run(sp, (spatial_ms || temporal_ms || kernel_launches) ? &t : nullptr);
            ddm::b200::check(cudaEventRecord(ev, eng.stream()), "event record");
            ddm::b200::check(cudaStreamWaitEvent(user, ev, 0), "stream wait");
            cudaEventDestroy(ev);
            if (spatial_ms) *spatial_ms = t.spatial_ms;
            if (temporal_ms) *temporal_ms = t.temporal_ms;
            if (kernel_launches) *kernel_launches = t.spatial_launches + t.temporal_launches;
            return 0;
        });
    });
}

int ddm_b200_shard_plan(int64_t q_count, int64_t frames, int ranks, int64_t* frame_begin,
                        int64_t* q_begin) {
    return guarded([&] {
        if (!frame_begin || !q_begin) throw ddm::InputError("null plan arrays");
        const auto p = ddm::plan_shards(q_count, frames, ranks);
        std::copy(p.frame_begin.begin(), p.frame_begin.end(), frame_begin);
        std::copy(p.q_begin.begin(), p.q_begin.end(), q_begin);
    });
}

int ddm_b200_spatial_shard_device(const void* d_frames, int pixel_bytes, int width, int height,
                                  int frames, int precision, void* d_spec, int device,
                                  void* stream, double* ms) {
    return guarded([&] {
        if (!d_frames || !d_spec) throw ddm::InputError("null device buffer");
        if (pixel_bytes != 1 && pixel_bytes != 2) throw ddm::InputError("pixel_bytes must be 1 or 2");
        if (width < 1 || height < 1 || frames < 1) throw ddm::InputError("dimensions must be positive");
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            on_engine_stream(eng, stream, [&] {
                ddm::b200::PhaseTimes t;
                eng.spatial_shard(d_frames, pixel_bytes, width, height, frames, precision != 0,
                                  d_spec, ms ? &t : nullptr);
                if (ms) *ms = t.spatial_ms;
            });
            return 0;
        });
    });
}

int ddm_b200_spatial_shard_p2p_device(const void* d_frames, int pixel_bytes, int width, int height,
                                      int frames, int precision, int ranks,
                                      const int64_t* q_begin, void* const* dest, int device,
                                      void* stream, double* ms) {
    return guarded([&] {
        if (!d_frames || !q_begin || !dest) throw ddm::InputError("null buffer");
        if (pixel_bytes != 1 && pixel_bytes != 2) throw ddm::InputError("pixel_bytes must be 1 or 2");
        if (width < 1 || height < 1 || frames < 1) throw ddm::InputError("dimensions must be positive");
        if (ranks < 1 || ranks > ddmk::PeerTable::kMax) throw ddm::InputError("ranks must be in [1, 8]");
        ddmk::PeerTable peers;
        peers.ranks = ranks;
        const int64_t plane = int64_t(height) * (width / 2 + 1);
        for (int d = 0; d <= ranks; ++d) peers.q_begin[d] = q_begin[d];
        if (peers.q_begin[0] != 0 || peers.q_begin[ranks] != plane)
            throw ddm::InputError("q_begin must cover the half plane");
        for (int d = 0; d < ranks; ++d) {
            if (peers.q_begin[d + 1] < peers.q_begin[d]) throw ddm::InputError("q_begin must ascend");
            if (!dest[d] && peers.q_begin[d + 1] > peers.q_begin[d]) throw ddm::InputError("null destination");
            peers.base[d] = dest[d];
        }
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            on_engine_stream(eng, stream, [&] {
                ddm::b200::PhaseTimes t;
                try {
                    eng.spatial_shard(d_frames, pixel_bytes, width, height, frames, precision != 0,
                                      nullptr, ms ? &t : nullptr, &peers);
                } catch (const std::invalid_argument& e) {
                    throw ddm::InputError(e.what());
                }
                if (ms) *ms = t.spatial_ms;
            });
            return 0;
        });
    });
}

int ddm_b200_temporal_segments_device(const void* d_recv, int64_t q_count, int n_segments,
                                      const int64_t* seg_frames, int precision,
                                      const int64_t* lags, int64_t n_lags, void* d_out,
                                      int64_t out_stride, int out_f64, int device, void* stream,
                                      double* ms) {
    return guarded([&] {
        if (!d_recv || !d_out || !seg_frames) throw ddm::InputError("null buffer");
        if (q_count < 1) throw ddm::InputError("need at least one wave vector");
        if (n_segments < 1 || n_segments > 8) throw ddm::InputError("1 to 8 frame segments");
        std::vector<int> segs((size_t)n_segments);
        int64_t frames = 0;
        for (int s = 0; s < n_segments; ++s) {
            if (seg_frames[s] < 1) throw ddm::InputError("empty frame segment");
            segs[(size_t)s] = (int)seg_frames[s];
            frames += seg_frames[s];
        }
        const bool f64 = precision != 0;
        if (frames > ddm::b200::max_frames(f64))
            throw ddm::PlanError("sequence longer than the device temporal engine limit");
        std::vector<int64_t> lag_list = (lags && n_lags > 0)
                                            ? ddm::normalize_lags({lags, lags + n_lags}, frames)
                                            : ddm::all_lags(frames);
        if (out_stride < q_count) throw ddm::InputError("out_stride smaller than q_count");
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            on_engine_stream(eng, stream, [&] {
                ddm::b200::PhaseTimes t;
                eng.temporal_segments(d_recv, q_count, segs, f64, lag_list, d_out, out_stride,
                                      out_f64 != 0, ms ? &t : nullptr);
                if (ms) *ms = t.temporal_ms;
            });
            return 0;
        });
    });
}

namespace {

// shared body of the azimuthal entry points: frames already on the device
void run_azimuthal_on_device(ddm::b200::Engine& eng, const void* d_frames, int pixel_bytes,
                             int width, int height, int frames, bool f64,
                             const std::vector<int64_t>& lag_list, int has_q_max, double q_max,
                             double* d_means, int64_t capacity, int64_t* counts,
                             int64_t* bin_count, ddm::b200::PhaseTimes* t, int* fused) {
    const int64_t plane = int64_t(height) * (width / 2 + 1);
    ddm::b200::RunSpec sp;
    sp.W = width;
    sp.H = height;
    sp.N = frames;
    sp.f64 = f64;
    sp.pixel_bytes = pixel_bytes;
    sp.d_frames = d_frames;
    sp.lags = lag_list;
    sp.identity = true;
    int64_t count = plane;
    if (has_q_max) {
        const auto wv = ddm::cutoff_set(width, height, std::optional<double>(q_max));
        count = wv.count();
        if (count < 1) throw ddm::InputError("wave-vector cutoff retains nothing");
        sp.flat.resize(size_t(count));
        for (int64_t k = 0; k < count; ++k) {
            sp.flat[size_t(k)] = wv.flat(k);
            if (sp.flat[size_t(k)] != k) sp.identity = false;
        }
    } else {
        sp.flat.resize(size_t(plane));
        for (int64_t k = 0; k < plane; ++k) sp.flat[size_t(k)] = k;
    }
    sp.groups = {{0, count}};
    sp.out_stride = plane;
    const auto& rp = eng.ring_plan(sp.flat, width, height);
    if (bin_count) *bin_count = rp.nbins;
    if (counts) std::copy(rp.counts.begin(), rp.counts.begin() + std::min(capacity, rp.nbins), counts);
    if (!d_means) return;  // size query
    if (capacity < rp.nbins) throw ddm::InputError("means capacity smaller than the bin count");
    // means are [lags][capacity]: run into [lags][nbins] then widen if the caller's pitch differs
    double* target = d_means;
    if (capacity != rp.nbins)
        target = static_cast<double*>(eng.buffer("ring_means", size_t(lag_list.size() * rp.nbins) * 8));
    const bool f = eng.run_rings(sp, rp, target, t);
    if (fused) *fused = f ? 1 : 0;
    if (target != d_means) {
        ddm::b200::check(cudaMemsetAsync(d_means, 0, size_t(lag_list.size() * capacity) * 8, eng.stream()), "memset");
        ddm::b200::check(cudaMemcpy2DAsync(d_means, size_t(capacity) * 8, target, size_t(rp.nbins) * 8,
                                           size_t(rp.nbins) * 8, lag_list.size(), cudaMemcpyDeviceToDevice,
                                           eng.stream()), "copy");
    }
}

}  // namespace

int ddm_b200_run_azimuthal_device(const void* d_frames, int pixel_bytes, int width, int height,
                                  int frames, int precision, const int64_t* lags, int64_t n_lags,
                                  int has_q_max, double q_max, double* d_means, int64_t capacity,
                                  int64_t* counts, int64_t* bin_count, int device, void* stream,
                                  double* spatial_ms, double* temporal_ms, int* fused) {
    return guarded([&] {
        if (!d_frames) throw ddm::InputError("null device buffer");
        if (pixel_bytes != 1 && pixel_bytes != 2) throw ddm::InputError("pixel_bytes must be 1 or 2");
        if (width < 1 || height < 1 || frames < 1) throw ddm::InputError("dimensions must be positive");
        const bool f64 = precision != 0;
        if (frames > ddm::b200::max_frames(f64))
            throw ddm::PlanError("sequence longer than the device temporal engine limit");
        std::vector<int64_t> lag_list = (lags && n_lags > 0)
                                            ? ddm::normalize_lags({lags, lags + n_lags}, frames)
                                            : ddm::all_lags(frames);
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            on_engine_stream(eng, stream, [&] {
                ddm::b200::PhaseTimes t;
                run_azimuthal_on_device(eng, d_frames, pixel_bytes, width, height, frames, f64,
                                        lag_list, has_q_max, q_max, d_means, capacity, counts,
                                        bin_count, (spatial_ms || temporal_ms) ? &t : nullptr, fused);
                if (spatial_ms) *spatial_ms = t.spatial_ms;
                if (temporal_ms) *temporal_ms = t.temporal_ms;
            });
            return 0;
        });
    });
}

int ddm_b200_run_azimuthal_u16(const uint16_t* pixels, int width, int height, int frames,
                               const ddm_b200_run_config* config, double* means, int64_t capacity,
                               int64_t* counts, int64_t* bin_count, int64_t* out_lags,
                               int64_t* out_n_lags) {
    return guarded([&] {
        if (!pixels) throw ddm::InputError("null pixel buffer");
        const ddm::RunConfig cfg = to_config(config);
        if (cfg.algorithm != ddm::Algorithm::WithFt)
            throw ddm::InputError("only the with_ft algorithm runs on the device");
        if (cfg.workers < 1) throw ddm::InputError("workers must be at least 1");
        if (width < 1 || height < 1 || frames < 1) throw ddm::InputError("dimensions must be positive");
        const bool f64 = cfg.precision == ddm::Precision::F64;
        if (frames > ddm::b200::max_frames(f64))
            throw ddm::PlanError("sequence longer than the device temporal engine limit");
        std::vector<int64_t> lag_list = cfg.lags.empty() ? ddm::all_lags(frames)
                                                         : ddm::normalize_lags(cfg.lags, frames);
        if (out_n_lags) *out_n_lags = int64_t(lag_list.size());
        if (out_lags) std::copy(lag_list.begin(), lag_list.end(), out_lags);
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(cfg.device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            const size_t fb = size_t(frames) * size_t(width) * size_t(height) * 2;
            void* d_frames = eng.frame_buffer(fb);
            if (!means) {  // size query only
                run_azimuthal_on_device(eng, d_frames, 2, width, height, frames, f64, lag_list,
                                        cfg.q_max.has_value(), cfg.q_max.value_or(0.0), nullptr,
                                        capacity, counts, bin_count, nullptr, nullptr);
                return 0;
            }
            ddm::b200::check(cudaMemcpyAsync(d_frames, pixels, fb, cudaMemcpyHostToDevice, eng.stream()),
                             "frame upload");
            int64_t nb = 0;
            run_azimuthal_on_device(eng, d_frames, 2, width, height, frames, f64, lag_list,
                                    cfg.q_max.has_value(), cfg.q_max.value_or(0.0), nullptr, 0,
                                    nullptr, &nb, nullptr, nullptr);
            if (capacity < nb) throw ddm::InputError("means capacity smaller than the bin count");
            double* d_means = static_cast<double*>(eng.buffer("ring_means_out", size_t(lag_list.size() * capacity) * 8));
            run_azimuthal_on_device(eng, d_frames, 2, width, height, frames, f64, lag_list,
                                    cfg.q_max.has_value(), cfg.q_max.value_or(0.0), d_means, capacity,
                                    counts, bin_count, nullptr, nullptr);
            ddm::b200::check(cudaMemcpyAsync(means, d_means, size_t(lag_list.size() * capacity) * 8,
                                             cudaMemcpyDeviceToHost, eng.stream()), "download");
            ddm::b200::check(cudaStreamSynchronize(eng.stream()), "sync");
            return 0;
        });
    });
}

int ddm_b200_ring_sums_device(const void* d_map, int map_f64, int64_t q_begin, int64_t q_count,
                              int64_t map_stride, int64_t n_lags, int width, int height, int has_q_max,
                              double q_max, double* d_sums, int64_t capacity, int64_t* counts,
                              int64_t* bin_count, int device, void* stream) {
    return guarded([&] {
        if (width < 1 || height < 1 || n_lags < 0 || q_begin < 0 || q_count < 0)
            throw ddm::InputError("ring sums: bad geometry");
        const int Wh = ddm::half_cols(width);
        const int64_t plane = int64_t(height) * Wh;
        if (q_begin + q_count > plane) throw ddm::InputError("ring sums: slice outside the plane");
        // rings of the whole plane (`analysis.cpp:61-97`): every rank agrees on the bin count
        auto bin_of = [&](int64_t k) {
            return std::llround(ddm::q_magnitude(int(k / Wh), int(k % Wh), height));
        };
        auto kept = [&](int64_t k) {
            return !has_q_max || ddm::q_magnitude(int(k / Wh), int(k % Wh), height) <= q_max;
        };
        int64_t nbins = 0;
        for (int64_t k = 0; k < plane; ++k)
            if (kept(k)) nbins = std::max<int64_t>(nbins, bin_of(k) + 1);
        if (bin_count) *bin_count = nbins;
        if (!d_sums) return;   // size query
        if (capacity < n_lags * nbins) throw ddm::InputError("ring sums: capacity too small");
        std::vector<int64_t> cnt(size_t(nbins), 0), off(size_t(nbins) + 1, 0), order;
        for (int64_t j = 0; j < q_count; ++j)
            if (kept(q_begin + j)) ++cnt[size_t(bin_of(q_begin + j))];
        for (int64_t b = 0; b < nbins; ++b) off[size_t(b) + 1] = off[size_t(b)] + cnt[size_t(b)];
        order.resize(size_t(off.back()));
        std::vector<int64_t> fill(off.begin(), off.end() - 1);
        for (int64_t j = 0; j < q_count; ++j)
            if (kept(q_begin + j)) order[size_t(fill[size_t(bin_of(q_begin + j))]++)] = j;
        if (counts) std::copy(cnt.begin(), cnt.end(), counts);
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            on_engine_stream(eng, stream, [&] {
                cudaStream_t st = eng.stream();
                auto* d_idx = static_cast<int64_t*>(
                    eng.buffer("ring_csr", (order.size() + off.size()) * sizeof(int64_t)));
                ddm::b200::check(cudaMemcpyAsync(d_idx, order.data(), order.size() * sizeof(int64_t),
                                                 cudaMemcpyHostToDevice, st), "upload");
                ddm::b200::check(cudaMemcpyAsync(d_idx + order.size(), off.data(), off.size() * sizeof(int64_t),
                                                 cudaMemcpyHostToDevice, st), "upload");
                ddm::b200::ring_sums(d_map, map_f64 != 0, n_lags, map_stride, d_idx, d_idx + order.size(),
                                     nbins, d_sums, st);
                ddm::b200::check(cudaStreamSynchronize(st), "sync");   // host CSR vectors
            });
            return 0;
        });
    });
}

int ddm_b200_fit_rings(const double* means, const int64_t* lags, int64_t n_lags,
                       const int64_t* counts, int64_t nbins, double frame_interval, int device,
                       double* amplitude, double* baseline, double* tau, double* residual,
                       int* flag) {
    return guarded([&] {
        if (!means || !lags || !counts || !amplitude || !baseline || !tau || !residual || !flag)
            throw ddm::InputError("null buffer");
        if (n_lags < 1 || nbins < 1) throw ddm::InputError("empty profile");
        if (!(frame_interval > 0.0)) throw ddm::InputError("frame interval must be positive");
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            cudaStream_t st = eng.stream();
            const size_t L = size_t(n_lags), B = size_t(nbins);
            char* base = static_cast<char*>(eng.buffer("fit_io", L * B * 8 + L * 8 + B * 8 + 4 * B * 8 + B * 4));
            double* d_means = reinterpret_cast<double*>(base);
            int64_t* d_lags = reinterpret_cast<int64_t*>(d_means + L * B);
            int64_t* d_counts = d_lags + L;
            double* d_out = reinterpret_cast<double*>(d_counts + B);
            int* d_flag = reinterpret_cast<int*>(d_out + 4 * B);
            ddm::b200::check(cudaMemcpyAsync(d_means, means, L * B * 8, cudaMemcpyHostToDevice, st), "upload");
            ddm::b200::check(cudaMemcpyAsync(d_lags, lags, L * 8, cudaMemcpyHostToDevice, st), "upload");
            ddm::b200::check(cudaMemcpyAsync(d_counts, counts, B * 8, cudaMemcpyHostToDevice, st), "upload");
            ddm::b200::check(ddmk::launch_fit_rings(d_means, d_lags, int(n_lags), d_counts, nbins, frame_interval,
                                                    d_out, d_out + B, d_out + 2 * B, d_out + 3 * B, d_flag, st),
                             "fit kernel");
            ddm::b200::check(cudaMemcpyAsync(amplitude, d_out, B * 8, cudaMemcpyDeviceToHost, st), "download");
            ddm::b200::check(cudaMemcpyAsync(baseline, d_out + B, B * 8, cudaMemcpyDeviceToHost, st), "download");
            ddm::b200::check(cudaMemcpyAsync(tau, d_out + 2 * B, B * 8, cudaMemcpyDeviceToHost, st), "download");
            ddm::b200::check(cudaMemcpyAsync(residual, d_out + 3 * B, B * 8, cudaMemcpyDeviceToHost, st), "download");
            ddm::b200::check(cudaMemcpyAsync(flag, d_flag, B * 4, cudaMemcpyDeviceToHost, st), "download");
            ddm::b200::check(cudaStreamSynchronize(st), "sync");
            return 0;
        });
    });
}

int ddm_b200_estimate_diffusion(const double* tau, const int* flag, int64_t nbins, int64_t width,
                                int64_t q_lo, int64_t q_hi, double* coefficient,
                                int64_t* bins_used) {
    return guarded([&] {
        // `analysis.cpp:242-271`: least squares through the origin of 1/tau against q^2,
        // q = 2 pi bin / width, over the ok fits of bins [q_lo, q_hi]
        if (!tau || !flag || !coefficient || !bins_used) throw ddm::InputError("null buffer");
        if (width < 1) throw ddm::InputError("estimate_diffusion: bad width");
        const double two_pi = 2.0 * std::acos(-1.0);
        double sxx = 0.0, sxy = 0.0;
        int64_t used = 0;
        for (int64_t b = std::max<int64_t>(q_lo, 0); b <= q_hi && b < nbins; ++b) {
            if (flag[b] != 0) continue;
            const double q = two_pi * double(b) / double(width);
            const double x = q * q;
            sxx += x * x;
            sxy += x * (1.0 / tau[b]);
            ++used;
        }
        *bins_used = used;
        *coefficient = (used > 0 && sxx > 0.0) ? sxy / sxx : 0.0;
    });
}

int ddm_b200_sequences_with_ft(const double* seq, int64_t q, int64_t n, int precision, int device,
                               double* d, double* d_a, double* corr, uint64_t* temporal_ffts) {
    return guarded([&] {
        if (!seq || !d) throw ddm::InputError("null buffer");
        if (q < 1 || n < 1) throw ddm::InputError("need at least one sequence of one value");
        const bool f64 = precision != 0;
        if (n > ddm::b200::max_frames(f64))
            throw ddm::PlanError("sequence longer than the device temporal engine limit");
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            const size_t cnt = size_t(q) * size_t(n);
            std::vector<unsigned char> host;
            if (f64) {
                host.resize(cnt * 16);
                std::memcpy(host.data(), seq, cnt * 16);
            } else {
                host.resize(cnt * 8);
                float* f = reinterpret_cast<float*>(host.data());
                for (size_t i = 0; i < 2 * cnt; ++i) f[i] = float(seq[i]);
            }
            const size_t outs = cnt * sizeof(double);
            char* dev = static_cast<char*>(eng.buffer("seq_io", host.size() + 3 * outs));
            double* dd = reinterpret_cast<double*>(dev + host.size());
            double* dda = dd + cnt;
            double* dco = dda + cnt;
            ddm::b200::check(cudaMemcpy(dev, host.data(), host.size(), cudaMemcpyHostToDevice), "upload");
            eng.sequences(dev, q, n, f64, dd, d_a ? dda : nullptr, corr ? dco : nullptr);
            ddm::b200::check(cudaMemcpy(d, dd, outs, cudaMemcpyDeviceToHost), "download");
            if (d_a) ddm::b200::check(cudaMemcpy(d_a, dda, outs, cudaMemcpyDeviceToHost), "download");
            if (corr) ddm::b200::check(cudaMemcpy(corr, dco, outs, cudaMemcpyDeviceToHost), "download");
            return 0;
        });
        if (temporal_ffts) *temporal_ffts = 2 * uint64_t(q);
    });
}

int ddm_b200_spectra_u16(const uint16_t* pixels, int width, int height, int frames, int precision,
                         int device, double* out) {
    return guarded([&] {
        if (!pixels || !out) throw ddm::InputError("null buffer");
        if (width < 1 || height < 1 || frames < 1) throw ddm::InputError("dimensions must be positive");
        ddm::detail::guard_device([&] {
            auto& eng = ddm::b200::Engine::instance(device);
            std::lock_guard<std::mutex> lock(eng.mutex());
            const bool f64 = precision != 0;
            const size_t np = size_t(height) * (width / 2 + 1) * size_t(frames);
            const size_t inb = (size_t(width) * height * frames * 2 + 255) / 256 * 256;
            const size_t cs = f64 ? 16 : 8;
            char* dev = static_cast<char*>(eng.buffer("spectra_io", inb + np * cs));
            ddm::b200::check(cudaMemcpy(dev, pixels, size_t(width) * height * frames * 2, cudaMemcpyHostToDevice), "upload");
            eng.spectra(dev, 2, width, height, frames, f64, dev + inb);
            if (f64) {
                ddm::b200::check(cudaMemcpy(out, dev + inb, np * 16, cudaMemcpyDeviceToHost), "download");
            } else {
                std::vector<float> tmp(2 * np);
                ddm::b200::check(cudaMemcpy(tmp.data(), dev + inb, np * 8, cudaMemcpyDeviceToHost), "download");
                for (size_t i = 0; i < 2 * np; ++i) out[i] = tmp[i];
            }
            return 0;
        });
    });
}

int ddm_b200_forward_spectrum(const double* frame, int width, int height, int precision, int device,
                              double* out) {
    (void)device;
    return guarded([&] {
        if (!frame || !out) throw ddm::InputError("null buffer");
        const size_t n = size_t(width) * size_t(height);
        if (precision != 0) {
            const auto s = ddm::forward_spectrum<double>({frame, n}, width, height);
            std::memcpy(out, s.data(), s.size() * sizeof(s[0]));
        } else {
            std::vector<float> f(frame, frame + n);
            const auto s = ddm::forward_spectrum<float>({f.data(), n}, width, height);
            for (size_t i = 0; i < s.size(); ++i) {
                out[2 * i] = s[i].real();
                out[2 * i + 1] = s[i].imag();
            }
        }
    });
}

int ddm_b200_azimuthal(const double* values, int64_t n_lags, int width, int height, int has_q_max,
                       double q_max, int device, double* means, int64_t* counts, int64_t capacity,
                       int64_t* bin_count) {
    (void)device;
    return guarded([&] {
        ddm::ResultMap map;
        map.width = width;
        map.height = height;
        map.lags.resize(size_t(n_lags));
        for (int64_t i = 0; i < n_lags; ++i) map.lags[size_t(i)] = i;
        map.values.assign(values, values + size_t(map.plane_size() * n_lags));
        const auto wv = ddm::cutoff_set(width, height,
                                        has_q_max ? std::optional<double>(q_max) : std::nullopt);
        const auto p = ddm::azimuthal_average(map, wv);
        *bin_count = p.bin_count;
        if (p.bin_count > capacity) throw ddm::InputError("bin capacity too small");
        std::copy(p.counts.begin(), p.counts.end(), counts);
        std::copy(p.means.begin(), p.means.end(), means);
    });
}

int ddm_b200_generate(int64_t particles, double diffusion, double psf_sigma, double amplitude,
                      double background, int width, int height, int frames, double frame_interval,
                      uint64_t seed, uint16_t* out) {
    return guarded([&] {
        ddm::SynthConfig c;
        c.particles = particles;
        c.diffusion = diffusion;
        c.psf_sigma = psf_sigma;
        c.amplitude = amplitude;
        c.background = background;
        c.width = width;
        c.height = height;
        c.frames = frames;
        c.frame_interval = frame_interval;
        c.seed = seed;
        const auto st = ddm::generate(c);
        std::copy(st.pixels.begin(), st.pixels.end(), out);
    });
}

int ddm_b200_generate_device(int64_t particles, double diffusion, double psf_sigma,
                             double amplitude, double background, int width, int height,
                             int frames, double frame_interval, uint64_t seed, uint16_t* d_out,
                             int device, void* stream) {
    return guarded([&] {
        ddm::SynthConfig c;
        c.particles = particles;
        c.diffusion = diffusion;
        c.psf_sigma = psf_sigma;
        c.amplitude = amplitude;
        c.background = background;
        c.width = width;
        c.height = height;
        c.frames = frames;
        c.frame_interval = frame_interval;
        c.seed = seed;
        ddm::generate_device(c, d_out, device, stream);
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------- sessions
struct ddm_b200 {
    ddm::detail::Session s;
    ddm_b200(int w, int h, int n, int p, int d) : s(w, h, n, p, d) {}
};

extern "C" {

int ddm_b200_create(int width, int height, int frames, int precision, int device, ddm_b200** out) {
    return guarded([&] {
        if (!out) throw ddm::InputError("null session pointer");
        *out = nullptr;
        *out = ddm::detail::guard_device([&] { return new ddm_b200(width, height, frames, precision, device); });
    });
}

int ddm_b200_destroy(ddm_b200* session) {
    return guarded([&] { delete session; });
}

int ddm_b200_stage_frames(ddm_b200* session, const uint16_t* host, int first, int count) {
    return guarded([&] {
        if (!session) throw ddm::InputError("null session");
        ddm::detail::guard_device([&] {
            session->s.stage(host, 2, first, count);
            return 0;
        });
    });
}

int ddm_b200_stage_frames_u8(ddm_b200* session, const uint8_t* host, int first, int count) {
    return guarded([&] {
        if (!session) throw ddm::InputError("null session");
        ddm::detail::guard_device([&] {
            session->s.stage(host, 1, first, count);
            return 0;
        });
    });
}

int ddm_b200_run_with_ft(ddm_b200* session, const int64_t* wv_flat, int64_t q_count, const int64_t* lags,
                         int64_t n_lags, double* out_lag_major, int64_t out_capacity,
                         ddm_b200_counters* counters, ddm_b200_timing* timing) {
    return guarded([&] {
        if (!session) throw ddm::InputError("null session");
        ddm::RunCounters c;
        const ddm::TimingBreakdown t = ddm::detail::guard_device([&] {
            return session->s.run_with_ft(wv_flat, q_count, lags, n_lags, out_lag_major, out_capacity, &c);
        });
        if (counters) *counters = {c.spatial_ffts, c.temporal_ffts, c.pairs};
        if (timing) *timing = {t.disk, t.step1, t.step2, t.merge, t.other, t.total};
    });
}

int ddm_b200_session_engines(ddm_b200* session, char* buf, int64_t capacity) {
    return guarded([&] {
        if (!session || !buf || capacity < 1) throw ddm::InputError("null session or buffer");
        const std::string& e = session->s.last_engines();
        const std::size_t n = std::min<std::size_t>(e.size(), std::size_t(capacity - 1));
        std::memcpy(buf, e.data(), n);
        buf[n] = '\0';
    });
}

}  // extern "C"
