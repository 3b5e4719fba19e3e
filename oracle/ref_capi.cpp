// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" veneer over the UNMODIFIED reference library (compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/libddmref.so) so the
// Python tests and bench.py's reference arm can call the reference's own code paths via
// ctypes. Nothing here re-implements reference arithmetic; every function forwards to the
// reference symbol named in its comment.  Status codes mirror the product C-ABI:
// 0 ok, 1 InputError, 2 PlanError/bad_alloc, 3 IoError, 5 other.

#include <ddm/analysis.hpp>
#include <ddm/archive.hpp>
#include <ddm/bench.hpp>
#include <ddm/errors.hpp>
#include <ddm/frame_source.hpp>
#include <ddm/scheduler.hpp>
#include <ddm/spectrum.hpp>
#include <ddm/synth.hpp>
#include <ddm/temporal.hpp>

#include <algorithm>
#include <complex>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <new>
#include <string>
#include <vector>

namespace {

int fail(char* err, int errlen, const std::string& what, int code) {
    if (err && errlen > 0) {
        std::strncpy(err, what.c_str(), static_cast<std::size_t>(errlen - 1));
        err[errlen - 1] = '\0';
    }
    return code;
}

template <class Fn>
int guarded(char* err, int errlen, Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const ddm::InputError& e) {
        return fail(err, errlen, e.what(), 1);
    } catch (const ddm::PlanError& e) {
        return fail(err, errlen, e.what(), 2);
    } catch (const ddm::IoError& e) {
        return fail(err, errlen, e.what(), 3);
    } catch (const std::bad_alloc& e) {
        return fail(err, errlen, e.what(), 2);
    } catch (const std::exception& e) {
        return fail(err, errlen, e.what(), 5);
    }
}

template <class S>
std::vector<std::complex<S>> to_complex(const double* inter, std::int64_t n) {
    std::vector<std::complex<S>> v(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i)
        v[static_cast<std::size_t>(i)] = {static_cast<S>(inter[2 * i]),
                                          static_cast<S>(inter[2 * i + 1])};
    return v;
}

} // namespace

extern "C" {

// ddm::pad_length, proj/core/src/temporal.cpp:10-17
std::int64_t ref_pad_length(std::int64_t n) {
    try {
        return ddm::pad_length(n);
    } catch (...) {
        return -1;
    }
}

// ddm::run, proj/core/src/scheduler.cpp:413-483 (MemoryFrameSource, frame_source.cpp:15-25)
int ref_run(const std::uint16_t* pixels, int width, int height, int frames,
            double frame_interval, int algorithm, int precision, const std::int64_t* lags,
            std::int64_t n_lags, int has_q_max, double q_max, std::int64_t memory_bytes,
            int workers, double* out_values, std::int64_t out_capacity,
            std::int64_t* out_lags, std::int64_t* out_n_lags, std::uint64_t* counters3,
            double* timing6, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ddm::ImageStack stack;
        stack.width = width;
        stack.height = height;
        stack.frames = frames;
        stack.frame_interval = frame_interval;
        stack.pixels.assign(pixels, pixels + static_cast<std::size_t>(width) * height * frames);
        ddm::MemoryFrameSource source(std::move(stack));
        ddm::RunConfig config;
        config.algorithm = algorithm == 0   ? ddm::Algorithm::WithFt
                           : algorithm == 1 ? ddm::Algorithm::WithoutFt
                                            : ddm::Algorithm::Direct;
        config.precision = precision == 0 ? ddm::Precision::F32 : ddm::Precision::F64;
        config.lags.assign(lags, lags + n_lags);
        if (has_q_max)
            config.q_max = q_max;
        config.memory_bytes = memory_bytes;
        config.workers = workers;
        const ddm::ResultArchive archive = ddm::run(source, config);
        if (static_cast<std::int64_t>(archive.map.values.size()) > out_capacity)
            throw ddm::InputError("ref_run: output capacity too small");
        std::copy(archive.map.values.begin(), archive.map.values.end(), out_values);
        std::copy(archive.map.lags.begin(), archive.map.lags.end(), out_lags);
        *out_n_lags = static_cast<std::int64_t>(archive.map.lags.size());
        counters3[0] = archive.counters.spatial_ffts;
        counters3[1] = archive.counters.temporal_ffts;
        counters3[2] = archive.counters.pairs;
        timing6[0] = archive.timing.disk;
        timing6[1] = archive.timing.step1;
        timing6[2] = archive.timing.step2;
        timing6[3] = archive.timing.merge;
        timing6[4] = archive.timing.other;
        timing6[5] = archive.timing.total;
    });
}

// ddm::with_ft_sequence<S>, proj/core/src/temporal.cpp:141-148 (SequenceEngine::with_ft :77-112)
int ref_with_ft_sequence(const double* seq, std::int64_t n, int precision, double* d,
                         double* d_a, double* corr, std::uint64_t* temporal_ffts, char* err,
                         int errlen) {
    return guarded(err, errlen, [&] {
        ddm::RunCounters counters;
        ddm::LagProfile p;
        if (precision == 0) {
            const auto v = to_complex<float>(seq, n);
            p = ddm::with_ft_sequence<float>(v, &counters);
        } else {
            const auto v = to_complex<double>(seq, n);
            p = ddm::with_ft_sequence<double>(v, &counters);
        }
        std::copy(p.d.begin(), p.d.end(), d);
        std::copy(p.d_a.begin(), p.d_a.end(), d_a);
        std::copy(p.corr.begin(), p.corr.end(), corr);
        *temporal_ffts = counters.temporal_ffts;
    });
}

// ddm::correlation_term<S>, proj/core/src/temporal.cpp:131-139
int ref_correlation_term(const double* seq, std::int64_t n, int precision, double* corr,
                         char* err, int errlen) {
    return guarded(err, errlen, [&] {
        std::vector<double> c;
        if (precision == 0)
            c = ddm::correlation_term<float>(to_complex<float>(seq, n));
        else
            c = ddm::correlation_term<double>(to_complex<double>(seq, n));
        std::copy(c.begin(), c.end(), corr);
    });
}

// ddm::averages_term<S>, proj/core/src/temporal.cpp:19-42
int ref_averages_term(const double* seq, std::int64_t n, int precision, double* d_a,
                      char* err, int errlen) {
    return guarded(err, errlen, [&] {
        std::vector<double> a;
        if (precision == 0)
            a = ddm::averages_term<float>(to_complex<float>(seq, n));
        else
            a = ddm::averages_term<double>(to_complex<double>(seq, n));
        std::copy(a.begin(), a.end(), d_a);
    });
}

// ddm::direct_sequence_oracle, proj/core/src/temporal.cpp:150-177
int ref_direct_sequence_oracle(const double* seq, std::int64_t n, double* d, double* d_a,
                               double* corr, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const auto p = ddm::direct_sequence_oracle(to_complex<double>(seq, n));
        std::copy(p.d.begin(), p.d.end(), d);
        std::copy(p.d_a.begin(), p.d_a.end(), d_a);
        std::copy(p.corr.begin(), p.corr.end(), corr);
    });
}

// ddm::forward_spectrum<S>, proj/core/src/spectrum.cpp:12-27 (SpatialTransform, fft.cpp:67-140)
int ref_forward_spectrum(const double* frame, int width, int height, int precision,
                         double* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const std::size_t np = static_cast<std::size_t>(width) * height;
        if (precision == 0) {
            std::vector<float> f(frame, frame + np);
            const auto s = ddm::forward_spectrum<float>(f, width, height);
            for (std::size_t k = 0; k < s.size(); ++k) {
                out[2 * k] = s[k].real();
                out[2 * k + 1] = s[k].imag();
            }
        } else {
            std::vector<double> f(frame, frame + np);
            const auto s = ddm::forward_spectrum<double>(f, width, height);
            for (std::size_t k = 0; k < s.size(); ++k) {
                out[2 * k] = s[k].real();
                out[2 * k + 1] = s[k].imag();
            }
        }
    });
}

// ddm::generate, proj/core/src/synth.cpp:98-132
int ref_generate(std::int64_t particles, double diffusion, double psf_sigma, double amplitude,
                 double background, int width, int height, int frames, double frame_interval,
                 std::uint64_t seed, std::uint16_t* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
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
        const auto stack = ddm::generate(c);
        std::copy(stack.pixels.begin(), stack.pixels.end(), out);
    });
}

// ddm::cutoff_set, proj/core/src/spectrum.cpp:65-84 (flat indices, spectrum.hpp:63-68)
int ref_cutoff_set(int width, int height, int has_q_max, double q_max, std::int64_t* count,
                   std::int64_t* flat_out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const auto set = ddm::cutoff_set(width, height,
                                         has_q_max ? std::optional<double>(q_max) : std::nullopt);
        *count = set.count();
        if (flat_out)
            for (std::int64_t k = 0; k < set.count(); ++k)
                flat_out[k] = set.flat(k);
    });
}

// ddm::plan_with_ft, proj/core/src/scheduler.cpp:365-384
int ref_plan_with_ft(std::int64_t q_count, std::int64_t frames, std::int64_t bytes,
                     int precision, std::int64_t* capacity, std::int64_t* groups, char* err,
                     int errlen) {
    return guarded(err, errlen, [&] {
        const auto plan = ddm::plan_with_ft(
            q_count, frames,
            {bytes, precision == 0 ? ddm::Precision::F32 : ddm::Precision::F64});
        *capacity = plan.capacity;
        *groups = plan.group_count();
    });
}

// ddm::azimuthal_average, proj/core/src/analysis.cpp:61-97
int ref_azimuthal(const double* values, const std::int64_t* lags, std::int64_t n_lags,
                  int width, int height, int has_q_max, double q_max, double* means,
                  std::int64_t* counts, std::int64_t capacity_bins, std::int64_t* bin_count,
                  char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ddm::ResultMap map;
        map.width = width;
        map.height = height;
        map.lags.assign(lags, lags + n_lags);
        map.values.assign(values, values + static_cast<std::size_t>(map.plane_size() * n_lags));
        const auto wv =
            ddm::cutoff_set(width, height, has_q_max ? std::optional<double>(q_max) : std::nullopt);
        const auto prof = ddm::azimuthal_average(map, wv);
        *bin_count = prof.bin_count;
        if (prof.bin_count > capacity_bins)
            throw ddm::InputError("ref_azimuthal: bin capacity too small");
        std::copy(prof.counts.begin(), prof.counts.end(), counts);
        std::copy(prof.means.begin(), prof.means.end(), means);
    });
}

} // extern "C"

extern "C" {

// The `ddm analyze` artefact set, composed exactly as tools/ddm_cli.cpp:206-240 composes it
// (open_frame_source, run with out_dir, write_results, azimuthal_average + write_radial_csv,
// fit_all_bins + write_fits_csv); run.json is the CLI's option echo and is not written.
// format: 0 raw_stack, 1 pgm_dir.
int ref_analyze(const char* path, int format, int algorithm, int precision,
                const std::int64_t* lags, std::int64_t n_lags, int has_q_max, double q_max,
                std::int64_t memory_bytes, int workers, const char* out_dir, char* err,
                int errlen) {
    return guarded(err, errlen, [&] {
        const auto source = ddm::open_frame_source(
            path, format == 1 ? ddm::StackFormat::PgmDir : ddm::StackFormat::RawStack);
        ddm::RunConfig config;
        config.algorithm = algorithm == 0   ? ddm::Algorithm::WithFt
                           : algorithm == 1 ? ddm::Algorithm::WithoutFt
                                            : ddm::Algorithm::Direct;
        config.precision = precision == 0 ? ddm::Precision::F32 : ddm::Precision::F64;
        config.lags.assign(lags, lags + n_lags);
        if (has_q_max)
            config.q_max = q_max;
        config.memory_bytes = memory_bytes;
        config.workers = workers;
        config.out_dir = out_dir;
        const ddm::ResultArchive archive = ddm::run(*source, config);
        ddm::write_results(archive, out_dir);
        const auto wv = ddm::cutoff_set(static_cast<int>(archive.map.width),
                                        static_cast<int>(archive.map.height), archive.q_max);
        const ddm::RadialProfile profile = ddm::azimuthal_average(archive.map, wv);
        ddm::write_radial_csv(profile, std::filesystem::path(out_dir) / "radial.csv");
        const auto fits = ddm::fit_all_bins(profile);
        if (!fits.empty())
            ddm::write_fits_csv(fits, std::filesystem::path(out_dir) / "fits.csv");
    });
}

} // extern "C"

extern "C" {

// ddm::sweep + write_bench_csv + crossover (proj/core/src/bench.cpp), as tools/ddm_cli.cpp:338-385
// drives them with the synthetic stack factory.
int ref_bench_sweep(const int* frame_counts, int n_frame_counts, const int* sizes, int n_sizes,
                    const int* algorithms, int n_algorithms, const int* workers, int n_workers,
                    const std::int64_t* budgets, int n_budgets, int repetitions, int warmup,
                    const char* out_csv, int* crossover_n, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ddm::SweepSpec spec;
        spec.frame_counts.assign(frame_counts, frame_counts + n_frame_counts);
        spec.sizes.assign(sizes, sizes + n_sizes);
        for (int i = 0; i < n_algorithms; ++i)
            spec.algorithms.push_back(algorithms[i] == 0   ? ddm::Algorithm::WithFt
                                      : algorithms[i] == 1 ? ddm::Algorithm::WithoutFt
                                                           : ddm::Algorithm::Direct);
        spec.worker_counts.assign(workers, workers + n_workers);
        if (n_budgets > 0)
            spec.budgets.assign(budgets, budgets + n_budgets);
        spec.repetitions = repetitions;
        spec.warmup = warmup;
        const auto table = ddm::sweep(spec, ddm::synthetic_stack_factory());
        ddm::write_bench_csv(table, out_csv);
        const auto xs = ddm::crossover(table);
        for (std::size_t i = 0; i < xs.size(); ++i)
            crossover_n[i] = xs[i].n_star ? *xs[i].n_star : -1;
    });
}

} // extern "C"
