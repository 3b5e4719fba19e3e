// Ring fits on the host side of the boundary, the analysis CSV writers and the `ddm analyze`
// artefact set as a library call (reference `analysis.cpp:99-304`, `tools/ddm_cli.cpp:206-240`).
#include "ddm/analysis.hpp"
#include "ddm/archive.hpp"
#include "ddm/errors.hpp"
#include "ddm/scheduler.hpp"
#include "run_internal.hpp"

#include <cmath>
#include <cstdio>
#include <fstream>

namespace fs = std::filesystem;

namespace ddm {

std::string to_string(ExponentialFit::Flag flag) {
    switch (flag) {
    case ExponentialFit::Flag::Ok: return "ok";
    case ExponentialFit::Flag::Degenerate: return "degenerate";
    case ExponentialFit::Flag::NoConverge: return "no_converge";
    }
    return "?";
}

namespace {

// fit_all_bins on a chosen device (analyze passes RunConfig::device)
std::vector<ExponentialFit> fit_all_bins_on(const RadialProfile& p, int device) {
    std::vector<ExponentialFit> fits;
    std::int64_t usable = 0;
    for (const auto m : p.lags)
        if (m >= 1) ++usable;
    if (usable < 4 || p.bin_count < 1) return fits;
    const std::size_t L = p.lags.size(), B = std::size_t(p.bin_count);
    std::vector<double> out(4 * B);
    std::vector<int> flag(B);
    detail::guard_device([&] {
        b200::Engine& eng = b200::Engine::instance(device);
        std::lock_guard<std::mutex> lock(eng.mutex());
        cudaStream_t st = eng.stream();
        char* base = static_cast<char*>(eng.buffer("fit_io", L * B * 8 + L * 8 + B * 8 + 4 * B * 8 + B * 4));
        double* d_means = reinterpret_cast<double*>(base);
        std::int64_t* d_lags = reinterpret_cast<std::int64_t*>(d_means + L * B);
        std::int64_t* d_counts = d_lags + L;
        double* d_out = reinterpret_cast<double*>(d_counts + B);
        int* d_flag = reinterpret_cast<int*>(d_out + 4 * B);
        b200::check(cudaMemcpyAsync(d_means, p.means.data(), L * B * 8, cudaMemcpyHostToDevice, st), "upload");
        b200::check(cudaMemcpyAsync(d_lags, p.lags.data(), L * 8, cudaMemcpyHostToDevice, st), "upload");
        b200::check(cudaMemcpyAsync(d_counts, p.counts.data(), B * 8, cudaMemcpyHostToDevice, st), "upload");
        b200::check(ddmk::launch_fit_rings(d_means, d_lags, int(L), d_counts, std::int64_t(B), p.frame_interval,
                                           d_out, d_out + B, d_out + 2 * B, d_out + 3 * B, d_flag, st),
                    "fit kernel");
        b200::check(cudaMemcpyAsync(out.data(), d_out, 4 * B * 8, cudaMemcpyDeviceToHost, st), "download");
        b200::check(cudaMemcpyAsync(flag.data(), d_flag, B * 4, cudaMemcpyDeviceToHost, st), "download");
        b200::check(cudaStreamSynchronize(st), "sync");
        return 0;
    });
    for (std::size_t b = 0; b < B; ++b) {
        if (flag[b] < 0) continue;
        ExponentialFit f;
        f.q_bin = std::int64_t(b);
        f.amplitude = out[b];
        f.baseline = out[B + b];
        f.tau = out[2 * B + b];
        f.residual = out[3 * B + b];
        f.flag = flag[b] == 0 ? ExponentialFit::Flag::Ok
                              : flag[b] == 1 ? ExponentialFit::Flag::Degenerate : ExponentialFit::Flag::NoConverge;
        fits.push_back(f);
    }
    return fits;
}

}  // namespace

std::vector<ExponentialFit> fit_all_bins(const RadialProfile& p) { return fit_all_bins_on(p, 0); }

ExponentialFit fit_exponential(const RadialProfile& p, std::int64_t q_bin) {
    if (q_bin < 0 || q_bin >= p.bin_count) throw InputError("fit_exponential: bin out of range");
    if (p.counts[std::size_t(q_bin)] < 1) throw InputError("fit_exponential: empty bin");
    RadialProfile one;
    one.bin_count = 1;
    one.frame_interval = p.frame_interval;
    one.lags = p.lags;
    one.counts = {p.counts[std::size_t(q_bin)]};
    one.means.resize(p.lags.size());
    std::size_t usable = 0;
    for (std::size_t li = 0; li < p.lags.size(); ++li) {
        one.means[li] = p.mean(std::int64_t(li), q_bin);
        if (p.lags[li] >= 1 && std::isfinite(one.means[li])) ++usable;
    }
    if (usable < 4) throw InputError("fit_exponential: need at least 4 usable lags");
    auto fits = fit_all_bins_on(one, 0);
    if (fits.empty()) throw InputError("fit_exponential: need at least 4 usable lags");
    fits.front().q_bin = q_bin;
    return fits.front();
}

DiffusionEstimate estimate_diffusion(const std::vector<ExponentialFit>& fits, std::int64_t width,
                                     std::int64_t q_lo, std::int64_t q_hi) {
    if (width < 1) throw InputError("estimate_diffusion: bad width");
    const double two_pi = 2.0 * std::acos(-1.0);
    double sxx = 0.0, sxy = 0.0;
    DiffusionEstimate e;
    for (const auto& f : fits) {
        if (f.flag != ExponentialFit::Flag::Ok || f.q_bin < q_lo || f.q_bin > q_hi) continue;
        const double q = two_pi * double(f.q_bin) / double(width);
        const double x = q * q;
        sxx += x * x;
        sxy += x * (1.0 / f.tau);
        ++e.bins_used;
    }
    if (e.bins_used > 0 && sxx > 0.0) e.coefficient = sxy / sxx;
    return e;
}

namespace {

// "%.17g" = the reference's ostream precision(17) in default float format
void put_double(std::FILE* f, double v) { std::fprintf(f, "%.17g", v); }

}  // namespace

void write_radial_csv(const RadialProfile& p, const fs::path& path) {
    // rows formatted per lag on the host pool (a C2 profile is ~370k rows), written in order
    std::vector<std::string> blocks(p.lags.size());
    detail::parallel_for(p.lags.size(), [&](std::size_t li) {
        std::string& b = blocks[li];
        char line[96];
        for (std::int64_t bin = 0; bin < p.bin_count; ++bin) {
            const auto c = p.counts[std::size_t(bin)];
            if (c < 1) continue;
            const int n = std::snprintf(line, sizeof line, "%lld,%lld,%.17g,%lld\n", (long long)p.lags[li],
                                        (long long)bin, p.mean(std::int64_t(li), bin), (long long)c);
            b.append(line, std::size_t(n));
        }
    });
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open " + path.string() + " for writing");
    std::fputs("lag,q_bin,mean,count\n", f);
    for (const auto& b : blocks) std::fwrite(b.data(), 1, b.size(), f);
    if (std::ferror(f) || std::fclose(f) != 0) throw IoError("write failed for " + path.string());
}

void write_fits_csv(const std::vector<ExponentialFit>& fits, const fs::path& path) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open " + path.string() + " for writing");
    std::fputs("q_bin,A,B,tau_seconds,residual,flag\n", f);
    for (const auto& x : fits) {
        std::fprintf(f, "%lld,", (long long)x.q_bin);
        put_double(f, x.amplitude);
        std::fputc(',', f);
        put_double(f, x.baseline);
        std::fputc(',', f);
        put_double(f, x.tau);
        std::fputc(',', f);
        put_double(f, x.residual);
        std::fprintf(f, ",%s\n", to_string(x.flag).c_str());
    }
    if (std::fclose(f) != 0) throw IoError("write failed for " + path.string());
}

ResultArchive analyze(FrameSource& source, RunConfig config, const fs::path& out_dir) {
    detail::Trace trace("analyze");
    config.out_dir = out_dir;  // as `ddm analyze`: the run's workspace is the output directory
    ResultArchive a = run(source, config);
    trace.lap("run");
    write_results(a, out_dir);
    trace.lap("write");
    const auto wv = cutoff_set(int(a.map.width), int(a.map.height), a.q_max);
    const RadialProfile profile = azimuthal_average(a.map, wv);
    trace.lap("azimuthal");
    write_radial_csv(profile, out_dir / "radial.csv");
    const auto fits = fit_all_bins_on(profile, config.device);
    if (!fits.empty()) write_fits_csv(fits, out_dir / "fits.csv");
    trace.lap("fits+csv");
    return a;
}

}  // namespace ddm

namespace ddm {

double b200::relative_deviation(const ResultMap& a, const ResultMap& b) {
    double peak = 0.0;
    for (const double v : a.values) peak = std::max(peak, std::abs(v));
    for (const double v : b.values) peak = std::max(peak, std::abs(v));
    return peak == 0.0 ? 0.0 : max_abs_difference(a, b) / peak;
}

CompareReport compare(FrameSource& source, const RunConfig& config, Algorithm a, Algorithm b) {
    CompareReport r;
    ResultArchive out[2];
    const Algorithm algs[2] = {a, b};
    for (int i = 0; i < 2; ++i) {
        RunConfig c = config;
        c.algorithm = algs[i];
        out[i] = run(source, c);
        r.algorithms[i] = out[i].algorithm;
        r.timing[i] = out[i].timing;
    }
    r.deviation = b200::relative_deviation(out[0].map, out[1].map);
    r.tolerance = config.precision == Precision::F32 ? 1e-4 : 1e-9;
    r.pass = r.deviation <= r.tolerance;
    return r;
}

}  // namespace ddm
