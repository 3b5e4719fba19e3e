// Reference-mirroring entry points around the hot path:
//   pad_length / combine            (`temporal.cpp:10-17,114-129`, host arithmetic)
//   SequenceEngine / with_ft_sequence (`temporal.cpp:44-148`, evaluated on the GPU)
//   forward_spectrum / compute_spectra (`spectrum.cpp:12-63`, evaluated on the GPU)
//   azimuthal_average               (`analysis.cpp:61-97`, GPU ring reduction)
//   generate                        (`synth.cpp:98-132`, host input generator, bit-exact)
#include "ddm/analysis.hpp"
#include "ddm/errors.hpp"
#include "ddm/spectrum.hpp"
#include "ddm/synth.hpp"
#include "ddm/temporal.hpp"
#include "run_internal.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

namespace ddm {

namespace {

// Scoped device allocation on the engine stream.
struct DevMem {
    void* p = nullptr;
    explicit DevMem(std::size_t bytes) { b200::check(cudaMalloc(&p, std::max<std::size_t>(bytes, 16)), "cudaMalloc"); }
    ~DevMem() { cudaFree(p); }
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
};

}  // namespace

std::int64_t pad_length(std::int64_t frames) {
    if (frames < 1) throw InputError("pad_length: sequence must have at least one frame");
    std::int64_t n2 = 1;
    while (n2 < frames) n2 <<= 1;
    return n2 << 1;
}

LagProfile combine(std::vector<double> d_a, std::vector<double> corr) {
    if (d_a.size() != corr.size()) throw InputError("combine: term lengths differ");
    const auto n = std::int64_t(d_a.size());
    LagProfile out;
    out.d.resize(d_a.size());
    for (std::int64_t m = 0; m < n; ++m)
        out.d[std::size_t(m)] = d_a[std::size_t(m)] - 2.0 * corr[std::size_t(m)] / double(n - m);
    out.d_a = std::move(d_a);
    out.corr = std::move(corr);
    return out;
}

template <typename Scalar>
SequenceEngine<Scalar>::SequenceEngine(std::int64_t frames, int device)
    : frames_(frames), device_(device) {
    if (frames < 1) throw InputError("pad_length: sequence must have at least one frame");
    if (frames > b200::max_frames(sizeof(Scalar) == 8))
        throw PlanError("sequence length beyond the device temporal engine limit");
}

template <typename Scalar>
LagProfile SequenceEngine<Scalar>::with_ft(std::span<const std::complex<Scalar>> seq) {
    if (std::int64_t(seq.size()) != frames_)
        throw InputError("SequenceEngine: sequence length does not match engine");
    return detail::guard_device([&] {
        b200::Engine& eng = b200::Engine::instance(device_);
        std::lock_guard<std::mutex> lock(eng.mutex());
        const std::size_t n = seq.size();
        DevMem in(n * sizeof(std::complex<Scalar>)), out(3 * n * sizeof(double));
        b200::check(cudaMemcpy(in.p, seq.data(), n * sizeof(std::complex<Scalar>),
                               cudaMemcpyHostToDevice), "upload");
        double* d = static_cast<double*>(out.p);
        eng.sequences(in.p, 1, frames_, sizeof(Scalar) == 8, d, d + n, d + 2 * n);
        LagProfile p;
        p.d.resize(n);
        p.d_a.resize(n);
        p.corr.resize(n);
        std::vector<double> host(3 * n);
        b200::check(cudaMemcpy(host.data(), d, 3 * n * sizeof(double), cudaMemcpyDeviceToHost), "download");
        std::copy(host.begin(), host.begin() + n, p.d.begin());
        std::copy(host.begin() + n, host.begin() + 2 * n, p.d_a.begin());
        std::copy(host.begin() + 2 * n, host.end(), p.corr.begin());
        temporal_ffts_ += 2;
        return p;
    });
}

template <typename Scalar>
std::vector<double> SequenceEngine<Scalar>::correlation(std::span<const std::complex<Scalar>> seq) {
    // the engine's corr is restored to the original basis: the raw sum of `temporal.cpp:48-75`
    return with_ft(seq).corr;
}

template <typename Scalar>
std::vector<double> SequenceEngine<Scalar>::with_ft_batch(std::span<const std::complex<Scalar>> seqs) {
    if (seqs.size() % std::size_t(frames_) != 0)
        throw InputError("SequenceEngine: batch is not a whole number of sequences");
    const std::int64_t q = std::int64_t(seqs.size()) / frames_;
    return detail::guard_device([&] {
        b200::Engine& eng = b200::Engine::instance(device_);
        std::lock_guard<std::mutex> lock(eng.mutex());
        DevMem in(seqs.size() * sizeof(std::complex<Scalar>)), out(seqs.size() * sizeof(double));
        b200::check(cudaMemcpy(in.p, seqs.data(), seqs.size() * sizeof(std::complex<Scalar>),
                               cudaMemcpyHostToDevice), "upload");
        eng.sequences(in.p, q, frames_, sizeof(Scalar) == 8, static_cast<double*>(out.p), nullptr, nullptr);
        std::vector<double> d(seqs.size());
        b200::check(cudaMemcpy(d.data(), out.p, d.size() * sizeof(double), cudaMemcpyDeviceToHost), "download");
        temporal_ffts_ += 2 * std::uint64_t(q);
        return d;
    });
}

template <typename Scalar>
LagProfile with_ft_sequence(std::span<const std::complex<Scalar>> seq, RunCounters* counters) {
    SequenceEngine<Scalar> engine(std::int64_t(seq.size()));
    LagProfile p = engine.with_ft(seq);
    if (counters) counters->temporal_ffts += engine.temporal_fft_count();
    return p;
}

template <typename Scalar>
std::vector<double> averages_term(std::span<const std::complex<Scalar>> seq) {
    SequenceEngine<Scalar> engine(std::int64_t(seq.size()));
    return engine.with_ft(seq).d_a;
}

template <typename Scalar>
std::vector<double> correlation_term(std::span<const std::complex<Scalar>> seq, RunCounters* counters) {
    SequenceEngine<Scalar> engine(std::int64_t(seq.size()));
    std::vector<double> c = engine.correlation(seq);
    if (counters) counters->temporal_ffts += engine.temporal_fft_count();
    return c;
}

LagProfile direct_sequence_oracle(std::span<const std::complex<double>> seq) {
    const auto n = std::int64_t(seq.size());
    if (n < 1) throw InputError("direct_sequence_oracle: empty sequence");
    LagProfile out;
    out.d.resize(seq.size());
    out.d_a.resize(seq.size());
    out.corr.resize(seq.size());
    for (std::int64_t m = 0; m < n; ++m) {
        double sd = 0.0, sa = 0.0, sc = 0.0;
        for (std::int64_t k = m; k < n; ++k) {
            const auto a = seq[std::size_t(k - m)], b = seq[std::size_t(k)];
            sd += std::norm(a - b);
            sa += std::norm(a) + std::norm(b);
            sc += a.real() * b.real() + a.imag() * b.imag();
        }
        const double ramp = double(n - m);
        out.d[std::size_t(m)] = sd / ramp;
        out.d_a[std::size_t(m)] = sa / ramp;
        out.corr[std::size_t(m)] = sc;
    }
    return out;
}

template std::vector<double> averages_term<float>(std::span<const std::complex<float>>);
template std::vector<double> averages_term<double>(std::span<const std::complex<double>>);
template std::vector<double> correlation_term<float>(std::span<const std::complex<float>>, RunCounters*);
template std::vector<double> correlation_term<double>(std::span<const std::complex<double>>, RunCounters*);
template class SequenceEngine<float>;
template class SequenceEngine<double>;
template LagProfile with_ft_sequence<float>(std::span<const std::complex<float>>, RunCounters*);
template LagProfile with_ft_sequence<double>(std::span<const std::complex<double>>, RunCounters*);

template <typename Scalar>
std::vector<std::complex<Scalar>> forward_spectrum(std::span<const Scalar> frame, int width,
                                                   int height) {
    if (width < 1 || height < 1) throw InputError("fft: frame dimensions must be positive");
    if (frame.size() != std::size_t(width) * height)
        throw InputError("forward_spectrum: frame size does not match dimensions");
    for (const Scalar v : frame)
        if (!std::isfinite(v)) throw InputError("forward_spectrum: non-finite input value");
    return detail::guard_device([&] {
        b200::Engine& eng = b200::Engine::instance(0);
        std::lock_guard<std::mutex> lock(eng.mutex());
        const std::size_t np = std::size_t(height) * half_cols(width);
        DevMem in(frame.size_bytes()), out(np * sizeof(std::complex<Scalar>));
        b200::check(cudaMemcpy(in.p, frame.data(), frame.size_bytes(), cudaMemcpyHostToDevice), "upload");
        eng.spectra(in.p, int(sizeof(Scalar)), width, height, 1, sizeof(Scalar) == 8, out.p);
        std::vector<std::complex<Scalar>> spec(np);
        b200::check(cudaMemcpy(spec.data(), out.p, np * sizeof(std::complex<Scalar>), cudaMemcpyDeviceToHost),
                    "download");
        return spec;
    });
}

template <typename Scalar>
SpectrumStack<Scalar> compute_spectra(const FrameSource& source, int workers, RunCounters* counters) {
    if (workers < 1) throw InputError("workers must be at least 1");
    SpectrumStack<Scalar> st;
    st.width = source.width();
    st.height = source.height();
    st.frames = source.frames();
    const std::size_t ppf = std::size_t(source.pixels_per_frame());
    std::vector<std::uint16_t> staged;
    const std::uint16_t* px = source.contiguous();
    if (!px) {
        staged.resize(ppf * std::size_t(st.frames));
        for (int n = 0; n < st.frames; ++n) source.read_frame(n, {staged.data() + n * ppf, ppf});
        px = staged.data();
    }
    st.amplitudes.resize(std::size_t(st.frames) * std::size_t(st.plane_size()));
    detail::guard_device([&] {
        b200::Engine& eng = b200::Engine::instance(0);
        std::lock_guard<std::mutex> lock(eng.mutex());
        DevMem in(ppf * 2 * st.frames), out(st.amplitudes.size() * sizeof(std::complex<Scalar>));
        b200::check(cudaMemcpy(in.p, px, ppf * 2 * st.frames, cudaMemcpyHostToDevice), "upload");
        eng.spectra(in.p, 2, st.width, st.height, st.frames, sizeof(Scalar) == 8, out.p);
        b200::check(cudaMemcpy(st.amplitudes.data(), out.p, st.amplitudes.size() * sizeof(std::complex<Scalar>),
                               cudaMemcpyDeviceToHost), "download");
        return 0;
    });
    if (counters) counters->spatial_ffts += std::uint64_t(st.frames);
    return st;
}

template std::vector<std::complex<float>> forward_spectrum<float>(std::span<const float>, int, int);
template std::vector<std::complex<double>> forward_spectrum<double>(std::span<const double>, int, int);
template SpectrumStack<float> compute_spectra<float>(const FrameSource&, int, RunCounters*);
template SpectrumStack<double> compute_spectra<double>(const FrameSource&, int, RunCounters*);

RadialProfile azimuthal_average(const ResultMap& map, const WaveVectorSet& wv) {
    if (wv.width != map.width || wv.height != map.height)
        throw InputError("azimuthal_average: wave-vector set does not match maps");
    const std::int64_t q = wv.count();
    std::vector<std::int64_t> bin(static_cast<std::size_t>(q));
    std::int64_t bmax = 0;
    for (std::int64_t k = 0; k < q; ++k) {
        const auto& v = wv.indices[std::size_t(k)];
        bin[std::size_t(k)] = std::llround(q_magnitude(v.row, v.col, int(map.height)));
        bmax = std::max(bmax, bin[std::size_t(k)]);
    }
    RadialProfile prof;
    prof.bin_count = bmax + 1;
    prof.frame_interval = map.frame_interval;
    prof.lags = map.lags;
    prof.counts.assign(std::size_t(prof.bin_count), 0);
    for (auto b : bin) ++prof.counts[std::size_t(b)];
    // CSR of plane positions grouped by bin, k-ascending within a bin (geometry only)
    std::vector<std::int64_t> off(std::size_t(prof.bin_count) + 1, 0);
    for (std::int64_t b = 0; b < prof.bin_count; ++b) off[std::size_t(b) + 1] = off[std::size_t(b)] + prof.counts[std::size_t(b)];
    std::vector<std::int64_t> order(static_cast<std::size_t>(q));
    {
        std::vector<std::int64_t> fill(off.begin(), off.end() - 1);
        for (std::int64_t k = 0; k < q; ++k) order[std::size_t(fill[std::size_t(bin[std::size_t(k)])]++)] = wv.flat(k);
    }
    const std::int64_t L = std::int64_t(map.lags.size());
    prof.means.assign(std::size_t(L * prof.bin_count), 0.0);
    if (L == 0) return prof;
    detail::guard_device([&] {
        b200::Engine& eng = b200::Engine::instance(0);
        std::lock_guard<std::mutex> lock(eng.mutex());
        DevMem dv(map.values.size() * sizeof(double)), dor(order.size() * sizeof(std::int64_t)),
            doff(off.size() * sizeof(std::int64_t)), dm(prof.means.size() * sizeof(double));
        cudaStream_t st = eng.stream();
        detail::upload_pageable(eng, dv.p, map.values.data(), map.values.size() * sizeof(double), st);
        b200::check(cudaMemcpyAsync(dor.p, order.data(), order.size() * sizeof(std::int64_t),
                                    cudaMemcpyHostToDevice, st), "upload");
        b200::check(cudaMemcpyAsync(doff.p, off.data(), off.size() * sizeof(std::int64_t),
                                    cudaMemcpyHostToDevice, st), "upload");
        b200::radial_means(static_cast<const double*>(dv.p), L, map.plane_size(),
                           static_cast<const std::int64_t*>(dor.p), static_cast<const std::int64_t*>(doff.p),
                           prof.bin_count, static_cast<double*>(dm.p), st);
        b200::check(cudaMemcpyAsync(prof.means.data(), dm.p, prof.means.size() * sizeof(double),
                                    cudaMemcpyDeviceToHost, st), "download");
        b200::check(cudaStreamSynchronize(st), "sync");
        return 0;
    });
    return prof;
}

// ---------------------------------------------------------------- synthetic stacks

void SynthConfig::validate() const {
    if (particles < 0) throw InputError("synth: particle count must be non-negative");
    if (diffusion < 0.0) throw InputError("synth: diffusion must be non-negative");
    if (psf_sigma <= 0.0) throw InputError("synth: psf sigma must be positive");
    if (width < 1 || height < 1 || frames < 1) throw InputError("synth: degenerate stack dimensions");
    if (amplitude < 0.0 || background < 0.0) throw InputError("synth: negative intensities");
    if (frame_interval <= 0.0) throw InputError("synth: frame interval must be positive");
}

namespace {

// Draw sequence pinned to the mt19937_64 output stream (top 53 bits -> [0,1)).
double draw01(std::mt19937_64& g) { return double(g() >> 11) * 0x1.0p-53; }

double periodic(double x, double period) {
    x = std::fmod(x, period);
    return x < 0.0 ? x + period : x;
}

void splat(const std::vector<double>& xs, const std::vector<double>& ys, const SynthConfig& c,
           std::uint16_t* out, std::vector<double>& canvas) {
    canvas.assign(std::size_t(c.width) * c.height, c.background);
    const double reach = 4.0 * c.psf_sigma;
    const double k = 1.0 / (2.0 * c.psf_sigma * c.psf_sigma);
    for (std::size_t p = 0; p < xs.size(); ++p) {
        const double cx = xs[p], cy = ys[p];
        const int y0 = int(std::floor(cy - reach)), y1 = int(std::ceil(cy + reach));
        const int x0 = int(std::floor(cx - reach)), x1 = int(std::ceil(cx + reach));
        for (int iy = y0; iy <= y1; ++iy) {
            const double dy = double(iy) - cy;
            const int row = ((iy % c.height) + c.height) % c.height;
            for (int ix = x0; ix <= x1; ++ix) {
                const double dx = double(ix) - cx;
                const double r2 = dx * dx + dy * dy;
                if (r2 > reach * reach) continue;
                const int col = ((ix % c.width) + c.width) % c.width;
                canvas[std::size_t(row) * c.width + col] += c.amplitude * std::exp(-r2 * k);
            }
        }
    }
    for (std::size_t i = 0; i < canvas.size(); ++i) {
        const double v = double(std::llround(canvas[i]));
        out[i] = std::uint16_t(std::clamp(v, 0.0, 65535.0));
    }
}

// Particle positions of every frame, [frames][particles][2] (x, y): the reference's draw
// sequence (`synth.cpp:98-132`): uniform starts, then per frame and particle one Box-Muller
// pair, periodic wrap.
std::vector<double> trajectories(const SynthConfig& c) {
    const auto np = std::size_t(c.particles);
    std::vector<double> pos(std::size_t(c.frames) * np * 2);
    std::mt19937_64 g(c.seed);
    std::vector<double> xs(np), ys(np);
    for (std::size_t p = 0; p < np; ++p) {
        xs[p] = draw01(g) * c.width;
        ys[p] = draw01(g) * c.height;
    }
    const double step = std::sqrt(2.0 * c.diffusion);
    const double two_pi = 2.0 * std::acos(-1.0);
    for (int n = 0; n < c.frames; ++n) {
        if (n > 0) {
            for (std::size_t p = 0; p < np; ++p) {
                // Box-Muller pair: u1 in (0, 1], u2 in [0, 1)
                const double u1 = (double(g() >> 11) + 1.0) * 0x1.0p-53;
                const double u2 = draw01(g);
                const double rad = std::sqrt(-2.0 * std::log(u1));
                const double th = two_pi * u2;
                xs[p] = periodic(xs[p] + step * (rad * std::cos(th)), c.width);
                ys[p] = periodic(ys[p] + step * (rad * std::sin(th)), c.height);
            }
        }
        double* f = pos.data() + std::size_t(n) * np * 2;
        for (std::size_t p = 0; p < np; ++p) {
            f[2 * p] = xs[p];
            f[2 * p + 1] = ys[p];
        }
    }
    return pos;
}

}  // namespace

ImageStack generate(const SynthConfig& c) {
    c.validate();
    ImageStack st;
    st.width = c.width;
    st.height = c.height;
    st.frames = c.frames;
    st.frame_interval = c.frame_interval;
    st.pixels.resize(std::size_t(c.frames) * std::size_t(st.pixels_per_frame()));
    const auto np = std::size_t(c.particles);
    const std::vector<double> pos = trajectories(c);
    std::vector<double> xs(np), ys(np), canvas;
    for (int n = 0; n < c.frames; ++n) {
        const double* f = pos.data() + std::size_t(n) * np * 2;
        for (std::size_t p = 0; p < np; ++p) {
            xs[p] = f[2 * p];
            ys[p] = f[2 * p + 1];
        }
        splat(xs, ys, c, st.frame(n).data(), canvas);
    }
    return st;
}

void generate_device(const SynthConfig& c, std::uint16_t* d_out, int device, void* stream) {
    c.validate();
    if (!d_out) throw InputError("null device buffer");
    const std::vector<double> pos = trajectories(c);
    detail::guard_device([&] {
        b200::Engine& eng = b200::Engine::instance(device);
        std::lock_guard<std::mutex> lock(eng.mutex());
        cudaStream_t st = eng.stream();
        cudaEvent_t ev;
        b200::check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        b200::check(cudaEventRecord(ev, static_cast<cudaStream_t>(stream)), "event record");
        b200::check(cudaStreamWaitEvent(st, ev, 0), "stream wait");
        void* d_pos = eng.buffer("synth_pos", std::max<std::size_t>(pos.size(), 1) * sizeof(double));
        b200::check(cudaMemcpyAsync(d_pos, pos.data(), pos.size() * sizeof(double), cudaMemcpyHostToDevice, st),
                    "upload");
        b200::check(ddmk::launch_render_frames(static_cast<const double*>(d_pos), int(c.particles), c.width,
                                               c.height, c.frames, c.psf_sigma, c.amplitude, c.background,
                                               d_out, st), "render kernel");
        b200::check(cudaEventRecord(ev, st), "event record");
        b200::check(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ev, 0), "stream wait");
        b200::check(cudaStreamSynchronize(st), "sync");   // `pos` is host memory
        cudaEventDestroy(ev);
        return 0;
    });
}

void write_synth_manifest(const SynthConfig& c, const std::filesystem::path& path) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open " + path.string() + " for writing");
    std::fprintf(f,
                 "{\n  \"amplitude\": %.17g,\n  \"background\": %.17g,\n  \"diffusion\": %.17g,\n"
                 "  \"frame_interval\": %.17g,\n  \"frames\": %d,\n  \"generator\": \"mt19937_64/box-muller\",\n"
                 "  \"height\": %d,\n  \"particles\": %lld,\n  \"psf_sigma\": %.17g,\n  \"seed\": %llu,\n"
                 "  \"tool_version\": \"0.1.0-b200\",\n  \"width\": %d\n}\n",
                 c.amplitude, c.background, c.diffusion, c.frame_interval, c.frames, c.height,
                 (long long)c.particles, c.psf_sigma, (unsigned long long)c.seed, c.width);
    if (std::fclose(f) != 0) throw IoError("write failed for " + path.string());
}

}  // namespace ddm
