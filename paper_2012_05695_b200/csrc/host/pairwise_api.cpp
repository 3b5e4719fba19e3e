// The reference's classical-engine entry points (`pairwise.cpp:11-117`) on the device:
// spectra (given, or computed on the GPU for direct_eq1) are gathered wave-vector-major and
// run through the pairwise kernel, which keeps the reference's f64 accumulation order.
#include "ddm/errors.hpp"
#include "ddm/pairwise.hpp"
#include "run_internal.hpp"

#include <algorithm>

namespace ddm {

template <typename Scalar>
void accumulate_difference(std::span<const std::complex<Scalar>> earlier,
                           std::span<const std::complex<Scalar>> later,
                           std::span<const std::int64_t> idx, std::span<double> acc) {
    for (std::size_t j = 0; j < idx.size(); ++j) {
        const auto k = std::size_t(idx[j]);
        const double re = double(earlier[k].real()) - double(later[k].real());
        const double im = double(earlier[k].imag()) - double(later[k].imag());
        acc[j] += re * re + im * im;
    }
}

namespace {

std::uint64_t pair_count(const std::vector<std::int64_t>& lags, std::int64_t frames) {
    std::uint64_t pairs = 0;
    for (const auto m : lags)
        if (m > 0) pairs += std::uint64_t(frames - m);
    return pairs;
}

// d_spec: frame-major [N][plane] spectra on the device (working precision f64 or f32) ->
// out.values (lag-major f64, zeros outside wv)
void pairwise_on_device(b200::Engine& eng, const void* d_spec, bool f64, int N, std::int64_t plane,
                        const WaveVectorSet& wv, ResultMap& out) {
    cudaStream_t st = eng.stream();
    const std::int64_t count = wv.count();
    const std::size_t cs = f64 ? 16 : 8;
    std::vector<std::int64_t> flat(static_cast<std::size_t>(count));
    for (std::int64_t k = 0; k < count; ++k) flat[std::size_t(k)] = wv.flat(k);
    std::vector<int> lags(out.lags.begin(), out.lags.end());
    const std::size_t total = out.values.size();
    auto* d_flat = static_cast<std::int64_t*>(eng.buffer("pw_flat", std::max<std::size_t>(flat.size(), 1) * 8));
    auto* d_lags = static_cast<int*>(eng.buffer("pw_lags", std::max<std::size_t>(lags.size(), 1) * 4));
    void* d_seq = eng.buffer("pw_seq", std::max<std::size_t>(std::size_t(count) * N * cs, 16));
    auto* d_map = static_cast<double*>(eng.buffer("pw_map", std::max<std::size_t>(total, 1) * 8));
    b200::check(cudaMemcpyAsync(d_flat, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, st), "upload");
    b200::check(cudaMemcpyAsync(d_lags, lags.data(), lags.size() * 4, cudaMemcpyHostToDevice, st), "upload");
    b200::check(cudaMemsetAsync(d_map, 0, total * 8, st), "memset");
    b200::check(f64 ? ddmk::launch_gather_sequences<double>(d_spec, N, plane, d_flat, count, d_seq, st)
                    : ddmk::launch_gather_sequences<float>(d_spec, N, plane, d_flat, count, d_seq, st),
                "gather kernel");
    int lag0 = lags.empty() ? -1 : lags[0];
    for (std::size_t i = 1; i < lags.size() && lag0 >= 0; ++i)
        if (lags[i] != lags[0] + int(i)) lag0 = -1;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, eng.device());
    b200::check(f64 ? ddmk::launch_pairwise<double>(d_seq, N, count, d_lags, int(lags.size()), d_map,
                                                    plane, d_flat, sms, st, lag0)
                    : ddmk::launch_pairwise<float>(d_seq, N, count, d_lags, int(lags.size()), d_map,
                                                   plane, d_flat, sms, st, lag0),
                "pairwise kernel");
    b200::check(cudaMemcpyAsync(out.values.data(), d_map, total * 8, cudaMemcpyDeviceToHost, st), "download");
    b200::check(cudaStreamSynchronize(st), "sync");
}

}  // namespace

template <typename Scalar>
ResultMap without_ft(const SpectrumStack<Scalar>& spectra, std::vector<std::int64_t> lags,
                     const WaveVectorSet& wave_vectors, int workers, RunCounters* counters) {
    if (wave_vectors.width != spectra.width || wave_vectors.height != spectra.height)
        throw InputError("without_ft: wave-vector set does not match spectra");
    lags = normalize_lags(std::move(lags), spectra.frames);
    if (workers < 1) throw InputError("workers must be at least 1");
    ResultMap out;
    out.width = spectra.width;
    out.height = spectra.height;
    out.lags = lags;
    out.values.assign(std::size_t(out.plane_size()) * lags.size(), 0.0);
    const int N = spectra.frames;
    if (std::int64_t(N) * 16 > 227 * 1024)
        throw PlanError("sequence of " + std::to_string(N) + " frames exceeds the device pairwise "
                        "engine limit of " + std::to_string(227 * 1024 / 16));
    if (N > 0 && wave_vectors.count() > 0 && !out.values.empty()) {
        detail::guard_device([&] {
            b200::Engine& eng = b200::Engine::instance(0);
            std::lock_guard<std::mutex> lock(eng.mutex());
            const std::size_t bytes = spectra.amplitudes.size() * sizeof(std::complex<Scalar>);
            void* d_spec = eng.buffer("pw_spectra", std::max<std::size_t>(bytes, 16));
            detail::upload_pageable(eng, d_spec, spectra.amplitudes.data(), bytes, eng.stream());
            pairwise_on_device(eng, d_spec, sizeof(Scalar) == 8, N, spectra.plane_size(), wave_vectors, out);
            return 0;
        });
    }
    if (counters) counters->pairs += pair_count(lags, N);
    return out;
}

ResultMap direct_eq1(const ImageStack& stack, std::vector<std::int64_t> lags, RunCounters* counters) {
    stack.validate();
    lags = normalize_lags(std::move(lags), stack.frames);
    ResultMap out;
    out.width = stack.width;
    out.height = stack.height;
    out.frame_interval = stack.frame_interval;
    out.lags = lags;
    out.values.assign(std::size_t(out.plane_size()) * lags.size(), 0.0);
    const int N = stack.frames;
    if (std::int64_t(N) * 16 > 227 * 1024)
        throw PlanError("sequence of " + std::to_string(N) + " frames exceeds the device pairwise "
                        "engine limit of " + std::to_string(227 * 1024 / 16));
    const WaveVectorSet wv = cutoff_set(stack.width, stack.height, std::nullopt);
    detail::guard_device([&] {
        b200::Engine& eng = b200::Engine::instance(0);
        std::lock_guard<std::mutex> lock(eng.mutex());
        const std::size_t px = stack.pixels.size() * 2;
        void* d_frames = eng.buffer("pw_frames", std::max<std::size_t>(px, 16));
        detail::upload_pageable(eng, d_frames, stack.pixels.data(), px, eng.stream());
        const std::int64_t plane = out.plane_size();
        void* d_spec = eng.buffer("pw_spectra", std::size_t(N) * plane * 16);
        eng.spectra(d_frames, 2, stack.width, stack.height, N, true, d_spec);
        pairwise_on_device(eng, d_spec, true, N, plane, wv, out);
        return 0;
    });
    const std::uint64_t transforms = pair_count(lags, N);
    if (counters) {
        counters->spatial_ffts += transforms;
        counters->pairs += transforms;
    }
    return out;
}

template void accumulate_difference<float>(std::span<const std::complex<float>>,
                                           std::span<const std::complex<float>>,
                                           std::span<const std::int64_t>, std::span<double>);
template void accumulate_difference<double>(std::span<const std::complex<double>>,
                                            std::span<const std::complex<double>>,
                                            std::span<const std::int64_t>, std::span<double>);
template ResultMap without_ft<float>(const SpectrumStack<float>&, std::vector<std::int64_t>,
                                     const WaveVectorSet&, int, RunCounters*);
template ResultMap without_ft<double>(const SpectrumStack<double>&, std::vector<std::int64_t>,
                                      const WaveVectorSet&, int, RunCounters*);

}  // namespace ddm
