// ddm-b200: half-plane geometry and the retained wave-vector list
// (reference `proj/core/include/ddm/spectrum.hpp:16-84`), plus the batched spatial
// transform computed on the GPU (`compute_spectra`, `forward_spectrum`).
#ifndef DDM_B200_SPECTRUM_HPP
#define DDM_B200_SPECTRUM_HPP

#include "ddm/frame_source.hpp"
#include "ddm/timing.hpp"

#include <cmath>
#include <complex>
#include <cstdint>
#include <optional>
#include <span>
#include <vector>

namespace ddm {

inline int half_cols(int width) { return width / 2 + 1; }

/// |q| of a half-plane position; rows past H/2 are negative vertical frequencies.
inline double q_magnitude(int row, int col, int height) {
    const int qr = row <= height / 2 ? row : row - height;
    return std::sqrt(double(qr) * qr + double(col) * col);
}

struct WaveVector {
    int row = 0;
    int col = 0;
};

/// Retained positions in row-major order; this order is the wave-vector index space of
/// groups and partial files.
struct WaveVectorSet {
    int width = 0;
    int height = 0;
    std::optional<double> q_max;
    std::vector<WaveVector> indices;

    std::int64_t count() const { return std::int64_t(indices.size()); }
    std::int64_t flat(std::int64_t k) const {
        const auto& v = indices[std::size_t(k)];
        return std::int64_t(v.row) * half_cols(width) + v.col;
    }
};

WaveVectorSet cutoff_set(int width, int height, std::optional<double> q_max);

/// Frame-major half-plane spectra (unnormalised forward transforms; DC = pixel sum).
template <typename Scalar>
struct SpectrumStack {
    int width = 0;
    int height = 0;
    int frames = 0;
    std::vector<std::complex<Scalar>> amplitudes;  // frames x height x half_cols

    std::int64_t plane_size() const { return std::int64_t(height) * half_cols(width); }
    std::span<const std::complex<Scalar>> frame(int n) const {
        return {amplitudes.data() + std::size_t(n) * plane_size(), std::size_t(plane_size())};
    }
};

/// One frame of finite real values -> height x half_cols spectrum (computed on the GPU).
template <typename Scalar>
std::vector<std::complex<Scalar>> forward_spectrum(std::span<const Scalar> frame, int width,
                                                   int height);

/// Every frame of the source, one batched GPU pass; `workers` is accepted for signature
/// compatibility and has no effect on values. Adds frames() to counters->spatial_ffts.
template <typename Scalar>
SpectrumStack<Scalar> compute_spectra(const FrameSource& source, int workers,
                                      RunCounters* counters = nullptr);

} // namespace ddm

#endif
