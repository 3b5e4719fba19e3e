// ddm::SpatialTransform / ddm::TemporalTransform (include/ddm/fft.hpp), the reference's
// per-frame and per-sequence transform objects (`fft.hpp:20-70`, `fft.cpp:72-205`) with the
// transforms on the GPU: SpatialTransform::run is the batched spatial engine over one frame
// (Engine::spectra, the path of forward_spectrum), TemporalTransform::forward/backward one
// complex transform of any length (Engine::transform1d, csrc/fft1d.cu). Each instance owns
// its host buffers and device buffers; the engine is shared under its mutex. Same argument
// checks as the reference: InputError for non-positive sizes.
#include "ddm/errors.hpp"
#include "ddm/fft.hpp"
#include "run_internal.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

namespace ddm {

namespace {

struct DeviceBlock {
    void* p = nullptr;
    explicit DeviceBlock(std::size_t bytes) {
        b200::check(cudaMalloc(&p, std::max<std::size_t>(bytes, 16)), "cudaMalloc");
    }
    ~DeviceBlock() { cudaFree(p); }
    DeviceBlock(const DeviceBlock&) = delete;
    DeviceBlock& operator=(const DeviceBlock&) = delete;
};

}  // namespace

template <typename Scalar>
struct SpatialTransform<Scalar>::Impl {
    std::vector<Scalar> in;
    std::vector<std::complex<Scalar>> out;
    DeviceBlock d_in, d_out;
    Impl(std::size_t n_in, std::size_t n_out)
        : in(n_in), out(n_out), d_in(n_in * sizeof(Scalar)), d_out(n_out * sizeof(std::complex<Scalar>)) {}
};

template <typename Scalar>
SpatialTransform<Scalar>::SpatialTransform(int width, int height) : width_(width), height_(height) {
    if (width < 1 || height < 1) throw InputError("fft: frame dimensions must be positive");
    impl_ = detail::guard_device([&] {
        return std::make_unique<Impl>(std::size_t(width) * height, std::size_t(height) * (width / 2 + 1));
    });
}

template <typename Scalar>
SpatialTransform<Scalar>::~SpatialTransform() = default;
template <typename Scalar>
SpatialTransform<Scalar>::SpatialTransform(SpatialTransform&&) noexcept = default;
template <typename Scalar>
SpatialTransform<Scalar>& SpatialTransform<Scalar>::operator=(SpatialTransform&&) noexcept = default;

template <typename Scalar>
std::span<Scalar> SpatialTransform<Scalar>::input() {
    return impl_->in;
}

template <typename Scalar>
std::span<const std::complex<Scalar>> SpatialTransform<Scalar>::output() const {
    return impl_->out;
}

template <typename Scalar>
void SpatialTransform<Scalar>::run() {
    detail::guard_device([&] {
        Impl& m = *impl_;
        b200::Engine& eng = b200::Engine::instance(0);
        std::lock_guard<std::mutex> lock(eng.mutex());
        b200::check(cudaMemcpy(m.d_in.p, m.in.data(), m.in.size() * sizeof(Scalar), cudaMemcpyHostToDevice),
                    "upload");
        eng.spectra(m.d_in.p, int(sizeof(Scalar)), width_, height_, 1, sizeof(Scalar) == 8, m.d_out.p);
        b200::check(cudaMemcpy(m.out.data(), m.d_out.p, m.out.size() * sizeof(std::complex<Scalar>),
                               cudaMemcpyDeviceToHost),
                    "download");
    });
}

template <typename Scalar>
struct TemporalTransform<Scalar>::Impl {
    std::vector<std::complex<Scalar>> buf;
    DeviceBlock d_buf;
    explicit Impl(std::size_t n) : buf(n), d_buf(n * sizeof(std::complex<Scalar>)) {}

    void transform(int sign) {
        detail::guard_device([&] {
            const std::size_t bytes = buf.size() * sizeof(std::complex<Scalar>);
            b200::Engine& eng = b200::Engine::instance(0);
            std::lock_guard<std::mutex> lock(eng.mutex());
            b200::check(cudaMemcpy(d_buf.p, buf.data(), bytes, cudaMemcpyHostToDevice), "upload");
            eng.transform1d(d_buf.p, int(buf.size()), sizeof(Scalar) == 8, sign);
            b200::check(cudaMemcpy(buf.data(), d_buf.p, bytes, cudaMemcpyDeviceToHost), "download");
        });
    }
};

template <typename Scalar>
TemporalTransform<Scalar>::TemporalTransform(std::int64_t length) : length_(length) {
    if (length < 1) throw InputError("fft: transform length must be positive");
    if (length > std::int64_t(1) << 30) throw PlanError("fft: transform length beyond the device plan");
    impl_ = detail::guard_device([&] { return std::make_unique<Impl>(std::size_t(length)); });
}

template <typename Scalar>
TemporalTransform<Scalar>::~TemporalTransform() = default;
template <typename Scalar>
TemporalTransform<Scalar>::TemporalTransform(TemporalTransform&&) noexcept = default;
template <typename Scalar>
TemporalTransform<Scalar>& TemporalTransform<Scalar>::operator=(TemporalTransform&&) noexcept = default;

template <typename Scalar>
std::span<std::complex<Scalar>> TemporalTransform<Scalar>::buffer() {
    return impl_->buf;
}

template <typename Scalar>
void TemporalTransform<Scalar>::forward() {
    impl_->transform(-1);
}

template <typename Scalar>
void TemporalTransform<Scalar>::backward() {
    impl_->transform(+1);
}

template class SpatialTransform<float>;
template class SpatialTransform<double>;
template class TemporalTransform<float>;
template class TemporalTransform<double>;

}  // namespace ddm
