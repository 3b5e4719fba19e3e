// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// Implements the FFTW3 entry points declared in fftw3.h so that the unmodified reference
// core (`/root/reference/proj/core/src/fft.cpp:23-63`) can be compiled here, where no
// libfftw3 exists.  FFTW itself (unpinned; the paper used 3.3.3,
// `PAPER.md:60`) is a third-party dependency absent from /root/reference; what it
// computes is the textbook unnormalised DFT, restated here as:
//   * complex length-n transforms: recursive mixed-radix decimation in time (radix 4, 2,
//     and generic small odd primes), Bluestein's chirp-z for lengths with a prime factor
//     above 13;
//   * r2c 2D (rows x cols): each real row through a half-length complex FFT plus the
//     standard even/odd split, then complex column transforms of the kept half plane.
// Twiddles are generated in double and rounded once to the working precision, as FFTW
// does. Plans own their scratch, so distinct plans may execute concurrently (the
// reference runs one plan per worker thread, `fft.cpp:13-18`).

#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <vector>

namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;

template <class T>
using cx = std::complex<T>;

template <class T>
class Dft {
public:
    Dft(int n, int sign) : n_(n), sign_(sign) {
        if (n < 1)
            throw std::bad_alloc();
        int rest = n;
        while (rest % 4 == 0) { radix_.push_back(4); rest /= 4; }
        while (rest % 2 == 0) { radix_.push_back(2); rest /= 2; }
        for (int p = 3; p <= 13 && rest > 1; p += 2)
            while (rest % p == 0) { radix_.push_back(p); rest /= p; }
        if (rest > 1) {
            init_bluestein();
            return;
        }
        tw_.resize(static_cast<std::size_t>(n));
        for (int k = 0; k < n; ++k) {
            const double a = sign * 2.0 * kPi * static_cast<double>(k) / n;
            tw_[static_cast<std::size_t>(k)] = cx<T>(static_cast<T>(std::cos(a)),
                                                     static_cast<T>(std::sin(a)));
        }
        scratch_.resize(16);
    }

    int size() const { return n_; }

    // out-of-place; in and out must not alias
    void run(const cx<T>* in, cx<T>* out) const {
        if (blue_) {
            run_bluestein(in, out);
            return;
        }
        if (n_ == 1) {
            out[0] = in[0];
            return;
        }
        rec(out, in, 1, 0, n_);
    }

private:
    int n_;
    int sign_;
    std::vector<int> radix_;
    std::vector<cx<T>> tw_;
    mutable std::vector<cx<T>> scratch_;

    bool blue_ = false;
    int m_ = 0;
    std::unique_ptr<Dft<T>> conv_fwd_, conv_bwd_;
    std::vector<cx<T>> chirp_;
    std::vector<cx<T>> kernel_hat_;
    mutable std::vector<cx<T>> a_, ahat_;

    void rec(cx<T>* out, const cx<T>* in, std::size_t fstride, std::size_t level,
             int len) const {
        const int p = radix_[level];
        const int m = len / p;
        if (m == 1) {
            for (int k = 0; k < p; ++k)
                out[k] = in[static_cast<std::size_t>(k) * fstride];
        } else {
            for (int q = 0; q < p; ++q)
                rec(out + static_cast<std::size_t>(q) * m, in + q * fstride, fstride * p,
                    level + 1, m);
        }
        switch (p) {
        case 2: bfly2(out, fstride, m); break;
        case 4: bfly4(out, fstride, m); break;
        default: bfly_generic(out, fstride, m, p); break;
        }
    }

    void bfly2(cx<T>* out, std::size_t fstride, int m) const {
        for (int u = 0; u < m; ++u) {
            const cx<T> t = out[u + m] * tw_[static_cast<std::size_t>(u) * fstride];
            out[u + m] = out[u] - t;
            out[u] += t;
        }
    }

    void bfly4(cx<T>* out, std::size_t fstride, int m) const {
        const T s = static_cast<T>(sign_);
        for (int u = 0; u < m; ++u) {
            const std::size_t j = static_cast<std::size_t>(u) * fstride;
            const cx<T> a0 = out[u];
            const cx<T> a1 = out[u + m] * tw_[j];
            const cx<T> a2 = out[u + 2 * m] * tw_[2 * j];
            const cx<T> a3 = out[u + 3 * m] * tw_[3 * j];
            const cx<T> b0 = a0 + a2;
            const cx<T> b1 = a0 - a2;
            const cx<T> b2 = a1 + a3;
            const cx<T> d = a1 - a3;
            const cx<T> rot(-s * d.imag(), s * d.real()); // (sign * i) * d
            out[u] = b0 + b2;
            out[u + 2 * m] = b0 - b2;
            out[u + m] = b1 + rot;
            out[u + 3 * m] = b1 - rot;
        }
    }

    void bfly_generic(cx<T>* out, std::size_t fstride, int m, int p) const {
        if (scratch_.size() < static_cast<std::size_t>(p))
            scratch_.resize(static_cast<std::size_t>(p));
        const std::size_t step = static_cast<std::size_t>(n_ / p); // W_p = tw[step]
        for (int u = 0; u < m; ++u) {
            for (int q = 0; q < p; ++q)
                scratch_[static_cast<std::size_t>(q)] =
                    out[u + q * m] * tw_[static_cast<std::size_t>(q) * u * fstride];
            for (int k = 0; k < p; ++k) {
                cx<T> acc = scratch_[0];
                for (int q = 1; q < p; ++q)
                    acc += scratch_[static_cast<std::size_t>(q)] *
                           tw_[static_cast<std::size_t>((k * q) % p) * step];
                out[u + k * m] = acc;
            }
        }
    }

    void init_bluestein() {
        blue_ = true;
        m_ = 1;
        while (m_ < 2 * n_ - 1)
            m_ <<= 1;
        conv_fwd_ = std::make_unique<Dft<T>>(m_, -1);
        conv_bwd_ = std::make_unique<Dft<T>>(m_, +1);
        chirp_.resize(static_cast<std::size_t>(n_));
        const long long two_n = 2LL * n_;
        for (int j = 0; j < n_; ++j) {
            const long long jj = (static_cast<long long>(j) * j) % two_n;
            const double a = sign_ * kPi * static_cast<double>(jj) / n_;
            chirp_[static_cast<std::size_t>(j)] =
                cx<T>(static_cast<T>(std::cos(a)), static_cast<T>(std::sin(a)));
        }
        std::vector<cx<T>> b(static_cast<std::size_t>(m_), cx<T>(0, 0));
        for (int j = 0; j < n_; ++j) {
            b[static_cast<std::size_t>(j)] = std::conj(chirp_[static_cast<std::size_t>(j)]);
            if (j > 0)
                b[static_cast<std::size_t>(m_ - j)] = b[static_cast<std::size_t>(j)];
        }
        kernel_hat_.resize(static_cast<std::size_t>(m_));
        conv_fwd_->run(b.data(), kernel_hat_.data());
        a_.resize(static_cast<std::size_t>(m_));
        ahat_.resize(static_cast<std::size_t>(m_));
    }

    void run_bluestein(const cx<T>* in, cx<T>* out) const {
        std::fill(a_.begin(), a_.end(), cx<T>(0, 0));
        for (int j = 0; j < n_; ++j)
            a_[static_cast<std::size_t>(j)] = in[j] * chirp_[static_cast<std::size_t>(j)];
        conv_fwd_->run(a_.data(), ahat_.data());
        for (int j = 0; j < m_; ++j)
            ahat_[static_cast<std::size_t>(j)] *= kernel_hat_[static_cast<std::size_t>(j)];
        conv_bwd_->run(ahat_.data(), a_.data());
        const T inv = static_cast<T>(1.0 / m_);
        for (int k = 0; k < n_; ++k)
            out[k] = a_[static_cast<std::size_t>(k)] * chirp_[static_cast<std::size_t>(k)] * inv;
    }
};

template <class T>
struct Plan1D {
    Dft<T> dft;
    cx<T>* in;
    cx<T>* out;
    mutable std::vector<cx<T>> tmp;
    Plan1D(int n, cx<T>* i, cx<T>* o, int sign)
        : dft(n, sign), in(i), out(o), tmp(static_cast<std::size_t>(n)) {}
    void execute() const {
        std::memcpy(static_cast<void*>(tmp.data()), in, tmp.size() * sizeof(cx<T>));
        dft.run(tmp.data(), out);
    }
};

template <class T>
struct PlanR2C2D {
    int rows, cols, half;
    T* in;
    cx<T>* out;
    bool packed;                      // even cols: half-length complex row transform
    std::unique_ptr<Dft<T>> row_dft;  // cols/2 (packed) or cols
    Dft<T> col_dft;
    std::vector<cx<T>> post;          // exp(-2 pi i k / cols), k <= cols/2
    static constexpr int kColBlock = 8;
    mutable std::vector<cx<T>> row_in, row_out, col_in, col_out;

    PlanR2C2D(int r, int c, T* i, cx<T>* o)
        : rows(r), cols(c), half(c / 2 + 1), in(i), out(o), packed(c % 2 == 0),
          col_dft(r, -1) {
        row_dft = std::make_unique<Dft<T>>(packed ? c / 2 : c, -1);
        post.resize(static_cast<std::size_t>(half));
        for (int k = 0; k < half; ++k) {
            const double a = -2.0 * kPi * static_cast<double>(k) / c;
            post[static_cast<std::size_t>(k)] =
                cx<T>(static_cast<T>(std::cos(a)), static_cast<T>(std::sin(a)));
        }
        row_in.resize(static_cast<std::size_t>(c));
        row_out.resize(static_cast<std::size_t>(c));
        col_in.resize(static_cast<std::size_t>(r) * kColBlock);
        col_out.resize(static_cast<std::size_t>(r));
    }

    void execute() const {
        const T half_t = static_cast<T>(0.5);
        for (int r = 0; r < rows; ++r) {
            const T* x = in + static_cast<std::size_t>(r) * cols;
            cx<T>* dst = out + static_cast<std::size_t>(r) * half;
            if (packed) {
                const int m = cols / 2;
                for (int k = 0; k < m; ++k)
                    row_in[static_cast<std::size_t>(k)] = cx<T>(x[2 * k], x[2 * k + 1]);
                row_dft->run(row_in.data(), row_out.data());
                for (int k = 0; k <= m; ++k) {
                    const cx<T> zk = row_out[static_cast<std::size_t>(k % m)];
                    const cx<T> zc = std::conj(row_out[static_cast<std::size_t>((m - k) % m)]);
                    const cx<T> e = (zk + zc) * half_t;
                    const cx<T> diff = zk - zc; // odd = diff / (2i)
                    const cx<T> o(diff.imag() * half_t, -diff.real() * half_t);
                    dst[k] = e + post[static_cast<std::size_t>(k)] * o;
                }
            } else {
                for (int k = 0; k < cols; ++k)
                    row_in[static_cast<std::size_t>(k)] = cx<T>(x[k], T(0));
                row_dft->run(row_in.data(), row_out.data());
                for (int k = 0; k < half; ++k)
                    dst[k] = row_out[static_cast<std::size_t>(k)];
            }
        }
        if (rows == 1)
            return;
        for (int c0 = 0; c0 < half; c0 += kColBlock) {
            const int nb = std::min(kColBlock, half - c0);
            for (int r = 0; r < rows; ++r) {
                const cx<T>* src = out + static_cast<std::size_t>(r) * half + c0;
                for (int b = 0; b < nb; ++b)
                    col_in[static_cast<std::size_t>(b) * rows + r] = src[b];
            }
            for (int b = 0; b < nb; ++b) {
                col_dft.run(col_in.data() + static_cast<std::size_t>(b) * rows, col_out.data());
                for (int r = 0; r < rows; ++r)
                    out[static_cast<std::size_t>(r) * half + c0 + b] =
                        col_out[static_cast<std::size_t>(r)];
            }
        }
    }
};

template <class T>
struct AnyPlan {
    virtual ~AnyPlan() = default;
    std::unique_ptr<Plan1D<T>> p1;
    std::unique_ptr<PlanR2C2D<T>> p2;
    void execute() const {
        if (p1)
            p1->execute();
        else
            p2->execute();
    }
};

} // namespace

struct ddm_shim_plan_d : AnyPlan<double> {};
struct ddm_shim_plan_f : AnyPlan<float> {};

namespace {

void* aligned(std::size_t n) {
    void* p = nullptr;
    if (posix_memalign(&p, 64, n ? n : 64) != 0)
        return nullptr;
    return p;
}

template <class P, class T>
P* make_1d(int n, T (*in)[2], T (*out)[2], int sign) {
    try {
        auto* plan = new P();
        plan->p1 = std::make_unique<Plan1D<T>>(n, reinterpret_cast<cx<T>*>(in),
                                               reinterpret_cast<cx<T>*>(out), sign);
        return plan;
    } catch (...) {
        return nullptr;
    }
}

template <class P, class T>
P* make_r2c(int n0, int n1, T* in, T (*out)[2]) {
    try {
        auto* plan = new P();
        plan->p2 = std::make_unique<PlanR2C2D<T>>(n0, n1, in, reinterpret_cast<cx<T>*>(out));
        return plan;
    } catch (...) {
        return nullptr;
    }
}

} // namespace

extern "C" {

void* fftw_malloc(size_t n) { return aligned(n); }
void fftw_free(void* p) { std::free(p); }
void* fftwf_malloc(size_t n) { return aligned(n); }
void fftwf_free(void* p) { std::free(p); }

fftw_plan fftw_plan_dft_r2c_2d(int n0, int n1, double* in, fftw_complex* out, unsigned) {
    return make_r2c<ddm_shim_plan_d>(n0, n1, in, out);
}
fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned) {
    return make_1d<ddm_shim_plan_d>(n, in, out, sign);
}
void fftw_execute(const fftw_plan p) { p->execute(); }
void fftw_destroy_plan(fftw_plan p) { delete p; }

fftwf_plan fftwf_plan_dft_r2c_2d(int n0, int n1, float* in, fftwf_complex* out, unsigned) {
    return make_r2c<ddm_shim_plan_f>(n0, n1, in, out);
}
fftwf_plan fftwf_plan_dft_1d(int n, fftwf_complex* in, fftwf_complex* out, int sign, unsigned) {
    return make_1d<ddm_shim_plan_f>(n, in, out, sign);
}
void fftwf_execute(const fftwf_plan p) { p->execute(); }
void fftwf_destroy_plan(fftwf_plan p) { delete p; }

} // extern "C"
