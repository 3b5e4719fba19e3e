// ddm::SpatialTransform / ddm::TemporalTransform on the device against a direct DFT in long
// double (tests/test_cpp_api.py, GPU). Prints "OK" or the first failure.
#include <ddm/errors.hpp>
#include <ddm/fft.hpp>

#include <cmath>
#include <complex>
#include <cstdio>
#include <random>
#include <vector>

using cld = std::complex<long double>;

static int failures = 0;

static void expect(bool ok, const char* what, double err) {
    if (!ok) {
        std::printf("FAIL %s err=%.3g\n", what, err);
        ++failures;
    }
}

template <typename S>
static void spatial_case(int W, int H, double tol, std::mt19937_64& rng) {
    ddm::SpatialTransform<S> fft(W, H);
    std::uniform_real_distribution<double> u(0.0, 4096.0);
    auto in = fft.input();
    for (auto& v : in) v = S(u(rng));
    fft.run();
    const auto out = fft.output();
    const int Wh = W / 2 + 1;
    if (out.size() != std::size_t(H) * Wh) return expect(false, "spatial size", 0);
    const long double two_pi = 2.0L * 3.14159265358979323846264338327950288L;
    double err = 0, scale = 0;
    for (int ky = 0; ky < H; ++ky)
        for (int kx = 0; kx < Wh; ++kx) {
            cld acc = 0;
            for (int y = 0; y < H; ++y)
                for (int x = 0; x < W; ++x) {
                    const long double ph = -two_pi * ((long double)(ky * y % H) / H + (long double)(kx * x % W) / W);
                    acc += (long double)in[std::size_t(y) * W + x] * cld(std::cos(ph), std::sin(ph));
                }
            const auto got = out[std::size_t(ky) * Wh + kx];
            err = std::max(err, (double)std::abs(cld(got.real(), got.imag()) - acc));
            scale = std::max(scale, (double)std::abs(acc));
        }
    char name[64];
    std::snprintf(name, sizeof name, "spatial<%zu> %dx%d", sizeof(S), W, H);
    expect(err <= tol * scale, name, err / scale);
}

template <typename S>
static void temporal_case(long L, double tol, std::mt19937_64& rng) {
    ddm::TemporalTransform<S> fft(L);
    std::normal_distribution<double> g;
    auto buf = fft.buffer();
    std::vector<std::complex<S>> x(buf.size());
    for (auto& v : x) v = {S(g(rng)), S(g(rng))};
    std::copy(x.begin(), x.end(), buf.begin());
    fft.forward();
    const long double two_pi = 2.0L * 3.14159265358979323846264338327950288L;
    double err = 0, scale = 0;
    for (long k = 0; k < L; ++k) {
        cld acc = 0;
        for (long n = 0; n < L; ++n) {
            const long double ph = -two_pi * (long double)(k * n % L) / L;
            acc += cld(x[n].real(), x[n].imag()) * cld(std::cos(ph), std::sin(ph));
        }
        err = std::max(err, (double)std::abs(cld(buf[k].real(), buf[k].imag()) - acc));
        scale = std::max(scale, (double)std::abs(acc));
    }
    char name[64];
    std::snprintf(name, sizeof name, "temporal<%zu> forward L=%ld", sizeof(S), L);
    expect(err <= tol * scale, name, err / scale);
    // backward(forward(x)) = L x (unnormalised, like the reference's FFTW plans)
    fft.backward();
    double rerr = 0, rscale = 0;
    for (long n = 0; n < L; ++n) {
        rerr = std::max(rerr, (double)std::abs(std::complex<double>(buf[n]) - (double)L * std::complex<double>(x[n])));
        rscale = std::max(rscale, (double)L * std::abs(std::complex<double>(x[n])));
    }
    std::snprintf(name, sizeof name, "temporal<%zu> round trip L=%ld", sizeof(S), L);
    expect(rerr <= tol * rscale, name, rerr / rscale);
}

// Long transforms: a direct sum for 16 spot bins, Parseval, and the round trip
template <typename S>
static void temporal_long_case(long L, double tol, std::mt19937_64& rng) {
    ddm::TemporalTransform<S> fft(L);
    std::normal_distribution<double> g;
    auto buf = fft.buffer();
    std::vector<std::complex<S>> x(buf.size());
    for (auto& v : x) v = {S(g(rng)), S(g(rng))};
    std::copy(x.begin(), x.end(), buf.begin());
    fft.forward();
    const long double two_pi = 2.0L * 3.14159265358979323846264338327950288L;
    double err = 0, scale = 0;
    for (int s = 0; s < 16; ++s) {
        const long k = (long)((unsigned long)rng() % (unsigned long)L);
        cld acc = 0;
        for (long n = 0; n < L; ++n) {
            const long double ph = -two_pi * (long double)((long long)k * n % L) / L;
            acc += cld(x[n].real(), x[n].imag()) * cld(std::cos(ph), std::sin(ph));
        }
        err = std::max(err, (double)std::abs(cld(buf[k].real(), buf[k].imag()) - acc));
        scale = std::max(scale, (double)std::sqrt((long double)L));
    }
    char name[80];
    std::snprintf(name, sizeof name, "temporal<%zu> spot bins L=%ld", sizeof(S), L);
    expect(err <= 8 * tol * scale, name, err / scale);
    long double ex = 0, eX = 0;
    for (long n = 0; n < L; ++n) {
        ex += std::norm(std::complex<long double>(x[n].real(), x[n].imag()));
        eX += std::norm(std::complex<long double>(buf[n].real(), buf[n].imag()));
    }
    std::snprintf(name, sizeof name, "temporal<%zu> Parseval L=%ld", sizeof(S), L);
    expect(std::fabs((double)(eX / (L * ex)) - 1.0) <= 8 * tol, name, (double)(eX / (L * ex)) - 1.0);
    fft.backward();
    double rerr = 0;
    for (long n = 0; n < L; ++n)
        rerr = std::max(rerr, std::abs(std::complex<double>(buf[n]) / (double)L - std::complex<double>(x[n])));
    std::snprintf(name, sizeof name, "temporal<%zu> round trip L=%ld", sizeof(S), L);
    expect(rerr <= 8 * tol * 6.0, name, rerr);
}

int main() {
    std::mt19937_64 rng(2012'05695);
    for (auto [W, H] : {std::pair{64, 64}, {1, 1}, {5, 8}, {37, 20}, {32, 48}, {128, 16}}) {
        spatial_case<float>(W, H, 2e-6, rng);
        spatial_case<double>(W, H, 1e-13, rng);
    }
    for (long L : {1L, 2L, 3L, 8L, 12L, 60L, 7L, 11L, 77L, 1000L, 1024L, 2048L, 3000L, 4096L}) {
        temporal_case<float>(L, 3e-6, rng);
        temporal_case<double>(L, 1e-13, rng);
    }
    for (long L : {12288L, 65536L, 100000L, 10007L}) {
        temporal_long_case<float>(L, 3e-6, rng);
        temporal_long_case<double>(L, 1e-13, rng);
    }
    if (failures == 0) std::printf("OK\n");
    return failures == 0 ? 0 : 1;
}
