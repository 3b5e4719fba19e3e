// Host-side analysis API (include/ddm/analysis.hpp) as the reference's unit tests pin it
// (`proj/tests/unit/test_analysis.cpp:209-270`): CSV tables, flag names, the diffusion slope.
// The ring average and the fits themselves run on the device and are checked in
// tests/test_analysis_gpu.py / tests/test_analyze_gpu.py.
#include "ddm/analysis.hpp"
#include "ddm/errors.hpp"

#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <string>
#include <vector>

namespace fs = std::filesystem;
using namespace ddm;

static int g_failed = 0;
#define EXPECT(cond)                                                                  \
    do {                                                                              \
        if (!(cond)) {                                                                \
            std::fprintf(stderr, "%s:%d: EXPECT(%s)\n", __FILE__, __LINE__, #cond);   \
            ++g_failed;                                                               \
        }                                                                             \
    } while (0)

static std::vector<std::string> lines_of(const fs::path& p) {
    std::ifstream in(p);
    std::vector<std::string> out;
    for (std::string l; std::getline(in, l);) out.push_back(l);
    return out;
}

int main(int argc, char** argv) {
    const fs::path root = argc > 1 ? fs::path(argv[1]) : fs::temp_directory_path() / "ddm_analysis_api";
    fs::remove_all(root);
    fs::create_directories(root);

    {   // radial.csv: header, one row per (lag, populated bin), full precision
        RadialProfile p;
        p.lags = {0, 1};
        p.bin_count = 4;
        p.counts = {1, 0, 6, 2};
        p.frame_interval = 1.0;
        p.means = {0.0, 0.0, 0.0, 0.0, 0.1, 0.0, 2.5, 1.0 / 3.0};
        write_radial_csv(p, root / "radial.csv");
        const auto l = lines_of(root / "radial.csv");
        EXPECT(l.size() == 1 + 2 * 3);
        if (l.size() == 7) {
            EXPECT(l[0] == "lag,q_bin,mean,count");
            EXPECT(l[1] == "0,0,0,1");
            EXPECT(l[4] == "1,0,0.10000000000000001,1");   // precision(17)
            EXPECT(l[5] == "1,2,2.5,6");
            EXPECT(l[6] == "1,3,0.33333333333333331,2");
        }
    }
    {   // fits.csv: header, one row per fit, flag names
        std::vector<ExponentialFit> fits(2);
        fits[0].q_bin = 3;
        fits[0].amplitude = 2.0;
        fits[0].baseline = 0.5;
        fits[0].tau = 5.0;
        fits[0].residual = 1e-17;
        fits[1].q_bin = 4;
        fits[1].flag = ExponentialFit::Flag::Degenerate;
        fits[1].tau = 1.0;
        write_fits_csv(fits, root / "fits.csv");
        const auto l = lines_of(root / "fits.csv");
        EXPECT(l.size() == 3);
        if (l.size() == 3) {
            EXPECT(l[0] == "q_bin,A,B,tau_seconds,residual,flag");
            EXPECT(l[1] == "3,2,0.5,5,1.0000000000000001e-17,ok");
            EXPECT(l[2] == "4,0,0,1,0,degenerate");
        }
        EXPECT(to_string(ExponentialFit::Flag::Ok) == "ok");
        EXPECT(to_string(ExponentialFit::Flag::Degenerate) == "degenerate");
        EXPECT(to_string(ExponentialFit::Flag::NoConverge) == "no_converge");
    }
    {   // diffusion slope from ideal rates: 1/tau = D q^2, q = 2 pi bin / width (:209-230)
        const double D = 0.7;
        std::vector<ExponentialFit> fits;
        for (int b = 1; b <= 12; ++b) {
            ExponentialFit f;
            f.q_bin = b;
            const double q = 2.0 * std::acos(-1.0) * b / 64.0;
            f.tau = 1.0 / (D * q * q);
            if (b == 4) f.flag = ExponentialFit::Flag::Degenerate;   // excluded
            fits.push_back(f);
        }
        const auto e = estimate_diffusion(fits, 64, 2, 10);
        EXPECT(e.bins_used == 8);
        EXPECT(std::abs(e.coefficient - D) <= D * 1e-12);
        EXPECT(estimate_diffusion(fits, 64, 20, 30).bins_used == 0);
        bool threw = false;
        try {
            estimate_diffusion(fits, 0, 2, 10);
        } catch (const InputError&) {
            threw = true;
        }
        EXPECT(threw);
    }
    fs::remove_all(root);
    std::printf("%s (%d failures)\n", g_failed ? "FAIL" : "OK", g_failed);
    return g_failed ? 1 : 0;
}
