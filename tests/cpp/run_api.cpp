// A C++ caller of the reference-named API on the device, as INTEGRATION.md §1 describes
// (`ddm::run`, `ddm::analyze`, `ddm::compare` from include/ddm/*.hpp, linked against
// libddm_b200.so): WITH_FT against WITHOUT_FT on a generated stack within the CLI's compare
// tolerances, the counters the reference pins, and the analyze artefacts on disk.
#include "ddm/analysis.hpp"
#include "ddm/archive.hpp"
#include "ddm/errors.hpp"
#include "ddm/frame_source.hpp"
#include "ddm/scheduler.hpp"
#include "ddm/synth.hpp"

#include <cstdio>
#include <filesystem>

namespace fs = std::filesystem;

static int g_failed = 0;
#define EXPECT(cond)                                                                  \
    do {                                                                              \
        if (!(cond)) {                                                                \
            std::fprintf(stderr, "%s:%d: EXPECT(%s)\n", __FILE__, __LINE__, #cond);   \
            ++g_failed;                                                               \
        }                                                                             \
    } while (0)

int main(int argc, char** argv) {
    const fs::path root = argc > 1 ? fs::path(argv[1]) : fs::temp_directory_path() / "ddm_run_api";
    fs::remove_all(root);
    ddm::SynthConfig sc;
    sc.width = sc.height = 48;
    sc.frames = 96;
    sc.particles = 30;
    sc.seed = 7;
    ddm::MemoryFrameSource src(ddm::generate(sc));

    ddm::RunConfig cfg;
    cfg.precision = ddm::Precision::F64;
    cfg.memory_bytes = std::int64_t(1) << 34;
    cfg.workers = 2;
    const ddm::ResultArchive a = ddm::run(src, cfg);
    EXPECT(a.map.lags.size() == 96 && a.map.width == 48 && a.map.height == 48);
    EXPECT(a.counters.spatial_ffts == 96 && a.counters.temporal_ffts == 2ull * 48 * 25);
    EXPECT(a.algorithm == "with_ft" && a.precision == "f64");
    a.validate();

    ddm::RunConfig pw = cfg;
    pw.algorithm = ddm::Algorithm::WithoutFt;
    const ddm::ResultArchive b = ddm::run(src, pw);
    EXPECT(b.counters.pairs == 96ull * 95 / 2);
    EXPECT(ddm::b200::relative_deviation(a.map, b.map) <= 1e-9);

    const ddm::CompareReport r = ddm::compare(src, cfg, ddm::Algorithm::WithFt, ddm::Algorithm::WithoutFt);
    EXPECT(r.pass && r.tolerance == 1e-9 && r.algorithms[0] == "with_ft" && r.algorithms[1] == "without_ft");

    ddm::RunConfig f32 = cfg;
    f32.precision = ddm::Precision::F32;
    const ddm::ResultArchive c = ddm::analyze(src, f32, root / "out");
    EXPECT(ddm::b200::relative_deviation(a.map, c.map) <= 1e-4);
    for (const char* f : {"index.json", "d_m0.bin", "d_m95.bin", "radial.csv", "fits.csv", "partials/group0.bin"})
        EXPECT(fs::exists(root / "out" / f));
    const ddm::ResultArchive back = ddm::read_results(root / "out");
    EXPECT(back.map.values == c.map.values && back.precision == "f32");

    bool threw = false;
    try {
        ddm::RunConfig bad = cfg;
        bad.memory_bytes = 16;
        ddm::run(src, bad);
    } catch (const ddm::PlanError&) {
        threw = true;
    }
    EXPECT(threw);
    fs::remove_all(root);
    std::printf("%s (%d failures)\n", g_failed ? "FAIL" : "OK", g_failed);
    return g_failed ? 1 : 0;
}
