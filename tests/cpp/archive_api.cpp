// C++ API checks of the result / partial archive (include/ddm/archive.hpp) against the
// behaviour the reference's unit tests pin (`proj/tests/unit/test_archive.cpp:56-230`).
// Host-only: built and run by tests/test_cpp_api.py on CPU (no device calls).
#include "ddm/archive.hpp"
#include "ddm/errors.hpp"
#include "ddm/scheduler.hpp"

#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <random>
#include <sstream>
#include <string>

namespace fs = std::filesystem;
using namespace ddm;

static int g_failed = 0;
#define EXPECT(cond)                                                        \
    do {                                                                    \
        if (!(cond)) {                                                      \
            std::fprintf(stderr, "%s:%d: EXPECT(%s)\n", __FILE__, __LINE__, #cond); \
            ++g_failed;                                                     \
        }                                                                   \
    } while (0)

template <class E>
static bool throws_as(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static ResultArchive make_archive(unsigned seed) {
    ResultArchive a;
    a.map.width = 6;
    a.map.height = 4;
    a.map.frame_interval = 0.5;
    a.map.lags = {0, 1, 3};
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 100.0);
    a.map.values.resize(3 * std::size_t(a.map.plane_size()));
    for (double& v : a.map.values) v = u(rng);
    a.frames = 8;
    a.algorithm = "with_ft";
    a.precision = "f64";
    a.workers = 2;
    a.counters.spatial_ffts = 8;
    a.counters.temporal_ffts = 48;
    a.timing.disk = 0.25;
    a.timing.finish(1.0);
    return a;
}

static std::string slurp(const fs::path& p) {
    std::ifstream in(p, std::ios::binary);
    std::ostringstream s;
    s << in.rdbuf();
    return s.str();
}

static PartialResult make_partial(std::int64_t group, std::int64_t b, std::int64_t e,
                                  std::vector<std::int64_t> lags, std::vector<double> values) {
    PartialResult p;
    p.group = group;
    p.wv_begin = b;
    p.wv_end = e;
    p.width = 6;
    p.height = 4;
    p.frames = 8;
    p.frame_interval = 0.5;
    p.lags = std::move(lags);
    p.values = std::move(values);
    return p;
}

int main(int argc, char** argv) {
    const fs::path root = argc > 1 ? fs::path(argv[1]) : fs::temp_directory_path() / "ddm_archive_api";
    fs::remove_all(root);
    fs::create_directories(root);

    {   // results round trip exactly (test_archive.cpp:56-78)
        const auto a = make_archive(3);
        const auto manifest = write_results(a, root / "r1");
        EXPECT(fs::exists(manifest) && fs::exists(root / "r1" / "d_m0.bin") && fs::exists(root / "r1" / "d_m3.bin"));
        const auto b = read_results(root / "r1");
        EXPECT(b.map.width == 6 && b.map.height == 4 && b.map.frame_interval == 0.5);
        EXPECT(b.map.lags == a.map.lags && b.map.values == a.map.values);
        EXPECT(b.frames == 8 && b.algorithm == "with_ft" && b.precision == "f64" && b.workers == 2);
        EXPECT(b.counters.spatial_ffts == 8 && b.counters.temporal_ffts == 48 && !b.q_max.has_value());
    }
    {   // map files byte-stable; manifests equal outside "timing" (:80-102)
        auto a = make_archive(5), b = make_archive(5);
        b.timing = TimingBreakdown{};
        b.timing.disk = 9.0;
        b.timing.finish(40.0);
        write_results(a, root / "s1");
        write_results(b, root / "s2");
        for (const char* f : {"d_m0.bin", "d_m1.bin", "d_m3.bin"})
            EXPECT(slurp(root / "s1" / f) == slurp(root / "s2" / f));
        auto strip = [](std::string j) {   // drop the "timing" object
            const auto i = j.find("\"timing\"");
            if (i == std::string::npos) return j;
            const auto e = j.find('}', i);
            return j.erase(i, e - i + 1);
        };
        const auto ja = slurp(root / "s1" / "index.json"), jb = slurp(root / "s2" / "index.json");
        EXPECT(ja != jb);
        EXPECT(strip(ja) == strip(jb));
    }
    {   // empty lag list rejected (:104-111)
        auto a = make_archive(7);
        a.map.lags.clear();
        a.map.values.clear();
        EXPECT(throws_as<InputError>([&] { write_results(a, root / "e"); }));
    }
    {   // validation rejects poisoned maps, tolerates round-off (:113-129)
        const auto a = make_archive(9);
        a.validate();
        auto bad = a;
        bad.map.values[5] = std::nan("");
        EXPECT(throws_as<InputError>([&] { bad.validate(); }));
        bad = a;
        bad.map.values[5] = -1.0;
        EXPECT(throws_as<InputError>([&] { bad.validate(); }));
        bad = a;
        bad.map.values[5] = -1e-12 * 100.0;
        EXPECT(!throws_as<InputError>([&] { bad.validate(); }));
    }
    {   // garbage manifests: InputError; missing directory: IoError (:131-137)
        fs::create_directories(root / "g");
        std::ofstream(root / "g" / "index.json") << "{not json";
        EXPECT(throws_as<InputError>([&] { read_results(root / "g"); }));
        EXPECT(throws_as<IoError>([&] { read_results(root / "g" / "missing"); }));
    }
    {   // partials round trip exactly (:139-169)
        auto p = make_partial(2, 10, 14, {1, 2}, {1, 2, 3, 4, 5, 6, 7, 8});
        p.q_max = 3.5;
        const auto f = write_partial(p, root / "p1");
        EXPECT(f.filename() == "group2.bin");
        const auto b = read_partial(f);
        EXPECT(b.group == 2 && b.wv_begin == 10 && b.wv_end == 14 && b.width == 6 && b.height == 4);
        EXPECT(b.frames == 8 && b.frame_interval == 0.5 && b.q_max && *b.q_max == 3.5);
        EXPECT(b.lags == p.lags && b.values == p.values);
    }
    {   // inconsistent payload rejected (:171-184)
        const auto p = make_partial(0, 0, 3, {1}, {1.0, 2.0});
        EXPECT(throws_as<InputError>([&] { write_partial(p, root / "p2"); }));
    }
    {   // listing sorts numerically by group (:186-206)
        for (std::int64_t g : {0, 2, 10}) write_partial(make_partial(g, 0, 1, {1}, {1.0}), root / "p3");
        const auto files = list_partials(root / "p3");
        EXPECT(files.size() == 3);
        if (files.size() == 3)
            EXPECT(files[0].filename() == "group0.bin" && files[1].filename() == "group2.bin" &&
                   files[2].filename() == "group10.bin");
    }
    {   // truncated header: InputError; truncated payload: IoError (:208-223, archive.cpp:26-31)
        const auto f = write_partial(make_partial(0, 0, 2, {1}, {1.0, 2.0}), root / "p4");
        const auto full = fs::file_size(f);
        fs::resize_file(f, 10);
        EXPECT(throws_as<InputError>([&] { read_partial(f); }));
        const auto g = write_partial(make_partial(1, 0, 2, {1}, {1.0, 2.0}), root / "p5");
        fs::resize_file(g, full - 4);
        EXPECT(throws_as<IoError>([&] { read_partial(g); }));
    }
    {   // no partials directory: empty listing (:225-230)
        fs::create_directories(root / "p6");
        EXPECT(list_partials(root / "p6").empty());
    }
    {   // merge_partials of the written groups reassembles the map (scheduler.cpp:485-542)
        fs::remove_all(root / "m");
        // 6 x 4 geometry, all 16 wave vectors, two groups of 8, lags {1}
        std::vector<double> v0(8), v1(8);
        for (int i = 0; i < 8; ++i) {
            v0[std::size_t(i)] = i;
            v1[std::size_t(i)] = 8 + i;
        }
        write_partial(make_partial(1, 8, 16, {1}, v1), root / "m");
        write_partial(make_partial(0, 0, 8, {1}, v0), root / "m");
        const auto map = merge_partials(list_partials(root / "m"));
        EXPECT(map.lags == std::vector<std::int64_t>{1});
        bool ok = map.values.size() == 16;
        for (std::size_t i = 0; ok && i < 16; ++i) ok = map.values[i] == double(i);
        EXPECT(ok);
        write_partial(make_partial(2, 4, 8, {1}, {0, 0, 0, 0}), root / "m");   // overlap
        EXPECT(throws_as<InputError>([&] { merge_partials(list_partials(root / "m")); }));
    }
    fs::remove_all(root);
    std::printf("%s (%d failures)\n", g_failed ? "FAIL" : "OK", g_failed);
    return g_failed ? 1 : 0;
}
