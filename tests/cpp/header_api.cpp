// Host-only checks of the reference-named utility headers (tests/test_cpp_api.py, CPU):
// ddm::parallel_blocks partition and error propagation, version constants, and the transform
// objects' argument checks (thrown before any device work).
#include <ddm/errors.hpp>
#include <ddm/fft.hpp>
#include <ddm/parallel.hpp>
#include <ddm/version.hpp>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            return 1;                                              \
        }                                                          \
    } while (0)

int main() {
    CHECK(std::strcmp(ddm::kVersion, "0.1.0") == 0);
    CHECK(ddm::kFormatVersion == 1);

    // 10 items over 4 workers: 3, 3, 2, 2 contiguous
    std::vector<std::pair<long, long>> parts(4, {-1, -1});
    ddm::parallel_blocks(0, 10, 4, [&](int w, std::int64_t b, std::int64_t e) { parts[w] = {long(b), long(e)}; });
    CHECK((parts == std::vector<std::pair<long, long>>{{0, 3}, {3, 6}, {6, 8}, {8, 10}}));
    // more workers than items: one item each, no empty calls
    std::atomic<int> calls{0};
    ddm::parallel_blocks(5, 8, 16, [&](int, std::int64_t b, std::int64_t e) {
        if (e - b == 1) ++calls;
    });
    CHECK(calls == 3);
    // empty range: body never runs
    bool ran = false;
    ddm::parallel_blocks(4, 4, 3, [&](int, std::int64_t, std::int64_t) { ran = true; });
    CHECK(!ran);
    // every element covered once
    std::vector<int> seen(1000, 0);
    ddm::parallel_blocks(0, 1000, 7, [&](int, std::int64_t b, std::int64_t e) {
        for (auto i = b; i < e; ++i) ++seen[i];
    });
    for (int s : seen) CHECK(s == 1);
    // the first failing worker's exception reaches the caller
    bool caught = false;
    try {
        ddm::parallel_blocks(0, 8, 4, [&](int w, std::int64_t, std::int64_t) {
            if (w >= 2) throw std::runtime_error(w == 2 ? "worker 2" : "worker 3");
        });
    } catch (const std::runtime_error& e) {
        caught = std::strcmp(e.what(), "worker 2") == 0;
    }
    CHECK(caught);

    bool bad = false;
    try { ddm::SpatialTransform<float>(0, 4); } catch (const ddm::InputError&) { bad = true; }
    CHECK(bad);
    bad = false;
    try { ddm::SpatialTransform<double>(4, -1); } catch (const ddm::InputError&) { bad = true; }
    CHECK(bad);
    bad = false;
    try { ddm::TemporalTransform<float>(0); } catch (const ddm::InputError&) { bad = true; }
    CHECK(bad);
    std::printf("OK\n");
    return 0;
}
