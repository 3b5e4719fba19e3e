// ddm-b200: Brownian-colloid stack generator, bit-identical to the reference
// (`proj/core/src/synth.cpp:98-132`: mt19937_64, explicit Box-Muller, periodic wrap,
// Gaussian blobs truncated at 4 sigma, llround + clamp to u16).
#ifndef DDM_B200_SYNTH_HPP
#define DDM_B200_SYNTH_HPP

#include "ddm/image_stack.hpp"

#include <cstdint>
#include <filesystem>

namespace ddm {

struct SynthConfig {
    std::int64_t particles = 100;
    double diffusion = 0.5;
    double psf_sigma = 1.0;
    double amplitude = 1000.0;
    double background = 100.0;
    int width = 64;
    int height = 64;
    int frames = 256;
    double frame_interval = 1.0;
    std::uint64_t seed = 0;
    void validate() const;
};

ImageStack generate(const SynthConfig& config);

/// The same stack rendered on the device into d_out ([frames][height][width] u16 in HBM,
/// b200 extension): trajectories from the reference's draw sequence on the host, frames by
/// the render kernel (csrc/synth.cu) with the reference's per-pixel addition order. Ordered
/// after `stream` (cudaStream_t, may be null); returns when the frames are written.
void generate_device(const SynthConfig& config, std::uint16_t* d_out, int device = 0,
                     void* stream = nullptr);

/// synth.json beside a generated stack (`synth.cpp:134-155`): tool version, generator name and
/// every SynthConfig field.
void write_synth_manifest(const SynthConfig& config, const std::filesystem::path& path);

} // namespace ddm

#endif
