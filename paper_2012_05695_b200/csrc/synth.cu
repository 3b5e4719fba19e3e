// Synthetic Brownian-colloid frames rendered on the device (the generator staging u16 frames
// to HBM, BASELINE north_star; reference `synth.cpp:42-79` `render_frame`).
//
// The particle trajectories come from the host (mt19937_64 + Box-Muller, `synth.cpp:98-132`,
// O(particles x frames), cheap); each frame is rendered here with the reference's per-pixel
// arithmetic and addition order:
//     canvas = background; for p in order, for (iy, ix) of p's 4-sigma window in row-major
//     order with r2 <= reach^2: canvas[wrap(iy), wrap(ix)] += amplitude * exp(-r2 k)
//     pixel = clamp(llround(canvas), 0, 65535)
// Pixels no window touches are llround(background). A touched pixel is rendered once, by the
// thread that meets it in the window of its lowest-index particle; that thread replays every
// particle's contributions to the pixel in the reference's order (so the double sum is the
// same sequence of additions).
#include <cstdint>

#include "kernels.cuh"

namespace ddmk {

namespace {

struct Win {
    int y0, y1, x0, x1;
};

__device__ __forceinline__ Win window(double cx, double cy, double reach) {
    return {(int)floor(cy - reach), (int)ceil(cy + reach), (int)floor(cx - reach), (int)ceil(cx + reach)};
}

// the host's arithmetic without contraction (x86-64 baseline has no FMA)
__device__ __forceinline__ double r2_of(double dx, double dy) {
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

__device__ __forceinline__ int floordiv(int a, int b) {
    const int q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// contributions of particle (cx, cy) to pixel (row, col), in the reference's (iy, ix) order;
// returns whether any (iy, ix) of the window hits the pixel within reach
__device__ __forceinline__ bool add_particle(double cx, double cy, int row, int col, int W, int H,
                                             double reach, double k, double amp, double& sum) {
    const Win w = window(cx, cy, reach);
    bool hit = false;
    // iy = row + a H in [y0, y1], ix = col + b W in [x0, x1]
    for (int a = floordiv(w.y0 - row + H - 1, H); row + a * H <= w.y1; ++a) {
        const int iy = row + a * H;
        const double dy = (double)iy - cy;
        for (int b = floordiv(w.x0 - col + W - 1, W); col + b * W <= w.x1; ++b) {
            const int ix = col + b * W;
            const double dx = (double)ix - cx;
            const double r2 = r2_of(dx, dy);
            if (r2 > reach * reach) continue;
            hit = true;
            sum = __dadd_rn(sum, __dmul_rn(amp, exp(__dmul_rn(-r2, k))));
        }
    }
    return hit;
}

__global__ void fill_kernel(uint16_t* __restrict__ out, int64_t n, uint16_t v) {
    const uint32_t v2 = (uint32_t)v | ((uint32_t)v << 16);
    uint32_t* o = reinterpret_cast<uint32_t*>(out);
    const int64_t n2 = n / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = v2;
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) out[n - 1] = v;
}

// one CTA per frame; pos: [frames][particles][2] (x, y)
__global__ void splat_kernel(const double* __restrict__ pos, int particles, int W, int H,
                             double reach, double k, double amp, double background,
                             uint16_t* __restrict__ out) {
    const int n = blockIdx.x;
    const double* fp = pos + (int64_t)n * particles * 2;
    uint16_t* frame = out + (int64_t)n * W * H;
    for (int p = 0; p < particles; ++p) {
        const double cx = fp[2 * p], cy = fp[2 * p + 1];
        const Win w = window(cx, cy, reach);
        const int ww = w.x1 - w.x0 + 1;
        const int cells = ww * (w.y1 - w.y0 + 1);
        for (int i = threadIdx.x; i < cells; i += blockDim.x) {
            const int iy = w.y0 + i / ww, ix = w.x0 + i % ww;
            const double dx = (double)ix - cx, dy = (double)iy - cy;
            if (r2_of(dx, dy) > reach * reach) continue;
            const int row = ((iy % H) + H) % H, col = ((ix % W) + W) % W;
            // rendered by the lowest-index particle touching it, and only once within that
            // particle's window (the first (iy, ix) that maps to it)
            bool owned = true;
            double scratch = 0.0;
            for (int q = 0; q < p && owned; ++q)
                if (add_particle(fp[2 * q], fp[2 * q + 1], row, col, W, H, reach, k, amp, scratch)) owned = false;
            if (!owned) continue;
            {
                // the first (yy, xx) of p's window (row-major) within reach that maps here
                bool first = false, found = false;
                for (int yy = row + floordiv(w.y0 - row + H - 1, H) * H; yy <= w.y1 && !found; yy += H) {
                    const double ddy = (double)yy - cy;
                    for (int xx = col + floordiv(w.x0 - col + W - 1, W) * W; xx <= w.x1; xx += W) {
                        const double ddx = (double)xx - cx;
                        if (r2_of(ddx, ddy) > reach * reach) continue;
                        found = true;
                        first = (yy == iy && xx == ix);
                        break;
                    }
                }
                if (!first) continue;
            }
            double sum = background;
            for (int q = p; q < particles; ++q)
                add_particle(fp[2 * q], fp[2 * q + 1], row, col, W, H, reach, k, amp, sum);
            const double v = (double)llround(sum);
            frame[(int64_t)row * W + col] = (uint16_t)fmin(fmax(v, 0.0), 65535.0);
        }
    }
}

}  // namespace

cudaError_t launch_render_frames(const double* d_pos, int particles, int W, int H, int frames,
                                 double psf_sigma, double amplitude, double background,
                                 uint16_t* d_out, cudaStream_t stream) {
    const int64_t n = (int64_t)W * H * frames;
    const double bg = (double)llround(background);
    const uint16_t fill = (uint16_t)(bg < 0.0 ? 0.0 : bg > 65535.0 ? 65535.0 : bg);
    fill_kernel<<<148 * 8, 256, 0, stream>>>(d_out, n, fill);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || particles == 0) return e;
    const double reach = 4.0 * psf_sigma;
    const double k = 1.0 / (2.0 * psf_sigma * psf_sigma);
    splat_kernel<<<frames, 128, 0, stream>>>(d_pos, particles, W, H, reach, k, amplitude, background, d_out);
    return cudaGetLastError();
}

}  // namespace ddmk
