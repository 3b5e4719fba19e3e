// Relaxation fits of the ring-averaged structure function (`analysis.cpp:108-224`) and the
// diffusion estimate (`:242-271`) — the `ddm analyze` artefacts after d(q, m), §8f rank 4.
//
// Model per ring: d(q, t) = A (1 - exp(-t / tau)) + B, t = m * dt for the lags m >= 1 with a
// finite mean. The reference's Levenberg-Marquardt is restated: deterministic start (B = 0,
// A = max, tau at the sample nearest A (1 - 1/e)), normal equations in (A, B, ln tau), damping
// lambda * diag, lambda /3 on success and x5 on failure, stop on relative improvement
// <= 1e-14, 200 iterations, degenerate rings (flat within 1e-12) and the ok / no_converge
// flags. On the device one warp fits one ring: lanes stride over the lags, every sum is a
// fixed-order warp tree, the 3x3 solve runs redundantly in every lane.
#include <cmath>

#include "kernels.cuh"

namespace ddmk {

namespace {

constexpr int kFitIter = 200;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Gaussian elimination with partial pivoting; false when singular (|pivot| < 1e-300)
__device__ bool solve3(double m[3][3], double r[3], double x[3]) {
#pragma unroll
    for (int col = 0; col < 3; ++col) {
        int piv = col;
        for (int row = col + 1; row < 3; ++row)
            if (fabs(m[row][col]) > fabs(m[piv][col])) piv = row;
        if (fabs(m[piv][col]) < 1e-300) return false;
        if (piv != col) {
            for (int k = 0; k < 3; ++k) {
                const double t = m[col][k];
                m[col][k] = m[piv][k];
                m[piv][k] = t;
            }
            const double t = r[col];
            r[col] = r[piv];
            r[piv] = t;
        }
        for (int row = col + 1; row < 3; ++row) {
            const double f = m[row][col] / m[col][col];
            for (int k = col; k < 3; ++k) m[row][k] -= f * m[col][k];
            r[row] -= f * r[col];
        }
    }
    for (int row = 2; row >= 0; --row) {
        double v = r[row];
        for (int k = row + 1; k < 3; ++k) v -= m[row][k] * x[k];
        x[row] = v / m[row][row];
    }
    return true;
}

// flag: 0 ok, 1 degenerate, 2 no_converge, -1 not fitted (empty ring / < 4 usable lags)
__global__ void fit_rings_kernel(const double* __restrict__ means, const int64_t* __restrict__ lags,
                                 int n_lags, const int64_t* __restrict__ counts, int64_t nbins,
                                 double dt, double* __restrict__ amp, double* __restrict__ base,
                                 double* __restrict__ tau_out, double* __restrict__ resid,
                                 int* __restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const int64_t bin = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (bin >= nbins) return;
    auto usable = [&](int li, double& t, double& y) {
        if (li >= n_lags || lags[li] < 1) return false;
        y = means[(int64_t)li * nbins + bin];
        if (!isfinite(y)) return false;
        t = (double)lags[li] * dt;
        return true;
    };
    // usable points, extremes, knee (first index at the minimal distance)
    int count = 0;
    double ymax = -INFINITY, ymin = INFINITY, ysum = 0.0;
    for (int l0 = 0; l0 < n_lags; l0 += 32) {
        double t, y;
        const bool ok = usable(l0 + lane, t, y);
        count += __popc(__ballot_sync(0xffffffffu, ok));
        if (ok) {
            ymax = fmax(ymax, y);
            ymin = fmin(ymin, y);
            ysum += y;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ymax = fmax(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
        ymin = fmin(ymin, __shfl_xor_sync(0xffffffffu, ymin, o));
    }
    ysum = warp_sum(ysum);
    if (counts[bin] < 1 || count < 4) {
        if (lane == 0) flag[bin] = -1;
        return;
    }
    const double scale = fmax(fmax(fabs(ymax), fabs(ymin)), 1e-300);
    if (ymax - ymin <= 1e-12 * scale) {
        if (lane == 0) {
            amp[bin] = 0.0;
            base[bin] = ysum / (double)count;
            tau_out[bin] = dt;
            resid[bin] = 0.0;
            flag[bin] = 1;
        }
        return;
    }
    double a = ymax, b = 0.0;
    const double knee = a * (1.0 - exp(-1.0));
    double best = INFINITY, tau = 0.0;
    int best_i = 1 << 30;
    for (int l0 = 0; l0 < n_lags; l0 += 32) {
        double t, y;
        if (usable(l0 + lane, t, y)) {
            const double e = fabs(y - knee);
            if (e < best) {
                best = e;
                best_i = l0 + lane;
                tau = t;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        const double ot = __shfl_xor_sync(0xffffffffu, tau, o);
        if (ob < best || (ob == best && oi < best_i)) {
            best = ob;
            best_i = oi;
            tau = ot;
        }
    }
    auto cost_of = [&](double aa, double bb, double tt) {
        double s = 0.0;
        for (int l0 = 0; l0 < n_lags; l0 += 32) {
            double t, y;
            if (usable(l0 + lane, t, y)) {
                const double r = aa * (1.0 - exp(-t / tt)) + bb - y;
                s += r * r;
            }
        }
        return warp_sum(s);
    };
    double lambda = 1e-3;
    double cost = cost_of(a, b, tau);
    bool converged = false;
    for (int iter = 0; iter < kFitIter; ++iter) {
        double jj[6] = {0, 0, 0, 0, 0, 0}, jr[3] = {0, 0, 0};
        for (int l0 = 0; l0 < n_lags; l0 += 32) {
            double t, y;
            if (usable(l0 + lane, t, y)) {
                const double e = exp(-t / tau);
                const double r = a * (1.0 - e) + b - y;
                const double j0 = 1.0 - e, j1 = 1.0, j2 = -a * e * t / tau;
                jj[0] += j0 * j0; jj[1] += j0 * j1; jj[2] += j0 * j2;
                jj[3] += j1 * j1; jj[4] += j1 * j2; jj[5] += j2 * j2;
                jr[0] += j0 * r; jr[1] += j1 * r; jr[2] += j2 * r;
            }
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) jj[k] = warp_sum(jj[k]);
#pragma unroll
        for (int k = 0; k < 3; ++k) jr[k] = warp_sum(jr[k]);
        double m[3][3] = {{jj[0], jj[1], jj[2]}, {jj[1], jj[3], jj[4]}, {jj[2], jj[4], jj[5]}};
        const double d0 = m[0][0], d1 = m[1][1], d2 = m[2][2];
        m[0][0] += lambda * fmax(d0, 1e-300);
        m[1][1] += lambda * fmax(d1, 1e-300);
        m[2][2] += lambda * fmax(d2, 1e-300);
        double rhs[3] = {-jr[0], -jr[1], -jr[2]}, step[3] = {0, 0, 0};
        if (!solve3(m, rhs, step)) {
            lambda *= 5.0;
            continue;
        }
        const double a2 = a + step[0], b2 = b + step[1];
        const double tau2 = tau * exp(fmin(fmax(step[2], -5.0), 5.0));
        const double cost2 = cost_of(a2, b2, tau2);
        if (cost2 <= cost) {
            const double gain = cost - cost2;
            a = a2;
            b = b2;
            tau = tau2;
            cost = cost2;
            lambda = fmax(lambda / 3.0, 1e-12);
            if (gain <= 1e-14 * (cost + 1e-300)) {
                converged = true;
                break;
            }
        } else {
            lambda *= 5.0;
            if (lambda > 1e12) {
                converged = true;   // flat basin: accept (as the reference)
                break;
            }
        }
    }
    if (lane == 0) {
        amp[bin] = a;
        base[bin] = b;
        tau_out[bin] = tau;
        resid[bin] = sqrt(cost / (double)count);
        flag[bin] = converged ? 0 : 2;
    }
}

}  // namespace

cudaError_t launch_fit_rings(const double* means, const int64_t* lags, int n_lags,
                             const int64_t* counts, int64_t nbins, double dt, double* amp,
                             double* base, double* tau, double* resid, int* flag,
                             cudaStream_t stream) {
    if (nbins < 1) return cudaSuccess;
    const int threads = 128;
    const int64_t blocks = (nbins * 32 + threads - 1) / threads;
    fit_rings_kernel<<<(unsigned)blocks, threads, 0, stream>>>(means, lags, n_lags, counts, nbins, dt,
                                                               amp, base, tau, resid, flag);
    return cudaGetLastError();
}

}  // namespace ddmk
