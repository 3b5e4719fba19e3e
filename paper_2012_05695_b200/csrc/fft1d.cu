// Single complex 1D transforms for the per-sequence seam `ddm::TemporalTransform`
// (include/ddm/fft.hpp; the reference's `fft.hpp:48-70` / `fft.cpp:142-205`). Not on the hot
// path (the batched engines fuse their transforms); any length: out-of-place Stockham passes
// of radix 4/2/5/3 through global memory (ping-pong between the data and a scratch buffer),
// or a direct f64-accumulated DFT for lengths with other prime factors. Unnormalised,
// SIGN = -1 forward, +1 backward, twiddles exp(-2 pi i j / L) from the engine's table.
#include "fft_core.cuh"
#include "kernels.cuh"

namespace ddmk {

namespace {

template <int R, int SIGN, typename S>
__global__ void stockham_pass_kernel(const cpx<S>* __restrict__ in, cpx<S>* __restrict__ out, int L,
                                     int p, const cpx<S>* __restrict__ tw) {
    const int nb = L / R;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb) return;
    const int k = i % p, twstep = L / (p * R);
    cpx<S> v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        cpx<S> x = in[i + r * nb];
        if (r > 0 && k > 0) x = cmul(x, twiddle<SIGN>(tw, r * k * twstep));
        v[r] = x;
    }
    Dft<R, SIGN, S>::run(v);
    const int base = (i - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) out[base + r * p] = v[r];
}

template <int SIGN, typename S>
__global__ void direct_dft_kernel(const cpx<S>* __restrict__ in, cpx<S>* __restrict__ out, int L,
                                  const cpx<S>* __restrict__ tw) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= L) return;
    double ax = 0.0, ay = 0.0;
    int j = 0;
    for (int n = 0; n < L; ++n) {
        const cpx<S> w = twiddle<SIGN>(tw, j);
        const cpx<S> x = in[n];
        ax += (double)x.x * (double)w.x - (double)x.y * (double)w.y;
        ay += (double)x.x * (double)w.y + (double)x.y * (double)w.x;
        j += k;
        if (j >= L) j -= L;
    }
    out[k] = {(S)ax, (S)ay};
}

template <int SIGN, typename S>
cudaError_t run_fft1d(cpx<S>* data, cpx<S>* scratch, int L, const cpx<S>* tw, cudaStream_t st) {
    const FftPlan plan = make_rt_plan(L);
    const int threads = 256;
    if (plan.naive) {
        direct_dft_kernel<SIGN, S><<<(L + threads - 1) / threads, threads, 0, st>>>(data, scratch, L, tw);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        return cudaMemcpyAsync(data, scratch, sizeof(cpx<S>) * L, cudaMemcpyDeviceToDevice, st);
    }
    cpx<S>* src = data;
    cpx<S>* dst = scratch;
    int p = 1;
    for (int s = 0; s < plan.npass; ++s) {
        const int R = plan.radix(s);
        const int blocks = (L / R + threads - 1) / threads;
        if (R == 2) stockham_pass_kernel<2, SIGN, S><<<blocks, threads, 0, st>>>(src, dst, L, p, tw);
        else if (R == 3) stockham_pass_kernel<3, SIGN, S><<<blocks, threads, 0, st>>>(src, dst, L, p, tw);
        else if (R == 5) stockham_pass_kernel<5, SIGN, S><<<blocks, threads, 0, st>>>(src, dst, L, p, tw);
        else stockham_pass_kernel<4, SIGN, S><<<blocks, threads, 0, st>>>(src, dst, L, p, tw);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        p *= R;
        std::swap(src, dst);
    }
    if (src != data) return cudaMemcpyAsync(data, src, sizeof(cpx<S>) * L, cudaMemcpyDeviceToDevice, st);
    return cudaSuccess;
}

}  // namespace

cudaError_t launch_fft1d(void* data, void* scratch, int len, bool f64, int sign, const void* tw,
                         cudaStream_t stream) {
    if (len < 1) return cudaErrorInvalidValue;
    if (len == 1) return cudaSuccess;
    if (f64) {
        auto* d = static_cast<cpx<double>*>(data);
        auto* s = static_cast<cpx<double>*>(scratch);
        auto* t = static_cast<const cpx<double>*>(tw);
        return sign < 0 ? run_fft1d<-1>(d, s, len, t, stream) : run_fft1d<1>(d, s, len, t, stream);
    }
    auto* d = static_cast<cpx<float>*>(data);
    auto* s = static_cast<cpx<float>*>(scratch);
    auto* t = static_cast<const cpx<float>*>(tw);
    return sign < 0 ? run_fft1d<-1>(d, s, len, t, stream) : run_fft1d<1>(d, s, len, t, stream);
}

}  // namespace ddmk
