// Step 1 of the WITH_FT pipeline on B200: batched r2c 2D spatial FFT of u16/u8 frames,
// with the frame-major -> wave-vector-major corner turn fused into the column pass.
//
// Replaces, per frame, the reference's u16->Scalar conversion (`scheduler.cpp:115-119`),
// FFTW r2c 2D (`fft.cpp:34-37,86-87,128-132`, unnormalised, H x (W/2+1) half plane) and
// the stride-N gather into group sequences (`scheduler.cpp:122-126`).
//
//   rows_kernel : one CTA = RB rows of one frame. Pixels are converted on load; a real row
//                 of even W goes through a W/2 complex FFT plus the even/odd split. Output
//                 is written column-major per frame (`mid[f][col][row]`), RB-row runs.
//   cols_kernel : one CTA = CB adjacent columns of one frame (contiguous in `mid`),
//                 H-point complex FFT, epilogue scatters every retained wave vector of the
//                 current group into the tile-major spectra layout (kernels.cuh).
// The host runs them over chunks of frames sized so `mid` stays L2 resident.
// Transform lengths in DDMK_LENGTH_CASES get compile-time pass plans; others take the
// runtime radix-4/2/5/3 plan (or a direct DFT for other prime factors).
#include <algorithm>
#include <type_traits>

#include "kernels.cuh"

namespace ddmk {

namespace {

constexpr int kThreads = 256;

template <int SIGN, int LC, typename S>
__device__ __forceinline__ void batch_fft(cpx<S>* buf, int L, int nbatch, const FftPlan& plan,
                                          const cpx<S>* __restrict__ tw, cpx<S>* scratch) {
    if constexpr (LC > 0)
        smem_fft_ct<LC, 1, SIGN, 2>(buf, LC, nbatch, tw);
    else
        smem_fft_rt<SIGN>(buf, L, nbatch, plan, tw, scratch);
}

template <typename S, typename Pix, int LC>
__global__ void __launch_bounds__(kThreads)
rows_kernel(const Pix* __restrict__ frames, int W, int H, int frame0, int RB, FftPlan plan,
            const cpx<S>* __restrict__ tw_row, const cpx<S>* __restrict__ tw_post,
            cpx<S>* __restrict__ mid) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cpx<S>* buf = reinterpret_cast<cpx<S>*>(smem_raw);
    const int L = LC > 0 ? LC : plan.len;
    const bool packed = (W % 2) == 0;
    const int Wh = W / 2 + 1;
    const int rblocks = (H + RB - 1) / RB;
    const int fi = blockIdx.x / rblocks;
    const int r0 = (blockIdx.x - fi * rblocks) * RB;
    const int nr = min(RB, H - r0);
    const Pix* src = frames + ((size_t)(frame0 + fi) * H + r0) * W;

    if constexpr (std::is_same_v<Pix, uint16_t>) {
      if (packed) {
        // pairs of u16 pixels as one 32-bit word; rows are contiguous: idx = rr*L + k
        const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
        for (int idx = threadIdx.x; idx < nr * L; idx += blockDim.x) {
            const uint32_t w2 = __ldg(s32 + idx);
            buf[idx] = {(S)(w2 & 0xFFFFu), (S)(w2 >> 16)};
        }
        goto loaded;
      }
    }
    if constexpr (std::is_same_v<Pix, uint8_t>) {
      if (packed) {
        const uint16_t* s16 = reinterpret_cast<const uint16_t*>(src);
        for (int idx = threadIdx.x; idx < nr * L; idx += blockDim.x) {
            const uint16_t w2 = __ldg(s16 + idx);
            buf[idx] = {(S)(w2 & 0xFFu), (S)(w2 >> 8)};
        }
        goto loaded;
      }
    }
    for (int idx = threadIdx.x; idx < nr * L; idx += blockDim.x) {
        const int rr = idx / L, k = idx - rr * L;
        if (packed) buf[idx] = {(S)src[rr * W + 2 * k], (S)src[rr * W + 2 * k + 1]};
        else buf[idx] = {(S)src[rr * W + k], S(0)};
    }
loaded:
    __syncthreads();
    batch_fft<-1, LC>(buf, L, nr, plan, tw_row, buf + RB * L);

    const S half = S(0.5);
    cpx<S>* dst = mid + (size_t)fi * Wh * H + r0;
    for (int idx = threadIdx.x; idx < nr * Wh; idx += blockDim.x) {
        const int c = idx / nr, rr = idx - c * nr;
        cpx<S> X;
        if (packed) {
            const cpx<S> zk = buf[rr * L + (c % L)];
            cpx<S> zc = buf[rr * L + (L - c) % L];
            zc.y = -zc.y;
            const cpx<S> e = {(zk.x + zc.x) * half, (zk.y + zc.y) * half};
            const cpx<S> o = {(zk.y - zc.y) * half, -(zk.x - zc.x) * half};  // (zk-zc)/(2i)
            X = cadd(e, cmul(tw_post[c], o));
        } else {
            X = buf[rr * L + c];
        }
        dst[(size_t)c * H + rr] = X;
    }
}

// F frames x CB columns per CTA (CB adjacent columns of each frame are contiguous in `mid`):
// the epilogue then writes each retained wave vector's F consecutive frames as one run
// (F complex = 128 B at F = 16 in f32), instead of one 8-byte value per sequence per CTA
template <typename S, int LC>
__global__ void __launch_bounds__(kThreads)
cols_kernel(const cpx<S>* __restrict__ mid, int H, int Wh, int CB, int F, int nframes, int N, int frame0,
            FftPlan plan, const cpx<S>* __restrict__ tw_col, cpx<S>* __restrict__ spec,
            SpecLayout lay, const int* __restrict__ slot_of_flat) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cpx<S>* buf = reinterpret_cast<cpx<S>*>(smem_raw);
    const int cblocks = (Wh + CB - 1) / CB;
    const int fb = blockIdx.x / cblocks;
    const int c0 = (blockIdx.x - fb * cblocks) * CB;
    const int nc = min(CB, Wh - c0);
    const int f0 = fb * F;                      // within the chunk
    const int nf = min(F, nframes - f0);
    // buf[(fl * nc + cc) * H + r]: frame fl's columns are one contiguous run of nc * H
    for (int idx = threadIdx.x; idx < nf * nc * H; idx += blockDim.x) {
        const int fl = idx / (nc * H), rest = idx - fl * nc * H;
        buf[idx] = mid[((size_t)(f0 + fl) * Wh + c0) * H + rest];
    }
    __syncthreads();
    batch_fft<-1, LC>(buf, H, nf * nc, plan, tw_col, buf + (size_t)F * CB * H);

    const int n0 = frame0 + f0;
    const int T = lay.T;
    // consecutive threads: consecutive frames of one wave vector
    for (int idx = threadIdx.x; idx < nf * nc * H; idx += blockDim.x) {
        const int fl = idx % nf, rc = idx / nf;
        const int r = rc / nc, cc = rc - r * nc;
        const int64_t fl_flat = (int64_t)r * Wh + c0 + cc;
        const int64_t k = slot_of_flat ? (int64_t)slot_of_flat[fl_flat] : fl_flat;
        const int64_t sl = k - lay.g_begin;
        if (k < 0 || sl < 0 || sl >= lay.g_count) continue;
        const int64_t tile = sl / T;
        spec[(tile * N + n0 + fl) * T + (sl - tile * T)] = buf[(fl * nc + cc) * H + r];
    }
}

// transforms per CTA: <= 16, <= 96 KB of shared memory, and at most 8192 points per CTA
// (2 radix-16 butterflies per thread at 256 threads)
int pick_rows(int L, size_t scalar_bytes, bool naive) {
    if (L > 8192) return 0;
    int rb = 16;
    const size_t cap = 96 * 1024;
    while (rb > 1 && ((size_t)rb * L * 2 * scalar_bytes * (naive ? 2 : 1) > cap || rb * L > 8192))
        rb >>= 1;
    return rb;
}

template <typename S, typename Pix, int LC>
void launch_rows(const SpatialArgs& a, int RB, const FftPlan& plan, size_t smem, cudaStream_t st) {
    auto k = rows_kernel<S, Pix, LC>;
    // a failed attribute stays the last error (the caller's cudaGetLastError reports it):
    // no launch that would fail later with an unrelated message
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return;
    const int grid = a.nframes * ((a.H + RB - 1) / RB);
    k<<<grid, kThreads, smem, st>>>(static_cast<const Pix*>(a.frames), a.W, a.H, a.frame0, RB,
                                    plan, static_cast<const cpx<S>*>(a.tw_row.ptr),
                                    static_cast<const cpx<S>*>(a.tw_post.ptr),
                                    static_cast<cpx<S>*>(a.mid));
}

template <typename S, int LC>
void launch_cols(const SpatialArgs& a, int CB, int F, const FftPlan& plan, size_t smem, cudaStream_t st) {
    auto k = cols_kernel<S, LC>;
    // a failed attribute stays the last error (the caller's cudaGetLastError reports it):
    // no launch that would fail later with an unrelated message
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return;
    const int Wh = a.W / 2 + 1;
    const int grid = ((a.nframes + F - 1) / F) * ((Wh + CB - 1) / CB);
    k<<<grid, kThreads, smem, st>>>(static_cast<const cpx<S>*>(a.mid), a.H, Wh, CB, F, a.nframes, a.N,
                                    a.frame0, plan, static_cast<const cpx<S>*>(a.tw_col.ptr),
                                    static_cast<cpx<S>*>(a.spec), a.layout, a.slot_of_flat);
}

}  // namespace

template <typename S>
cudaError_t launch_spatial(const SpatialArgs& a, cudaStream_t stream) {
    const int Lr = a.tw_row.len, Lc = a.tw_col.len;
    const FftPlan prow = make_rt_plan(Lr);
    const FftPlan pcol = make_rt_plan(Lc);
    const size_t cs = 2 * sizeof(S);
    const int RB = pick_rows(Lr, sizeof(S), prow.naive);
    // column CTAs: F frames x CB columns, the same transform budget as a row CTA, frames first
    const int CT = pick_rows(Lc, sizeof(S), pcol.naive);
    if (RB == 0 || CT == 0) return cudaErrorInvalidValue;
    const int F = std::min(CT, std::max(1, a.nframes));
    const int CB = std::max(1, CT / F);
    const size_t smem_r = (size_t)RB * Lr * cs * (prow.naive ? 2 : 1);
    const size_t smem_c = (size_t)F * CB * Lc * cs * (pcol.naive ? 2 : 1);

#define DDMK_ROWS_CASE(LEN)                                                             \
    case LEN:                                                                           \
        if (a.pixel_bytes == 2) launch_rows<S, uint16_t, LEN>(a, RB, prow, smem_r, stream); \
        else if (a.pixel_bytes == 1) launch_rows<S, uint8_t, LEN>(a, RB, prow, smem_r, stream); \
        else if (a.pixel_bytes == 4) launch_rows<S, float, 0>(a, RB, prow, smem_r, stream); \
        else launch_rows<S, double, 0>(a, RB, prow, smem_r, stream);                  \
        break;
    switch (Lr) {
        DDMK_LENGTH_CASES(DDMK_ROWS_CASE)
    default:
        if (a.pixel_bytes == 2) launch_rows<S, uint16_t, 0>(a, RB, prow, smem_r, stream);
        else if (a.pixel_bytes == 1) launch_rows<S, uint8_t, 0>(a, RB, prow, smem_r, stream);
        else if (a.pixel_bytes == 4) launch_rows<S, float, 0>(a, RB, prow, smem_r, stream);
        else launch_rows<S, double, 0>(a, RB, prow, smem_r, stream);
    }
#undef DDMK_ROWS_CASE
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;

#define DDMK_COLS_CASE(LEN) \
    case LEN: launch_cols<S, LEN>(a, CB, F, pcol, smem_c, stream); break;
    switch (Lc) {
        DDMK_LENGTH_CASES(DDMK_COLS_CASE)
    default: launch_cols<S, 0>(a, CB, F, pcol, smem_c, stream);
    }
#undef DDMK_COLS_CASE
    return cudaGetLastError();
}

template cudaError_t launch_spatial<float>(const SpatialArgs&, cudaStream_t);
template cudaError_t launch_spatial<double>(const SpatialArgs&, cudaStream_t);

}  // namespace ddmk
