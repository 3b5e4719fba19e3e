// Spatial step v2 (sm_100a): register-resident group FFTs (warp_fft.cuh) for power-of-two
// frame sizes, writing the wave-vector-major spectra the warp temporal engine streams.
//
// Same contract as spatial.cu (FFTW r2c 2D, `fft.cpp:34-37,86-87,128-132`, unnormalised,
// rows=H x cols=W -> H x (W/2+1); conversion `scheduler.cpp:115-119`; corner turn
// `scheduler.cpp:122-126`), specialised on the transform lengths:
//   rows2  : one group of A lanes per image row. Pixel pairs (x[2k], x[2k+1]) are read as
//            32-bit words (u16) and form the L = W/2 complex input; the even/odd split after
//            the FFT needs Z[k] and Z[L-k], so rows pass through shared memory once and are
//            written column-major per frame, mid[f][col][row], RB = 256/A rows per run.
//   cols2  : one CTA = one column x F = 256/A frames; every group transforms the column of
//            one frame; the CTA transposes through shared memory so that each retained wave
//            vector receives F consecutive frames as one contiguous run:
//            spec[slot * N + frame] (layout T = 1, consumed by temporal_warp.cu).
// Packed f32x2 products (FMUL2/FFMA2, fft_core.cuh) but scalar sums in the row and column
// passes: measured at C2 / C3 / C4 (tools/gpu_ab3.sh, profiles/r02z_f32x2_ab.txt) spatial
// 0.737 / 6.96 / 66.6 ms scalar, 0.718 / 6.83 / 66.5 all packed, 0.707 / 6.76 / 65.6 with
// products only (FADD2 alone: 0.777 at C2). K3L (temporal_long2.cu) keeps both packed.
#ifndef DDM_F32X2_ADD
#define DDM_F32X2_ADD 0
#endif
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "warp_fft.cuh"

namespace ddmk {

namespace {

constexpr int kThreads = 256;

template <int L>
struct Split {  // L = A * B with A | B, A <= 32
    static constexpr int log2L = L <= 1 ? 0 : 1 + Split<(L > 1 ? L / 2 : 1)>::log2L;
};
template <>
struct Split<1> {
    static constexpr int log2L = 0;
};
template <int L>
__host__ __device__ constexpr int split_a() {
    constexpr int e = Split<L>::log2L;
    constexpr int a = 1 << (e / 2);
    return a > 32 ? 32 : a;
}

// ---------------------------------------------------------------------------- rows
template <typename S, typename Pix, int L>
__device__ __forceinline__ void rows2_body(const Pix* __restrict__ frames, int H, int frame0,
                                           const cpx<S>* __restrict__ tw_row,
                                           const cpx<S>* __restrict__ tw_post,
                                           cpx<S>* __restrict__ mid, int item,
                                           unsigned char* smem_raw) {
    constexpr int A = split_a<L>(), B = L / A;
    constexpr int W = 2 * L, Wh = L + 1;
    constexpr int RB = kThreads / A;                 // rows per CTA (one per group)
    constexpr int REG = B * (A + 1) + 1;             // group region (odd stride: banks)
    cpx<S>* region_base = reinterpret_cast<cpx<S>*>(smem_raw);

    const int g = threadIdx.x / A, a = threadIdx.x % A;
    const int rblocks = (H + RB - 1) / RB;
    const int fi = item / rblocks;
    const int r0 = (item - fi * rblocks) * RB;
    constexpr int nr = RB;  // H % RB == 0 (spatial_warp_supported)
    cpx<S>* reg = region_base + g * REG;

    LaneTw<B, S> tw;
    tw.init_from(tw_row, a, L);

    cpx<S> v[B];
    if (g < nr) {
        const Pix* row = frames + ((size_t)(frame0 + fi) * H + r0 + g) * W;
        if constexpr (std::is_same_v<Pix, uint16_t>) {
            const uint32_t* w32 = reinterpret_cast<const uint32_t*>(row);
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t p = __ldcs(w32 + a + A * b);   // read once: evict first
                v[b] = {(S)(p & 0xFFFFu), (S)(p >> 16)};
            }
        } else {
            const uint16_t* w16 = reinterpret_cast<const uint16_t*>(row);
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint16_t p = __ldcs(w16 + a + A * b);
                v[b] = {(S)(p & 0xFFu), (S)(p >> 8)};
            }
        }
        group_fft<A, B, -1, S>(v, reg, a, tw);
        // natural order into the group region: Z[k] at k
#pragma unroll
        for (int i = 0; i < B / A; ++i)
#pragma unroll
            for (int d = 0; d < A; ++d) reg[(a + i * A) + B * d] = v[i * A + d];
    }
    __syncthreads();

    // even/odd split: X[c] = (Z[c] + conj Z[L-c]) / 2 + W_W^c (Z[c] - conj Z[L-c]) / (2i)
    // thread (rq, cb) owns rows RV rq .. RV rq + RV - 1 and the columns c = cb + CS j: fixed
    // strides, no division, one twiddle load per column for its rows, and those rows' values
    // of a column (adjacent in mid[f][col][row]) leave as one store: 32 bytes (RV = 4,
    // st.global.v8) in f32, 16 bytes per two rows in f64
    constexpr int RV = sizeof(S) == 4 ? 4 : 2;       // rows per thread
    constexpr int RQ = RB / RV;
    constexpr int CS = kThreads / RQ;                // column stride
    constexpr int NJ = (Wh + CS - 1) / CS;
    const S half = S(0.5);
    const int rq = threadIdx.x % RQ, cb = threadIdx.x / RQ;
    const cpx<S>* z0 = region_base + (RV * rq) * REG;
    cpx<S>* dst = mid + (size_t)fi * Wh * H + r0 + RV * rq + (size_t)cb * H;
    const size_t step = (size_t)CS * H;
    auto split = [&](const cpx<S>* z, int c, cpx<S> w) {
        const cpx<S> zk = z[c < L ? c : c - L];
        cpx<S> zc = z[c == 0 ? 0 : L - c];
        zc.y = -zc.y;
        const cpx<S> e = {(zk.x + zc.x) * half, (zk.y + zc.y) * half};
        const cpx<S> o = {(zk.y - zc.y) * half, -(zk.x - zc.x) * half};
        return cadd(e, cmul(w, o));
    };
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int c = cb + CS * j;
        if (j == NJ - 1 && c >= Wh) break;
        const cpx<S> w = tw_post[c];
        cpx<S> x[RV];
#pragma unroll
        for (int r = 0; r < RV; ++r) x[r] = split(z0 + r * REG, c, w);
        if constexpr (sizeof(S) == 4) {
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + j * step),
                         "f"(x[0].x), "f"(x[0].y), "f"(x[1].x), "f"(x[1].y), "f"(x[2].x), "f"(x[2].y),
                         "f"(x[3].x), "f"(x[3].y)
                         : "memory");
        } else {
            dst[j * step] = x[0];
            dst[j * step + 1] = x[1];
        }
    }
}

template <typename S, typename Pix, int L>
__global__ void __launch_bounds__(kThreads)
rows2_kernel(const Pix* __restrict__ frames, int H, int frame0, const cpx<S>* __restrict__ tw_row,
             const cpx<S>* __restrict__ tw_post, cpx<S>* __restrict__ mid) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    rows2_body<S, Pix, L>(frames, H, frame0, tw_row, tw_post, mid, blockIdx.x, smem_raw);
}

// streaming store (evict-first in L2): spectra are not re-read until the temporal step, so
// they must not push the L2-resident row-pass buffers out
template <typename S>
__device__ __forceinline__ void st_stream(cpx<S>* p, cpx<S> v) {
    if constexpr (sizeof(S) == 4) __stcs(reinterpret_cast<float2*>(p), make_float2(v.x, v.y));
    else *p = v;
}

template <typename S>
__device__ __forceinline__ cpx<S> ld_cg(const cpx<S>* p) {
    if constexpr (sizeof(S) == 4) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(p));
        return {v.x, v.y};
    } else {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
        return {v.x, v.y};
    }
}

// ---------------------------------------------------------------------------- cols
// Column-pass epilogue: the CTA's transposed stage sm[r * (F + 1) + f] (wave-vector row r,
// frame f of this CTA's nf frames starting at n0, column c) -> the spectra, a peer's receive
// buffer, or a cutoff / group subset.
template <typename S, int HL, int F = kThreads / split_a<HL>(), int NT = kThreads>
__device__ __forceinline__ void cols_epilogue(const cpx<S>* sm, int Wh, int N, int n0, int nf, int c,
                                              cpx<S>* __restrict__ spec, const SpecLayout& lay,
                                              const int* __restrict__ slot_of_flat,
                                              const PeerTable& peers) {
    constexpr int SP = F + 1;
    const int64_t plane = (int64_t)HL * Wh;
    if (peers.ranks > 0) {
        // fused corner turn: every wave vector goes to its owner's receive buffer (a peer
        // pointer over NVLink); rows ascend with j, so the owner index only moves forward
        constexpr int RS = NT / F;
        const int f = threadIdx.x % F, rb = threadIdx.x / F;
        if (f < nf) {
            const int64_t kstep = (int64_t)RS * Wh;
            int64_t k = (int64_t)rb * Wh + c;
            int d = 0;
            int64_t k_end = -1;   // owner slice [.., k_end) of the current destination
            cpx<S>* dst = nullptr;
#pragma unroll 4
            for (int j = 0; j < HL / RS; ++j, k += kstep, dst += kstep * N) {
                if (k >= k_end) {  // crossed into the next rank's slice (rare)
                    while (d + 1 < peers.ranks && k >= peers.q_begin[d + 1]) ++d;
                    k_end = peers.q_begin[d + 1];
                    dst = static_cast<cpx<S>*>(peers.base[d]) + (k - peers.q_begin[d]) * N + n0 + f;
                }
                st_stream(dst, sm[(rb + RS * j) * SP + f]);
            }
        }
        return;
    }
    if constexpr (sizeof(S) == 4) {
    if (!slot_of_flat && lay.g_begin == 0 && lay.g_count == plane && ((N | n0) & 1) == 0) {
        // every wave vector of the plane, identity slots, f32: thread (fp, rb + RS j) copies
        // frames fp, fp + 1 of wave vector (r, c) as one 16-byte store; TPR consecutive
        // threads fill an F-frame run
        constexpr int TPR = F / 2, RS = NT / TPR;
        const int fp = 2 * (threadIdx.x % TPR), rb = threadIdx.x / TPR;
        if (fp < nf) {
            cpx<S>* dst = spec + ((int64_t)rb * Wh + c) * N + n0 + fp;
            const int64_t step = (int64_t)RS * Wh * N;
            const bool pair = fp + 1 < nf;
#pragma unroll 8
            for (int j = 0; j < HL / RS; ++j) {
                const cpx<S>* src = sm + (rb + RS * j) * SP + fp;
                if (pair) {
                    const cpx<S> u = src[0], w = src[1];
                    __stcs(reinterpret_cast<float4*>(dst + j * step), make_float4(u.x, u.y, w.x, w.y));
                } else {
                    st_stream(dst + j * step, src[0]);
                }
            }
        }
        return;
    }
    }
    if (!slot_of_flat && lay.g_begin == 0 && lay.g_count == plane) {
        // every wave vector of the plane, identity slots: thread (f, rb + RS j) copies one
        // frame of wave vector (r, c); consecutive threads fill F-frame runs
        constexpr int RS = NT / F;                   // row stride
        const int f = threadIdx.x % F, rb = threadIdx.x / F;
        if (f < nf) {
            cpx<S>* dst = spec + ((int64_t)rb * Wh + c) * N + n0 + f;
            const int64_t step = (int64_t)RS * Wh * N;
#pragma unroll 8
            for (int j = 0; j < HL / RS; ++j) st_stream(dst + j * step, sm[(rb + RS * j) * SP + f]);
        }
        return;
    }
    for (int idx = threadIdx.x; idx < HL * F; idx += NT) {
        const int r = idx / F, f = idx - r * F;
        if (f >= nf) continue;
        const int64_t flat = (int64_t)r * Wh + c;
        const int64_t k = slot_of_flat ? (int64_t)slot_of_flat[flat] : flat;
        const int64_t s = k - lay.g_begin;
        if (k < 0 || s < 0 || s >= lay.g_count) continue;
        spec[s * N + n0 + f] = sm[r * SP + f];
    }
}

// column c of the frames [f0, f0 + F) of the chunk held in `mid` (frame0 = the chunk's first
// frame of the stack)
template <typename S, int HL>
__device__ __forceinline__ void cols2_core(const cpx<S>* __restrict__ mid, int Wh, int N, int frame0,
                                           int nframes, const cpx<S>* __restrict__ tw_col,
                                           cpx<S>* __restrict__ spec, const SpecLayout& lay,
                                           const int* __restrict__ slot_of_flat,
                                           const PeerTable& peers, int c, int f0,
                                           unsigned char* smem_raw) {
    constexpr int A = split_a<HL>(), B = HL / A;
    constexpr int F = kThreads / A;                  // frames per CTA (one per group)
    constexpr int REG = B * (A + 1);
    constexpr int SP = F + 1;                        // stage pitch (complex)
    cpx<S>* sm = reinterpret_cast<cpx<S>*>(smem_raw);

    const int g = threadIdx.x / A, a = threadIdx.x % A;
    const int nf = min(F, nframes - f0);

    LaneTw<B, S> tw;
    tw.init_from(tw_col, a, HL);

    cpx<S> v[B];
    if (g < nf) {
        const cpx<S>* col = mid + ((size_t)(f0 + g) * Wh + c) * HL;
        // L2 loads (ld.global.cg): read exactly once
#pragma unroll
        for (int b = 0; b < B; ++b) v[b] = ld_cg(col + a + A * b);
        group_fft<A, B, -1, S>(v, sm + g * REG, a, tw);
        {
            // the row-pass buffer has been consumed: drop its L2 lines without writing
            // them back to DRAM (HL * 8 bytes per column, 128-byte lines)
            const char* base = reinterpret_cast<const char*>(col);
            for (int l = a; l < HL * (int)sizeof(cpx<S>) / 128; l += A)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + 128 * l) : "memory");
        }
    }
    __syncthreads();  // exchange regions are reused as the transpose stage
    if (g < nf) {
#pragma unroll
        for (int i = 0; i < B / A; ++i)
#pragma unroll
            for (int d = 0; d < A; ++d) sm[((a + i * A) + B * d) * SP + g] = v[i * A + d];
    }
    __syncthreads();

    cols_epilogue<S, HL>(sm, Wh, N, frame0 + f0, nf, c, spec, lay, slot_of_flat, peers);
}

template <typename S, int HL>
__device__ __forceinline__ void cols2_body(const cpx<S>* __restrict__ mid, int Wh, int N, int frame0,
                                           int nframes, const cpx<S>* __restrict__ tw_col,
                                           cpx<S>* __restrict__ spec, const SpecLayout& lay,
                                           const int* __restrict__ slot_of_flat,
                                           const PeerTable& peers, int item,
                                           unsigned char* smem_raw) {
    constexpr int F = kThreads / split_a<HL>();
    const int fblocks = (nframes + F - 1) / F;
    const int c = item / fblocks;
    const int f0 = (item - c * fblocks) * F;         // within the chunk
    cols2_core<S, HL>(mid, Wh, N, frame0, nframes, tw_col, spec, lay, slot_of_flat, peers, c, f0,
                      smem_raw);
}

template <typename S, int HL>
__global__ void __launch_bounds__(kThreads)
cols2_kernel(const cpx<S>* __restrict__ mid, int Wh, int N, int frame0, int nframes,
             const cpx<S>* __restrict__ tw_col, cpx<S>* __restrict__ spec, SpecLayout lay,
             const int* __restrict__ slot_of_flat, const __grid_constant__ PeerTable peers) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cols2_body<S, HL>(mid, Wh, N, frame0, nframes, tw_col, spec, lay, slot_of_flat, peers,
                             blockIdx.x, smem_raw);
}

// ---------------------------------------------------------------------------- cols, H = 2048
// The 2048-point column pass with two warps per column (cols2<2048>:pair). With one warp per
// column a lane holds 64 values (187 registers, one 8-warp CTA per SM: latency-bound, 52% of
// HBM at C4). Here lane a < 64 of a column group holds x[a + 64 b], b < 32:
//   Y[a][k1]  = W_2048^{a k1} sum_b x[a + 64 b] W_32^{b k1}                 (DFT_32 in registers)
//   lane (k1, a1), a1 = a & 1, reads Y[2 a2 + a1][k1] through shared memory (pitch 66: the
//   half-warp's 16 loads hit 16 distinct bank pairs) and forms
//   Z_a1[k] = sum_a2 Y[2 a2 + a1][k1] W_32^{a2 k}                            (DFT_32)
//   X[k1 + 32 k]        = Z_0[k] + W_64^k Z_1[k]
//   X[k1 + 32 (k + 32)] = Z_0[k] - W_64^k Z_1[k]                            (lane-pair radix 2)
// 32 values per lane (~110 registers), 16 warps per SM; 8 frames per CTA as before, so the
// corner-turn runs stay 64 bytes.
constexpr int kPairThreads = 512;
constexpr int kPairF = kPairThreads / 64;   // frames per CTA
constexpr int kPairP = 66;                  // exchange pitch (complex)

template <typename S>
__global__ void __launch_bounds__(kPairThreads, 1)
cols2_pair_kernel(const cpx<S>* __restrict__ mid, int Wh, int N, int frame0, int nframes,
                  const cpx<S>* __restrict__ tw_col, cpx<S>* __restrict__ spec, SpecLayout lay,
                  const int* __restrict__ slot_of_flat, const __grid_constant__ PeerTable peers) {
    constexpr int HL = 2048, B = 32, F = kPairF, P = kPairP, SP = F + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cpx<S>* sm = reinterpret_cast<cpx<S>*>(smem_raw);
    const int g = threadIdx.x >> 6, a = threadIdx.x & 63;
    const int fblocks = (nframes + F - 1) / F;
    const int c = blockIdx.x / fblocks;
    const int f0 = (blockIdx.x - c * fblocks) * F;
    const int nf = min(F, nframes - f0);
    const bool act = g < nf;
    const int k1 = a >> 1, a1 = a & 1;

    cpx<S> v[B];
    if (act) {
        LaneTw<B, S> tw;
        tw.init_from(tw_col, a, HL);
        const cpx<S>* col = mid + ((size_t)(f0 + g) * Wh + c) * HL;
#pragma unroll
        for (int b = 0; b < B; ++b) v[b] = ld_cg(col + a + 64 * b);
        RegDft<B, -1, S>::run(v);
#pragma unroll
        for (int k = 1; k < B; ++k) v[k] = cmul(v[k], tw.template get<-1>(k));
        cpx<S>* ex = sm + g * B * P;
#pragma unroll
        for (int k = 0; k < B; ++k) ex[k * P + a] = v[k];
        asm volatile("bar.sync %0, 64;" ::"r"(1 + g) : "memory");   // this column group only
        {
            // both warps of the group have their column values (the barrier): drop the
            // row-pass buffer's L2 lines without write-back
            const char* base = reinterpret_cast<const char*>(col);
            for (int l = a; l < HL * (int)sizeof(cpx<S>) / 128; l += 64)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + 128 * l) : "memory");
        }
#pragma unroll
        for (int a2 = 0; a2 < B; ++a2) v[a2] = ex[k1 * P + 2 * a2 + a1];
        RegDft<B, -1, S>::run(v);
        // odd lanes: W_64^k Z_1[k] (compile-time constants, selected per lane)
        const S one = a1 ? S(0) : S(1), sel = a1 ? S(1) : S(0);
#pragma unroll
        for (int k = 1; k < B; ++k) {
            const cpx<S> w = ct_w<-1, S>(k, 64);
            v[k] = cmul(v[k], cpx<S>{one + sel * w.x, sel * w.y});
        }
        // pair butterfly: even lane Z0 + t, odd lane Z0 - t (t = its own value)
        const S sgn = a1 ? S(-1) : S(1);
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const S px = __shfl_xor_sync(0xffffffffu, v[k].x, 1);
            const S py = __shfl_xor_sync(0xffffffffu, v[k].y, 1);
            v[k] = {fma(sgn, v[k].x, px), fma(sgn, v[k].y, py)};
        }
    }
    __syncthreads();  // every group's exchange reads are done: the area becomes the stage
    if (act) {
#pragma unroll
        for (int k = 0; k < B; ++k) sm[(k1 + 32 * (k + 32 * a1)) * SP + g] = v[k];
    }
    __syncthreads();
    cols_epilogue<S, HL, F, kPairThreads>(sm, Wh, N, frame0 + f0, nf, c, spec, lay, slot_of_flat, peers);
}

constexpr size_t pair_smem(size_t cs) {
    const size_t ex = (size_t)kPairF * 32 * kPairP, st = (size_t)2048 * (kPairF + 1);
    return (ex > st ? ex : st) * cs;
}

template <typename S>
cudaError_t launch_cols2_pair(const SpatialArgs& a, cudaStream_t st) {
    auto k = cols2_pair_kernel<S>;
    const size_t smem = pair_smem(sizeof(cpx<S>));
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int Wh = a.W / 2 + 1;
    const int grid = Wh * ((a.nframes + kPairF - 1) / kPairF);
    k<<<grid, kPairThreads, smem, st>>>(static_cast<const cpx<S>*>(a.mid), Wh, a.N, a.frame0,
                                        a.nframes, static_cast<const cpx<S>*>(a.tw_col.ptr),
                                        static_cast<cpx<S>*>(a.spec), a.layout, a.slot_of_flat,
                                        a.peers);
    return cudaGetLastError();
}

// complex slots of the column pass's exchange / transpose area
template <int HL>
__host__ __device__ constexpr int cols_area() {
    constexpr int A = split_a<HL>(), B = HL / A;
    constexpr int ex = (kThreads / A) * B * (A + 1);
    constexpr int st = HL * (kThreads / A + 1);
    return ex > st ? ex : st;
}

template <int L>
__host__ __device__ constexpr size_t rows_smem(size_t cs) {
    constexpr int A = split_a<L>(), B = L / A;
    return (size_t)(kThreads / A) * (B * (A + 1) + 1) * cs;
}
template <int HL>
__host__ __device__ constexpr size_t cols_smem(size_t cs) {
    constexpr int A = split_a<HL>(), B = HL / A;
    const size_t ex = (size_t)(kThreads / A) * B * (A + 1);
    const size_t st = (size_t)HL * (kThreads / A + 1);
    return (ex > st ? ex : st) * cs;
}

template <typename S, typename Pix, int L>
cudaError_t launch_rows2(const SpatialArgs& a, cudaStream_t st) {
    auto k = rows2_kernel<S, Pix, L>;
    const size_t smem = rows_smem<L>(sizeof(cpx<S>));
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    constexpr int RB = kThreads / split_a<L>();
    const int grid = a.nframes * ((a.H + RB - 1) / RB);
    k<<<grid, kThreads, smem, st>>>(static_cast<const Pix*>(a.frames), a.H, a.frame0,
                                    static_cast<const cpx<S>*>(a.tw_row.ptr),
                                    static_cast<const cpx<S>*>(a.tw_post.ptr),
                                    static_cast<cpx<S>*>(a.mid));
    return cudaGetLastError();
}

template <typename S, int HL>
cudaError_t launch_cols2(const SpatialArgs& a, cudaStream_t st) {
    auto k = cols2_kernel<S, HL>;
    const size_t smem = cols_smem<HL>(sizeof(cpx<S>));
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    constexpr int F = kThreads / split_a<HL>();
    const int Wh = a.W / 2 + 1;
    const int grid = Wh * ((a.nframes + F - 1) / F);
    k<<<grid, kThreads, smem, st>>>(static_cast<const cpx<S>*>(a.mid), Wh, a.N, a.frame0,
                                    a.nframes, static_cast<const cpx<S>*>(a.tw_col.ptr),
                                    static_cast<cpx<S>*>(a.spec), a.layout,
                                    a.slot_of_flat, a.peers);
    return cudaGetLastError();
}

bool pow2_in(int x, int lo, int hi) { return x >= lo && x <= hi && (x & (x - 1)) == 0; }

}  // namespace

bool spatial_warp_supported(int W, int H, int pixel_bytes, int scalar_bytes) {
    if (scalar_bytes != 4 || (pixel_bytes != 1 && pixel_bytes != 2)) return false;
    if (!(W % 2 == 0 && pow2_in(W / 2, 16, 1024) && pow2_in(H, 16, 2048))) return false;
    const int e = 31 - __builtin_clz(W / 2);
    const int A = std::min(1 << (e / 2), 32);
    return H % (kThreads / A) == 0;  // whole row blocks per CTA
}

bool spatial_cols_pair() {
    // DDM_COLS2_PAIR=0: the one-warp 2048-point column pass (A/B)
    static const bool on = [] {
        const char* e = std::getenv("DDM_COLS2_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}

int spatial_warp_col_frames(int H) {
    const int e = 31 - __builtin_clz(H);
    return kThreads / std::min(1 << (e / 2), 32);
}

template <typename S>
cudaError_t launch_spatial_warp(const SpatialArgs& a, cudaStream_t stream, int parts) {
    const int L = a.W / 2;
    cudaError_t e = cudaSuccess;
    if (parts & 1) {
#define DDMK_R2(LEN)                                                               \
    case LEN:                                                                      \
        e = a.pixel_bytes == 2 ? launch_rows2<S, uint16_t, LEN>(a, stream)          \
                               : launch_rows2<S, uint8_t, LEN>(a, stream);          \
        break;
    switch (L) {
        DDMK_R2(16) DDMK_R2(32) DDMK_R2(64) DDMK_R2(128) DDMK_R2(256) DDMK_R2(512) DDMK_R2(1024)
    default: return cudaErrorInvalidValue;
    }
#undef DDMK_R2
    if (e != cudaSuccess) return e;
    }
    if (!(parts & 2)) return cudaSuccess;
    if constexpr (std::is_same_v<S, float>) {
        if (a.H == 2048 && spatial_cols_pair()) return launch_cols2_pair<S>(a, stream);
    }
#define DDMK_C2(LEN) \
    case LEN: e = launch_cols2<S, LEN>(a, stream); break;
    switch (a.H) {
        DDMK_C2(16) DDMK_C2(32) DDMK_C2(64) DDMK_C2(128) DDMK_C2(256) DDMK_C2(512) DDMK_C2(1024)
        DDMK_C2(2048)
    default: return cudaErrorInvalidValue;
    }
#undef DDMK_C2
    return e;
}

template cudaError_t launch_spatial_warp<float>(const SpatialArgs&, cudaStream_t, int);
template cudaError_t launch_spatial_warp<double>(const SpatialArgs&, cudaStream_t, int);

bool spatial_warp_f64_supported(int W, int H, int pixel_bytes) {
    // register budget of the f64 instantiations: rows up to W = 1024, columns up to H = 1024
    return spatial_warp_supported(W, H, pixel_bytes, 4) && W <= 1024 && H <= 1024;
}

}  // namespace ddmk
