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
    // thread (rr, cb) owns row rr and the columns c = cb + CS j: fixed strides, no division,
    // all twiddle loads hoisted by the unrolled loop
    constexpr int CS = kThreads / RB;                // column stride
    constexpr int NJ = (Wh + CS - 1) / CS;
    const S half = S(0.5);
    const int rr = threadIdx.x % RB, cb = threadIdx.x / RB;
    const cpx<S>* z = region_base + rr * REG;
    cpx<S>* dst = mid + (size_t)fi * Wh * H + r0 + rr + (size_t)cb * H;
    const size_t step = (size_t)CS * H;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int c = cb + CS * j;
        if (j == NJ - 1 && c >= Wh) break;
        const cpx<S> zk = z[c < L ? c : c - L];
        cpx<S> zc = z[c == 0 ? 0 : L - c];
        zc.y = -zc.y;
        const cpx<S> e = {(zk.x + zc.x) * half, (zk.y + zc.y) * half};
        const cpx<S> o = {(zk.y - zc.y) * half, -(zk.x - zc.x) * half};
        dst[j * step] = cadd(e, cmul(tw_post[c], o));
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

// ---------------------------------------------------------------------------- cols
// kCoherent: `mid` was written by other CTAs of the same launch (the fused spatial kernel),
// so it is read through L2 (ld.global.cg), never a stale L1 line.
// Column-pass epilogue: the CTA's transposed stage sm[r * (F + 1) + f] (wave-vector row r,
// frame f of this CTA's nf frames starting at n0, column c) -> the spectra, a peer's receive
// buffer, or a cutoff / group subset.
template <typename S, int HL>
__device__ __forceinline__ void cols_epilogue(const cpx<S>* sm, int Wh, int N, int n0, int nf, int c,
                                              cpx<S>* __restrict__ spec, const SpecLayout& lay,
                                              const int* __restrict__ slot_of_flat,
                                              const PeerTable& peers) {
    constexpr int A = split_a<HL>();
    constexpr int F = kThreads / A;
    constexpr int SP = F + 1;
    const int64_t plane = (int64_t)HL * Wh;
    if (peers.ranks > 0) {
        // fused corner turn: every wave vector goes to its owner's receive buffer (a peer
        // pointer over NVLink); rows ascend with j, so the owner index only moves forward
        constexpr int RS = kThreads / F;
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
    if (!slot_of_flat && lay.g_begin == 0 && lay.g_count == plane) {
        // every wave vector of the plane, identity slots: thread (f, rb + RS j) copies one
        // frame of wave vector (r, c); consecutive threads fill F-frame runs
        constexpr int RS = kThreads / F;             // row stride
        const int f = threadIdx.x % F, rb = threadIdx.x / F;
        if (f < nf) {
            cpx<S>* dst = spec + ((int64_t)rb * Wh + c) * N + n0 + f;
            const int64_t step = (int64_t)RS * Wh * N;
#pragma unroll 8
            for (int j = 0; j < HL / RS; ++j) st_stream(dst + j * step, sm[(rb + RS * j) * SP + f]);
        }
        return;
    }
    for (int idx = threadIdx.x; idx < HL * F; idx += kThreads) {
        const int r = idx / F, f = idx - r * F;
        if (f >= nf) continue;
        const int64_t flat = (int64_t)r * Wh + c;
        const int64_t k = slot_of_flat ? (int64_t)slot_of_flat[flat] : flat;
        const int64_t s = k - lay.g_begin;
        if (k < 0 || s < 0 || s >= lay.g_count) continue;
        spec[s * N + n0 + f] = sm[r * SP + f];
    }
}

template <typename S, int HL, bool kCoherent>
__device__ __forceinline__ void cols2_body(const cpx<S>* __restrict__ mid, int Wh, int N, int frame0,
                                           int nframes, const cpx<S>* __restrict__ tw_col,
                                           cpx<S>* __restrict__ spec, const SpecLayout& lay,
                                           const int* __restrict__ slot_of_flat,
                                           const PeerTable& peers, int item,
                                           unsigned char* smem_raw) {
    constexpr int A = split_a<HL>(), B = HL / A;
    constexpr int F = kThreads / A;                  // frames per CTA (one per group)
    constexpr int REG = B * (A + 1);
    constexpr int SP = F + 1;                        // stage pitch (complex)
    cpx<S>* sm = reinterpret_cast<cpx<S>*>(smem_raw);

    const int g = threadIdx.x / A, a = threadIdx.x % A;
    const int fblocks = (nframes + F - 1) / F;
    const int c = item / fblocks;
    const int f0 = (item - c * fblocks) * F;         // within the chunk
    const int nf = min(F, nframes - f0);

    LaneTw<B, S> tw;
    tw.init_from(tw_col, a, HL);

    cpx<S> v[B];
    if (g < nf) {
        const cpx<S>* col = mid + ((size_t)(f0 + g) * Wh + c) * HL;
        if constexpr (kCoherent && sizeof(S) == 4) {
            const float2* c2 = reinterpret_cast<const float2*>(col);
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const float2 t = __ldcs(c2 + a + A * b);      // L2, last use
                v[b] = {t.x, t.y};
            }
        } else {
#pragma unroll
            for (int b = 0; b < B; ++b) v[b] = col[a + A * b];
        }
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
__global__ void __launch_bounds__(kThreads)
cols2_kernel(const cpx<S>* __restrict__ mid, int Wh, int N, int frame0, int nframes,
             const cpx<S>* __restrict__ tw_col, cpx<S>* __restrict__ spec, SpecLayout lay,
             const int* __restrict__ slot_of_flat, const __grid_constant__ PeerTable peers) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cols2_body<S, HL, false>(mid, Wh, N, frame0, nframes, tw_col, spec, lay, slot_of_flat, peers,
                             blockIdx.x, smem_raw);
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
constexpr size_t rows_smem(size_t cs) {
    constexpr int A = split_a<L>(), B = L / A;
    return (size_t)(kThreads / A) * (B * (A + 1) + 1) * cs;
}
template <int HL>
constexpr size_t cols_smem(size_t cs) {
    constexpr int A = split_a<HL>(), B = HL / A;
    const size_t ex = (size_t)(kThreads / A) * B * (A + 1);
    const size_t st = (size_t)HL * (kThreads / A + 1);
    return (ex > st ? ex : st) * cs;
}

template <typename S, typename Pix, int L>
void launch_rows2(const SpatialArgs& a, cudaStream_t st) {
    auto k = rows2_kernel<S, Pix, L>;
    const size_t smem = rows_smem<L>(sizeof(cpx<S>));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    constexpr int RB = kThreads / split_a<L>();
    const int grid = a.nframes * ((a.H + RB - 1) / RB);
    k<<<grid, kThreads, smem, st>>>(static_cast<const Pix*>(a.frames), a.H, a.frame0,
                                    static_cast<const cpx<S>*>(a.tw_row.ptr),
                                    static_cast<const cpx<S>*>(a.tw_post.ptr),
                                    static_cast<cpx<S>*>(a.mid));
}

template <typename S, int HL>
void launch_cols2(const SpatialArgs& a, cudaStream_t st) {
    auto k = cols2_kernel<S, HL>;
    const size_t smem = cols_smem<HL>(sizeof(cpx<S>));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    constexpr int F = kThreads / split_a<HL>();
    const int Wh = a.W / 2 + 1;
    const int grid = Wh * ((a.nframes + F - 1) / F);
    k<<<grid, kThreads, smem, st>>>(static_cast<const cpx<S>*>(a.mid), Wh, a.N, a.frame0,
                                    a.nframes, static_cast<const cpx<S>*>(a.tw_col.ptr),
                                    static_cast<cpx<S>*>(a.spec), a.layout,
                                    a.slot_of_flat, a.peers);
}

// ---------------------------------------------------------------------------- fused
// One persistent launch for the whole spatial step: CTAs take work items from a global
// counter in the order R0 | R1 C0 | R2 C1 | ... | C(K-1), where R(k) are the row-pass items
// of frame chunk k and C(k) its column-pass items. Chunk k's `mid` is ring buffer k % NB.
// C(k) waits until every R(k) item is done; R(k) waits until C(k - NB) has released its
// buffer. Every dependency points to items dequeued earlier, so the queue always drains;
// there are no launch gaps or per-chunk tails, and row and column work overlap freely.
struct FusedSched {
    int K, F, N, nbuf, lead, rblocks, Wh, Fc;
    size_t buf_elems;               // complex values per mid buffer
    int* sync;                      // [0] work counter, [1..K] rows done, [K+1..2K] cols done
    __device__ int nf(int k) const { return min(F, N - k * F); }
    __device__ int n_rows(int k) const { return nf(k) * rblocks; }
    __device__ int n_cols(int k) const { return Wh * ((nf(k) + Fc - 1) / Fc); }
    // segment s -> (is_cols, chunk): R(0..D-1), then pairs (R(j + D), C(j)), then the last
    // D column segments; D = lead (rows run D chunks ahead of the columns)
    __device__ void seg(int s, bool& cols, int& k) const {
        const int D = min(lead, K), P = K - D;
        if (s < D) { cols = false; k = s; return; }
        const int t = s - D;
        if (t < 2 * P) { cols = (t & 1); k = (t & 1) ? t / 2 : t / 2 + D; return; }
        cols = true;
        k = P + (t - 2 * P);
    }
    __device__ int seg_size(int s) const {
        bool c; int k;
        seg(s, c, k);
        return c ? n_cols(k) : n_rows(k);
    }
    __device__ int total() const {
        int t = 0;
        for (int k = 0; k < K; ++k) t += n_rows(k) + n_cols(k);
        return t;
    }
};

__device__ __forceinline__ void wait_count(const int* p, int target) {
    while (atomicAdd(const_cast<int*>(p), 0) < target) __nanosleep(64);
    __threadfence();
}

template <typename S, typename Pix, int L, int HL>
__global__ void __launch_bounds__(kThreads, 2)
spatial_fused_kernel(const Pix* __restrict__ frames, int H, const cpx<S>* __restrict__ tw_row,
                     const cpx<S>* __restrict__ tw_post, const cpx<S>* __restrict__ tw_col,
                     cpx<S>* __restrict__ mid, cpx<S>* __restrict__ spec, SpecLayout lay,
                     const int* __restrict__ slot_of_flat, const __grid_constant__ PeerTable peers,
                     const FusedSched sc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_item, s_cols, s_chunk, s_idx;
    const int total = sc.total();
    int seg = 0, seg_start = 0;     // thread 0's cursor (items only increase)
    // thread 0 claims the following item while the current one is processed, so the atomic's
    // round trip never stalls the CTA (the smallest unfinished item is always running or
    // queued behind a smaller one: the queue still drains)
    int next = threadIdx.x == 0 ? atomicAdd(sc.sync, 1) : 0;
    for (;;) {
        if (threadIdx.x == 0) {
            const int item = next;
            if (item < total) next = atomicAdd(sc.sync, 1);
            s_item = item;
            if (item < total) {
                while (item >= seg_start + sc.seg_size(seg)) {
                    seg_start += sc.seg_size(seg);
                    ++seg;
                }
                bool c; int k;
                sc.seg(seg, c, k);
                s_cols = c;
                s_chunk = k;
                s_idx = item - seg_start;
                if (c) wait_count(sc.sync + 1 + k, sc.n_rows(k));
                else if (k >= sc.nbuf) wait_count(sc.sync + 1 + sc.K + (k - sc.nbuf), sc.n_cols(k - sc.nbuf));
            }
        }
        __syncthreads();
        if (s_item >= total) break;
        const int k = s_chunk, idx = s_idx;
        cpx<S>* buf = mid + (size_t)(k % sc.nbuf) * sc.buf_elems;
        if (s_cols) {
            cols2_body<S, HL, true>(buf, sc.Wh, sc.N, k * sc.F, sc.nf(k), tw_col, spec, lay,
                                    slot_of_flat, peers, idx, smem_raw);
        } else {
            rows2_body<S, Pix, L>(frames, H, k * sc.F, tw_row, tw_post, buf, idx, smem_raw);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(sc.sync + 1 + (s_cols ? sc.K : 0) + k, 1);
        }
    }
}

template <typename S, typename Pix, int L, int HL>
cudaError_t launch_fused_t(const SpatialArgs& a, int F, int nbuf, int lead, int* sync, int num_sms,
                           cudaStream_t st) {
    auto k = spatial_fused_kernel<S, Pix, L, HL>;
    const size_t smem = std::max(rows_smem<L>(sizeof(cpx<S>)), cols_smem<HL>(sizeof(cpx<S>)));
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, smem);
    if (e != cudaSuccess) return e;
    FusedSched sc;
    sc.N = a.N;
    sc.F = F;
    sc.K = (a.N + F - 1) / F;
    sc.nbuf = nbuf;
    sc.lead = lead;
    sc.rblocks = a.H / (kThreads / split_a<L>());
    sc.Wh = a.W / 2 + 1;
    sc.Fc = kThreads / split_a<HL>();
    sc.buf_elems = (size_t)F * sc.Wh * a.H;
    sc.sync = sync;
    e = cudaMemsetAsync(sync, 0, (size_t)(1 + 2 * sc.K) * sizeof(int), st);
    if (e != cudaSuccess) return e;
    k<<<std::max(1, occ) * num_sms, kThreads, smem, st>>>(
        static_cast<const Pix*>(a.frames), a.H, static_cast<const cpx<S>*>(a.tw_row.ptr),
        static_cast<const cpx<S>*>(a.tw_post.ptr), static_cast<const cpx<S>*>(a.tw_col.ptr),
        static_cast<cpx<S>*>(a.mid), static_cast<cpx<S>*>(a.spec), a.layout, a.slot_of_flat,
        a.peers, sc);
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

int spatial_warp_col_frames(int H) {
    const int e = 31 - __builtin_clz(H);
    return kThreads / std::min(1 << (e / 2), 32);
}

template <typename S>
cudaError_t launch_spatial_warp(const SpatialArgs& a, cudaStream_t stream, int parts) {
    const int L = a.W / 2;
    if (parts & 1) {
#define DDMK_R2(LEN)                                                               \
    case LEN:                                                                      \
        if (a.pixel_bytes == 2) launch_rows2<S, uint16_t, LEN>(a, stream);         \
        else launch_rows2<S, uint8_t, LEN>(a, stream);                             \
        break;
    switch (L) {
        DDMK_R2(16) DDMK_R2(32) DDMK_R2(64) DDMK_R2(128) DDMK_R2(256) DDMK_R2(512) DDMK_R2(1024)
    default: return cudaErrorInvalidValue;
    }
#undef DDMK_R2
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    }
    if (!(parts & 2)) return cudaSuccess;
#define DDMK_C2(LEN) \
    case LEN: launch_cols2<S, LEN>(a, stream); break;
    switch (a.H) {
        DDMK_C2(16) DDMK_C2(32) DDMK_C2(64) DDMK_C2(128) DDMK_C2(256) DDMK_C2(512) DDMK_C2(1024)
        DDMK_C2(2048)
    default: return cudaErrorInvalidValue;
    }
#undef DDMK_C2
    return cudaGetLastError();
}

template cudaError_t launch_spatial_warp<float>(const SpatialArgs&, cudaStream_t, int);

cudaError_t launch_spatial_fused(const SpatialArgs& a, int F, int nbuf, int lead, int* sync,
                                 int num_sms, cudaStream_t stream) {
    // R(k) waits for C(k - nbuf), which the queue must hold earlier: nbuf > lead >= 1
    if (lead < 1 || nbuf <= lead) return cudaErrorInvalidValue;
    const int L = a.W / 2;
#define DDMK_F(LEN, HLEN)                                                                   \
    if (L == LEN && a.H == HLEN)                                                            \
        return a.pixel_bytes == 2                                                           \
                   ? launch_fused_t<float, uint16_t, LEN, HLEN>(a, F, nbuf, lead, sync, num_sms, stream) \
                   : launch_fused_t<float, uint8_t, LEN, HLEN>(a, F, nbuf, lead, sync, num_sms, stream);
    DDMK_F(256, 512) DDMK_F(512, 1024) DDMK_F(128, 256)
#undef DDMK_F
    return cudaErrorNotSupported;
}

}  // namespace ddmk
