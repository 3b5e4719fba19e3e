// Register/shared-memory FFT building blocks for the DDM kernels (sm_100a).
//
// All transforms are unnormalised DFTs, X[k] = sum_n x[n] exp(SIGN * 2 pi i n k / L),
// matching what the reference obtains from FFTW (`proj/core/src/fft.cpp:34-41`:
// FFTW_FORWARD = -1 for the spatial r2c and the temporal forward, +1 for the temporal
// backward). Passes are Stockham autosort (decimation in time): pass with radix R and
// running sub-length p reads x[i + r L/R], twiddles by W_{pR}^{r k} (k = i mod p), does an
// in-register R-point DFT and writes y[(i-k) R + k + r p]; after all passes the data are in
// natural order.  Twiddles come from a per-length table tw[j] = exp(-2 pi i j / L) built in
// double on the host and rounded once to the working precision (as FFTW does).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ddmk {

template <typename S>
struct alignas(2 * sizeof(S)) cpx {
    S x, y;
};

// ---------------------------------------------------------------- packed f32x2 (sm_100a)
// Blackwell issues two f32 lanes per instruction with FADD2 / FMUL2 / FFMA2 (PTX add/sub/
// mul/fma.rn.f32x2 on a 64-bit register pair). A complex<float> is exactly such a pair, and
// ptxas folds the FFT's operand shuffles into the instruction's source modifiers: a broadcast
// of one half (`R.F32`), the swap (`.LO_HI`), the one-half negation (`.NP`, the quarter-turn
// (-y, x)) and a broadcast immediate. So an add or subtract is one instruction instead of two,
// a product by a constant or runtime twiddle two instead of four, a + w b two instead of
// four. Every FFT kernel (spatial, temporal, long) is issue-bound on these, and the roundings
// are the same fused single-precision operations as the scalar forms. DDM_F32X2=0 restores
// the scalar code.
#ifndef DDM_F32X2
#define DDM_F32X2 1
#endif
namespace px {
using u64 = unsigned long long;
__device__ __forceinline__ u64 pk(float x, float y) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ cpx<float> up(u64 r) {
    cpx<float> a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
}  // namespace px

#ifndef DDM_F32X2_ADD
#define DDM_F32X2_ADD DDM_F32X2
#endif
#ifndef DDM_F32X2_MUL
#define DDM_F32X2_MUL DDM_F32X2
#endif
// kPacked: products (cmul, cfma, caxpy); kPackedAdd: sums (cadd, csub, creflect)
template <typename S>
constexpr bool kPacked = DDM_F32X2_MUL && sizeof(S) == 4;
template <typename S>
constexpr bool kPackedAdd = DDM_F32X2_ADD && sizeof(S) == 4;

template <typename S>
__device__ __forceinline__ cpx<S> cmul(cpx<S> a, cpx<S> b) {
    if constexpr (kPacked<S>) {   // b.x (a.x, a.y) + b.y (-a.y, a.x)
        using namespace px;
        return up(fma2(pk(-a.y, a.x), pk(b.y, b.y), mul2(pk(b.x, b.x), pk(a.x, a.y))));
    } else {
        return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
    }
}
// a + w b as two fused multiply-add chains (4 FMA instead of cmul's 4 plus 2 adds)
template <typename S>
__device__ __forceinline__ cpx<S> cfma(cpx<S> w, cpx<S> b, cpx<S> a) {
    if constexpr (kPacked<S>) {   // a + w.x (b.x, b.y) + w.y (-b.y, b.x)
        using namespace px;
        return up(fma2(pk(-b.y, b.x), pk(w.y, w.y), fma2(pk(w.x, w.x), pk(b.x, b.y), pk(a.x, a.y))));
    } else {
        return {fma(w.x, b.x, fma(-w.y, b.y, a.x)), fma(w.x, b.y, fma(w.y, b.x, a.y))};
    }
}
// 2 a - t: the other butterfly output once t = a + u is known (a - u, 2 FMA)
template <typename S>
__device__ __forceinline__ cpx<S> creflect(cpx<S> a, cpx<S> t) {
    if constexpr (kPackedAdd<S>) {
        using namespace px;
        return up(fma2(pk(a.x, a.y), pk(2.f, 2.f), pk(-t.x, -t.y)));
    } else {
        return {fma(S(2), a.x, -t.x), fma(S(2), a.y, -t.y)};
    }
}
template <typename S>
__device__ __forceinline__ cpx<S> cadd(cpx<S> a, cpx<S> b) {
    if constexpr (kPackedAdd<S>) return px::up(px::add2(px::pk(a.x, a.y), px::pk(b.x, b.y)));
    else return {a.x + b.x, a.y + b.y};
}
template <typename S>
__device__ __forceinline__ cpx<S> csub(cpx<S> a, cpx<S> b) {
    if constexpr (kPackedAdd<S>) return px::up(px::sub2(px::pk(a.x, a.y), px::pk(b.x, b.y)));
    else return {a.x - b.x, a.y - b.y};
}
// s a + b (real s)
template <typename S>
__device__ __forceinline__ cpx<S> caxpy(S s, cpx<S> a, cpx<S> b) {
    if constexpr (kPacked<S>) return px::up(px::fma2(px::pk(s, s), px::pk(a.x, a.y), px::pk(b.x, b.y)));
    else return {fma(s, a.x, b.x), fma(s, a.y, b.y)};
}
// multiply by SIGN * i  (the quarter-turn of the transform direction)
template <int SIGN, typename S>
__device__ __forceinline__ cpx<S> rot90(cpx<S> a) {
    return SIGN < 0 ? cpx<S>{a.y, -a.x} : cpx<S>{-a.y, a.x};
}
// twiddle from the forward table; conjugate for the backward direction
template <int SIGN, typename S>
__device__ __forceinline__ cpx<S> twiddle(const cpx<S>* __restrict__ tw, int j) {
    cpx<S> w = tw[j];
    if (SIGN > 0) w.y = -w.y;
    return w;
}

template <typename S>
struct consts;
template <>
struct consts<float> {
    static constexpr float r2 = 0.70710678118654752440f;
    static constexpr float c16_1 = 0.92387953251128675613f;  // cos(pi/8)
    static constexpr float s16_1 = 0.38268343236508977173f;  // sin(pi/8)
    static constexpr float c3 = -0.5f;
    static constexpr float s3 = 0.86602540378443864676f;
    static constexpr float c5_1 = 0.30901699437494742410f;   // cos(2pi/5)
    static constexpr float c5_2 = -0.80901699437494742410f;  // cos(4pi/5)
    static constexpr float s5_1 = 0.95105651629515357212f;   // sin(2pi/5)
    static constexpr float s5_2 = 0.58778525229247312917f;   // sin(4pi/5)
};
template <>
struct consts<double> {
    static constexpr double r2 = 0.70710678118654752440;
    static constexpr double c16_1 = 0.92387953251128675613;
    static constexpr double s16_1 = 0.38268343236508977173;
    static constexpr double c3 = -0.5;
    static constexpr double s3 = 0.86602540378443864676;
    static constexpr double c5_1 = 0.30901699437494742410;
    static constexpr double c5_2 = -0.80901699437494742410;
    static constexpr double s5_1 = 0.95105651629515357212;
    static constexpr double s5_2 = 0.58778525229247312917;
};

// ---------------------------------------------------------------- in-register DFTs

template <int SIGN, typename S>
__device__ __forceinline__ void dft2(cpx<S>& a, cpx<S>& b) {
    const cpx<S> t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <int SIGN, typename S>
__device__ __forceinline__ void dft4(cpx<S>& a0, cpx<S>& a1, cpx<S>& a2, cpx<S>& a3) {
    const cpx<S> b0 = cadd(a0, a2), b1 = csub(a0, a2);
    const cpx<S> b2 = cadd(a1, a3), b3 = rot90<SIGN>(csub(a1, a3));
    a0 = cadd(b0, b2);
    a2 = csub(b0, b2);
    a1 = cadd(b1, b3);
    a3 = csub(b1, b3);
}

// v[r] <- sum_s v[s] W_R^{r s}, W_R = exp(SIGN 2 pi i / R)
template <int R, int SIGN, typename S>
struct Dft;

template <int SIGN, typename S>
struct Dft<1, SIGN, S> {
    __device__ __forceinline__ static void run(cpx<S>*) {}
};

template <int SIGN, typename S>
struct Dft<2, SIGN, S> {
    __device__ __forceinline__ static void run(cpx<S>* v) { dft2<SIGN>(v[0], v[1]); }
};

template <int SIGN, typename S>
struct Dft<4, SIGN, S> {
    __device__ __forceinline__ static void run(cpx<S>* v) { dft4<SIGN>(v[0], v[1], v[2], v[3]); }
};

// DFT_4 of (a0, t1 a1, t2 a2, t3 a3) with the twiddles fused into the first butterflies
// (a0 untwiddled): 20 instructions instead of 24
template <int SIGN, typename S>
__device__ __forceinline__ void dft4_tw(cpx<S>& a0, cpx<S>& a1, cpx<S>& a2, cpx<S>& a3, cpx<S> t1,
                                        cpx<S> t2, cpx<S> t3) {
    const cpx<S> b0 = cfma(t2, a2, a0), b1 = creflect(a0, b0);
    const cpx<S> p = cmul(a1, t1);
    const cpx<S> b2 = cfma(t3, a3, p), b3 = rot90<SIGN>(creflect(p, b2));
    a0 = cadd(b0, b2);
    a2 = csub(b0, b2);
    a1 = cadd(b1, b3);
    a3 = csub(b1, b3);
}
// same with a0 twiddled too
template <int SIGN, typename S>
__device__ __forceinline__ void dft4_tw(cpx<S>& a0, cpx<S>& a1, cpx<S>& a2, cpx<S>& a3, cpx<S> t0,
                                        cpx<S> t1, cpx<S> t2, cpx<S> t3) {
    const cpx<S> p0 = cmul(a0, t0);
    const cpx<S> b0 = cfma(t2, a2, p0), b1 = creflect(p0, b0);
    const cpx<S> p = cmul(a1, t1);
    const cpx<S> b2 = cfma(t3, a3, p), b3 = rot90<SIGN>(creflect(p, b2));
    a0 = cadd(b0, b2);
    a2 = csub(b0, b2);
    a1 = cadd(b1, b3);
    a3 = csub(b1, b3);
}

// second half of DFT_8 once the even (v0, v2, v4, v6) and odd (v1, v3, v5, v7) DFT_4s are done
template <int SIGN, typename S>
__device__ __forceinline__ void dft8_finish(cpx<S>* v);

template <int SIGN, typename S>
struct Dft<8, SIGN, S> {
    __device__ __forceinline__ static void run(cpx<S>* v) {
        // radix-2 x radix-4 split: even/odd halves, then twiddles W8^k
        dft4<SIGN>(v[0], v[2], v[4], v[6]);
        dft4<SIGN>(v[1], v[3], v[5], v[7]);
        dft8_finish<SIGN>(v);
    }
};

template <int SIGN, typename S>
__device__ __forceinline__ void dft8_finish(cpx<S>* v) {
    {
        const S r = consts<S>::r2;
        // W8^1 = (1 + SIGN i)/sqrt2, W8^2 = SIGN i, W8^3 = (-1 + SIGN i)/sqrt2; the sqrt2
        // scalings are fused into the output butterflies: E +- r (O.x -+ ...) as FMAs
        const cpx<S> e1 = v[2], o1 = v[3], e3 = v[6], o3 = v[7];
        // W8^1 O / r  and  W8^3 O / r
        // u1 = o1 + rot(o1), u3 = rot(o3) - o3 (rot = the SIGN quarter-turn)
        const cpx<S> u1 = cadd(o1, rot90<SIGN>(o1));
        const cpx<S> u3 = csub(rot90<SIGN>(o3), o3);
        v[5] = rot90<SIGN>(v[5]);
        cpx<S> o[8];
        o[0] = cadd(v[0], v[1]);
        o[4] = csub(v[0], v[1]);
        o[1] = caxpy(r, u1, e1);
        o[5] = caxpy(-r, u1, e1);
        o[2] = cadd(v[4], v[5]);
        o[6] = csub(v[4], v[5]);
        o[3] = caxpy(r, u3, e3);
        o[7] = caxpy(-r, u3, e3);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = o[i];
    }
}

template <int SIGN, typename S>
struct Dft<16, SIGN, S> {
    __device__ __forceinline__ static void run(cpx<S>* v) {
        // 4 x 4: column DFT-4 over stride-4 groups, twiddle W16^{r s}, row DFT-4
#pragma unroll
        for (int s = 0; s < 4; ++s) dft4<SIGN>(v[s], v[s + 4], v[s + 8], v[s + 12]);
        // v[s + 4 r] now holds sub-DFT r of column s; twiddle by W16^{r s}
        const S c1 = consts<S>::c16_1, s1 = consts<S>::s16_1, r2 = consts<S>::r2;
        const S sg = SIGN < 0 ? S(-1) : S(1);
        const cpx<S> w1 = {c1, sg * s1}, w2 = {r2, sg * r2}, w3 = {s1, sg * c1};
        v[5] = cmul(v[5], w1);
        v[6] = cmul(v[6], w2);
        v[7] = cmul(v[7], w3);
        v[9] = cmul(v[9], w2);
        v[10] = rot90<SIGN>(v[10]);
        v[11] = cmul(v[11], cpx<S>{-r2, sg * r2});
        v[13] = cmul(v[13], w3);
        v[14] = cmul(v[14], cpx<S>{-r2, sg * r2});
        v[15] = cmul(v[15], cpx<S>{-c1, -sg * s1});
#pragma unroll
        for (int r = 0; r < 4; ++r) dft4<SIGN>(v[4 * r], v[4 * r + 1], v[4 * r + 2], v[4 * r + 3]);
        // output index k = r + 4 t sits at v[4 r + t]; transpose to natural order
        cpx<S> o[16];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int t = 0; t < 4; ++t) o[r + 4 * t] = v[4 * r + t];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = o[i];
    }
};

template <int SIGN, typename S>
struct Dft<3, SIGN, S> {
    __device__ __forceinline__ static void run(cpx<S>* v) {
        const S c = consts<S>::c3, s = (SIGN < 0 ? -consts<S>::s3 : consts<S>::s3);
        const cpx<S> a = cadd(v[1], v[2]), b = csub(v[1], v[2]);
        const cpx<S> m = {v[0].x + c * a.x, v[0].y + c * a.y};
        const cpx<S> j = {-s * b.y, s * b.x};  // i * s * b
        v[0] = cadd(v[0], a);
        v[1] = cadd(m, j);
        v[2] = csub(m, j);
    }
};

template <int SIGN, typename S>
struct Dft<5, SIGN, S> {
    __device__ __forceinline__ static void run(cpx<S>* v) {
        const S c1 = consts<S>::c5_1, c2 = consts<S>::c5_2;
        const S s1 = SIGN < 0 ? -consts<S>::s5_1 : consts<S>::s5_1;
        const S s2 = SIGN < 0 ? -consts<S>::s5_2 : consts<S>::s5_2;
        const cpx<S> a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
        const cpx<S> a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
        const cpx<S> m1 = {v[0].x + c1 * a1.x + c2 * a2.x, v[0].y + c1 * a1.y + c2 * a2.y};
        const cpx<S> m2 = {v[0].x + c2 * a1.x + c1 * a2.x, v[0].y + c2 * a1.y + c1 * a2.y};
        // i * (s1 b1 + s2 b2) and i * (s2 b1 - s1 b2)
        const cpx<S> n1 = {-(s1 * b1.y + s2 * b2.y), s1 * b1.x + s2 * b2.x};
        const cpx<S> n2 = {-(s2 * b1.y - s1 * b2.y), s2 * b1.x - s1 * b2.x};
        v[0] = cadd(v[0], cadd(a1, a2));
        v[1] = cadd(m1, n1);
        v[4] = csub(m1, n1);
        v[2] = cadd(m2, n2);
        v[3] = csub(m2, n2);
    }
};

// ---------------------------------------------------------------- plans

// A length-L transform split into passes of radix {2,3,4,5,8,16}; L == 1 has no passes.
// Lengths with other prime factors are flagged `naive` and use a direct O(L^2) sum.
struct FftPlan {
    int len = 1;
    int npass = 0;
    uint64_t radices = 0;  // 4 bits per pass, pass s at bits [4s, 4s+4): radix value - 1
    bool naive = false;
    __host__ __device__ int radix(int s) const { return (int)((radices >> (4 * s)) & 15) + 1; }
    __host__ void push(int r) { radices |= (uint64_t)(r - 1) << (4 * npass++); }
};

// ---------------------------------------------------------------- shared-memory passes
//
// `nbatch` independent transforms of length L live in shared memory at buf + b*stride.
// Each pass is done in place: every thread first pulls all the butterflies it owns into
// registers, the block synchronises, then the outputs are written back. MAXB bounds the
// butterflies per thread per pass (checked by the launcher).

template <int R, int SIGN, int MAXB, typename S>
__device__ __forceinline__ void smem_pass(cpx<S>* buf, int stride, int nbatch, int L, int p,
                          const cpx<S>* __restrict__ tw) {
    const int nb = L / R;               // butterflies per transform
    const int total = nb * nbatch;
    const int twstep = L / (p * R);      // W_{pR}^{rk} = tw[r k twstep]
    cpx<S> v[MAXB][R];
#pragma unroll
    for (int u = 0; u < MAXB; ++u) {
        const int item = threadIdx.x + u * blockDim.x;
        if (item < total) {
            const int b = item / nb, i = item - b * nb;
            const cpx<S>* src = buf + b * stride;
            const int k = i % p;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                cpx<S> x = src[i + r * nb];
                if (r > 0 && k > 0) x = cmul(x, twiddle<SIGN>(tw, r * k * twstep));
                v[u][r] = x;
            }
            Dft<R, SIGN, S>::run(v[u]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < MAXB; ++u) {
        const int item = threadIdx.x + u * blockDim.x;
        if (item < total) {
            const int b = item / nb, i = item - b * nb;
            cpx<S>* dst = buf + b * stride;
            const int k = i % p;
            const int base = (i - k) * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) dst[base + r * p] = v[u][r];
        }
    }
    __syncthreads();
}

// Direct O(L^2) DFT in place (lengths with prime factors > 5); scratch holds nbatch*L.
template <int SIGN, typename S>
__device__ __noinline__ void smem_naive(cpx<S>* buf, int stride, int nbatch, int L, cpx<S>* scratch,
                           const cpx<S>* __restrict__ tw) {
    const int total = L * nbatch;
    for (int item = threadIdx.x; item < total; item += blockDim.x) {
        const int b = item / L, k = item - b * L;
        const cpx<S>* src = buf + b * stride;
        // accumulate in double for either precision: this path is for rare odd lengths
        double ax = 0.0, ay = 0.0;
        int j = 0;
        for (int n = 0; n < L; ++n) {
            const cpx<S> w = twiddle<SIGN>(tw, j);
            const cpx<S> x = src[n];
            ax += (double)x.x * (double)w.x - (double)x.y * (double)w.y;
            ay += (double)x.x * (double)w.y + (double)x.y * (double)w.x;
            j += k;
            if (j >= L) j -= L;
        }
        scratch[item] = {(S)ax, (S)ay};
    }
    __syncthreads();
    for (int item = threadIdx.x; item < total; item += blockDim.x) {
        const int b = item / L, k = item - b * L;
        buf[b * stride + k] = scratch[item];
    }
    __syncthreads();
}

template <int R, int SIGN, int MAXB, typename S>
__device__ __noinline__ void smem_pass_ool(cpx<S>* buf, int stride, int nbatch, int L, int p,
                                           const cpx<S>* __restrict__ tw) {
    smem_pass<R, SIGN, MAXB>(buf, stride, nbatch, L, p, tw);
}

// Runtime plan (rare lengths): radix 4/2/3/5 passes, each an out-of-line call.
template <int SIGN, typename S>
__device__ void smem_fft_rt(cpx<S>* buf, int stride, int nbatch, const FftPlan& plan,
                            const cpx<S>* __restrict__ tw, cpx<S>* scratch) {
    if (plan.naive || plan.npass == 0) {
        if (plan.naive) smem_naive<SIGN>(buf, stride, nbatch, plan.len, scratch, tw);
        return;
    }
    int p = 1;
    for (int s = 0; s < plan.npass; ++s) {
        const int R = plan.radix(s);
        if (R == 2) smem_pass_ool<2, SIGN, 16>(buf, stride, nbatch, plan.len, p, tw);
        else if (R == 3) smem_pass_ool<3, SIGN, 12>(buf, stride, nbatch, plan.len, p, tw);
        else if (R == 5) smem_pass_ool<5, SIGN, 8>(buf, stride, nbatch, plan.len, p, tw);
        else smem_pass_ool<4, SIGN, 8>(buf, stride, nbatch, plan.len, p, tw);
        p *= R;
    }
}

// Runtime plan for smem_fft_rt: radix 4 first, then 2, 5, 3; capacity 2048 points per CTA
// at 256 threads (8 radix-4 butterflies per thread).
inline FftPlan make_rt_plan(int len) {
    FftPlan p;
    p.len = len;
    int rest = len;
    while (rest % 4 == 0) { p.push(4); rest /= 4; }
    while (rest % 2 == 0) { p.push(2); rest /= 2; }
    while (rest % 5 == 0) { p.push(5); rest /= 5; }
    while (rest % 3 == 0) { p.push(3); rest /= 3; }
    if (rest != 1) {
        p.npass = 0;
        p.radices = 0;
        p.naive = true;
    }
    return p;
}

// ---------------------------------------------------------------- compile-time plans
//
// Radix choice for the remaining length `rem` of a transform: balanced power-of-two radices
// (2^11 = 16*16*8, 2^9 = 8*8*8, ...), 5 before 4/2 for 5-smooth lengths.
__host__ __device__ constexpr int ct_radix(int rem) {
    if (rem % 5 == 0) return 5;
    if (rem % 3 == 0 && (rem & (rem - 1)) != 0 && rem % 2 != 0) return 3;
    if ((rem & (rem - 1)) == 0) {
        int e = 0;
        while ((1 << e) < rem) ++e;
        if (e <= 4) return rem;          // 2, 4, 8, 16 in one pass
        if (e % 4 == 0) return 16;
        if (e % 3 == 0) return 8;
        if (e == 5) return 8;            // 8 * 4
        if (e == 7) return 16;           // 16 * 8
        if (e == 10) return 16;          // 16 * 8 * 8
        if (e == 11) return 16;          // 16 * 16 * 8
        if (e == 13) return 16;          // 16 * 16 * 32 -> 16 * 16 * 8 * 4
        if (e == 14) return 16;
        return 16;
    }
    if (rem % 16 == 0) return 16;
    if (rem % 8 == 0) return 8;
    if (rem % 4 == 0) return 4;
    if (rem % 2 == 0) return 2;
    if (rem % 3 == 0) return 3;
    return 0;  // unsupported prime factor
}

__host__ __device__ constexpr bool ct_supported(int len) {
    int rem = len;
    while (rem > 1) {
        const int r = ct_radix(rem);
        if (r == 0 || rem % r != 0) return false;
        rem /= r;
    }
    return true;
}

// Passes of a length-L transform, p = product of radices already applied. MAXB16 is the
// butterfly budget per thread counted in radix-16 units (scaled up for smaller radices).
template <int L, int P, int SIGN, int MAXB16, typename S>
__device__ __forceinline__ void smem_fft_ct(cpx<S>* buf, int stride, int nbatch,
                                            const cpx<S>* __restrict__ tw) {
    if constexpr (P < L) {
        constexpr int R = ct_radix(L / P);
        static_assert(R > 0, "unsupported transform length");
        constexpr int MB = (MAXB16 * 16 + R - 1) / R;
        smem_pass<R, SIGN, MB>(buf, stride, nbatch, L, P, tw);
        smem_fft_ct<L, P * R, SIGN, MAXB16, S>(buf, stride, nbatch, tw);
    }
}

}  // namespace ddmk

// Dispatch a runtime transform length onto a compile-time instantiation: FN<L>(args...) for
// the lengths below, `fallback` otherwise.
#define DDMK_LENGTH_CASES(X)                                                                  \
    X(1) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192) \
    X(5) X(10) X(20) X(25) X(40) X(50) X(100) X(125) X(200) X(250) X(500) X(1000)
