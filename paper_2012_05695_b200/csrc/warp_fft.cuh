// Warp-level, register-resident FFT building blocks (sm_100a).
//
// A length-L transform is owned by a group of A lanes (A divides 32) and held as B values per
// lane, L = A * B ("four-step" / Bailey factorisation):
//   input : lane a of the group holds x[a + A*b],            b in [0, B)
//   step 1: in-register DFT_B over b                     -> Y_a[c], c in [0, B)
//   step 2: twiddle Y_a[c] *= W_L^{a c}
//   step 3: one exchange through the group's shared-memory scratch ([c][a], pitch A+1)
//   step 4: in-register DFT_A over a, for each of the lane's B/A columns c = a + i*A
//   output: lane a holds X[(a + i*A) + B*d] at v[i*A + d],    i in [0, B/A), d in [0, A)
// One exchange per transform, no block barriers (only __syncwarp), conflict-free pitch.
// Twiddles of step 2 come from a per-lane cache of w^j (j < 8) and w^{8i} computed once
// with double-precision sincospi, so every twiddle is one complex product of two
// correctly-rounded values.
#pragma once

#include "fft_core.cuh"

namespace ddmk {

// ---------------------------------------------------------------- compile-time cos/sin
// cos/sin(2 pi k / n) evaluated at compile time (Taylor series after octant reduction).
__host__ __device__ constexpr double ct_poly_sin(double x) {
    double term = x, sum = x;
    for (int i = 1; i < 14; ++i) {
        term *= -x * x / ((2 * i) * (2 * i + 1));
        sum += term;
    }
    return sum;
}
__host__ __device__ constexpr double ct_poly_cos(double x) {
    double term = 1.0, sum = 1.0;
    for (int i = 1; i < 14; ++i) {
        term *= -x * x / ((2 * i - 1) * (2 * i));
        sum += term;
    }
    return sum;
}
// returns {cos, sin} of 2 pi k / n
struct CS {
    double c, s;
};
__host__ __device__ constexpr CS ct_cis(long k, long n) {
    k %= n;
    if (k < 0) k += n;
    // reduce to the first octant using exact rational symmetries
    const long n8 = 8 * k;  // angle in units of 2pi/(8n): octant = n8 / n
    const double pi = 3.141592653589793238462643383279502884;
    const int oct = (int)(n8 / n);
    // angle within the octant, measured so |theta| <= pi/4
    double c = 0, s = 0;
    // theta = 2 pi k / n; write theta = oct * pi/4 + r, r in [0, pi/4)
    const double r = 2.0 * pi * ((double)(8 * k - (long)oct * n) / (8.0 * (double)n));
    const double cr = ct_poly_cos(r), sr = ct_poly_sin(r);
    const double h = 0.70710678118654752440084436210484903928;
    // rotate (cr, sr) by oct * 45 degrees
    switch (oct) {
    case 0: c = cr; s = sr; break;
    case 1: c = h * (cr - sr); s = h * (cr + sr); break;
    case 2: c = -sr; s = cr; break;
    case 3: c = -h * (cr + sr); s = h * (cr - sr); break;
    case 4: c = -cr; s = -sr; break;
    case 5: c = -h * (cr - sr); s = -h * (cr + sr); break;
    case 6: c = sr; s = -cr; break;
    default: c = h * (cr + sr); s = -h * (cr - sr); break;
    }
    return {c, s};
}

// W_n^{e} = exp(SIGN 2 pi i e / n) as a compile-time complex of the working precision
template <int SIGN, typename S>
__device__ __forceinline__ constexpr cpx<S> ct_w(long e, long n) {
    const CS v = ct_cis(e, n);
    return {(S)v.c, (S)(SIGN < 0 ? -v.s : v.s)};
}

// ---------------------------------------------------------------- in-register DFT_R
// Dft<2,4,8,16> live in fft_core.cuh; composites R = R1 * R2 are built generically.
template <int R1, int R2, int SIGN, typename S>
__device__ __forceinline__ void dft_composite(cpx<S>* v) {
    constexpr int R = R1 * R2;
    cpx<S> y[R];
    // n = a + R1 b, k = c + R2 d : X[c + R2 d] = sum_a W_R1^{ad} W_R^{ac} sum_b x[a + R1 b] W_R2^{bc}
#pragma unroll
    for (int a = 0; a < R1; ++a) {
        cpx<S> col[R2];
#pragma unroll
        for (int b = 0; b < R2; ++b) col[b] = v[a + R1 * b];
        Dft<R2, SIGN, S>::run(col);
#pragma unroll
        for (int c = 0; c < R2; ++c) {
            cpx<S> t = col[c];
            if (a != 0 && c != 0) t = cmul(t, ct_w<SIGN, S>((long)a * c, R));
            y[a * R2 + c] = t;
        }
    }
#pragma unroll
    for (int c = 0; c < R2; ++c) {
        cpx<S> row[R1];
#pragma unroll
        for (int a = 0; a < R1; ++a) row[a] = y[a * R2 + c];
        Dft<R1, SIGN, S>::run(row);
#pragma unroll
        for (int d = 0; d < R1; ++d) v[c + R2 * d] = row[d];
    }
}

// DFT_32 as 4 x 8 with the inner twiddles fused into the row DFT_4's first butterflies:
// b0 = y0 + w2 y2 (FMA chains), b1 = 2 y0 - b0, p = w1 y1, b2 = p + w3 y3, b3 = 2 p - b2
// (24 instructions per row instead of 28; W_32^8 = SIGN i is a rotation).
// TW: the input is v[n] tw(n) with tw(n) = twf(n) (a functor; tw(0) = 1 is skipped), fused
// into the first butterflies of the column DFT_8s
template <int SIGN, typename S, bool TW = false, class Tw = int>
__device__ __forceinline__ void dft32_fused(cpx<S>* v, const Tw& twf = 0) {
    cpx<S> y[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int b = 0; b < 8; ++b) y[a][b] = v[a + 4 * b];
        if constexpr (TW) {
            // even b (n = a + 8 j) and odd b (n = a + 4 + 8 j) DFT_4s with the input twiddles
            if (a == 0)
                dft4_tw<SIGN>(y[a][0], y[a][2], y[a][4], y[a][6], twf(8), twf(16), twf(24));
            else
                dft4_tw<SIGN>(y[a][0], y[a][2], y[a][4], y[a][6], twf(a), twf(a + 8), twf(a + 16),
                              twf(a + 24));
            dft4_tw<SIGN>(y[a][1], y[a][3], y[a][5], y[a][7], twf(a + 4), twf(a + 12), twf(a + 20),
                          twf(a + 28));
            dft8_finish<SIGN>(y[a]);
        } else {
            Dft<8, SIGN, S>::run(y[a]);
        }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        cpx<S> b0, b1, b2, b3;
        if (c == 0) {
            b0 = cadd(y[0][0], y[2][0]);
            b1 = csub(y[0][0], y[2][0]);
            b2 = cadd(y[1][0], y[3][0]);
            b3 = csub(y[1][0], y[3][0]);
        } else {
            if (c == 4) {
                const cpx<S> t = rot90<SIGN>(y[2][c]);  // W_32^8
                b0 = cadd(y[0][c], t);
                b1 = csub(y[0][c], t);
            } else {
                b0 = cfma(ct_w<SIGN, S>(2 * c, 32), y[2][c], y[0][c]);
                b1 = creflect(y[0][c], b0);
            }
            const cpx<S> p = cmul(y[1][c], ct_w<SIGN, S>(c, 32));
            b2 = cfma(ct_w<SIGN, S>(3 * c, 32), y[3][c], p);
            b3 = creflect(p, b2);
        }
        b3 = rot90<SIGN>(b3);
        v[c] = cadd(b0, b2);
        v[c + 16] = csub(b0, b2);
        v[c + 8] = cadd(b1, b3);
        v[c + 24] = csub(b1, b3);
    }
}

template <int R, int SIGN, typename S>
struct RegDft {
    __device__ __forceinline__ static void run(cpx<S>* v) {
        if constexpr (R == 1) {
        } else if constexpr (R <= 16) {
            Dft<R, SIGN, S>::run(v);
        } else if constexpr (R == 32) {
            dft32_fused<SIGN, S>(v);
        } else if constexpr (R == 64) {
            dft_composite<8, 8, SIGN, S>(v);
        } else {
            static_assert(R <= 64, "register DFT too large");
        }
    }
};

// ---------------------------------------------------------------- per-lane twiddle cache
// w^c for c in [0, B) with w = exp(-2 pi i a / L), from lo[c % 8] * hi[c / 8].
template <int B, typename S>
struct LaneTw {
    static constexpr int NLO = B < 8 ? B : 8;
    static constexpr int NHI = B < 8 ? 1 : B / 8;
    cpx<S> lo[NLO];
    cpx<S> hi[NHI];

    __device__ __forceinline__ void init(int a, int L) {
#pragma unroll
        for (int j = 0; j < NLO; ++j) {
            double s, c;
            sincospi(-2.0 * (double)((long)a * j % L) / (double)L, &s, &c);
            lo[j] = {(S)c, (S)s};
        }
#pragma unroll
        for (int i = 0; i < NHI; ++i) {
            double s, c;
            sincospi(-2.0 * (double)((long)a * 8 * i % L) / (double)L, &s, &c);
            hi[i] = {(S)c, (S)s};
        }
    }
    // same values from a precomputed table tab[j] = exp(-2 pi i j / L) (global, L1-resident)
    __device__ __forceinline__ void init_from(const cpx<S>* __restrict__ tab, int a, int L) {
#pragma unroll
        for (int j = 0; j < NLO; ++j) lo[j] = tab[(a * j) % L];
#pragma unroll
        for (int i = 0; i < NHI; ++i) hi[i] = tab[(a * 8 * i) % L];
    }
    // forward-direction twiddle W_L^{a c}; SIGN > 0 conjugates
    template <int SIGN>
    __device__ __forceinline__ cpx<S> get(int c) const {
        cpx<S> w = (c < 8) ? lo[c % NLO] : cmul(lo[c % 8], hi[c / 8]);
        if (SIGN > 0) w.y = -w.y;
        return w;
    }
};

// ---------------------------------------------------------------- group FFT
// scratch: this group's region, B * (A + 1) complex. `a` = lane index within the group.
template <int A, int B, int SIGN, typename S>
__device__ __forceinline__ void group_fft(cpx<S> (&v)[B], cpx<S>* scratch, int a,
                                          const LaneTw<B, S>& tw) {
    static_assert(B % A == 0, "B must be a multiple of A");
    constexpr int P = A + 1;
    RegDft<B, SIGN, S>::run(v);
#pragma unroll
    for (int c = 1; c < B; ++c) v[c] = cmul(v[c], tw.template get<SIGN>(c));
#pragma unroll
    for (int c = 0; c < B; ++c) scratch[c * P + a] = v[c];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < B / A; ++i)
#pragma unroll
        for (int ap = 0; ap < A; ++ap) v[i * A + ap] = scratch[(a + i * A) * P + ap];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < B / A; ++i) RegDft<A, SIGN, S>::run(v + i * A);
}

}  // namespace ddmk
