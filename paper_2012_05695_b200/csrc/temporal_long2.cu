// Long-sequence temporal engine, balanced (sm_100a): two independent warp groups per CTA,
// each transforming its own wave vector with G = R/2 warps (N2 = 1024 R; R = 4 for the
// 1024^2 x 2048 case, R = 8 for 2048^2 x 4096). Same arithmetic as temporal_long.cu — the
// forward FFT_N2 of the zero-padded sequence as R FFT_1024s on W_N2^{n' r}-twisted,
// W_R-combined chunks, |X|^2 in f32, the half-length real-input inverse as R/2 FFT_1024s
// combined by an R/2-point DFT, the reference's unfold and combine — with the work split so
// every warp does the same share: forward transforms r = w and r = w + G, inverse transform
// s = w. (The one-group engine runs R/2 of its warps idle through the inverse.)
//
// Per group, per sequence (group-local named barriers; the other group is never waited on):
//   TMA bulk copy of t -> stage; mean; shift written back; 2 x (build y_r, FFT_1024, P_r -> pu)
//   |t|^2 -> scratch (natural order), suffix sums S(m) -> stage (t is dead)
//   inverse: E_w = IFFT_1024(P_2w + i P_2w+1), twisted, written over P_2w / P_2w+1 in place
//   U(m' + 1024 p) = sum_s E'_s(m') e^{2 pi i s p / H}, in place; unfold; d(m) -> out
// Map mode writes the q-major staging block (transposed lag-major by the host side), ring
// mode adds d into its item's f64 partial row in global memory (one owner thread per m, the
// item's sequences in order: deterministic).
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "temporal_common.cuh"
#include "warp_fft.cuh"

namespace ddmk {

namespace {

using namespace tc;

constexpr int kF2 = 1024;

__device__ __forceinline__ int pad32b(int n) { return n + (n >> 5); }

__device__ __forceinline__ void group_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int R>
struct Geom2 {
    static constexpr int N2 = kF2 * R, L = N2 / 2, NMAX = L, H = R / 2, G = R / 2;
    static constexpr int TG = 32 * G;                      // threads per group
    static constexpr size_t stage = (size_t)NMAX * 8;      // t, then S(m) (floats, pad32b)
    static constexpr size_t pu = (size_t)L * 8;            // P (floats), then E' / U (complex)
    static constexpr size_t scratch = (size_t)G * kXS * 8; // FFT exchange; |t|^2 in between
    static constexpr size_t red = 32 * 8;
    static constexpr size_t group = stage + pu + scratch + red + 16;
    static constexpr size_t shared_tabs = (size_t)kXS * 8 + (size_t)R * 32 * 8 * 2 + (size_t)R * H * 8 +
                                          (size_t)H * 32 * 8;
    static constexpr size_t total = 2 * group + shared_tabs;
    static_assert((size_t)(NMAX + NMAX / 32) * 4 <= scratch, "|t|^2 must fit the exchange area");
};

template <int R, bool kRing, bool FULL>
__global__ void __launch_bounds__(64 * (R / 2), (R == 4 ? 2 : 1))
temporal_long2_kernel(const cpx<float>* __restrict__ spec, const __grid_constant__ SegTable segs,
                      int N_rt, int64_t q0, int64_t q1, float* __restrict__ out_q,
                      const __grid_constant__ RingArgs ring) {
    using G2 = Geom2<R>;
    constexpr int TG = G2::TG, H = G2::H, G = G2::G;
    const int N = FULL ? G2::NMAX : N_rt;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int grp = warp / G, w = warp % G, gtid = tid - grp * TG;

    // shared tables (after both group regions)
    unsigned char* tabs = smem + 2 * G2::group;
    cpx<float>* tw_even = reinterpret_cast<cpx<float>*>(tabs);
    cpx<float>* tw_pre = tw_even + kXS;            // [r][b]  W_N2^{32 b r}
    cpx<float>* tw_lane = tw_pre + R * 32;         // [r][l]  W_N2^{l r}
    cpx<float>* wj_tab = tw_lane + R * 32;         // [r][j]  W_R^{j r}
    cpx<float>* comb_d = wj_tab + R * H;           // [s][d]  e^{+2 pi i 32 s d / L}
    fill_fft1024_tables(tw_even, nullptr, tid, blockDim.x);
    for (int i = tid; i < R * 32; i += blockDim.x) {
        const int r = i >> 5, b = i & 31;
        double sn, cs;
        sincospi(-2.0 * (double)(32 * b * r) / G2::N2, &sn, &cs);
        tw_pre[i] = {(float)cs, (float)sn};
        sincospi(-2.0 * (double)(b * r) / G2::N2, &sn, &cs);
        tw_lane[i] = {(float)cs, (float)sn};
        if (r < H) {
            sincospi(2.0 * (double)(32 * r * b) / G2::L, &sn, &cs);
            comb_d[i] = {(float)cs, (float)sn};
        }
    }
    for (int i = tid; i < R * H; i += blockDim.x) {
        const int r = i / H, j = i % H;
        double sn, cs;
        sincospi(-2.0 * (double)((j * r) % R) / R, &sn, &cs);
        wj_tab[i] = {(float)cs, (float)sn};
    }

    // this group's region
    unsigned char* gbase = smem + grp * G2::group;
    cpx<float>* stage = reinterpret_cast<cpx<float>*>(gbase);
    float* sS = reinterpret_cast<float*>(gbase);                       // S(m) after the forward
    float* pf = reinterpret_cast<float*>(gbase + G2::stage);           // P_r[k'] at pf[r*1024+k']
    cpx<float>* pu = reinterpret_cast<cpx<float>*>(gbase + G2::stage); // E'_s / U
    cpx<float>* scratch = reinterpret_cast<cpx<float>*>(gbase + G2::stage + G2::pu);
    float* pw = reinterpret_cast<float*>(scratch);                     // |t|^2 between FFTs
    double* red = reinterpret_cast<double*>(gbase + G2::stage + G2::pu + G2::scratch);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(red + 32);
    cpx<float>* my_scratch = scratch + w * kXS;
    const int bid = 1 + grp;                                           // named barrier id

    if (gtid == 0) {
        mbar_init(bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cpx<float> comb_lane, unf_base;
    {
        double sn, cs;
        sincospi(2.0 * (double)(w * lane) / G2::L, &sn, &cs);
        comb_lane = {(float)cs, (float)sn};
        sincospi(2.0 * (double)gtid / G2::N2, &sn, &cs);
        unf_base = {(float)cs, (float)sn};
    }
    __syncthreads();

    // ---- work list of this group
    const int64_t gg = (int64_t)blockIdx.x * 2 + grp, ngroups = (int64_t)gridDim.x * 2;
    int64_t item = gg, idx = -1;   // ring cursor: slot index into ring.order
    auto ring_first = [&](int64_t it, int64_t& it_out, int64_t& i_out) {
        for (it_out = it; it_out < ring.nitems; it_out += ngroups)
            if (ring.item_off[it_out] < ring.item_off[it_out + 1]) {
                i_out = ring.item_off[it_out];
                return;
            }
        i_out = -1;
    };
    const uint32_t bytes = (uint32_t)N * 8u;
    auto prefetch = [&](int64_t q) {
        if (q < 0 || gtid != 0) return;
        if (segs.count == 0) {
            bulk_load(stage, spec + q * (int64_t)N, bytes, bar);
        } else {
            fence_expect(bar, bytes);
            for (int s = 0; s < segs.count; ++s)
                bulk_copy(stage + segs.off[s], spec + segs.base[s] + q * (int64_t)segs.n[s],
                          (uint32_t)segs.n[s] * 8u, bar);
        }
    };
    int64_t q;
    if (kRing) {
        ring_first(gg, item, idx);
        q = idx >= 0 ? ring.order[idx] : -1;
    } else {
        q = q0 + gg < q1 ? q0 + gg : -1;
    }
    prefetch(q);
    uint32_t phase = 0u;
    const float inv_nf = 1.0f / (float)N;
    constexpr float inv_n2 = 1.0f / (float)G2::N2;

    while (q >= 0) {
        int64_t qn, n_item = item, n_idx = idx;
        bool first_of_item = false;
        if (kRing) {
            first_of_item = (idx == ring.item_off[item]);
            n_idx = idx + 1;
            if (n_idx >= ring.item_off[item + 1]) ring_first(item + ngroups, n_item, n_idx);
            qn = n_idx >= 0 ? ring.order[n_idx] : -1;
        } else {
            qn = q + ngroups < q1 ? q + ngroups : -1;
        }
        // wait for the copy; back off between polls so a waiting group leaves the issue slots
        // to the other group of the SM
        {
            uint32_t ok = 0;
            while (true) {
                asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                             : "=r"(ok)
                             : "r"(smem_addr(bar)), "r"(phase)
                             : "memory");
                if (ok) break;
                __nanosleep(64);
            }
        }
        phase ^= 1u;

        // ---- mean (f32, fixed order)
        {
            float sx = 0.f, sy = 0.f;
            for (int n = gtid; n < N; n += TG) {
                sx += stage[n].x;
                sy += stage[n].y;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sx += __shfl_xor_sync(0xffffffffu, sx, o);
                sy += __shfl_xor_sync(0xffffffffu, sy, o);
            }
            if (lane == 0) {
                red[2 * w] = sx;
                red[2 * w + 1] = sy;
            }
        }
        group_bar(bid, TG);
        float mx = 0.f, my = 0.f;
#pragma unroll
        for (int k = 0; k < G; ++k) {
            mx += (float)red[2 * k];
            my += (float)red[2 * k + 1];
        }
        mx *= inv_nf;
        my *= inv_nf;
        // shift once and write t back: the forward transforms and |t|^2 read it shifted
        for (int n = gtid; n < N; n += TG) {
            const cpx<float> x = stage[n];
            stage[n] = {x.x - mx, x.y - my};
        }
        group_bar(bid, TG);

        // ---- forward: this warp's two residues r = w and r = w + G
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
            const int r = w + G * half;
            // sum_j t[n1 + 1024 j] W_R^{j r}: W_4^r = (-i)^r is a swap and two signs (warp-
            // uniform), so R = 4 needs no complex product and R = 8 one:
            // (t0 + W_4^r t2) + W_8^r (t1 + W_4^r t3)
            const bool sw = r & 1;
            const float sa = (r & 2) ? -1.f : 1.f, sb = ((r + 1) & 2) ? -1.f : 1.f;
            auto rot_add = [&](cpx<float> base, cpx<float> t) {   // base + W_4^r t
                return cpx<float>{fmaf(sa, sw ? t.y : t.x, base.x), fmaf(sb, sw ? t.x : t.y, base.y)};
            };
            const cpx<float> w8 = wj_tab[r * H + (H > 1 ? 1 : 0)];
            const cpx<float> tl = tw_lane[r * 32 + lane];
            auto tap = [&](int n) -> cpx<float> {
                return (FULL || n < N) ? stage[n] : cpx<float>{0.f, 0.f};
            };
            cpx<float> v[32];
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                const int n1 = lane + 32 * b;
                cpx<float> a;
                if constexpr (H == 2) {
                    a = rot_add(tap(n1), tap(n1 + kF2));
                } else {
                    static_assert(H == 4, "R = 4 or 8");
                    const cpx<float> A = rot_add(tap(n1), tap(n1 + 2 * kF2));
                    const cpx<float> B = rot_add(tap(n1 + kF2), tap(n1 + 3 * kF2));
                    a = cfma(w8, B, A);
                }
                v[b] = cmul(cmul(a, tl), tw_pre[r * 32 + b]);
            }
            fft1024<-1, false>(v, my_scratch, lane, tw_even);
#pragma unroll
            for (int d = 0; d < 32; ++d) pf[r * kF2 + lane + 32 * d] = v[d].x * v[d].x + v[d].y * v[d].y;
        }

        // ---- |t|^2 in natural order into the exchange area, once every warp's transforms
        //      are done with it
        group_bar(bid, TG);
        for (int n = gtid; n < G2::NMAX; n += TG) {
            float p = 0.f;
            if (FULL || n < N) {
                const cpx<float> x = stage[n];
                p = x.x * x.x + x.y * x.y;
            }
            pw[pad32b(n)] = p;
        }
        group_bar(bid, TG);   // P complete; |t|^2 complete; t no longer read

        // ---- S(m) = sum_{n >= m} (p_n + p_{N-1-n}): thread u scans n = 32 u + j
        {
            float qv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = 32 * gtid + j;
                qv[j] = (n < N) ? pw[pad32b(n)] + pw[pad32b(N - 1 - n)] : 0.f;
            }
            float rr = 0.f;
#pragma unroll
            for (int j = 31; j >= 0; --j) {
                rr += qv[j];
                qv[j] = rr;
            }
            double incl = (double)rr;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_down_sync(0xffffffffu, incl, o);
                if (lane + o < 32) incl += t;
            }
            if (lane == 0) red[16 + w] = incl;
            group_bar(bid, TG);
            double later = 0.0;
            for (int k = w + 1; k < G; ++k) later += red[16 + k];
            const float base = (float)(incl - (double)rr + later);
#pragma unroll
            for (int j = 0; j < 32; ++j) sS[pad32b(32 * gtid + j)] = qv[j] + base;
        }
        group_bar(bid, TG);   // S(m) in the stage; the exchange area is free again

        // ---- inverse: E_w = IFFT_1024(P_2w + i P_2w+1), twisted by e^{2 pi i w m' / L},
        //      written over this warp's own P pair
        {
            cpx<float> v[32];
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                const int j = lane + 32 * b;
                v[b] = {pf[(2 * w) * kF2 + j], pf[(2 * w + 1) * kF2 + j]};
            }
            __syncwarp();
            fft1024<+1, false>(v, my_scratch, lane, tw_even);
            if (w == 0) {   // twist e^{2 pi i 0 m' / L} = 1
#pragma unroll
                for (int d = 0; d < 32; ++d) pu[lane + 32 * d] = v[d];
            } else {
#pragma unroll
                for (int d = 0; d < 32; ++d)
                    pu[w * kF2 + lane + 32 * d] = cmul(v[d], cmul(comb_lane, comb_d[w * 32 + d]));
            }
        }
        group_bar(bid, TG);

        // ---- U(m' + 1024 p) = sum_s E'_s(m') e^{2 pi i s p / H}, in place per m'
#pragma unroll
        for (int i = 0; i < kF2 / TG; ++i) {
            const int m1 = gtid + TG * i;
            cpx<float> e[H];
#pragma unroll
            for (int s = 0; s < H; ++s) e[s] = pu[s * kF2 + m1];
            if constexpr (H == 2) {
                pu[m1] = cadd(e[0], e[1]);
                pu[m1 + kF2] = csub(e[0], e[1]);
            } else {
                dft4<+1>(e[0], e[1], e[2], e[3]);
#pragma unroll
                for (int p = 0; p < H; ++p) pu[m1 + kF2 * p] = e[p];
            }
        }
        group_bar(bid, TG);

        // ---- S(m) of this thread's lags into registers: the stage is then free and the next
        //      sequence's copy overlaps the unfold
        constexpr int NI = G2::NMAX / TG;
        float sreg[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) sreg[i] = sS[pad32b(gtid + TG * i)];
        group_bar(bid, TG);
        prefetch(qn);

        // ---- unfold + combine, m = gtid + TG i (TG / N2 = 1/64 of a turn per step)
        double* prow = kRing ? ring.partial + item * (int64_t)N : nullptr;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int m = gtid + TG * i;
            if (m < N) {
                const cpx<float> A = pu[m];
                const cpx<float> B = pu[(G2::L - m) & (G2::L - 1)];
                const cpx<float> ww = cmul(unf_base, ct_w<+1, float>(i, 64));
                const float re2 = (A.x + B.x) + (ww.x * (A.y + B.y) + ww.y * (A.x - B.x));
                float val = fmaf(-re2, inv_n2, sreg[i]) * __frcp_rn((float)(N - m));
                if (m == 0) val = 0.f;
                if constexpr (kRing) prow[m] = first_of_item ? (double)val : prow[m] + (double)val;
                else out_q[(q - q0) * (int64_t)N + m] = val;
            }
        }
        group_bar(bid, TG);   // pu consumed before the next sequence's P lands in it
        if (kRing) {
            item = n_item;
            idx = n_idx;
        }
        q = qn;
    }
}

template <int R>
cudaError_t launch_long2_r(const TemporalArgs& a, int64_t q0, int64_t q1, float* out_q,
                           int num_sms, cudaStream_t stream) {
    using G2 = Geom2<R>;
    const bool ring = a.ring.nitems > 0;
    const size_t smem = G2::total;
    const int per_sm = R == 4 ? 2 : 1;
    const int64_t work = ring ? a.ring.nitems : q1 - q0;
    const int grid = (int)std::min<int64_t>((work + 1) / 2, (int64_t)num_sms * per_sm);
    if (grid <= 0) return cudaSuccess;
    const bool full = a.N == G2::NMAX;
    auto k = ring ? (full ? temporal_long2_kernel<R, true, true> : temporal_long2_kernel<R, true, false>)
                  : (full ? temporal_long2_kernel<R, false, true> : temporal_long2_kernel<R, false, false>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 2 * G2::TG, smem, stream>>>(static_cast<const cpx<float>*>(a.spec), a.segs, a.N, q0, q1,
                                          out_q, a.ring);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_long2(const TemporalArgs& a, int64_t q0, int64_t q1, float* out_q, int num_sms,
                         cudaStream_t stream) {
    return a.N2 == 4 * kF2 ? launch_long2_r<4>(a, q0, q1, out_q, num_sms, stream)
                           : launch_long2_r<8>(a, q0, q1, out_q, num_sms, stream);
}

}  // namespace ddmk
