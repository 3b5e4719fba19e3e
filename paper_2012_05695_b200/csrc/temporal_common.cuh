// Shared device helpers of the temporal engines (temporal_warp.cu, temporal_long.cu):
// TMA bulk copies with mbarrier completion and the register-resident length-1024 transform.
#pragma once

#include <cstdint>

#include "kernels.cuh"
#include "warp_fft.cuh"

namespace ddmk {
namespace tc {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}

// lane 0: expect `bytes` on `bar` and start the bulk copy global -> shared
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          unsigned long long* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void fence_expect(unsigned long long* bar, uint32_t bytes) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes,
                                          unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// one-instruction L2 prefetch of a contiguous range by the bulk-copy engine (16-byte aligned,
// size a multiple of 16)
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// wait with backoff: a warp whose copy has not landed sleeps between polls instead of
// taking issue slots from the warps that have work
__device__ __forceinline__ void mbar_wait_backoff(unsigned long long* bar, uint32_t phase) {
    uint32_t ok = 0;
    while (true) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(phase)
            : "memory");
        if (ok) return;
        __nanosleep(64);
    }
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// v[b] *= W_64^{b} = exp(SIGN 2 pi i b / 64): compile-time constants after unrolling
template <int SIGN>
__device__ __forceinline__ void premul_w64(cpx<float> (&v)[32]) {
#pragma unroll
    for (int b = 1; b < 32; ++b) {
        if (b == 16) v[b] = rot90<SIGN>(v[b]);  // W_64^{16} = SIGN i
        else v[b] = cmul(v[b], ct_w<SIGN, float>(b, 64));
    }
}

// Exchange pitch of the length-1024 transforms: 34 complex per row keeps every row 16-byte
// aligned, so the transposed reads are 128-bit (two values per load) and stay conflict-free
// per quarter warp; a warp's exchange buffer holds kXS complex.
constexpr int kXP = 34;
constexpr int kXS = 32 * kXP;

// Length-1024 transform of the warp (lane a holds x[a + 32 b] in v[b]; on return lane c
// holds X[c + 32 d] in v[d]).  Four-step: DFT_32 over b, exchange, then DFT_32 over a of
// Y[a][c] W(a, c) with the twiddles fused into its first butterflies; lane c reads W(., c)
// from row c of a CTA table twt[c * kXP + a] (128-bit loads): W_1024^{a c}, or for ODD
// W_2048^{a (2c + 1)}, where the input is x[n] W_2048^{n}: its W_64^{b} part is applied
// before the first DFT_32 and its lane factor W_2048^{a} is folded into the table, so X =
// the odd outputs of the zero-padded FFT_2048.  W(0, c) = 1.
template <int SIGN, bool ODD>
__device__ __forceinline__ void fft1024(cpx<float> (&v)[32], cpx<float>* scratch, int lane,
                                        const cpx<float>* __restrict__ twt) {
    if constexpr (ODD)   // W_64^{b} fused into the first butterflies (compile-time constants)
        dft32_fused<SIGN, float, true>(v, [](int b) { return ct_w<SIGN, float>(b, 64); });
    else
        RegDft<32, SIGN, float>::run(v);
#pragma unroll
    for (int c = 0; c < 32; ++c) scratch[c * kXP + lane] = v[c];
    __syncwarp();
    const float4* row = reinterpret_cast<const float4*>(scratch + lane * kXP);
#pragma unroll
    for (int ap = 0; ap < 32; ap += 2) {
        const float4 t = row[ap / 2];
        v[ap] = {t.x, t.y};
        v[ap + 1] = {t.z, t.w};
    }
    __syncwarp();
    const cpx<float>* tw = twt + lane * kXP;
    auto twf = [tw](int a) {
        cpx<float> w = tw[a];
        if (SIGN > 0) w.y = -w.y;
        return w;
    };
    dft32_fused<SIGN, float, true>(v, twf);
}

// Twiddle tables of fft1024 (kXS complex each), row c = lane c: even W_1024^{a c}, odd
// W_2048^{a (2c + 1)}
__device__ __forceinline__ void fill_fft1024_tables(cpx<float>* tw_even, cpx<float>* tw_odd,
                                                    int tid, int nthreads) {
    for (int i = tid; i < 32 * 32; i += nthreads) {
        const int a = i >> 5, c = i & 31;
        double sn, cs;
        sincospi(-2.0 * (double)(a * c) / 1024, &sn, &cs);
        tw_even[a * kXP + c] = {(float)cs, (float)sn};   // symmetric in (a, c)
        if (tw_odd) {
            sincospi(-2.0 * (double)(a * (2 * c + 1)) / 2048, &sn, &cs);
            tw_odd[c * kXP + a] = {(float)cs, (float)sn};  // row c: the lane that applies it
        }
    }
}

}  // namespace tc
}  // namespace ddmk
