// K3 in ring mode (the fused azimuthal average, `analysis.cpp:61-97` on top of
// `temporal.cpp:77-129`): the same kernel as temporal_warp.cu, instantiated here with the
// packed f32x2 codelets (fft_core.cuh). Ring mode runs 8 warps per SM (its per-warp ring
// accumulators take the shared memory of the other 4), and at 8 warps the packed codelets
// fit without spills and win: C2 + ring average temporal 1.000 -> 0.835 ms, step 1.98 ->
// 1.76 ms (three interleaved A/B rounds, tools/gpu_ab_az.sh). Map mode (12 warps) is in
// temporal_warp.cu. DDM_F32X2_RING=0 selects the scalar codelets for A/B builds.
#ifndef DDM_F32X2
#ifdef DDM_F32X2_RING
#define DDM_F32X2 DDM_F32X2_RING
#else
#define DDM_F32X2 1
#endif
#endif
#include "temporal_warp_kernel.cuh"

namespace ddmk {

cudaError_t launch_temporal_warp_ring(const TemporalArgs& a, int num_sms, cudaStream_t stream) {
    return launch_w<float, false, true>(a, num_sms, stream);
}

}  // namespace ddmk
