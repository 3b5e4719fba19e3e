"""The device renderer (`ddm_b200_generate_device`, csrc/synth.cu) against the reference
generator (`ddm::generate`, bit-identical to `synth.cpp:98-132`; pinned by the golden in
tests/golden and test_gpu_parity.py). Same trajectories by construction; the per-pixel sum
replays the reference's addition order, so frames agree exactly except where CUDA's and
glibc's double exp() differ by an ulp on a pixel that rounds at .5 (then by 1 count)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    torch = pytest.importorskip("torch")
    from paper_2012_05695_b200 import ddm as D
    if D.device_count() < 1 or not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch, D


@pytest.mark.parametrize("W,H,N,P,sigma,seed", [
    (64, 64, 256, 100, 1.0, 7),        # the reference's default stack
    (128, 96, 50, 300, 1.5, 3),        # wrap across both edges
    (8, 6, 20, 5, 1.0, 11),            # windows wider than the frame: several images per pixel
    (500, 500, 8, 100, 1.0, 7),        # C5 geometry
    (33, 17, 9, 0, 1.0, 1),            # no particles: background only
])
def test_device_frames_match_host_generator(env, W, H, N, P, sigma, seed):
    torch, D = env
    host = D.generate(W, H, N, particles=P, diffusion=0.5, psf_sigma=sigma, seed=seed)
    dev = torch.empty((N, H, W), dtype=torch.int16, device="cuda")
    D.generate_device(dev.data_ptr(), W, H, N, particles=P, diffusion=0.5, psf_sigma=sigma, seed=seed)
    got = dev.cpu().numpy().view(np.uint16)
    diff = np.abs(got.astype(np.int64) - host.astype(np.int64))
    assert diff.max() <= 1
    assert np.count_nonzero(diff) <= max(1, host.size // 100000)
