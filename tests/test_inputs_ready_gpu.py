"""FLR_FLAG_INPUTS_READY (-m gpu): with resident inputs the moment kernel of call i+1 streams
while call i's apply drains; the library's own workspace must never be raced.  Many
back-to-back calls on ONE workspace alternate between frames (and shapes of work: a batch),
each output is copied out right after its call, and every one must equal the flag-free
result bit for bit (same kernels, same arithmetic) and meet the oracle bar."""
import pytest
import torch

from tests.parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def flr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_11625_b200 as m

    m.lib()
    return m


@pytest.mark.parametrize("W,H,n", [(1920, 1080, 1), (640, 360, 3)])
def test_inputs_ready_back_to_back(flr, oracle_mod, W, H, n):
    from paper_2410_11625_b200 import synth

    frames = [synth.batch(n, W, H, Q=8, seed0=1400 + 10 * k) for k in range(3)]
    dev = [(g.cuda(), y.cuda()) for g, y in frames]
    plain = flr.Denoiser(n, 8, W, H, device="cuda")
    fast = flr.Denoiser(n, 8, W, H, device="cuda", flags=flr.FLAG_INPUTS_READY)
    ref_gpu = [plain(g, y).clone() for g, y in dev]
    outs = []
    for i in range(24):  # back to back on one stream, one workspace
        g, y = dev[i % 3]
        outs.append(fast(g, y).clone())
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        assert torch.equal(o, ref_gpu[i % 3]), f"call {i} differs from the flag-free result"
    for k in range(2):
        ref = oracle_mod.denoise(frames[k][0].numpy(), frames[k][1].numpy(), D=8, sigma=10.0, R=3)
        assert_parity(ref_gpu[k].cpu().numpy(), ref, f"inputs-ready frame {k}")
