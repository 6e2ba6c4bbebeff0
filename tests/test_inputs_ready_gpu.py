"""FLR_FLAG_INPUTS_READY (-m gpu): with resident inputs the moment kernel of call i+1 streams
while the previous kernel on the stream drains; the library's own workspace must never be
raced.  Calls are issued BACK TO BACK on one stream and one workspace (no copy or any other
kernel between them: outputs go to preallocated rotating buffers and are compared only
after one final synchronise), and every result must equal the flag-free result bit for bit
(same kernels, same arithmetic) and meet the oracle bar.

Chains covered (the predecessor of each call's moment kernel differs):
  denoise -> denoise   (predecessor: the apply grid)
  fit -> fit           (predecessor: the blur+solve grid, which reads the moment field by TMA)
  fit -> denoise       (same, then an apply)
  modulated, unaligned albedo (the demodulated radiance is produced inside the call, so the
                       moment kernel must not stream it before its grid wait)
"""
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
def test_inputs_ready_denoise_chain(flr, oracle_mod, W, H, n):
    from paper_2410_11625_b200 import synth

    frames = [synth.batch(n, W, H, Q=8, seed0=1400 + 10 * k) for k in range(3)]
    dev = [(g.cuda(), y.cuda()) for g, y in frames]
    plain = flr.Denoiser(n, 8, W, H, device="cuda")
    fast = flr.Denoiser(n, 8, W, H, device="cuda", flags=flr.FLAG_INPUTS_READY)
    ref_gpu = [plain(g, y).clone() for g, y in dev]
    torch.cuda.synchronize()
    outs = [torch.empty_like(ref_gpu[0]) for _ in range(24)]
    for i in range(24):  # back to back on one stream, one workspace
        g, y = dev[i % 3]
        fast(g, y, out=outs[i])
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        assert torch.equal(o, ref_gpu[i % 3]), f"call {i} differs from the flag-free result"
    for k in range(2):
        ref = oracle_mod.denoise(frames[k][0].numpy(), frames[k][1].numpy(), D=8, sigma=10.0, R=3)
        assert_parity(ref_gpu[k].cpu().numpy(), ref, f"inputs-ready frame {k}")


# Q = 3 and 7: 3(Q+1) equals the padded model stride, the case the round-1 review found racy
@pytest.mark.parametrize("Q", [3, 7, 8])
def test_inputs_ready_fit_chains(flr, oracle_mod, Q):
    from paper_2410_11625_b200 import synth

    W, H, n = 1920, 1080, 1
    frames = [synth.batch(n, W, H, Q=Q, seed0=2400 + 10 * k) for k in range(2)]
    dev = [(g.cuda(), y.cuda()) for g, y in frames]
    ref_models = [flr.fit(g, y) for g, y in dev]
    ref_out = [flr.denoise(g, y) for g, y in dev]
    torch.cuda.synchronize()
    ws = torch.empty(flr.workspace_size(n, Q, W, H), dtype=torch.uint8, device="cuda")
    F = flr.FLAG_INPUTS_READY
    models = [torch.empty_like(ref_models[0]) for _ in range(16)]
    outs = [torch.empty_like(ref_out[0]) for _ in range(8)]
    for i in range(16):  # fit -> fit, one workspace
        g, y = dev[i % 2]
        flr.fit(g, y, flags=F, workspace=ws, out=models[i])
    for i in range(8):  # fit -> denoise -> fit -> denoise ...
        g, y = dev[i % 2]
        flr.fit(g, y, flags=F, workspace=ws, out=models[(i + 1) % 16])
        flr.denoise(g, y, flags=F, workspace=ws, out=outs[i])
    torch.cuda.synchronize()
    for i in range(16):
        if i in range(1, 9):  # overwritten by the second loop (frame (i-1) % 2)
            assert torch.equal(models[i], ref_models[(i - 1) % 2]), f"fit call {i}"
        else:
            assert torch.equal(models[i], ref_models[i % 2]), f"fit call {i}"
    for i in range(8):
        assert torch.equal(outs[i], ref_out[i % 2]), f"denoise call {i} after a fit"
    ref = oracle_mod.denoise(frames[0][0].numpy(), frames[0][1].numpy(), D=8, sigma=10.0, R=3)
    assert_parity(ref_out[0].cpu().numpy(), ref, f"fit chain Q={Q}")


def test_inputs_ready_modulated_unfused(flr):
    """Albedo 4 bytes off a 16-byte boundary: the unfused route demodulates into `out` first."""
    from paper_2410_11625_b200 import synth

    W, H, n, Q = 640, 360, 2, 8
    g, y = synth.batch(n, W, H, Q=Q, seed0=3100)
    g, y = g.cuda(), y.cuda()
    gen = torch.Generator().manual_seed(5)
    alb_buf = (0.05 + 0.9 * torch.rand(n * 3 * H * W + 1, generator=gen)).cuda()
    albedo = alb_buf[1:].view(n, 3, H, W)  # 4-byte aligned, not 16
    direct = torch.rand(n, 3, H, W, generator=gen).cuda()
    rmod = (y * albedo).contiguous()
    ref = flr.denoise_modulated(g, rmod, albedo, direct)
    torch.cuda.synchronize()
    ws = torch.empty(flr.workspace_size(n, Q, W, H), dtype=torch.uint8, device="cuda")
    outs = [torch.empty_like(ref) for _ in range(12)]
    for i in range(12):
        flr.denoise_modulated(g, rmod, albedo, direct, flags=flr.FLAG_INPUTS_READY, workspace=ws, out=outs[i])
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        assert torch.equal(o, ref), f"modulated call {i}"
    assert flr.last_launch_names()[0] == "k_demod"
