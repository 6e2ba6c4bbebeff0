"""C-ABI checks that need no GPU (-m "not gpu"): libflr.so loads, exports every function
include/flr.h declares, and rejects bad arguments before launching anything."""
import ctypes
import os
import re

import pytest

import paper_2410_11625_b200 as flr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    src = open(header).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(flr_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2410_11625_b200 import build

    build.build()
    return flr.lib()


def test_exports_every_declared_symbol(L):
    names = _declared(os.path.join(ROOT, "include", "flr.h"))
    assert {"flr_fit", "flr_apply", "flr_denoise", "flr_denoise_upsample", "flr_denoise_modulated",
            "flr_fit_f16", "flr_denoise_f16", "flr_denoise_upsample_f16"} <= set(names)
    for n in names:
        assert hasattr(L, n), n


def test_oracle_exports_every_declared_symbol(oracle_mod):
    L = oracle_mod.lib()
    for n in _declared(os.path.join(ROOT, "oracle", "flr_ref.h")):
        assert hasattr(L, n), n


def test_default_params(L):
    p = flr.Params()
    L.flr_default_params(ctypes.byref(p))
    assert (p.block, p.upsample, p.radius, p.variant) == (8, 1, 0, 0)
    assert (p.sigma, p.eps_add, p.eps_mul) == (10.0, 1e-5, 1e-4)
    L.flr_default_params(None)  # no-op


def test_status_strings(L):
    names = [L.flr_status_string(i).decode() for i in range(7)]
    assert names == ["FLR_OK", "FLR_ERR_INVALID_VALUE", "FLR_ERR_SHAPE", "FLR_ERR_ALIGNMENT",
                     "FLR_ERR_WORKSPACE", "FLR_ERR_UNSUPPORTED", "FLR_ERR_CUDA"]
    assert L.flr_status_string(99) is not None


def test_effective_radius():
    assert flr.effective_radius() == 3                      # ceil(2*10/8)
    assert flr.effective_radius(sigma=20.0) == 5            # C3
    assert flr.effective_radius(block=4, upsample=2) == 3   # C4: D_out = 8
    assert flr.effective_radius(radius=7) == 7
    with pytest.raises(ValueError):
        flr.effective_radius(block=3)


def test_workspace_size_grows_and_validates():
    a = flr.workspace_size(1, 8, 1920, 1080)
    b = flr.workspace_size(2, 8, 1920, 1080)
    assert 0 < a < b
    assert a % 256 == 0
    with pytest.raises(flr.FLRError):
        flr.workspace_size(1, 0, 64, 64)
    with pytest.raises(flr.FLRError):
        flr.workspace_size(0, 8, 64, 64)
    with pytest.raises(flr.FLRError):
        flr.workspace_size(1, 8, 64, 64, eps_mul=1.0)


FAKE = ctypes.c_void_p(0x7F0000000000)  # never dereferenced: every case fails validation first


def _p(**kw):
    return flr.Params.make(**kw)


@pytest.mark.parametrize("kw,status", [
    (dict(block=3), 1), (dict(sigma=0.0), 1), (dict(sigma=float("nan")), 1), (dict(eps_add=-1.0), 1),
    (dict(eps_mul=1.0), 1), (dict(radius=-1), 1), (dict(upsample=0), 1), (dict(variant=7), 5),
    (dict(radius=33), 5),
])
def test_fit_rejects_bad_params(L, kw, status):
    p = _p(**kw)
    st = L.flr_fit(1, 8, 64, 64, FAKE, FAKE, ctypes.byref(p), FAKE, FAKE, 1 << 30, None)
    assert st == status


def test_fit_rejects_bad_shapes_and_pointers(L):
    p = _p()
    big = 1 << 40
    assert L.flr_fit(1, 16, 64, 64, FAKE, FAKE, ctypes.byref(p), FAKE, FAKE, big, None) == 1
    assert L.flr_fit(0, 8, 64, 64, FAKE, FAKE, ctypes.byref(p), FAKE, FAKE, big, None) == 2
    assert L.flr_fit(1, 8, 0, 64, FAKE, FAKE, ctypes.byref(p), FAKE, FAKE, big, None) == 2
    assert L.flr_fit(1, 8, 64, 64, None, FAKE, ctypes.byref(p), FAKE, FAKE, big, None) == 1
    assert L.flr_fit(1, 8, 64, 64, ctypes.c_void_p(0x7F0000000001), FAKE, ctypes.byref(p), FAKE, FAKE,
                     big, None) == 3
    assert L.flr_fit(1, 8, 64, 64, FAKE, FAKE, None, FAKE, FAKE, big, None) == 1
    # workspace too small / misaligned
    assert L.flr_fit(1, 8, 64, 64, FAKE, FAKE, ctypes.byref(p), FAKE, FAKE, 16, None) == 4
    assert L.flr_fit(1, 8, 64, 64, FAKE, FAKE, ctypes.byref(p), FAKE, ctypes.c_void_p(0x7F0000000010),
                     big, None) == 3


def test_apply_and_upsample_shape_checks(L):
    p = _p(upsample=2, block=4)
    big = 1 << 40
    # model grid mismatch
    assert L.flr_apply(1, 8, 64, 64, 8, 7, 8, FAKE, FAKE, FAKE, None) == 2
    # hi-res size must be exactly U x lo-res
    assert L.flr_denoise_upsample(1, 8, 32, 32, FAKE, FAKE, 64, 63, FAKE, ctypes.byref(p), FAKE, FAKE,
                                  big, None) == 2
    # denoise requires upsample == 1
    assert L.flr_denoise(1, 8, 32, 32, FAKE, FAKE, ctypes.byref(p), FAKE, FAKE, big, None) == 1


def test_binding_refuses_cpu_tensors():
    import torch

    g = torch.zeros(1, 4, 8, 8)
    y = torch.zeros(1, 3, 8, 8)
    with pytest.raises(ValueError):
        flr.denoise(g, y)


def test_solver_field_validated(L):
    """flr_params.solver: APPENDIX (default) or TIKHONOV; anything else is rejected
    before any launch."""
    import paper_2410_11625_b200 as flr

    p = flr.Params()
    L.flr_default_params(ctypes.byref(p))
    assert p.solver == flr.SOLVER_APPENDIX
    for s, ok in ((0, True), (1, True), (2, False), (-1, False)):
        p.solver = s
        assert (L.flr_effective_radius(ctypes.byref(p)) >= 0) == ok


def test_flags_field_validated(L):
    p = flr.Params()
    L.flr_default_params(ctypes.byref(p))
    assert p.flags == 0
    p.flags = flr.FLAG_INPUTS_READY
    assert L.flr_effective_radius(ctypes.byref(p)) >= 0
    p.flags = 2  # unknown bit
    assert L.flr_effective_radius(ctypes.byref(p)) == -1


def test_modulated_argument_checks(L):
    """flr_denoise_modulated validates before launching (no GPU touched)."""
    p = _p()
    big = 1 << 40
    f = ctypes.c_float
    # NULL albedo, non-positive / NaN floor -> INVALID_VALUE
    assert L.flr_denoise_modulated(1, 8, 64, 64, FAKE, FAKE, None, None, f(1e-3), ctypes.byref(p), FAKE, FAKE,
                                   big, None) == 1
    assert L.flr_denoise_modulated(1, 8, 64, 64, FAKE, FAKE, FAKE, None, f(0.0), ctypes.byref(p), FAKE, FAKE,
                                   big, None) == 1
    assert L.flr_denoise_modulated(1, 8, 64, 64, FAKE, FAKE, FAKE, None, f(float("nan")), ctypes.byref(p), FAKE,
                                   FAKE, big, None) == 1
    # upsample must be 1; misaligned direct light
    pu = _p(upsample=2, block=4)
    assert L.flr_denoise_modulated(1, 8, 64, 64, FAKE, FAKE, FAKE, None, f(1e-3), ctypes.byref(pu), FAKE, FAKE,
                                   big, None) == 1
    assert L.flr_denoise_modulated(1, 8, 64, 64, FAKE, FAKE, FAKE, ctypes.c_void_p(0x7F0000000002), f(1e-3),
                                   ctypes.byref(p), FAKE, FAKE, big, None) == 3


def test_half_guide_entry_points_reject_unsupported_shapes(L):
    """The fp16-guide entry points run only the TMA kernels: W % 8, block 4/8/16 (fit) and
    output blocks of a multiple of 8 (apply); anything else is UNSUPPORTED before launch."""
    big = 1 << 40
    p = _p()
    assert L.flr_fit_f16(1, 8, 68, 64, FAKE, FAKE, ctypes.byref(p), FAKE, FAKE, big, None) == 5  # W % 8
    assert L.flr_fit_f16(1, 8, 64, 64, FAKE, FAKE, ctypes.byref(_p(block=2)), FAKE, FAKE, big, None) == 5
    assert L.flr_denoise_f16(1, 8, 64, 64, FAKE, FAKE, ctypes.byref(_p(block=4)), FAKE, FAKE, big, None) == 5
    assert L.flr_denoise_f16(1, 8, 64, 64, FAKE, FAKE, ctypes.byref(_p(variant=flr.VARIANT_FUSED)), FAKE, FAKE,
                             big, None) == 5
    assert L.flr_denoise_upsample_f16(1, 8, 32, 32, FAKE, FAKE, 64, 64, FAKE, ctypes.byref(_p(block=2, upsample=2)),
                                      FAKE, FAKE, big, None) == 5
