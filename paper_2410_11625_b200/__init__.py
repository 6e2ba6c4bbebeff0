"""Fast Local Regression (arXiv 2410.11625) on B200 -- thin Python binding of libflr.so.

Argument marshalling only: every step of the path (block moments, moment blur,
per-block solve, blended apply) runs in the sm_100a kernels behind the C ABI
declared in include/flr.h.  Tensors are torch CUDA tensors used as device
memory; the current torch stream is passed to the library.  There is no CPU
fallback: a missing library or a CPU tensor raises.

    import paper_2410_11625_b200 as flr
    out = flr.denoise(guides, radiance)                 # [n,Q,H,W], [n,3,H,W] -> [n,3,H,W]
    models = flr.fit(guides, radiance)                  # [n,By,Bx,Q+1,3], raw basis
    out = flr.apply(models, guides, block_out=8)
    out = flr.denoise_upsample(g_lo, y_lo, g_hi, block=4, upsample=2)
"""
from __future__ import annotations

import ctypes
import math
import os

__all__ = ["FLRError", "Params", "lib", "lib_path", "workspace_size", "effective_radius", "fit",
           "apply", "denoise", "denoise_upsample", "denoise_modulated", "Denoiser", "EventTrace", "last_launch_count", "last_launch_names",
           "VARIANT_AUTO", "VARIANT_STAGED", "VARIANT_FUSED", "SOLVER_APPENDIX", "SOLVER_TIKHONOV"]

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libflr.so")
_lib = None

VARIANT_AUTO = 0
VARIANT_STAGED = 1
VARIANT_FUSED = 2
SOLVER_APPENDIX = 0  # the paper's normalised solve
SOLVER_TIKHONOV = 1  # Eq. tikhonov, Fig. 3 semantics; eps_add is its epsilon
FLAG_INPUTS_READY = 1  # inputs complete before the preceding kernel began (streaming loops)


class EventTrace(ctypes.Structure):
    """Mirror of flr_event_trace (include/flr.h): caller-owned cudaEvent_t handles."""
    _fields_ = [("events", ctypes.POINTER(ctypes.c_void_p)), ("capacity", ctypes.c_int32),
                ("recorded", ctypes.c_int32)]

    @classmethod
    def from_events(cls, events):
        """`events`: torch.cuda.Event(enable_timing=True) objects, already created (recorded once)."""
        arr = (ctypes.c_void_p * len(events))(*[ctypes.c_void_p(e.cuda_event) for e in events])
        t = cls(ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)), len(events), 0)
        t._keep = (arr, list(events))
        return t


class FLRError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        name = lib().flr_status_string(status).decode() if _lib is not None else str(status)
        super().__init__(f"{what}: {name} ({status})")


class Params(ctypes.Structure):
    """Mirror of flr_params (include/flr.h)."""
    _fields_ = [("block", ctypes.c_int32), ("upsample", ctypes.c_int32), ("radius", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("sigma", ctypes.c_double), ("eps_add", ctypes.c_double),
                ("eps_mul", ctypes.c_double), ("solver", ctypes.c_int32), ("flags", ctypes.c_int32)]

    @classmethod
    def make(cls, block=8, upsample=1, sigma=10.0, radius=0, eps_add=1e-5, eps_mul=1e-4,
             variant=VARIANT_AUTO, solver=0, flags=0):
        return cls(int(block), int(upsample), int(radius), int(variant), float(sigma),
                   float(eps_add), float(eps_mul), int(solver), int(flags))


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Load libflr.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(
                f"{_LIB_PATH} is missing: run `python -m paper_2410_11625_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(_LIB_PATH)
        i32, sz, vp, dp = ctypes.c_int32, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p
        pp = ctypes.POINTER(Params)
        L.flr_default_params.argtypes = [pp]
        L.flr_default_params.restype = None
        L.flr_status_string.argtypes = [ctypes.c_int]
        L.flr_status_string.restype = ctypes.c_char_p
        L.flr_effective_radius.argtypes = [pp]
        L.flr_effective_radius.restype = i32
        L.flr_workspace_size.argtypes = [i32, i32, i32, i32, pp, ctypes.POINTER(sz)]
        L.flr_fit.argtypes = [i32, i32, i32, i32, dp, dp, pp, dp, vp, sz, vp]
        L.flr_apply.argtypes = [i32, i32, i32, i32, i32, i32, i32, dp, dp, dp, vp]
        L.flr_denoise.argtypes = [i32, i32, i32, i32, dp, dp, pp, dp, vp, sz, vp]
        L.flr_denoise_upsample.argtypes = [i32, i32, i32, i32, dp, dp, i32, i32, dp, pp, dp, vp, sz, vp]
        tp = ctypes.POINTER(EventTrace)
        L.flr_denoise_traced.argtypes = [i32, i32, i32, i32, dp, dp, pp, dp, vp, sz, vp, tp]
        L.flr_denoise_upsample_traced.argtypes = [i32, i32, i32, i32, dp, dp, i32, i32, dp, pp, dp, vp, sz,
                                                  vp, tp]
        L.flr_denoise_modulated.argtypes = [i32, i32, i32, i32, dp, dp, dp, dp, ctypes.c_float, pp, dp, vp, sz,
                                            vp]
        L.flr_denoise_modulated_traced.argtypes = [i32, i32, i32, i32, dp, dp, dp, dp, ctypes.c_float, pp, dp,
                                                   vp, sz, vp, tp]
        L.flr_fit_f16.argtypes = [i32, i32, i32, i32, dp, dp, pp, dp, vp, sz, vp]
        L.flr_denoise_f16.argtypes = [i32, i32, i32, i32, dp, dp, pp, dp, vp, sz, vp]
        L.flr_denoise_f16_traced.argtypes = [i32, i32, i32, i32, dp, dp, pp, dp, vp, sz, vp, tp]
        L.flr_denoise_upsample_f16.argtypes = [i32, i32, i32, i32, dp, dp, i32, i32, dp, pp, dp, vp, sz, vp]
        L.flr_denoise_upsample_f16_traced.argtypes = [i32, i32, i32, i32, dp, dp, i32, i32, dp, pp, dp, vp, sz,
                                                      vp, tp]
        L.flr_last_launch_count.argtypes = []
        L.flr_last_launch_count.restype = i32
        L.flr_last_launch_name.argtypes = [i32]
        L.flr_last_launch_name.restype = ctypes.c_char_p
        for f in ("flr_workspace_size", "flr_fit", "flr_apply", "flr_denoise", "flr_denoise_upsample",
                  "flr_denoise_traced", "flr_denoise_upsample_traced", "flr_denoise_modulated",
                  "flr_denoise_modulated_traced", "flr_fit_f16", "flr_denoise_f16", "flr_denoise_f16_traced",
                  "flr_denoise_upsample_f16", "flr_denoise_upsample_f16_traced"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        raise FLRError(status, what)


def last_launch_count() -> int:
    return int(lib().flr_last_launch_count())


def last_launch_names() -> list:
    """Kernel names of the launches the last call on this thread enqueued, in order."""
    L = lib()
    return [L.flr_last_launch_name(i).decode() for i in range(L.flr_last_launch_count())]


def effective_radius(**params) -> int:
    p = Params.make(**params)
    r = lib().flr_effective_radius(ctypes.byref(p))
    if r < 0:
        raise ValueError(f"invalid params {params}")
    return int(r)


def workspace_size(n: int, Q: int, W_fit: int, H_fit: int, **params) -> int:
    p = Params.make(**params)
    out = ctypes.c_size_t(0)
    _check(lib().flr_workspace_size(n, Q, W_fit, H_fit, ctypes.byref(p), ctypes.byref(out)),
           "flr_workspace_size")
    return int(out.value)


# ----------------------------------------------------------------- torch helpers
def _torch():
    import torch

    return torch


def _frames(t, name, C=None, half_ok=False):
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.float32 and not (half_ok and t.dtype == torch.float16):
        raise TypeError(f"{name} must be float32" + (" or float16" if half_ok else ""))
    if t.dim() == 3:
        t = t.unsqueeze(0)
    if t.dim() != 4:
        raise ValueError(f"{name} must be [n,C,H,W] or [C,H,W]")
    if C is not None and t.shape[1] != C:
        raise ValueError(f"{name} must have {C} channels")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _stream_ptr(device):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _workspace(nbytes, device, workspace):
    torch = _torch()
    if workspace is not None:
        if workspace.numel() * workspace.element_size() < nbytes:
            raise ValueError("workspace too small")
        return workspace
    # torch's caching allocator returns 512-byte aligned blocks
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def fit(guides, radiance, *, block=8, upsample=1, sigma=10.0, radius=0, eps_add=1e-5,
        eps_mul=1e-4, variant=VARIANT_AUTO, solver=SOLVER_APPENDIX, flags=0, out=None, workspace=None):
    """Per-block raw-basis models [n, By, Bx, Q+1, 3].
    float16 guides (the fp16 guide network's output) take the fp16 streaming path."""
    torch = _torch()
    g = _frames(guides, "guides", half_ok=True)
    y = _frames(radiance, "radiance", 3)
    n, Q, H, W = g.shape
    if tuple(y.shape) != (n, 3, H, W):
        raise ValueError("radiance must be [n,3,H,W] matching guides")
    p = Params.make(block, upsample, sigma, radius, eps_add, eps_mul, variant, solver, flags)
    Bx, By = math.ceil(W / block), math.ceil(H / block)
    if out is None:
        out = torch.empty((n, By, Bx, Q + 1, 3), dtype=torch.float32, device=g.device)
    ws_bytes = workspace_size(n, Q, W, H, block=block, upsample=upsample, sigma=sigma, radius=radius,
                              eps_add=eps_add, eps_mul=eps_mul, variant=variant)
    ws = _workspace(ws_bytes, g.device, workspace)
    fn = lib().flr_fit_f16 if g.dtype == torch.float16 else lib().flr_fit
    _check(fn(n, Q, W, H, _ptr(g), _ptr(y), ctypes.byref(p), _ptr(out), _ptr(ws),
              ws.numel() * ws.element_size(), _stream_ptr(g.device)), "flr_fit")
    return out


def apply(models, guides, block_out, *, out=None):
    """Blended apply of models [n,By,Bx,Q+1,3] at output resolution."""
    torch = _torch()
    g = _frames(guides, "guides")
    n, Q, H, W = g.shape
    m = models
    if m.dim() == 4:
        m = m.unsqueeze(0)
    if not m.is_cuda or m.dtype != torch.float32 or not m.is_contiguous():
        raise ValueError("models must be a contiguous float32 CUDA tensor")
    if m.shape[0] != n or m.shape[3] != Q + 1 or m.shape[4] != 3:
        raise ValueError("models must be [n,By,Bx,Q+1,3]")
    By, Bx = int(m.shape[1]), int(m.shape[2])
    if out is None:
        out = torch.empty((n, 3, H, W), dtype=torch.float32, device=g.device)
    _check(lib().flr_apply(n, Q, W, H, int(block_out), Bx, By, _ptr(m), _ptr(g), _ptr(out),
                           _stream_ptr(g.device)), "flr_apply")
    return out


def denoise(guides, radiance, *, block=8, sigma=10.0, radius=0, eps_add=1e-5, eps_mul=1e-4,
            variant=VARIANT_AUTO, solver=SOLVER_APPENDIX, flags=0, out=None, workspace=None):
    """FLR denoise: fit + apply with the same guides.  [n,Q,H,W], [n,3,H,W] -> [n,3,H,W].
    Guides may be float16 (fp16 streaming path)."""
    torch = _torch()
    g = _frames(guides, "guides", half_ok=True)
    y = _frames(radiance, "radiance", 3)
    n, Q, H, W = g.shape
    if tuple(y.shape) != (n, 3, H, W):
        raise ValueError("radiance must be [n,3,H,W] matching guides")
    p = Params.make(block, 1, sigma, radius, eps_add, eps_mul, variant, solver, flags)
    if out is None:
        out = torch.empty((n, 3, H, W), dtype=torch.float32, device=g.device)
    ws_bytes = workspace_size(n, Q, W, H, block=block, sigma=sigma, radius=radius, eps_add=eps_add,
                              eps_mul=eps_mul, variant=variant)
    ws = _workspace(ws_bytes, g.device, workspace)
    fn = lib().flr_denoise_f16 if g.dtype == torch.float16 else lib().flr_denoise
    _check(fn(n, Q, W, H, _ptr(g), _ptr(y), ctypes.byref(p), _ptr(out), _ptr(ws),
              ws.numel() * ws.element_size(), _stream_ptr(g.device)), "flr_denoise")
    return out


def denoise_upsample(guides_lo, radiance_lo, guides_hi, *, block=4, upsample=2, sigma=10.0, radius=0,
                     eps_add=1e-5, eps_mul=1e-4, variant=VARIANT_AUTO, solver=SOLVER_APPENDIX, flags=0, out=None,
                     workspace=None):
    """Joint denoise + upsample: fit on low-res radiance/guides, apply with hi-res guides.
    With upsample=1 this is FLNR's split-guide call (fit on X'_model, apply X'_map).
    Both guide sets float32, or both float16 (fp16 streaming path)."""
    torch = _torch()
    g = _frames(guides_lo, "guides_lo", half_ok=True)
    y = _frames(radiance_lo, "radiance_lo", 3)
    gh = _frames(guides_hi, "guides_hi", half_ok=True)
    if g.dtype != gh.dtype:
        raise TypeError("guides_lo and guides_hi must have the same dtype")
    n, Q, H, W = g.shape
    Hh, Wh = int(gh.shape[2]), int(gh.shape[3])
    if tuple(y.shape) != (n, 3, H, W) or gh.shape[0] != n or gh.shape[1] != Q:
        raise ValueError("shape mismatch between guides_lo, radiance_lo and guides_hi")
    p = Params.make(block, upsample, sigma, radius, eps_add, eps_mul, variant, solver, flags)
    if out is None:
        out = torch.empty((n, 3, Hh, Wh), dtype=torch.float32, device=g.device)
    ws_bytes = workspace_size(n, Q, W, H, block=block, upsample=upsample, sigma=sigma, radius=radius,
                              eps_add=eps_add, eps_mul=eps_mul, variant=variant)
    ws = _workspace(ws_bytes, g.device, workspace)
    fn = lib().flr_denoise_upsample_f16 if g.dtype == torch.float16 else lib().flr_denoise_upsample
    _check(fn(n, Q, W, H, _ptr(g), _ptr(y), Wh, Hh, _ptr(gh), ctypes.byref(p), _ptr(out), _ptr(ws),
              ws.numel() * ws.element_size(), _stream_ptr(g.device)), "flr_denoise_upsample")
    return out


def denoise_modulated(guides, radiance_mod, albedo, direct=None, *, block=8, sigma=10.0, radius=0,
                      eps_add=1e-5, eps_mul=1e-4, albedo_floor=1e-3, solver=SOLVER_APPENDIX, flags=0, out=None,
                      workspace=None):
    """The paper's protocol: demodulate by max(albedo, floor), FLR-denoise,
    remodulate, add the direct light.  All radiance-like tensors are [n,3,H,W]."""
    torch = _torch()
    g = _frames(guides, "guides")
    r = _frames(radiance_mod, "radiance_mod", 3)
    a = _frames(albedo, "albedo", 3)
    d = _frames(direct, "direct", 3) if direct is not None else None
    n, Q, H, W = g.shape
    for t, nm in ((r, "radiance_mod"), (a, "albedo")) + (((d, "direct"),) if d is not None else ()):
        if tuple(t.shape) != (n, 3, H, W):
            raise ValueError(f"{nm} must be [n,3,H,W] matching guides")
    p = Params.make(block, 1, sigma, radius, eps_add, eps_mul, VARIANT_AUTO, solver, flags)
    if out is None:
        out = torch.empty((n, 3, H, W), dtype=torch.float32, device=g.device)
    ws_bytes = workspace_size(n, Q, W, H, block=block, sigma=sigma, radius=radius, eps_add=eps_add,
                              eps_mul=eps_mul)
    ws = _workspace(ws_bytes, g.device, workspace)
    _check(lib().flr_denoise_modulated(n, Q, W, H, _ptr(g), _ptr(r), _ptr(a), _ptr(d) if d is not None else None,
                                       float(albedo_floor), ctypes.byref(p), _ptr(out), _ptr(ws),
                                       ws.numel() * ws.element_size(), _stream_ptr(g.device)),
           "flr_denoise_modulated")
    return out


class Denoiser:
    """Pre-sized workspace + output for repeated calls on one shape (bench / serving loop).

    Holds the ctypes argument objects so a call is one C-ABI call with no allocation."""

    def __init__(self, n, Q, W, H, device="cuda", block=8, upsample=1, sigma=10.0, radius=0,
                 eps_add=1e-5, eps_mul=1e-4, variant=VARIANT_AUTO, solver=SOLVER_APPENDIX, flags=0):
        torch = _torch()
        self.n, self.Q, self.W, self.H, self.U = n, Q, W, H, upsample
        self.params = Params.make(block, upsample, sigma, radius, eps_add, eps_mul, variant, solver, flags)
        nbytes = workspace_size(n, Q, W, H, block=block, upsample=upsample, sigma=sigma, radius=radius,
                                eps_add=eps_add, eps_mul=eps_mul, variant=variant)
        self.workspace = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        self.out = torch.empty((n, 3, H * upsample, W * upsample), dtype=torch.float32, device=device)
        self._L = lib()

    def modulated(self, guides, radiance_mod, albedo, direct=None, albedo_floor=1e-3, out=None, stream=None,
                  trace=None):
        """The albedo protocol (flr_denoise_modulated) on this shape: one C-ABI call."""
        torch = _torch()
        out = self.out if out is None else out
        s = ctypes.c_void_p(stream if stream is not None else torch.cuda.current_stream().cuda_stream)
        ws = self.workspace
        tr = ctypes.byref(trace) if trace is not None else None
        st = self._L.flr_denoise_modulated_traced(self.n, self.Q, self.W, self.H, guides.data_ptr(),
                                                  radiance_mod.data_ptr(), albedo.data_ptr(),
                                                  direct.data_ptr() if direct is not None else None,
                                                  float(albedo_floor), ctypes.byref(self.params), out.data_ptr(),
                                                  ws.data_ptr(), ws.numel(), s, tr)
        _check(st, "flr_denoise_modulated_traced")
        return out

    def __call__(self, guides, radiance, guides_hi=None, out=None, stream=None, trace=None):
        """One C-ABI call; `trace` is an optional EventTrace (per-launch CUDA events)."""
        torch = _torch()
        out = self.out if out is None else out
        s = ctypes.c_void_p(stream if stream is not None else torch.cuda.current_stream().cuda_stream)
        ws = self.workspace
        tr = ctypes.byref(trace) if trace is not None else None
        gh = guides if guides_hi is None else guides_hi
        if guides.dtype == torch.float16:  # fp16 guide planes (flr_*_f16)
            if guides_hi is None:
                st = self._L.flr_denoise_f16_traced(self.n, self.Q, self.W, self.H, guides.data_ptr(),
                                                    radiance.data_ptr(), ctypes.byref(self.params), out.data_ptr(),
                                                    ws.data_ptr(), ws.numel(), s, tr)
            else:
                st = self._L.flr_denoise_upsample_f16_traced(self.n, self.Q, self.W, self.H, guides.data_ptr(),
                                                             radiance.data_ptr(), self.W * self.U, self.H * self.U,
                                                             gh.data_ptr(), ctypes.byref(self.params),
                                                             out.data_ptr(), ws.data_ptr(), ws.numel(), s, tr)
            _check(st, "flr_denoise_f16")
            return out
        st = self._L.flr_denoise_upsample_traced(self.n, self.Q, self.W, self.H, guides.data_ptr(),
                                                 radiance.data_ptr(), self.W * self.U, self.H * self.U,
                                                 gh.data_ptr(), ctypes.byref(self.params), out.data_ptr(),
                                                 ws.data_ptr(), ws.numel(), s, tr)
        _check(st, "flr_denoise_upsample_traced")
        return out
