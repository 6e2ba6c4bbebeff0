"""Seeded synthetic FLR inputs: rasterised-style guide planes + 1spp-like noisy radiance.

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle's tests, and it holds none of the method's arithmetic: it draws scenes,
it does not fit or apply anything.  Inputs mirror the paper's workloads
(DESIGN.md section 4 states the recipe):

* guides: albedo luminance, unit normals, depth crowded
  towards the far plane, ambient occlusion, and two smooth sigmoid "neural"
  planes standing in for the optional network-generated guides;
* radiance: the demodulated indirect light of a Lambertian-looking scene
   times heavy-tailed multiplicative 1spp noise with 1 %
  fireflies (one indirect sample per pixel).

The scene is a floor, a back wall (large exactly-flat guide regions: the
paper's instability case) and 4-8 random spheres/boxes.  Per-pixel
random numbers come from a counter-based integer hash, so a frame is a pure
function of (seed, size, Q) on any device; parity tests draw on the CPU and
copy the same tensors to both sides.
"""
from __future__ import annotations

import math

import numpy as np
import torch

# Q=8 layout of BASELINE.json config 2; Q=4 layout of config 1.
GUIDES_Q8 = ("albedo", "normal_x", "normal_y", "normal_z", "depth", "ao", "neural_0", "neural_1")
GUIDES_Q4 = ("albedo", "facing", "depth", "ao")
POOL = ("albedo", "normal_x", "normal_y", "normal_z", "depth", "ao", "neural_0", "neural_1",
        "world_x", "world_y", "world_z", "facing", "neural_2", "neural_3", "checker", "neural_4")

_M32 = 0xFFFFFFFF


def guide_names(Q: int):
    if Q == 4:
        return GUIDES_Q4
    if Q == 8:
        return GUIDES_Q8
    if not 1 <= Q <= len(POOL):
        raise ValueError(f"Q must be in [1, {len(POOL)}]")
    return POOL[:Q]


def _mul32(x, m):
    """(x * m) mod 2^32 for int64 tensors x in [0, 2^32) without int64 overflow."""
    lo = x & 0xFFFF
    hi = x >> 16
    return ((lo * m) + (((hi * m) & 0xFFFF) << 16)) & _M32


def _hash32(x):
    x = x & _M32
    x = _mul32(x ^ (x >> 16), 0x7FEB352D)
    x = _mul32(x ^ (x >> 15), 0x846CA68B)
    return x ^ (x >> 16)


def _uniform(seed: int, stream: int, idx, device):
    """U(0,1) from a counter hash of (seed, stream, pixel index); never exactly 0."""
    base = _hash32(torch.tensor((seed * 0x9E3779B1 + stream * 0x85EBCA77) & _M32,
                                dtype=torch.int64, device=device))
    h = _hash32(idx ^ base)
    h = _hash32(h + stream + 1)
    return ((h >> 8).to(torch.float32) + 0.5) * (1.0 / 16777216.0)


class Scene:
    """Random scene parameters drawn from a numpy Generator seeded by `seed`."""

    def __init__(self, seed: int):
        rng = np.random.default_rng(seed)
        self.seed = seed
        self.cam = np.array([rng.uniform(-0.4, 0.4), rng.uniform(1.0, 1.6), 4.2])
        self.look = np.array([rng.uniform(-0.3, 0.3), 0.7, -1.0])
        self.fov = math.radians(rng.uniform(45.0, 60.0))
        self.wall_z = -3.0
        nobj = int(rng.integers(4, 9))
        self.spheres = []
        self.boxes = []
        for k in range(nobj):
            r = rng.uniform(0.25, 0.7)
            cx, cz = rng.uniform(-2.2, 2.2), rng.uniform(-2.6, 1.2)
            alb = rng.uniform(0.05, 0.95)
            if k % 3 == 2:
                h = rng.uniform(0.3, 1.2)
                self.boxes.append((np.array([cx - r, 0.0, cz - r]), np.array([cx + r, h, cz + r]), alb))
            else:
                self.spheres.append((np.array([cx, r, cz]), r, alb))
        self.floor_alb = (rng.uniform(0.2, 0.5), rng.uniform(0.5, 0.9))
        self.wall_alb = rng.uniform(0.3, 0.9)
        self.tint = rng.uniform(0.5, 1.0, size=3)
        self.light = rng.normal(size=3)
        self.light[1] = abs(self.light[1]) + 0.5
        self.light /= np.linalg.norm(self.light)
        self.blobs = [(rng.uniform(0.1, 0.9), rng.uniform(0.1, 0.9), rng.uniform(0.03, 0.12),
                       rng.uniform(0.3, 0.7)) for _ in range(int(rng.integers(2, 5)))]
        self.neural = rng.uniform(0.5, 3.0, size=(5, 4))


def _render(scene: Scene, W: int, H: int, device):
    """Primary-hit rasterisation at pixel centres: returns dict of float32 planes [H, W]."""
    f32 = torch.float32
    dev = torch.device(device)
    cam = torch.tensor(scene.cam, dtype=f32, device=dev)
    fwd = torch.tensor(scene.look - scene.cam, dtype=f32, device=dev)
    fwd = fwd / fwd.norm()
    up0 = torch.tensor([0.0, 1.0, 0.0], dtype=f32, device=dev)
    right = torch.linalg.cross(fwd, up0)
    right = right / right.norm()
    up = torch.linalg.cross(right, fwd)
    th = math.tan(scene.fov / 2)
    ys = (torch.arange(H, dtype=f32, device=dev) + 0.5) / H
    xs = (torch.arange(W, dtype=f32, device=dev) + 0.5) / W
    py = (1.0 - 2.0 * ys)[:, None] * th
    px = (2.0 * xs - 1.0)[None, :] * th * (W / H)
    d = fwd[None, None, :] + px[..., None] * right + py[..., None] * up
    d = d / d.norm(dim=-1, keepdim=True)
    dx, dy, dz = d[..., 0], d[..., 1], d[..., 2]
    inf = torch.full((H, W), float("inf"), dtype=f32, device=dev)

    t_best = inf.clone()
    nrm = torch.zeros(H, W, 3, dtype=f32, device=dev)
    alb = torch.zeros(H, W, dtype=f32, device=dev)
    kind = torch.zeros(H, W, dtype=torch.int64, device=dev)  # 0 wall, 1 floor, 2 object

    # back wall z = wall_z, normal +z (exactly flat guides)
    tw = torch.where(dz < 0, (scene.wall_z - cam[2]) / dz, inf)
    hit = tw < t_best
    t_best = torch.where(hit, tw, t_best)
    nrm[hit] = torch.tensor([0.0, 0.0, 1.0], dtype=f32, device=dev)
    alb = torch.where(hit, torch.full_like(alb, scene.wall_alb), alb)
    kind = torch.where(hit, torch.zeros_like(kind), kind)
    # floor y = 0, normal +y, checker albedo
    tf = torch.where(dy < 0, -cam[1] / dy, inf)
    hit = tf < t_best
    t_best = torch.where(hit, tf, t_best)
    nrm[hit] = torch.tensor([0.0, 1.0, 0.0], dtype=f32, device=dev)
    pfx = cam[0] + tf * dx
    pfz = cam[2] + tf * dz
    chk = ((torch.floor(pfx * 2.0) + torch.floor(pfz * 2.0)).remainder(2.0) > 0.5)
    falb = torch.where(chk, torch.full_like(alb, scene.floor_alb[0]), torch.full_like(alb, scene.floor_alb[1]))
    alb = torch.where(hit, falb, alb)
    kind = torch.where(hit, torch.ones_like(kind), kind)
    # spheres
    for c, r, a in scene.spheres:
        c = torch.tensor(c, dtype=f32, device=dev)
        oc = cam - c
        b = (d * oc).sum(-1)
        cc = (oc * oc).sum() - r * r
        disc = b * b - cc
        ts = torch.where(disc > 0, -b - torch.sqrt(disc.clamp_min(0)), inf)
        ts = torch.where(ts > 1e-3, ts, inf)
        hit = ts < t_best
        t_best = torch.where(hit, ts, t_best)
        p = cam + ts.clamp_max(1e6)[..., None] * d
        n_s = (p - c) / r
        nrm = torch.where(hit[..., None], n_s, nrm)
        alb = torch.where(hit, torch.full_like(alb, a), alb)
        kind = torch.where(hit, torch.full_like(kind, 2), kind)
    # axis-aligned boxes (slab test)
    for lo, hi_, a in scene.boxes:
        lo = torch.tensor(lo, dtype=f32, device=dev)
        hi_ = torch.tensor(hi_, dtype=f32, device=dev)
        inv = 1.0 / torch.where(d.abs() < 1e-9, torch.full_like(d, 1e-9), d)
        t0 = (lo - cam) * inv
        t1 = (hi_ - cam) * inv
        tmin = torch.minimum(t0, t1)
        tmax = torch.maximum(t0, t1)
        tn = tmin.max(-1).values
        tx = tmax.min(-1).values
        tb = torch.where((tx >= tn) & (tn > 1e-3), tn, inf)
        hit = tb < t_best
        t_best = torch.where(hit, tb, t_best)
        axis = tmin.argmax(-1)
        sgn = -torch.sign(torch.gather(d, -1, axis[..., None]))[..., 0]
        n_b = torch.zeros_like(d)
        n_b.scatter_(-1, axis[..., None], sgn[..., None])
        nrm = torch.where(hit[..., None], n_b, nrm)
        alb = torch.where(hit, torch.full_like(alb, a), alb)
        kind = torch.where(hit, torch.full_like(kind, 2), kind)

    t = torch.where(torch.isfinite(t_best), t_best, torch.full_like(t_best, 50.0))
    p = cam + t[..., None] * d
    # depth: hyperbolic z-buffer value, crowded near the far plane
    zview = t * (d * fwd).sum(-1)
    near, far = 0.5, 20.0
    depth = ((1.0 / near - 1.0 / zview.clamp(near, far)) / (1.0 / near - 1.0 / far)).clamp(0, 1)
    # ambient occlusion: analytic sphere occlusion + floor/wall crease
    ao = torch.ones(H, W, dtype=f32, device=dev)
    occluders = [(torch.tensor(c, dtype=f32, device=dev), r) for c, r, _ in scene.spheres]
    occluders += [(torch.tensor((lo + hi_) / 2, dtype=f32, device=dev), 0.5 * float(np.max(hi_ - lo)))
                  for lo, hi_, _ in scene.boxes]
    for c, r in occluders:
        v = c - p
        dist = v.norm(dim=-1).clamp_min(1e-3)
        cosv = ((nrm * v).sum(-1) / dist).clamp_min(0)
        occ = (r * r / (dist * dist)).clamp_max(1.0) * cosv
        ao = ao * (1.0 - 0.8 * occ.clamp(0, 1) * (dist > r * 1.01))
    crease = torch.exp(-torch.minimum(p[..., 1].abs(), (p[..., 2] - scene.wall_z).abs()) / 0.35)
    ao = ao * (1.0 - 0.45 * crease * (kind < 2))
    ao = ao.clamp(0.0, 1.0)
    facing = (-(nrm * d).sum(-1)).clamp(-1, 1)
    return dict(t=t, p=p, nrm=nrm, alb=alb, kind=kind, depth=depth, ao=ao, facing=facing,
                chk=chk.to(f32), xs=xs, ys=ys)


def _sig(x):
    return torch.sigmoid(x)


def _planes(scene: Scene, R: dict, names):
    p, nrm = R["p"], R["nrm"]
    nz = scene.neural
    out = []
    for name in names:
        if name == "albedo":
            out.append(R["alb"])
        elif name.startswith("normal_"):
            out.append(nrm[..., "xyz".index(name[-1])])
        elif name == "depth":
            out.append(R["depth"])
        elif name == "ao":
            out.append(R["ao"])
        elif name == "facing":
            out.append(R["facing"])
        elif name.startswith("world_"):
            out.append(p[..., "xyz".index(name[-1])] * 0.25)
        elif name == "checker":
            out.append(R["chk"])
        elif name.startswith("neural_"):
            k = int(name[-1])
            a, b, c, e = nz[k]
            out.append(_sig(a * torch.sin(b * p[..., 0] + c) + e * torch.cos(b * p[..., 2] - a)
                            + 2.0 * (R["ao"] - 0.6)))
        else:
            raise ValueError(name)
    return torch.stack(out).to(torch.float32).contiguous()


def _radiance(scene: Scene, R: dict, W: int, H: int, seed: int, noise: bool, device):
    """Demodulated indirect light: smooth in (normal, AO, depth) plus soft cast-shadow
    blobs the guides do not explain, times 1spp multiplicative noise."""
    dev = torch.device(device)
    f32 = torch.float32
    nrm, ao, depth = R["nrm"], R["ao"], R["depth"]
    light = torch.tensor(scene.light, dtype=f32, device=dev)
    sky = 0.35 + 0.25 * nrm[..., 1] + 0.15 * (nrm * light).sum(-1).clamp_min(0)
    base = ao.pow(1.5) * sky * (1.1 - 0.4 * depth)
    xs, ys = R["xs"], R["ys"]
    shadow = torch.ones(H, W, dtype=f32, device=dev)
    for bx, by, bs, bd in scene.blobs:
        g = torch.exp(-(((xs[None, :] - bx) ** 2) + ((ys[:, None] - by) ** 2)) / (2 * bs * bs))
        shadow = shadow * (1.0 - bd * g)
    L = torch.stack([base * shadow * float(scene.tint[c]) for c in range(3)])
    if not noise:
        return L.contiguous()
    idx = torch.arange(H * W, dtype=torch.int64, device=dev).reshape(H, W)
    u1 = _uniform(seed, 1, idx, dev)
    u2 = _uniform(seed, 2, idx, dev)
    u3 = _uniform(seed, 3, idx, dev)
    # Z = 2 Bernoulli(1/2) Exp(1), x20 with probability 1 % (fireflies); finite, >= 0
    z = 2.0 * (u1 < 0.5).to(f32) * (-torch.log(u2))
    z = z * torch.where(u3 < 0.01, torch.full_like(z, 20.0), torch.ones_like(z))
    chroma = torch.stack([_uniform(seed, 4 + c, idx, dev) for c in range(3)])
    z3 = z[None] * (0.85 + 0.3 * chroma)
    return (L * z3).to(f32).contiguous()


def frame(W: int, H: int, Q: int = 8, seed: int = 1000, device="cpu", noise: bool = True,
          duplicate_guide: bool = False):
    """One frame: (guides [Q,H,W] f32, radiance [3,H,W] f32) on `device`."""
    scene = Scene(seed)
    R = _render(scene, W, H, device)
    names = list(guide_names(Q))
    G = _planes(scene, R, names)
    if duplicate_guide and Q >= 2:
        G[Q - 1] = G[0]
    Y = _radiance(scene, R, W, H, seed, noise, device)
    return G, Y


def modulated_frame(W: int, H: int, Q: int = 8, seed: int = 1000, device="cpu"):
    """Inputs of the paper's albedo protocol, as a renderer would
    hand them over: (guides [Q,H,W], radiance_mod [3,H,W] = albedo x noisy indirect light,
    albedo [3,H,W] RGB in [0, 0.95], direct [3,H,W] noise-free direct light >= 0).
    No FLR arithmetic here: the modulation is the renderer's product A * L."""
    scene = Scene(seed)
    R = _render(scene, W, H, device)
    G = _planes(scene, R, list(guide_names(Q)))
    Y = _radiance(scene, R, W, H, seed, True, device)
    dev = torch.device(device)
    f32 = torch.float32
    alb = R["alb"].to(f32)
    tint = torch.stack([_uniform(seed, 20 + c, R["kind"].to(torch.int64), dev) for c in range(3)])
    A = (alb[None] * (0.7 + 0.3 * tint)).clamp(0.0, 0.95)
    light = torch.tensor(scene.light, dtype=f32, device=dev)
    lam = (R["nrm"] * light).sum(-1).clamp_min(0.0)
    Dl = torch.stack([2.0 * lam * R["ao"] * float(scene.tint[c]) for c in range(3)])
    return G, (A * Y).to(f32).contiguous(), A.to(f32).contiguous(), Dl.to(f32).contiguous()


def batch(n: int, W: int, H: int, Q: int = 8, seed0: int = 1000, device="cpu", **kw):
    """n frames with seeds seed0 .. seed0+n-1: (guides [n,Q,H,W], radiance [n,3,H,W])."""
    gs, ys = zip(*(frame(W, H, Q, seed0 + i, device, **kw) for i in range(n)))
    return torch.stack(gs).contiguous(), torch.stack(ys).contiguous()


def upsample_pair(W_lo: int, H_lo: int, U: int = 2, Q: int = 8, seed: int = 1000, device="cpu"):
    """Joint denoise+upsample inputs (Fig. 4): the same scene rasterised at
    low and high resolution; noisy radiance only at low resolution.
    Returns (guides_lo [Q,H,W], radiance_lo [3,H,W], guides_hi [Q,U*H,U*W])."""
    scene = Scene(seed)
    names = list(guide_names(Q))
    R_lo = _render(scene, W_lo, H_lo, device)
    G_lo = _planes(scene, R_lo, names)
    Y_lo = _radiance(scene, R_lo, W_lo, H_lo, seed, True, device)
    R_hi = _render(scene, W_lo * U, H_lo * U, device)
    G_hi = _planes(scene, R_hi, names)
    return G_lo, Y_lo, G_hi


def uniform_noise(shape, seed: int, device="cpu"):
    """Plain U(0,1) float32 tensor from the counter hash (random-guide test inputs)."""
    numel = int(np.prod(shape))
    idx = torch.arange(numel, dtype=torch.int64, device=torch.device(device))
    return _uniform(seed, 99, idx, device).reshape(shape).contiguous()
