"""Build libflr.so in-tree for sm_100a (nvcc; one object per guide count Q, in parallel).

    python -m paper_2410_11625_b200.build [--force] [--jobs N]

Objects go to paper_2410_11625_b200/build/ and are rebuilt only when a source or
header is newer.  The shared library is paper_2410_11625_b200/libflr.so; it links
cudart statically, so it only needs the NVIDIA driver at run time.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import hashlib
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libflr.so")
QS = range(1, 16)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                  "-I", os.path.join(ROOT, "include")]
# developer builds only: extra nvcc defines, e.g. FLR_DEFS="-DFLR_WATCHDOG" (hang diagnostics)
NVFLAGS += os.environ.get("FLR_DEFS", "").split()


def _nvcc():
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found: libflr.so cannot be built")
    return exe


def _deps():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "flr.h")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _digest(src, deps, defines):
    """Content hash of a unit's inputs: an object is rebuilt whenever what it was compiled
    from differs (mtimes alone miss edits made while a build was running)."""
    h = hashlib.sha1()
    for f in [src] + sorted(deps):
        with open(f, "rb") as fh:
            h.update(f.encode() + b"\0" + fh.read())
    h.update(" ".join(NVFLAGS + list(defines)).encode())
    return h.hexdigest()


def _unit_stale(obj, src, deps, defines):
    try:
        with open(obj + ".sha") as fh:
            return fh.read().strip() != _digest(src, deps, defines) or not os.path.exists(obj)
    except OSError:
        return True


def _compile(src, obj, defines=(), verbose=False):
    digest = _digest(src, _deps(), defines)  # of the inputs as they are when compilation starts
    cmd = [_nvcc()] + NVFLAGS + list(defines) + ["-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)}:\n{r.stdout}\n{r.stderr}")
    with open(obj + ".sha", "w") as fh:
        fh.write(digest)
    return obj


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    deps = _deps()
    units = []
    api = os.path.join(CSRC, "flr_api.cu")
    units.append((api, os.path.join(OBJ, "flr_api.o"), ()))
    inst = os.path.join(CSRC, "flr_inst.cu")
    # FLR_QS=4,8 builds only those guide counts (fast dev builds); the others report UNSUPPORTED
    only = os.environ.get("FLR_QS")
    keep = {int(x) for x in only.split(",")} if only else set(QS)
    for q in QS:
        stub = () if q in keep else ("-DFLR_STUB",)
        tag = "" if q in keep else "_stub"
        units.append((inst, os.path.join(OBJ, f"flr_inst_q{q}{tag}.o"), (f"-DFLR_Q={q}",) + stub))
    todo = [u for u in units if force or _unit_stale(u[1], u[0], deps, u[2])]
    if todo:
        jobs = jobs or max(1, min(len(todo), os.cpu_count() or 1))
        with cf.ThreadPoolExecutor(jobs) as ex:
            list(ex.map(lambda u: _compile(*u, verbose=verbose), todo))
    objs = [u[1] for u in units]
    if force or todo or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        cmd = [_nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.jobs, a.verbose))
