"""In-tree build of libvoxrf_b200.so for sm_100a (nvcc, no JIT cache).

The shared library lands in ``paper_2307_03404_b200/_lib/`` so it travels with
the repository snapshot to the GPU box (git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libvoxrf_b200.so"
SOURCES = ["vrf_kernels.cu", "vrf_order.cu", "vrf_track.cu", "vrf_capi.cu", "vrf_map.cu", "vrf_pose.cu",
           "vrf_eval.cu"]
HEADERS = ["vrf_device.cuh", "vrf_internal.h", "vrf_context.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
]
# experiments only (e.g. -DVRF_QSTATS); part of the build digest
NVCC_FLAGS += os.environ.get("VRF_EXTRA_NVCC_FLAGS", "").split()


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: cannot build libvoxrf_b200 for sm_100a")
    return cand


def _digest() -> str:
    h = hashlib.sha256()
    for name in SOURCES + HEADERS:
        h.update((CSRC / name).read_bytes())
    h.update((ROOT / "include" / "voxrf_b200.h").read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, libdir: Path = LIBDIR,
          defines=()) -> Path:
    """Compile every CUDA source for sm_100a and link the C-ABI library. libdir /
    defines: an A/B variant of the same sources (tools/ab/), loaded with VRF_LIB."""
    libdir = Path(libdir)
    libdir.mkdir(parents=True, exist_ok=True)
    lib = libdir / LIB.name
    flags = [*NVCC_FLAGS, *(f"-D{d}" for d in defines)]
    stamp = libdir / "build.sha256"
    digest = _digest() + " ".join(defines)
    if lib.exists() and stamp.exists() and stamp.read_text() == digest and not force:
        return lib
    nvcc = _nvcc()
    objdir = libdir / "obj"
    objdir.mkdir(exist_ok=True)
    log = []
    procs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc, *flags, "-c", str(CSRC / src), "-o", str(obj)]
        procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                 stderr=subprocess.STDOUT, text=True)))
    for src, cmd, p in procs:
        out, _ = p.communicate()
        log.append(f"$ {' '.join(cmd)}\n{out}")
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
    objs = [str(objdir / (Path(x).stem + ".o")) for x in SOURCES]
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib), *objs,
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.append(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}{r.stderr}")
    (libdir / "ptxas.log").write_text("\n".join(log))
    stamp.write_text(digest)
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    print(build(force=bool(os.environ.get("FORCE")), verbose=True))
