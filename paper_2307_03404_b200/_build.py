"""In-tree build of libvoxrf_b200.so for sm_100a (nvcc, no JIT cache).

The shared library lands in ``paper_2307_03404_b200/_lib/`` so it travels with
the repository snapshot to the GPU box (git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import hashlib
import os
import re
import shutil
import subprocess
import tempfile
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


_WIDTH = {".64": 8, ".128": 16, ".U8": 1, ".S8": 1, ".U16": 2, ".S16": 2}


def scan_local_slots(sass_lines) -> dict:
    """{kernel: [stack offsets loaded but never stored]} for one `nvdisasm -c`
    listing (see unwritten_local_loads)."""
    bad = {}
    kern, st, ld, computed = None, {}, {}, set()
    for raw in sass_lines:
        m = re.match(r"\s*\.text\.(\S+):", raw)
        if m:
            kern = m.group(1)
            continue
        m = re.search(r"\b(STL|LDL)((?:\.[A-Z0-9]+)*)\s+(.*?);", raw)
        if not (m and kern):
            continue
        w = next((v for k, v in _WIDTH.items() if m.group(2).endswith(k)), 4)
        a = re.search(r"\[R1(?:\+0x([0-9a-f]+))?\]", m.group(3))
        if not a:
            if m.group(1) == "STL":
                computed.add(kern)
            continue
        o = int(a.group(1) or "0", 16)
        (st if m.group(1) == "STL" else ld).setdefault(kern, []).append((o, w))
    for k, loads in ld.items():
        if k in computed:
            continue
        cov = set()
        for o, w in st.get(k, []):
            cov.update(range(o, o + w))
        miss = sorted({o for o, w in loads if not set(range(o, o + w)) <= cov})
        if miss:
            bad[k] = miss
    return bad


def unwritten_local_loads(lib: Path) -> dict:
    """Kernels whose SASS loads a stack slot ([R1 + off]) that no store of the
    kernel writes. r02 found ptxas (CUDA 12.9, sm_100a) spilling
    k_pose_group_u under a 128-register cap with LDL.LU from two slots and no
    STL to either (the ray origin was read back as garbage). Kernels that store
    through computed addresses (local arrays) are skipped: their slots cannot be
    matched statically. {} when clean or when cuobjdump / nvdisasm are absent."""
    cuobjdump, nvdisasm = shutil.which("cuobjdump"), shutil.which("nvdisasm")
    if not cuobjdump or not nvdisasm:
        return {}
    bad = {}
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([cuobjdump, "-xelf", "all", str(Path(lib).resolve())], cwd=d,
                           capture_output=True, text=True)
        if r.returncode != 0:
            return {}
        for cub in sorted(Path(d).glob("*.cubin")):
            sass = subprocess.run([nvdisasm, "-c", str(cub)], capture_output=True,
                                  text=True).stdout.split("\n")
            bad.update(scan_local_slots(sass))
    return bad


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
    bad = unwritten_local_loads(lib)
    if bad:
        lib.unlink()
        raise RuntimeError(
            "ptxas emitted local-memory loads from stack slots the kernel never stores "
            f"(the spill miscompile of DESIGN.md §5): {bad}")
    stamp.write_text(digest)
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    print(build(force=bool(os.environ.get("FORCE")), verbose=True))
