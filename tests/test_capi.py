"""The C-ABI library loads and exports every symbol include/voxrf_b200.h declares
(no compute calls: this runs without a GPU)."""
import re
from pathlib import Path

import numpy as np

from paper_2307_03404_b200 import _capi

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "voxrf_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vrf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _capi.load()
    names = declared_symbols()
    assert len(names) >= 35
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_capi.EXPORTED)


def test_abi_version_and_host_rng_matches_oracle(oracle):
    lib = _capi.load()
    assert lib.vrf_abi_version() == 1
    from paper_2307_03404_b200 import Rng
    r = Rng(1)
    b = r.draw_batch(3, 160, 120, 500)
    assert np.array_equal(b, oracle.draw_batch(1, 3, 160, 120, 500))


def test_context_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2307_03404_b200 import Context
    try:
        Context(0)
    except RuntimeError as e:
        assert "no CPU fallback" in str(e)
    else:
        raise AssertionError("context creation must fail without a CUDA device")


def test_bench_and_entry_compile():
    """bench.py and __graft_entry__.py are only run on the GPU box: at least
    byte-compile them here."""
    import py_compile
    root = Path(__file__).resolve().parent.parent
    for name in ("bench.py", "__graft_entry__.py"):
        py_compile.compile(str(root / name), doraise=True)


def test_spill_slot_scanner_flags_never_stored_loads():
    """_build.scan_local_slots (the build-time guard against the ptxas spill
    miscompile, profiles/r02_pose_spill_bug.md) on fabricated listings: a load
    from a slot no store writes is flagged; covered loads, and kernels that store
    through computed addresses, are not."""
    from paper_2307_03404_b200 import _build
    sass = """
        .text._Z3badv:
        /*0000*/  STL [R1+0x70], R0 ;
        /*0010*/  STL.128 [R1], R4 ;
        /*0020*/  LDL.LU.64 R16, [R1+0x68] ;
        /*0030*/  LDL.64 R18, [R1+0x8] ;
        /*0040*/  LDL R2, [R1+0x70] ;
        .text._Z4goodv:
        /*0000*/  STL.64 [R1+0x8], R2 ;
        /*0010*/  LDL.LU.64 R4, [R1+0x8] ;
        .text._Z8computedv:
        /*0000*/  STL [R7], R2 ;
        /*0010*/  LDL R4, [R1+0x20] ;
    """.split("\n")
    assert _build.scan_local_slots(sass) == {"_Z3badv": [0x68]}


def test_built_library_has_no_never_stored_stack_loads():
    """The product library as built: no kernel reads a stack slot it never
    writes (skipped when cuobjdump / nvdisasm are absent)."""
    import shutil
    from paper_2307_03404_b200 import _build
    lib = Path(_capi._LIB_PATH)
    if not lib.exists() or not shutil.which("nvdisasm"):
        import pytest
        pytest.skip("library or nvdisasm absent")
    assert _build.unwritten_local_loads(lib) == {}


def test_parallel_batch_draw_equals_the_sequential_stream():
    """vrf_rng_draw_batch draws batches of >= 65,536 rays in parallel chunks from
    jumped-ahead xoshiro256** states (GF(2) powers of the transition). The rays
    and the final state equal the sequential stream's (rng.hpp:20-41: one raw
    draw per uniform_index), here checked against the same stream drawn in
    sub-threshold pieces, which run sequentially."""
    from paper_2307_03404_b200 import Rng
    for n in (65536, 100003, 1 << 20):
        a = Rng(11)
        b = Rng(11)
        got = a.draw_batch(10, 1200, 680, n)
        parts, left = [], n
        while left:
            m = min(left, 40000)
            parts.append(b.draw_batch(10, 1200, 680, m))
            left -= m
        assert np.array_equal(got, np.concatenate(parts))
        assert list(a.state) == list(b.state)


def test_host_rng_matches_oracle_across_the_parallel_threshold(oracle):
    """The same, against the C oracle's sequential Rng (the reference stream)."""
    from paper_2307_03404_b200 import Rng
    n = 70000
    got = Rng(5).draw_batch(3, 64, 48, n)
    assert np.array_equal(got, oracle.draw_batch(5, 3, 64, 48, n))
