"""Builds A/B variants of libvoxrf_b200.so (same sources, extra -D defines) into
tools/ab/_lib_<name>/; a run selects one with VRF_LIB=tools/ab/_lib_<name>/libvoxrf_b200.so.
usage: python tools/ab/build_variants.py name=DEF1,DEF2 [name2=...]"""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2307_03404_b200 import _build  # noqa: E402


def one(spec):
    name, _, defs = spec.partition("=")
    d = [x for x in defs.split(",") if x]
    return _build.build(libdir=ROOT / "tools" / "ab" / f"_lib_{name}", defines=d)


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for p in ex.map(one, sys.argv[1:]):
            print(p)
