"""CPU checks of the boundary: libseeds.so builds, loads and exports every
symbol include/seeds.h declares; argument validation needs no GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "seeds.h")).read()
    return sorted(set(re.findall(r"^\s*(?:seeds_status|void|const char\s*\*)\s*(seeds_\w+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for n in ("seeds_create", "seeds_iterate", "seeds_batch"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1309_3848_b200 import build, seeds
    build.build()
    lib = seeds.load()
    for n in declared():
        assert hasattr(lib, n), n
    assert set(declared()) <= set(seeds.EXPORTS)


def test_create_validation_without_gpu():
    """Invalid arguments are rejected before any CUDA call (SEEDS_EINVAL / ERANGE)."""
    from paper_1309_3848_b200 import seeds
    lib = seeds.load()
    ctx = ctypes.c_void_p()
    bad = [
        (0, 10, 3, 10, 2, 5, 0, 2), (10, 10, 0, 10, 2, 5, 0, 2), (10, 10, 5, 10, 2, 5, 0, 2),
        (10, 10, 3, 0, 2, 5, 0, 2), (10, 10, 3, 10, -1, 5, 0, 2), (10, 10, 3, 10, 16, 5, 0, 2),
        (10, 10, 3, 10, 2, 0, 0, 2), (10, 10, 3, 10, 2, 257, 0, 2), (10, 10, 3, 10, 2, 5, 2, 2),
        (10, 10, 3, 10, 2, 5, 0, -1), (10, 10, 3, 10, 2, 17, 0, 2),  # B = 4913 > 4096
    ]
    for a in bad:
        assert lib.seeds_create(*a, ctypes.byref(ctx)) == -1, a
    assert lib.seeds_create(70000, 70000, 3, 10, 2, 5, 0, 2, ctypes.byref(ctx)) == -6
    assert lib.seeds_status_string(-6) == b"problem exceeds an integer width"


def test_product_path_has_no_oracle_import():
    """The product package never imports the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1309_3848_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "seeds_oracle" not in src, f


def test_persistent_kernels_use_no_local_memory():
    """The grid kernels keep their hot state in registers or shared
    memory (ptxas -v of the in-tree build, paper_1309_3848_b200/ptxas_info.txt):
    no stack at all for the default grid kernels
    (template flag 0) and the single-tile kernels (k_tile1); the extended-pixel instantiations (means post-processing,
    priors) may keep a cold loop counter (at most 16 bytes) in local memory --
    the grid barrier does not invalidate L1, which once made a spilled register
    unsafe across it."""
    from paper_1309_3848_b200 import build
    build.build()
    info = open(os.path.join(ROOT, "paper_1309_3848_b200", "ptxas_info.txt")).read()
    blocks = re.split(r"Compiling entry function '", info)[1:]
    seen = 0
    for b in blocks:
        name = b.split("'", 1)[0]
        if "k_grid" not in name and "k_tile1" not in name:
            continue
        seen += 1
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", b)
        assert m, name
        if "k_grid" in name and name.endswith("ELi1EEEvNS_10GridParamsE"):
            assert int(m.group(1)) <= 16, (name, m.group(0))
        else:
            assert m.groups() == ("0", "0", "0"), (name, m.group(0))
    assert seen >= 12
