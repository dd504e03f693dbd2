"""The C ABI from plain C (examples/seeds_c_demo.c): it compiles against
include/seeds.h and libseeds.so with gcc (CPU), and on a B200 its labels --
reported as a checksum -- equal the oracle's for the same two-tone frame, with
no superpixel straddling the colour seam."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1309_3848_b200")


def compile_demo(tmp_path):
    from paper_1309_3848_b200 import build
    build.build()
    exe = str(tmp_path / "seeds_c_demo")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "seeds_c_demo.c"), "-L", PKG, "-lseeds",
                           f"-Wl,-rpath,{PKG}", "-o", exe])
    return exe


def test_c_example_compiles(tmp_path):
    assert os.path.exists(compile_demo(tmp_path))


@pytest.mark.gpu
def test_c_example_matches_oracle(tmp_path, orc):
    out = subprocess.run([compile_demo(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    m = re.search(r"straddling the seam (\d+), checksum (\d+)", out.stdout)
    assert m and m.group(1) == "0", out.stdout
    W, H = 96, 64
    img = np.zeros((H, W, 3), np.uint8)
    img[:, :37] = [40, 60, 80]
    img[:, 37:] = 210
    r = orc.run(img, 24, 3, 5, 0, 4)
    s = 0
    for v in r.labels.ravel():
        s = (s * 1000003 + int(v)) % (1 << 64)
    assert int(m.group(2)) == s
