"""c5 (or CFG) through the cross-device row-band path with one rank
(seeds_create_banded(0, 1)) against the ordinary run: device time per frame."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds, SeedsBand, SeedsBands  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
f = configs.frames(cfg, n=1)[0]
p = configs.params(cfg)
H, W, C = f.shape
args = (W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"], p["smoothness_prior"], p["iters_per_level"])
d = torch.from_numpy(f).cuda()


def timeit(fn, n=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


s0 = Seeds(*args)
out0 = torch.empty((H, W), dtype=torch.int32, device="cuda")
t0 = timeit(lambda: s0.iterate(d, out0))
s1 = SeedsBand(*args, 0, 1)
out1 = torch.zeros((H, W), dtype=torch.int32, device="cuda")
t1 = timeit(lambda: s1.run(d, labels_out=out1))
assert torch.equal(out0, out1)
line = f"{cfg}: ordinary {t0:.3f} ms, cross-device band path world 1 {t1:.3f} ms ({100 * (t1 / t0 - 1):+.1f}%)"
for k in (1, 2, 4, 8):
    sk = SeedsBands(*args, k)
    ok = torch.zeros((H, W), dtype=torch.int32, device="cuda")
    tk = timeit(lambda: sk.run(d, labels_out=ok))
    assert torch.equal(out0, ok)
    line += f"; {k} bands in one launch {tk:.3f} ms (grid_ctas {sk.info.grid_ctas}, tiles {sk.info.grid_tiles})"
    sk.close()
print(line, f"; ordinary plan ctas {s0.info.grid_ctas} tiles {s0.info.grid_tiles}")
