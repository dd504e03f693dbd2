"""Determinism check: run a config several times (device entry point) and
compare labels/histograms; prints the plan."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1309_3848_b200 import configs
from paper_1309_3848_b200.seeds import Seeds
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
img = configs.frames(cfg, n=1)
p = configs.params(cfg)
n, H, W, C = img.shape
s = Seeds(W, H, C, *[p[k] for k in ("n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
print(cfg, "plan ctas", s.info.grid_ctas, "tiles", s.info.grid_tiles, "mode", s.info.exec_mode)
d = torch.from_numpy(img).cuda()
ref = None
for r in range(reps):
    lab = s.batch(d).clone()
    h, a = s.read_state(0)
    if ref is None:
        ref = (lab, h.clone())
    else:
        print("rep", r, "labels equal", torch.equal(lab, ref[0]), "hist equal", torch.equal(h, ref[1]),
              "label diffs", int((lab != ref[0]).sum()))
# host entry point against the device one
h_img = np.ascontiguousarray(img)
h_out = np.empty((n, H, W), np.int32)
for r in range(2):
    s.batch_host(h_img, h_out)
    dl = ref[0].cpu().numpy()
    print("host run", r, "equal to device", bool((h_out == dl).all()), "diffs", int((h_out != dl).sum()))
    lab = s.batch(d).clone()
    print("device again equal", torch.equal(lab, ref[0]))
