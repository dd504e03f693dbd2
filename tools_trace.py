import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1309_3848_b200 import configs
from paper_1309_3848_b200.seeds import Seeds
cfg = sys.argv[1] if len(sys.argv) > 1 else 'c2'
img = configs.frames(cfg, n=1)[0]; p = configs.params(cfg)
s = Seeds(img.shape[1], img.shape[0], 3, *[p[k] for k in ("n_superpixels","n_levels","bins_per_channel","smoothness_prior","iters_per_level")])
s.set_mode("resident")
s.debug_trace(True)
d = torch.from_numpy(img).cuda()
for _ in range(3): out = s.iterate(d)
torch.cuda.synchronize()
tr = s.debug_trace(True)
S = s.info.subsweeps
print("cluster", s.info.cluster_size, "S", S)
# per sub-sweep: work duration per CTA = stamp[s+1][0] - stamp[s][1]
for ph in range(1, S + 1):
    work = tr[:, ph, 0] - tr[:, ph - 1, 1]
    bar = tr[:, ph, 1] - tr[:, ph, 0]
    print(ph - 1, "work max/min (cycles)", int(work.max()), int(work.min()), "argmax", int(work.argmax()), "barrier max", int(bar.max()))
tot = tr[:, S, 1] - tr[:, 0, 1]
print("total cycles per CTA", tot)
