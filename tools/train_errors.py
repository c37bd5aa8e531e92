"""Per-group gradient error of cc_train_step vs the training oracle at full
size (prints max |g - g_oracle| / max |g_oracle| per parameter group)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2403_11651_b200 as P  # noqa: E402
import workload  # noqa: E402
from test_train_oracle import groups  # noqa: E402

cfg = workload.CONFIGS["ref"].replace(lam=0.02)
im = workload.make_image(cfg, 8)
rng = np.random.default_rng(1008)
y = workload.gen_continuous_latents(rng, im.latents)
u = workload.gen_noise(rng, im.latents.size)
tr = P.DeviceTrainer(cfg, y, im.arm_w, im.up_w, im.syn_w, im.image)
res = tr.step(noise=u, update=False).cpu().numpy()
g = tr.grad.cpu().numpy().astype(np.float64)
out, gr = oracle.train_grad(oracle.model(cfg), oracle.pack_params(y, im.arm_w, im.up_w, im.syn_w), u, im.image)
print("cost rel err", np.abs(res - out) / np.abs(out))
for name, a, b in groups(cfg):
    sc = np.abs(gr[a:b]).max()
    print(f"{name:10s} n={b - a:7d} max|g|={sc:.3e} rel err={np.abs(g[a:b] - gr[a:b]).max() / max(sc, 1e-300):.2e}")
