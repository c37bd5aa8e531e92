"""Per-phase timing of arm_tcg_kernel from the CCRD_TCG_TIMING experiment build
(tools/libccrd_tcgtime.so): one 2K image, warpgroup 0 / warp 0 of every CTA;
prints mean cycles per 128-latent block for each phase."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CCRD_LIB"] = os.path.join(ROOT, "tools", "libccrd_tcgtime.so")
import torch  # noqa: E402

import paper_2403_11651_b200 as P  # noqa: E402
import workload  # noqa: E402

cfg = workload.CONFIGS["batched2k"]
im = workload.make_image(cfg, 0)
d = P.desc_from_config(cfg)
lat = torch.from_numpy(im.latents).cuda()
rate = torch.zeros(1, dtype=torch.float64, device="cuda")
wsb = P.cc_workspace_bytes(d, 1)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
for _ in range(3):
    P.cc_arm_rate(d, lat.data_ptr(), im.arm_w, rate.data_ptr(), 0, 0, 0, ws.data_ptr(), wsb, 0)
torch.cuda.synchronize()
L = P.load()
buf = np.zeros((148, 12), np.uint64)
L.cc_debug_tcg_timing.argtypes = [C.c_void_p, C.c_int]
assert L.cc_debug_tcg_timing(buf.ctypes.data, 148) == 0
t = buf.astype(np.float64)
nb = t[:, 7]
names = ["gather+sttm", "barrier0", "mma0 issue+wait", "epi0", "barrier1", "mma1 issue+wait", "epi1"]
per = t[:, :7] / nb[:, None]
tot = per.sum(1)
print(f"blocks per warpgroup-0: mean {nb.mean():.1f}")
for k, n in enumerate(names):
    print(f"  {n:18s} {per[:, k].mean():8.0f} cyc  {100 * per[:, k].mean() / tot.mean():5.1f}%")
print(f"  {'total':18s} {tot.mean():8.0f} cyc per block")
print(f"tiles {t[:, 10].mean():.1f}, staging {(t[:, 8] / t[:, 10]).mean():.0f} cyc per tile; "
      f"warpgroup-0 lifetime {t[:, 9].mean():.0f} cyc = blocks {t[:, :7].sum(1).mean():.0f} + staging {t[:, 8].mean():.0f} + other")
