"""Per-phase timing of synth_kernel from the CCRD_SYN_TIMING experiment build
(tools/libccrd_timing.so): runs one 2K image and prints phase durations."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CCRD_LIB"] = os.path.join(ROOT, "tools", "libccrd_timing.so")
import torch  # noqa: E402

import paper_2403_11651_b200 as P  # noqa: E402
import workload  # noqa: E402

cfg = workload.CONFIGS["batched2k"]
ims = workload.make_batch(cfg, [0, 1])
b = P.DeviceBatch(cfg, ims)
for _ in range(3):
    b.forward()
torch.cuda.synchronize()
L = P.load()
n = 1376
buf = np.zeros((n, 8), np.uint64)
L.cc_debug_syn_timing.argtypes = [C.c_void_p, C.c_int]
assert L.cc_debug_syn_timing(buf.ctypes.data, n) == 0
t = buf.astype(np.int64)
names = ["loads", "chain", "mlp", "conv0", "conv1+sse"]
d = np.stack([t[:, 1] - t[:, 0], t[:, 2] - t[:, 1], t[:, 3] - t[:, 2], t[:, 4] - t[:, 3], t[:, 5] - t[:, 4]], 1)
tot = t[:, 5] - t[:, 0]
print("per-CTA cycles (mean / p10 / p90):")
for k, nm in enumerate(names):
    print(f"  {nm:10s} {d[:, k].mean():9.0f} {np.percentile(d[:, k], 10):9.0f} {np.percentile(d[:, k], 90):9.0f}  "
          f"{100 * d[:, k].mean() / tot.mean():5.1f}%")
print(f"  {'total':10s} {tot.mean():9.0f}")
sm = t[:, 6]
# per-SM: sum of CTA lifetimes vs SM busy span
spans = []
for s_ in np.unique(sm):
    m = sm == s_
    spans.append((t[m, 5].max() - t[m, 0].min(), tot[m].sum(), m.sum()))
spans = np.array(spans, dtype=np.float64)
print(f"SMs {len(spans)}, CTAs/SM {spans[:, 2].mean():.2f}, mean span {spans[:, 0].mean():.0f} cyc, "
      f"sum(CTA lifetimes)/span = {np.mean(spans[:, 1] / spans[:, 0]):.2f} (avg resident CTAs)")
