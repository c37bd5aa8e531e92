"""Where does the end-to-end host path's time go?  Pinned H2D bandwidth, the
host path's wall time vs. its enqueue time, for the batched 2K workload."""
import time

import numpy as np
import torch

import paper_2403_11651_b200 as P
import workload

cfg = workload.CONFIGS["batched2k"]
n = 16
ims = workload.make_batch(cfg, list(range(n)), threads=16)
for im in ims:
    im.image = workload.quantize_image_u8(im.image)
dev = torch.device("cuda", 0)
# raw pinned H2D
h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty_like(h, device=dev)
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print(f"pinned H2D: {10 * h.numel() / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
desc = P.desc_from_config(cfg)
desc.image_u8 = 1
desc.latents_i8 = 1
lat = [torch.from_numpy(im.latents.astype(np.int8)).pin_memory() for im in ims]
img = [torch.from_numpy(workload.to_u8(im.image)).pin_memory() for im in ims]
io = [P.CcImageIO(lat[i].data_ptr(), ims[i].arm_w.ctypes.data, ims[i].up_w.ctypes.data, ims[i].syn_w.ctypes.data,
                  img[i].data_ptr(), None) for i in range(n)]
ws_b = P.cc_workspace_bytes_host(desc, n)
ws = torch.empty(ws_b, dtype=torch.uint8, device=dev)
res = np.zeros((n, 4))
s = torch.cuda.current_stream().cuda_stream
P.cc_rd_forward_host(desc, io, res, ws.data_ptr(), ws_b, s)
torch.cuda.synchronize()
walls = []
for _ in range(5):
    t0 = time.perf_counter()
    P.cc_rd_forward_host(desc, io, res, ws.data_ptr(), ws_b, s)
    walls.append(time.perf_counter() - t0)
w = min(walls)
bytes_ = sum(l.numel() + i.numel() for l, i in zip(lat, img))
print(f"host path: {n} images {w * 1e3:.2f} ms -> {n * cfg.H * cfg.W / w / 1e9:.2f} Gpx/s, "
      f"H2D {bytes_ / w / 1e9:.1f} GB/s of {bytes_ / 1e6:.0f} MB")
# device path, same images
b = P.DeviceBatch(cfg, ims, with_xhat=False, image_u8=True)
b.forward()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    b.forward()
e1.record()
torch.cuda.synchronize()
dm = e0.elapsed_time(e1) / 3
print(f"device path: {dm:.2f} ms -> {n * cfg.H * cfg.W / dm / 1e6:.2f} Gpx/s")
# enqueue-only time of the device path (host side)
torch.cuda.synchronize()
t0 = time.perf_counter()
b.forward()
te = time.perf_counter() - t0
torch.cuda.synchronize()
print(f"device path host enqueue: {te * 1e3:.2f} ms for {n} images")
# device path, one image per call (the host path's compute structure, no PCIe)
bs = [P.DeviceBatch(cfg, [im], with_xhat=False, image_u8=True) for im in ims]
for bb in bs:
    bb.forward()
torch.cuda.synchronize()
e0.record()
for _ in range(3):
    for bb in bs:
        bb.forward()
e1.record()
torch.cuda.synchronize()
dm1 = e0.elapsed_time(e1) / 3
print(f"device path, 1 image per call: {dm1:.2f} ms -> {n * cfg.H * cfg.W / dm1 / 1e6:.2f} Gpx/s")
# H2D of the same bytes alone, and H2D concurrent with the device path's compute
cs = torch.cuda.Stream()
dl = [torch.empty_like(l, device=dev) for l in lat]
di = [torch.empty_like(i, device=dev) for i in img]
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(cs):
    for k in range(n):
        dl[k].copy_(lat[k], non_blocking=True)
        di[k].copy_(img[k], non_blocking=True)
torch.cuda.synchronize()
print(f"H2D alone: {(time.perf_counter() - t0) * 1e3:.2f} ms")
torch.cuda.synchronize()
t0 = time.perf_counter()
b.forward()
with torch.cuda.stream(cs):
    for k in range(n):
        dl[k].copy_(lat[k], non_blocking=True)
        di[k].copy_(img[k], non_blocking=True)
torch.cuda.synchronize()
print(f"device forward || H2D: {(time.perf_counter() - t0) * 1e3:.2f} ms")
