"""Upper bound of multi-image training concurrency: K trainers on K streams
(the constant weight bank is shared, so the numbers are timing-only)."""
import time

import numpy as np
import torch

import paper_2403_11651_b200 as P
import workload

cfg = workload.CONFIGS["ref"]
dev = torch.device("cuda", 0)
for K in (1, 2, 3, 4):
    trs, streams = [], []
    for k in range(K):
        im = workload.make_image(cfg, 100 + k)
        rng = np.random.default_rng(k)
        y = workload.gen_continuous_latents(rng, im.latents)
        trs.append(P.DeviceTrainer(cfg, y, im.arm_w, im.up_w, im.syn_w, im.image, device=dev))
        streams.append(torch.cuda.Stream())
    for _ in range(3):
        for tr, st in zip(trs, streams):
            tr.step(lr=1e-3, stream_ptr=st.cuda_stream)
    torch.cuda.synchronize()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        for tr, st in zip(trs, streams):
            tr.step(lr=1e-3, stream_ptr=st.cuda_stream)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"K={K}: {K * n / dt:.0f} image-iterations/s")
