#!/usr/bin/env python
"""Benchmark of the B200-native Cool-chic RD forward (BASELINE.json metric:
"decoded pixels/sec (RD forward incl. ARM rate) and fraction of B200 roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full RD forward (ARM rate over every latent, upsampling,
synthesis, MSE, RD cost) of the BASELINE.json configs[3] batch -- 64 images of
1365x2048 at the ~2000 MAC/pixel architecture -- per GPU (weak scaling: each
rank owns 64 independent images; the per-image results are all-reduced).  Rank
0 prints one JSON line.  ``--impl reference`` times the fp64 CPU oracle on the
host cores (the tier's reference arm; rank 0 only).
"""
from __future__ import annotations

import argparse
import faulthandler
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload  # noqa: E402

METRIC = "decoded pixels/sec (RD forward incl. ARM rate) and fraction of B200 roofline"
UNIT = "pixels/s"
# FP32 FMA roofline: 148 SMs x 128 FP32 lanes x 2 FLOP x
# 1.965 GHz (B200_PROFILING.md SM count, clocks.max.sm).  The FFMA2 probe
# (tools/microbench/ffma_probe.cu) measured 126.9 FMA/clk/SM = 99.2 % of it.
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def tf32_peak_tflops():
    """Dense TF32 tensor peak: the measured cuBLAS bf16 GEMM peak
    (MEASURED_PEAKS.json; burst figure, a kernel timed alone) x the nominal
    TF32 / BF16 ratio of B200_PROFILING.md (1.1 / 2.25 PFLOP/s dense)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16 = float(json.load(f)["bf16_tflops"])
        src = "measured bf16 %.1f TF/s (MEASURED_PEAKS.json, burst) x 1.1/2.25" % bf16
    except Exception:
        bf16 = 1590.0
        src = "fallback bf16 1590 TF/s (B200_PROFILING.md) x 1.1/2.25"
    return bf16 * 1.1 / 2.25, src


def arm_tc_mac_per_latent(cfg):
    """tcgen05 multiply-accumulates the tensor-core ARM issues per latent
    (arm_tc.cu arm_tcp_kernel / arm_tcg_kernel): layer 0 = context (K0 = C + 8 columns incl. the
    bias block) x (W_hi + W_lo); hidden layer = A_hi (K1 = NH + 8) x (W_hi +
    W_lo) + A_lo (NH) x W_hi; N = NH.  The 2-wide output layer runs on the CUDA
    cores."""
    C, NH = cfg.n_ctx, cfg.arm_widths[1]
    return 2 * (C + 8) * NH + 2 * (NH + 8) * NH + NH * NH
REASONS = [(0x1, "gpu_idle"), (0x2, "applications_clocks_setting"), (0x4, "sw_power_cap"),
           (0x8, "hw_slowdown"), (0x10, "sync_boost"), (0x20, "sw_thermal_slowdown"),
           (0x40, "hw_thermal_slowdown"), (0x80, "hw_power_brake_slowdown")]


class ClockSampler(threading.Thread):
    """Samples the SM clock and clock-event reasons through NVML while the
    timed region runs (B200_PROFILING.md clocks rule)."""

    def __init__(self, cuda_index: int, period: float = 0.01):
        super().__init__(daemon=True)
        self.period = period
        self.samples = []
        self.max_mhz = None
        self._halt = threading.Event()
        self.ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            h = None
            try:  # match the CUDA device to its NVML handle by UUID
                import torch
                want = str(torch.cuda.get_device_properties(cuda_index).uuid)
                for i in range(N.nvmlDeviceGetCount()):
                    hi = N.nvmlDeviceGetHandleByIndex(i)
                    u = N.nvmlDeviceGetUUID(hi)
                    u = u.decode() if isinstance(u, bytes) else u
                    if u.replace("GPU-", "") == want.replace("GPU-", ""):
                        h = hi
                        break
            except Exception:
                h = None
            if h is None:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                idx = int(vis.split(",")[cuda_index]) if vis and vis.split(",")[0].isdigit() else cuda_index
                h = N.nvmlDeviceGetHandleByIndex(idx)
            self.h = h
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - reported in the JSON
            self.err = repr(e)

    def run(self):
        if not self.ok:
            return
        N = self.N
        while not self._halt.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                try:
                    rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    rs = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def stop(self):
        self._halt.set()
        self.join(timeout=2)

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mask = 0
        for _, r in self.samples:
            mask |= r
        return {"sm_mhz": float(statistics.median(s for s, _ in self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in REASONS if mask & b and n != "gpu_idle"], "samples": len(self.samples)}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def load_traffic(kernel: str):
    """Per-launch DRAM bytes of `kernel` from the committed ncu --set full
    summary (profiles/), or None."""
    for name in sorted(os.listdir(os.path.join(ROOT, "profiles")), reverse=True) if os.path.isdir(
            os.path.join(ROOT, "profiles")) else []:
        if name.startswith("ncu_full_") and name.endswith(".json"):
            try:
                with open(os.path.join(ROOT, "profiles", name)) as f:
                    d = json.load(f)
                k = d.get("kernels", {}).get(kernel)
                if k and k.get("dram_bytes_per_launch"):
                    return float(k["dram_bytes_per_launch"])
            except Exception:
                pass
    return None


# --------------------------------------------------------------------------- ours
def run_ours(args, rk):
    import torch

    import paper_2403_11651_b200 as P
    from paper_2403_11651_b200 import dist

    cfg = workload.CONFIGS[args.config]
    n_img = args.images or cfg.n_img
    dev = torch.device("cuda", rk.local_rank)
    torch.cuda.set_device(dev)
    P.load()
    seeds = [workload.image_seed(args.seed, g) for g in dist.owned_images(rk.rank, n_img)]
    t0 = time.perf_counter()
    images = workload.make_batch(cfg, seeds, threads=min(16, host_cores()))
    if args.image == "u8":   # 8-bit sources (the paper's Kodak / CLIC images are 8-bit RGB)
        for im in images:
            im.image = workload.quantize_image_u8(im.image)
    gen_s = time.perf_counter() - t0
    log(f"generated {len(images)} images in {gen_s:.1f}s")
    batch = P.DeviceBatch(cfg, images, device=dev, with_xhat=True, image_u8=args.image == "u8")
    desc = batch.desc
    macs = P.cc_mac_per_pixel(desc)
    log("device batch ready")
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def step():
        res = batch.forward(sptr)
        if rk.world > 1:
            dist.allreduce_results(dist.scatter_results(res, rk.rank, rk.world, n_img))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    log("warm-up done")
    sampler = ClockSampler(rk.local_rank)
    log(f"sampler ok={sampler.ok}")
    dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    for _ in range(args.steps):
        step()
        launches += P.ccrd.cc_last_launch_count()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    sampler.stop()
    log("timed region done")
    ms = ev0.elapsed_time(ev1)
    # per-kernel roofline: the production path runs the ARM and the synthesis
    # kernels concurrently on two streams (their event times overlap), so each
    # kernel's own launch duration is measured in a short SERIAL pass of the
    # same workload (same kernels, CCRD_SERIAL=1), inputs resident
    os.environ["CCRD_SERIAL"] = "1"
    step()
    torch.cuda.synchronize(dev)
    P.ccrd.cc_profile_begin()
    for _ in range(args.profile_steps):
        step()
    torch.cuda.synchronize(dev)
    prof = P.ccrd.cc_profile_end()
    os.environ.pop("CCRD_SERIAL", None)
    ms_max = dist.max_over_ranks(ms, device=dev)
    P_img = cfg.H * cfg.W
    px_total = rk.world * n_img * P_img * args.steps
    value = px_total / (ms_max / 1e3)

    # per-kernel rooflines; the headline `roofline` is the kernel with the
    # largest share of the serial step
    arm_tc = P.cc_arm_path_for(desc) == P.CC_ARM_TC
    # the tensor-core ARM's default kernel is the ping-pong one (arm_tc.cu;
    # CCRD_ARM_TC_PP=0 selects the one-block arm_tcg_kernel)
    arm_name = (("arm_tcg_kernel" if os.environ.get("CCRD_ARM_TC_PP", "1") == "0" else "arm_tcp_kernel")
                if arm_tc else "arm_rate_kernel")
    arm_avg_s = prof.arm_ms / max(1, prof.arm_launches) / 1e3
    syn_avg_s = prof.syn_ms / max(1, prof.syn_launches) / 1e3
    arm_tflops = 2.0 * macs.arm_macs / arm_avg_s / 1e12            # fp32-accurate algorithmic FLOP
    syn_tflops = 2.0 * (macs.up_macs + macs.syn_macs) / syn_avg_s / 1e12
    path_tflops = 2.0 * macs.total * value / rk.world / 1e12
    serial_ms = prof.arm_ms + prof.syn_ms + prof.pyr_ms + prof.reduce_ms
    arm_mac_latent = sum(cfg.arm_widths[k] * cfg.arm_widths[k + 1] for k in range(len(cfg.arm_widths) - 1))
    timing = (f"launch durations from CUDA events in a {args.profile_steps}-step serial pass "
              "(the timed steps run ARM || synthesis on two streams)")
    fp32_src = "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (B200_PROFILING.md); FFMA2 probe measured 99.2 % of it"
    kern = {}
    if arm_tc:
        tf32_peak, tf32_src = tf32_peak_tflops()
        tc_macs = arm_tc_mac_per_latent(cfg) * macs.n_latents
        tc_tflops = 2.0 * tc_macs / arm_avg_s / 1e12
        kern[arm_name] = {
            "bound": "tensor", "achieved": tc_tflops, "peak": tf32_peak, "unit": "TFLOP/s", "frac": tc_tflops / tf32_peak,
            "algorithmic": f"{tc_macs} TF32 tensor MAC (2 FLOP) per launch = 1 image's {macs.n_latents} latents x "
                           f"{arm_tc_mac_per_latent(cfg)} MAC (3xTF32 split of the {arm_mac_latent}-MAC fp32 ARM)",
            "peak_source": tf32_src, "fp32_equiv_tflops": arm_tflops,
            "fp32_equiv_frac_of_fp32_peak": arm_tflops / FP32_PEAK_TFLOPS}
    else:
        kern[arm_name] = {
            "bound": "alu", "achieved": arm_tflops, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": arm_tflops / FP32_PEAK_TFLOPS,
            "algorithmic": f"{macs.arm_macs} FP32 FMA (2 FLOP) per launch = 1 image's latents x {arm_mac_latent} MAC",
            "peak_source": fp32_src}
    kern[arm_name].update({"avg_launch_ms": arm_avg_s * 1e3, "launches": prof.arm_launches,
                           "share": prof.arm_ms / serial_ms, "traffic": load_traffic(arm_name)})
    kern["synth_kernel"] = {
        "bound": "alu", "achieved": syn_tflops, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
        "frac": syn_tflops / FP32_PEAK_TFLOPS,
        "algorithmic": f"{macs.up_macs + macs.syn_macs} FP32 FMA (2 FLOP) per launch = 1 image's pixels x "
                       f"{(macs.up_macs + macs.syn_macs) / (cfg.H * cfg.W):.2f} MAC (last upsampling step + synthesis)",
        "peak_source": fp32_src, "avg_launch_ms": syn_avg_s * 1e3, "launches": prof.syn_launches,
        "share": prof.syn_ms / serial_ms, "traffic": load_traffic("synth_kernel")}
    for e in kern.values():  # DRAM bytes of the ncu capture / this run's launch duration (HBM is not binding)
        if e.get("traffic"):
            e["dram_gbs"] = e["traffic"] / (e["avg_launch_ms"] * 1e-3) / 1e9
    dom = max(kern, key=lambda k: kern[k]["share"])
    roofline = {"kernel": dom, "timing": timing}
    roofline.update({k: kern[dom][k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "algorithmic",
                                               "avg_launch_ms", "peak_source")})
    kern["pyramid_kernel"] = {"ms_total": prof.pyr_ms, "launches": prof.pyr_launches, "share": prof.pyr_ms / serial_ms}
    kern["reduce_batch_kernel"] = {"ms_total": prof.reduce_ms, "launches": prof.reduce_launches}
    kern["serial_ms_per_step"] = serial_ms / args.profile_steps

    # end to end: host (pinned) buffers through cc_rd_forward_host
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, images, desc, dev, stream, rk, n_img)

    # sanity: results finite, rate positive
    res = batch.results.cpu().numpy()
    if not os.environ.get("CCRD_LIB"):
        assert np.isfinite(res).all() and (res[:, 0] > 0).all(), "non-finite or empty results"

    log("e2e done")
    clocks = sampler.summary()
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": rk.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {
            "workload": f"{args.config}: {n_img} x {cfg.H}x{cfg.W} RGB images per GPU, L={cfg.L}, "
                        f"ARM {list(cfg.arm_widths)} C={cfg.n_ctx}, synthesis {list(cfg.syn_widths)}+{cfg.syn_n_res}x"
                        f"res3x3, {cfg.up_taps}-tap separable upsampling (BASELINE.json configs[3])",
            "images_per_gpu": n_img, "H": cfg.H, "W": cfg.W, "mac_per_pixel": round(macs.total, 3),
            "image": "uint8 planar, x = v / 255 (desc.image_u8)" if args.image == "u8" else "fp32 planar",
            "l2": f"inputs larger than L2: {(sum(im.latents.nbytes + im.image.size * (1 if args.image == 'u8' else 4) for im in images)) / 1e9:.2f} GB "
                  "read per step per GPU (126 MB L2)",
            "parallelism": f"image-sharded x{rk.world}",
        },
        "roofline": roofline,
        "kernels": kern,  # serial pass (see roofline.timing); share = of the serial step
        "streams": "ARM kernels || (pyramid -> synthesis) kernels on two CUDA streams, joined per step",
        "path_roofline": {"achieved_tflops_per_gpu": path_tflops, "frac": path_tflops / FP32_PEAK_TFLOPS,
                          "note": "whole step, fp32-equivalent: pixels/s x closed-form MAC/px x 2 / FP32 CUDA-core "
                                  "peak (the ARM's MACs run on the tensor cores when arm_path = tc)"},
        "arm_path": "tc" if arm_tc else "ffma2",
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "input_gen_s": round(gen_s, 2),
    }
    if rk.rank == 0 and rk.world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = run_cpu_baseline(cfg, images)
    if rk.rank == 0:
        print(json.dumps(out), flush=True)


def run_strip(args, rk):
    """BASELINE.json configs[4]: ONE 4320x7680 image split into horizontal
    strips, one per rank (strong scaling).  A step = the halo exchange of
    latent rows (grouped NCCL send/recv into the window buffers; none at N=1),
    cc_rd_forward_strip on every rank, and the all-reduce of the additive
    (rate, sse, mse, cost) shares."""
    import torch
    import torch.distributed as tdist

    import paper_2403_11651_b200 as P
    from paper_2403_11651_b200 import dist

    cfg = workload.CONFIGS[args.config]
    dev = torch.device("cuda", rk.local_rank)
    torch.cuda.set_device(dev)
    P.load()
    desc = P.desc_from_config(cfg)
    strips, lays = dist.strip_layouts(desc, rk.world)
    st, lay = strips[rk.rank], lays[rk.rank]
    t0 = time.perf_counter()
    im = workload.make_image(cfg, workload.image_seed(args.seed, 0))
    gen_s = time.perf_counter() - t0
    dims = cfg.level_dims()
    off = [sum(h * w for h, w in dims[:l]) for l in range(cfg.L)]
    ds = P.ccrd.DeviceStrip(cfg, st, im.arm_w, im.up_w, im.syn_w, image_rows=im.image[:, st.r0:st.r1], device=dev)
    # this rank's bitstream share: its owned latent rows only; halos arrive by exchange
    ds.lat.copy_(dist.pack_window(torch.from_numpy(im.latents), off, lay, owned_only=True).to(dev))
    macs = P.cc_mac_per_pixel(desc)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    halo_bytes = [0]

    def step():
        halo_bytes[0] = dist.exchange_halos(ds.lat, lays, rk.rank)
        r = ds.forward(sptr)
        if rk.world > 1:
            tdist.all_reduce(r, op=tdist.ReduceOp.SUM)
        return r

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(rk.local_rank)
    dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    P.ccrd.cc_profile_begin()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    for _ in range(args.steps):
        res = step()
        launches += P.ccrd.cc_last_launch_count()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    sampler.stop()
    prof = P.ccrd.cc_profile_end()
    ms = ev0.elapsed_time(ev1)
    ms_max = dist.max_over_ranks(ms, device=dev)
    value = cfg.H * cfg.W * args.steps / (ms_max / 1e3)
    resn = res.cpu().numpy()
    assert np.isfinite(resn).all() and resn[0] > 0
    arm_avg_s = prof.arm_ms / max(1, prof.arm_launches) / 1e3
    own_lat = sum((st.own_hi[l] - st.own_lo[l]) * dims[l][1] for l in range(cfg.L))
    arm_pl = sum(cfg.arm_widths[k] * cfg.arm_widths[k + 1] for k in range(len(cfg.arm_widths) - 1))
    arm_tflops = 2.0 * own_lat * arm_pl / arm_avg_s / 1e12
    path_tflops = 2.0 * macs.total * value / rk.world / 1e12
    if P.cc_arm_path_for(desc) == P.CC_ARM_TC:
        # the tensor-core ARM against the TF32 tensor peak with the executed
        # 3xTF32 MACs (as the headline's `kernels` entry), fp32-equivalent beside
        tf32_peak, tf32_src = tf32_peak_tflops()
        tc_tflops = 2.0 * own_lat * arm_tc_mac_per_latent(cfg) / arm_avg_s / 1e12
        arm_roof = {"bound": "tensor", "kernel": "arm_tcp_kernel", "achieved": tc_tflops, "peak": tf32_peak,
                    "unit": "TFLOP/s", "frac": tc_tflops / tf32_peak, "traffic": None,
                    "algorithmic": f"{own_lat} latents x {arm_tc_mac_per_latent(cfg)} TF32 tensor MAC per launch "
                                   f"(3xTF32 split of the {arm_pl}-MAC fp32 ARM)",
                    "peak_source": tf32_src, "fp32_equiv_tflops": arm_tflops,
                    "fp32_equiv_frac_of_fp32_peak": arm_tflops / FP32_PEAK_TFLOPS, "avg_launch_ms": arm_avg_s * 1e3}
    else:
        arm_roof = {"bound": "alu", "kernel": "arm_rate_kernel", "achieved": arm_tflops, "peak": FP32_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": arm_tflops / FP32_PEAK_TFLOPS, "traffic": None,
                    "avg_launch_ms": arm_avg_s * 1e3}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": rk.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"8k: one {cfg.H}x{cfg.W} RGB image in {rk.world} horizontal strip(s), L={cfg.L}, "
                               f"ARM {list(cfg.arm_widths)} C={cfg.n_ctx}, synthesis {list(cfg.syn_widths)}+"
                               f"{cfg.syn_n_res}xres3x3 (BASELINE.json configs[4])",
                   "H": cfg.H, "W": cfg.W, "mac_per_pixel": round(macs.total, 3),
                   "strip_rows": [st.r0, st.r1], "halo_bytes_recv_per_step_rank0": halo_bytes[0],
                   "l2": "inputs larger than L2 (0.4 GB of image + latents per step)",
                   "parallelism": f"strips x{rk.world}, NCCL halo exchange + all-reduce"},
        "roofline": arm_roof,
        "path_roofline": {"achieved_tflops_per_gpu": path_tflops, "frac": path_tflops / FP32_PEAK_TFLOPS},
        "e2e": None, "gpu_launches": launches, "clocks": sampler.summary(), "input_gen_s": round(gen_s, 2),
    }
    if rk.rank == 0:
        print(json.dumps(out), flush=True)


def run_decode(args, rk):
    """NEXT-3: the decoder's data-parallel output stage (cc_decode: latents ->
    upsampling -> synthesis -> clamp -> 8-bit RGB) over the batched 2K
    workload, one cc_decode per image.  The sequential entropy decoding of the
    latents is out of scope, so this is not a full decode time."""
    import torch

    import paper_2403_11651_b200 as P
    from paper_2403_11651_b200 import dist

    cfg = workload.CONFIGS[args.config]
    n_img = args.images or cfg.n_img
    dev = torch.device("cuda", rk.local_rank)
    torch.cuda.set_device(dev)
    P.load()
    images = workload.make_batch(cfg, [workload.image_seed(args.seed, g) for g in dist.owned_images(rk.rank, n_img)],
                                 threads=min(16, host_cores()))
    desc = P.desc_from_config(cfg)
    lats = [torch.from_numpy(im.latents).to(dev) for im in images]
    outs = [torch.empty((cfg.H, cfg.W, 3), dtype=torch.uint8, device=dev) for _ in images]
    ws_b = P.cc_workspace_bytes(desc, 1)
    ws = torch.empty(ws_b, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        for i, im in enumerate(images):
            P.cc_decode(desc, lats[i].data_ptr(), im.up_w, im.syn_w, outs[i].data_ptr(), ws.data_ptr(), ws_b,
                        stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(rk.local_rank)
    dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    sampler.stop()
    ms = dist.max_over_ranks(ev0.elapsed_time(ev1), device=dev)
    value = rk.world * n_img * cfg.H * cfg.W * args.steps / (ms / 1e3)
    macs = P.cc_mac_per_pixel(desc)
    flops = 2.0 * (macs.up + macs.syn) * value / rk.world
    out = {
        "metric": "decoder output stage (upsampling + synthesis + clamp + 8-bit) pixels/s", "value": value,
        "unit": "pixels/s", "n_gpus": rk.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"decode_{cfg.name}: {n_img} x {cfg.H}x{cfg.W} per GPU, 8-bit RGB output",
                   "H": cfg.H, "W": cfg.W, "mac_per_pixel_up_syn": round(macs.up + macs.syn, 3)},
        "path_roofline": {"achieved_tflops_per_gpu": flops / 1e12, "frac": flops / 1e12 / FP32_PEAK_TFLOPS},
        "context": "paper: ~100 ms per 512x768 decode on one CPU core incl. the sequential ARM (BASELINE.md)",
        "e2e": None, "clocks": sampler.summary(),
    }
    if rk.rank == 0:
        print(json.dumps(out), flush=True)


def run_arm_decode(args, rk):
    """NEXT-3: the decoder's autoregressive ARM as an anti-diagonal wavefront
    (cc_arm_decode) over the BASELINE.json configs[3] batch -- all images and
    grids in one call; the entropy decoder is played by the true latents
    (include/ccrd.h).  Also times one image alone (decode latency)."""
    import torch

    import paper_2403_11651_b200 as P
    from paper_2403_11651_b200 import dist

    cfg = workload.CONFIGS[args.config]
    n_img = args.images or cfg.n_img
    dev = torch.device("cuda", rk.local_rank)
    torch.cuda.set_device(dev)
    P.load()
    ims = workload.make_batch(cfg, [workload.image_seed(args.seed, g) for g in dist.owned_images(rk.rank, n_img)],
                              threads=min(16, host_cores()))
    d = P.desc_from_config(cfg)
    lat = [torch.from_numpy(im.latents).to(dev) for im in ims]
    dec = [torch.empty_like(t) for t in lat]
    rate = torch.zeros(n_img, dtype=torch.float64, device=dev)
    io = [P.CcImageIO(lat[i].data_ptr(), ims[i].arm_w.ctypes.data, 0, 0, 0, 0) for i in range(n_img)]
    wsb = P.cc_arm_decode_workspace_bytes(d, n_img)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    dptr = [t.data_ptr() for t in dec]

    def step(k=n_img):
        P.cc_arm_decode(d, io[:k], dptr[:k], rate.data_ptr(), None, None, None, 0, ws.data_ptr(), wsb,
                        stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(rk.local_rank)
    dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    sampler.stop()
    ms = dist.max_over_ranks(ev0.elapsed_time(ev1), device=dev)
    # one image alone: the decode latency
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        step(1)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    lat1_ms = e0.elapsed_time(e1) / 3
    assert all(torch.equal(a, b) for a, b in zip(dec, lat)), "decoded latents differ from the encoded ones"
    value = rk.world * n_img * cfg.H * cfg.W * args.steps / (ms / 1e3)
    macs = P.cc_mac_per_pixel(d)
    arm_tflops = 2.0 * macs.arm_macs * n_img * args.steps / (ms / 1e3) / 1e12
    out = {
        "metric": "autoregressive latent decode (wavefront ARM) pixels/s", "value": value, "unit": "pixels/s",
        "n_gpus": rk.world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"decode_{args.config}: {n_img} x {cfg.H}x{cfg.W} per GPU, all grids in one call; "
                               "entropy decoder played by the true latents (include/ccrd.h)",
                   "latents_per_image": int(ims[0].latents.size)},
        "latency_one_image_ms": lat1_ms,
        "arm_tflops": arm_tflops, "arm_frac_of_fp32_peak": arm_tflops / FP32_PEAK_TFLOPS,
        "context": "paper: ~100 ms per 512x768 decode on one CPU core (ARM + upsampling + synthesis), BASELINE.md",
        "e2e": None, "gpu_launches": P.ccrd.cc_last_launch_count() * args.steps, "clocks": sampler.summary(),
    }
    if rk.rank == 0:
        print(json.dumps(out), flush=True)


def run_analysis(args, rk):
    """NEXT-4: the N-O analysis transform forward (encoding = one forward pass,
    PAPER.md:422-449, 483-484) on Kodak-sized images (no_kodak) by default;
    --tf32 runs the point-wise GEMMs on TF32 tensor cores."""
    import torch

    import paper_2403_11651_b200 as P
    from paper_2403_11651_b200 import dist

    acfg = workload.ANALYSIS[args.analysis]
    n_img = args.images or 8
    dev = torch.device("cuda", rk.local_rank)
    torch.cuda.set_device(dev)
    P.load()
    ad = P.analysis_desc(acfg, args.tf32, n_img)   # ONE call encodes this GPU's n_img images
    ins = [workload.make_analysis_input(acfg, workload.image_seed(args.seed, g))
           for g in dist.owned_images(rk.rank, n_img)]
    imgs = torch.from_numpy(np.stack([i for i, _ in ins])).to(dev)   # [N][3][H][W]
    w = torch.from_numpy(ins[0][1]).to(dev)   # N-O: one shared network
    n_lat = sum(-(-acfg.H // (1 << l)) * -(-acfg.W // (1 << l)) for l in range(acfg.L))
    lats = torch.empty(n_img, n_lat, device=dev)
    ws_b = P.cc_analysis_workspace_bytes(ad)
    ws = torch.empty(ws_b, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(src=imgs, dst=lats):
        P.cc_analysis_forward(ad, src.data_ptr(), w.data_ptr(), dst.data_ptr(), ws.data_ptr(), ws_b,
                              stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(rk.local_rank)
    dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    sampler.stop()
    # end to end: pinned host images in, host latents out, copies inside the timed region
    h_img = imgs.cpu().pin_memory()
    h_lat = torch.empty(n_img, n_lat).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(args.steps):
        imgs.copy_(h_img, non_blocking=True)
        step()
        h_lat.copy_(lats, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = dist.max_over_ranks(e0.elapsed_time(e1), device=dev)
    ms = dist.max_over_ranks(ev0.elapsed_time(ev1), device=dev)
    px = acfg.H * acfg.W
    value = rk.world * n_img * px * args.steps / (ms / 1e3)
    C = acfg.C
    macs = 3 * C * px
    for l in range(acfg.L):
        hl, wl = -(-acfg.H // (1 << l)), -(-acfg.W // (1 << l))
        macs += acfg.blocks * (C * 49 + 8 * C * C) * hl * wl + (C * C * hl * wl if l > 0 else 0) + C * hl * wl
    tflops = 2.0 * macs / px * value / rk.world / 1e12
    out = {
        "metric": "N-O analysis transform (encoding forward) pixels/s", "value": value, "unit": "pixels/s",
        "n_gpus": rk.world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": ["f32", "tf32", "tf32", "f16-operand/f32-accumulate"][args.tf32],
        "mode": ["fp32 cuBLASLt", "TF32 fused tcgen05 block kernels", "TF32 cuBLASLt unfused",
                 "fused tcgen05 block kernels, FP16 operands, TMA-staged depth-wise"][args.tf32],
        "data": "synthetic",
        "config": {"workload": f"{acfg.name}: {n_img} x {acfg.H}x{acfg.W} per GPU in one call, C={C}, L={acfg.L}, "
                               f"{acfg.blocks} blocks/level", "kmac_per_pixel": round(macs / px / 1e3, 2),
                   "l2": f"inputs {n_img * acfg.H * acfg.W * 12 / 1e6:.0f} MB, activations "
                         f"{n_img * acfg.H * acfg.W * C * 4 / 1e6:.0f} MB per block pass"},
        "achieved_tflops_per_gpu": tflops,
        "context": "paper: N-O encoding < 1 s per image (one forward pass, ~160 kMAC/px), hardware not stated",
        "e2e": {"value": rk.world * n_img * acfg.H * acfg.W * args.steps / (e2e_ms / 1e3), "unit": "pixels/s",
                "h2d_bytes_per_step": h_img.numel() * 4, "d2h_bytes_per_step": h_lat.numel() * 4},
        "gpu_launches": P.ccrd.cc_last_launch_count() * args.steps,
        "clocks": sampler.summary(),
    }
    if rk.rank == 0:
        print(json.dumps(out), flush=True)


def run_train(args, rk):
    """NEXT-2: the encoder training iteration (forward on the noise proxy,
    backward, Adam) of ONE image per GPU (BASELINE.json configs[2] by default:
    the 512x768 ~2000 MAC/px model, the size the paper's encoding times are
    for).  value = training iterations/s x pixels (forward+backward pixels/s,
    whole job); also iterations/s and the encoding MAC/s with the paper's
    kappa_enc = 3 kappa_dec accounting."""
    import torch

    import paper_2403_11651_b200 as P
    from paper_2403_11651_b200 import dist

    cfg = workload.CONFIGS[args.config if args.config != "batched2k" else "ref"]
    dev = torch.device("cuda", rk.local_rank)
    torch.cuda.set_device(dev)
    P.load()
    # --images N: N independent encoders per GPU, each on its own stream (the
    # paper encodes every image separately; one 512x768 iteration does not
    # fill 148 SMs, so concurrent encoders raise the aggregate rate)
    n_img = max(1, args.images or 1)
    trs, noises = [], []
    for i in range(n_img):
        im = workload.make_image(cfg, workload.image_seed(args.seed, rk.rank * n_img + i))
        rng = np.random.default_rng(args.seed + 77 + rk.rank * n_img + i)
        y = workload.gen_continuous_latents(rng, im.latents)
        trs.append(P.DeviceTrainer(cfg, y, im.arm_w, im.up_w, im.syn_w, im.image, device=dev))
        noises.append([torch.from_numpy(workload.gen_noise(rng, y.size)).to(dev) for _ in range(4)])
    tr = trs[0]
    macs = P.cc_mac_per_pixel(tr.desc)
    stream = torch.cuda.current_stream(dev)
    streams = [stream] if n_img == 1 else [torch.cuda.Stream(dev) for _ in range(n_img)]

    def step(k):
        res = None
        for t, nz, st in zip(trs, noises, streams):
            with torch.cuda.stream(st):
                t.noise.copy_(nz[k % len(nz)])   # on-device copy: the noise is an input of the iteration
                res = t.step(lr=1e-3)
        return res

    def join():   # the side streams' work joins the timing stream
        for st in streams:
            if st is not stream:
                stream.wait_stream(st)

    def fork():
        for st in streams:
            if st is not stream:
                st.wait_stream(stream)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(rk.local_rank)
    dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    fork()
    launches = 0
    for k in range(args.steps):
        res = step(k)
        launches += n_img * P.ccrd.cc_last_launch_count()
    join()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    sampler.stop()
    ms = dist.max_over_ranks(ev0.elapsed_time(ev1), device=dev)
    its = rk.world * n_img * args.steps / (ms / 1e3)
    r = res.cpu().numpy()
    assert np.isfinite(r).all()
    px = cfg.H * cfg.W
    enc_flops = 3.0 * macs.total * px * its * 2
    out = {
        "metric": "encoder training iterations (forward + backward + Adam) as pixels/s", "value": its * px,
        "unit": "pixels/s", "n_gpus": rk.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"train_{cfg.name}: {n_img} x {cfg.H}x{cfg.W} image(s) per GPU"
                               f"{' on concurrent streams' if n_img > 1 else ''}, ARM {list(cfg.arm_widths)}, "
                               f"synthesis {list(cfg.syn_widths)}+{cfg.syn_n_res}xres3x3, noise proxy, Adam",
                   "H": cfg.H, "W": cfg.W, "mac_per_pixel_dec": round(macs.total, 3),
                   "l2": "per-step working set ~200 MB > 126 MB L2", "parallelism": f"image per GPU x{rk.world}", "images_per_gpu": n_img},
        "iterations_per_s": its,
        "path_roofline": {"achieved_tflops_per_gpu": enc_flops / rk.world / 1e12,
                          "frac": enc_flops / rk.world / 1e12 / FP32_PEAK_TFLOPS,
                          "note": "kappa_enc = 3 kappa_dec MAC per pixel per iteration (PAPER.md:389-394)"},
        "context": "paper: ~30 min for ~102950 iterations on a 512x768 image (~57 it/s), hardware not stated "
                   "(BASELINE.md section 1)",
        "e2e": None, "gpu_launches": launches, "clocks": sampler.summary(),
    }
    if rk.rank == 0:
        print(json.dumps(out), flush=True)


def run_e2e(args, cfg, images, desc, dev, stream, rk, n_img):
    import torch

    import paper_2403_11651_b200 as P
    from paper_2403_11651_b200 import dist
    # latents travel as int8 when every value fits (the workload clips them to
    # +-lat_clip); the host path widens them to int16 on the device
    hd = P.CcModelDesc.from_buffer_copy(desc)
    hd.latents_i8 = int(args.e2e_i8 and max(int(np.abs(im.latents).max()) for im in images) <= 127)
    lat = [torch.from_numpy(im.latents.astype(np.int8) if hd.latents_i8 else im.latents).pin_memory()
           for im in images]
    img = [torch.from_numpy(workload.to_u8(im.image) if desc.image_u8 else im.image).pin_memory() for im in images]
    # the step's result is the per-image (rate, sse, mse, cost); x_hat is an
    # optional output, read back only with --e2e-xhat
    xh = [torch.empty(im.image.shape, dtype=torch.float32).pin_memory() for im in images] if args.e2e_xhat else None
    io = [P.CcImageIO(lat[i].data_ptr(), images[i].arm_w.ctypes.data, images[i].up_w.ctypes.data,
                      images[i].syn_w.ctypes.data, img[i].data_ptr(), xh[i].data_ptr() if xh else None)
          for i in range(n_img)]
    ws_b = P.cc_workspace_bytes_host(hd, n_img)
    ws = torch.empty(ws_b, dtype=torch.uint8, device=dev)
    res = np.zeros((n_img, 4))
    steps = max(2, min(args.steps, args.e2e_steps))
    P.cc_rd_forward_host(hd, io, res, ws.data_ptr(), ws_b, stream.cuda_stream)   # warm-up
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(steps):
        P.cc_rd_forward_host(hd, io, res, ws.data_ptr(), ws_b, stream.cuda_stream)
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    wall = dist.max_over_ranks(wall, device=dev)
    h2d = sum(lat[i].numel() * lat[i].element_size() + img[i].numel() * img[i].element_size() for i in range(n_img))
    d2h = 32 * n_img + (sum(t.numel() * 4 for t in xh) if xh else 0)
    return {"value": rk.world * n_img * cfg.H * cfg.W * steps / wall, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "api": "cc_rd_forward_host (pinned host " + ("int8" if hd.latents_i8 else "int16") + " latents + "
                   + ("8-bit" if desc.image_u8 else "fp32")
                   + " image in, per-image results" + (" + x_hat" if xh else "") + " out, synchronous)"}


def run_cpu_baseline(cfg, images):
    import oracle
    cores = host_cores()
    oracle.set_threads(cores)
    done, wall = 0, 0.0
    for im in images:
        t, _ = oracle.time_rd_forward(cfg, im, cores)
        wall += t
        done += 1
        if wall * cores >= 10.0 or done >= 4:
            break
    return {"value": done * cfg.H * cfg.W / wall, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{done} full {cfg.H}x{cfg.W} image(s) of the same workload, fp64 C oracle "
                      f"(OpenMP over rows, {cores} threads), {wall:.2f} s wall"}


# ---------------------------------------------------------------------- reference
def run_reference(args, rk):
    """The tier's reference arm: the fp64 CPU oracle, as it stands, on the host
    cores; each step = one image of the same workload (bounded sample)."""
    if rk.rank != 0:
        return
    import oracle
    cfg = workload.CONFIGS[args.config]
    cores = host_cores()
    oracle.set_threads(cores)
    n = args.steps + args.warmup
    ims = workload.make_batch(cfg, [workload.image_seed(args.seed, g) for g in range(min(n, 4))],
                              threads=min(16, cores))
    if args.image == "u8":   # the same 8-bit images our arm encodes
        for im in ims:
            im.image = workload.quantize_image_u8(im.image)
    for i in range(args.warmup):
        oracle.rd_forward_image(cfg, ims[i % len(ims)])
    t0 = time.perf_counter()
    for i in range(args.steps):
        oracle.rd_forward_image(cfg, ims[(args.warmup + i) % len(ims)])
    wall = time.perf_counter() - t0
    value = args.steps * cfg.H * cfg.W / wall
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": rk.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{args.config}: one {cfg.H}x{cfg.W} image of the same workload per step "
                               f"(bounded sample of the {cfg.n_img}-image batch)", "H": cfg.H, "W": cfg.W},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{args.steps} timed steps x 1 image, fp64 C oracle, {cores} OpenMP threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def log(msg):
    if os.environ.get("CCRD_BENCH_VERBOSE"):
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def main():
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="batched2k", choices=list(workload.CONFIGS))
    ap.add_argument("--images", type=int, default=0, help="images per GPU (default: the config's)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--profile-steps", type=int, default=3, help="serial pass for per-kernel timing")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-xhat", action="store_true", help="e2e also reads x_hat back (fp32, 12 B/px)")
    ap.add_argument("--e2e-i8", type=int, default=1, help="e2e sends latents as int8 when they fit (1) or int16 (0)")
    ap.add_argument("--image", choices=("u8", "f32"), default="u8",
                    help="image format of the RD forward: 8-bit planes (x = v/255) or fp32")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--train", action="store_true", help="time the encoder training iteration (NEXT-2)")
    ap.add_argument("--decode", action="store_true", help="time the decoder output stage (NEXT-3)")
    ap.add_argument("--arm-decode", action="store_true", help="time the wavefront autoregressive ARM decode (NEXT-3)")
    ap.add_argument("--analysis", default="", help="time the N-O analysis transform (NEXT-4): no_kodak | no_2k")
    ap.add_argument("--tf32", type=int, default=1, choices=(0, 1, 2, 3),
                    help="analysis arithmetic: 0 fp32 cuBLASLt | 1 TF32 fused tcgen05 blocks | 2 TF32 cuBLASLt "
                         "unfused | 3 fused, FP16 operands, TMA-staged depth-wise")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 breaks the timing rules", file=sys.stderr)
    from paper_2403_11651_b200 import dist
    if args.impl == "reference":
        rk = dist.rank_from_env()
        run_reference(args, rk)
        return
    rk = dist.init("nccl")
    if args.train:
        run_train(args, rk)
    elif args.decode:
        run_decode(args, rk)
    elif args.analysis:
        run_analysis(args, rk)
    elif args.arm_decode:
        run_arm_decode(args, rk)
    elif args.config == "8k":
        run_strip(args, rk)
    else:
        run_ours(args, rk)
    import torch.distributed as tdist
    if tdist.is_initialized():
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
