"""Subprocess helper of tests/test_arm_tc_gpu.py: with CCRD_ARM_PATH=tc (set
by the caller before the library loads) checks the tensor-core ARM against the
fp64 oracle -- per-latent bits / mu / scale and the full RD forward."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2403_11651_b200 as P  # noqa: E402
import workload  # noqa: E402

assert os.environ.get("CCRD_ARM_PATH") == "tc"
# (W = 512 / 1024: every grid's rows 16-byte strided -> the TMA window path of
# arm_tcg_kernel; the other widths take its LDG staging path)
cases = [("ref", 70, 101, None), ("ref", 64, 200, None), ("ref", 71, 133, workload.TABLE1[1079]["arm"]),
         ("ref", 53, 61, workload.TABLE1[2300]["arm"]), ("ref", 77, 512, None),
         ("ref", 45, 1024, workload.TABLE1[2300]["arm"]), ("ref", 37, 512, workload.TABLE1[1079]["arm"])]
# + latents outside +-2048 (not exact in tf32): the kernel detects them per
# window and runs that tile's layer 0 in fp32 on the CUDA cores
cases += [("ref", 45, 512, "big"), ("ref", 38, 200, "big")]
for name, H, W, arm in cases:
    cfg = workload.CONFIGS[name].replace(H=H, W=W)
    if arm is not None and arm != "big":
        cfg = cfg.replace(n_ctx=arm[0], arm_widths=arm)
    im = workload.make_image(cfg, 5)
    if arm == "big":
        rng = np.random.default_rng(77)
        lat = im.latents.astype(np.int64)
        pick = rng.random(lat.size) < 0.01
        lat[pick] = rng.integers(-30000, 30001, int(pick.sum()))
        im.latents = lat.astype(np.int16)
    d = P.desc_from_config(cfg)
    lat = torch.from_numpy(im.latents).cuda()
    n = im.latents.size
    mu, sc, bits = (torch.zeros(n, device="cuda") for _ in range(3))
    rate = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws_b = P.cc_workspace_bytes(d, 1)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    def arm_rate():
        P.cc_arm_rate(d, lat.data_ptr(), im.arm_w, rate.data_ptr(), mu.data_ptr(), sc.data_ptr(), bits.data_ptr(),
                      ws.data_ptr(), ws_b, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        return mu.cpu().numpy(), sc.cpu().numpy(), bits.cpu().numpy()
    R, mu_o, b_o, bits_o, _ = oracle.rate(oracle.model(cfg), im.latents, im.arm_w, per_latent=True)
    if arm == "big":
        # contexts up to 3e4: pre-activations ~1e3, so plain fp32 itself errs by
        # ~1e-4 on mu; the bar is the FFMA2 path's own error (a wrong exact
        # path would err by O(1)), per latent, plus the usual tolerances
        with P.arm_path(P.CC_ARM_FFMA2):
            mu_f, sc_f, bits_f = arm_rate()
        mu_g, sc_g, bits_g = arm_rate()
        e_f, e_g = np.abs(mu_f - mu_o), np.abs(mu_g - mu_o)
        assert e_g.max() <= 1e-5 + 4 * e_f.max(), (e_g.max(), e_f.max())
        assert np.percentile(e_g, 50) <= 1e-5, np.percentile(e_g, 50)
        eb_f, eb_g = np.abs(bits_f - bits_o), np.abs(bits_g - bits_o)
        assert eb_g.max() <= 1e-3 + 4 * eb_f.max(), (eb_g.max(), eb_f.max())
        np.testing.assert_allclose(sc_g, b_o, rtol=1e-4, atol=0)
        assert abs(rate.item() - R) <= 1e-5 * R, (rate.item(), R)
        continue
    mu_g, sc_g, bits_g = arm_rate()
    np.testing.assert_allclose(mu_g, mu_o, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(sc_g, b_o, rtol=1e-5, atol=0)
    np.testing.assert_allclose(bits_g, bits_o, rtol=0, atol=1e-3)
    assert abs(rate.item() - R) <= 1e-5 * R, (rate.item(), R)
    b = P.DeviceBatch(cfg, [im])
    res = b.forward()
    torch.cuda.synchronize()
    ref = oracle.rd_forward_image(cfg, im)
    got = res.cpu().numpy()[0]
    assert abs(got[0] - ref["rate_bits"]) <= 1e-4 * ref["rate_bits"]
    assert abs(got[3] - ref["cost"]) <= 1e-4 * ref["cost"]
print("arm_tc parity ok")
