"""GPU parity of the strip path (cc_rd_forward_strip; SURVEY.md §8e,
BASELINE.json configs[4]).

Each strip runs on the device from its own window buffer (owned rows + the
halo the exchange would deliver, packed here from the full pyramid: one GPU,
so the strips run one after another -- the exchange itself is tested with
gloo in test_strips_cpu.py).  Checks:
  * stitched strip x_hat == the full-image CUDA x_hat, BIT-IDENTICAL (same
    kernels, same per-pixel FMA order, window = receptive field);
  * the strips' additive shares sum to the full-image result (1e-7 relative:
    the per-warp / per-thread fp32 partial sums group latents and pixels by
    tile, and strip tiles start at the strip's first row; measured ~1e-9) and
    to the fp64 oracle within
    north_star's 1e-4 relative; stitched x_hat within 1e-5 of the oracle;
  * the full 4320x7680 image at G = 8 (the launch configuration of
    bench.py --config 8k --gpus 8, one strip per rank).
"""
import numpy as np
import pytest

import oracle
import workload
from test_strips_cpu import STRIP_CASES, _full_off, strip_cfg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run_strips(cfg, im, world):
    import paper_2403_11651_b200 as P
    from paper_2403_11651_b200 import dist as ccdist
    d = P.desc_from_config(cfg)
    strips, lays = ccdist.strip_layouts(d, world)
    off = _full_off(cfg)
    full_lat = torch.from_numpy(im.latents).cuda()
    xh = np.zeros((3, cfg.H, cfg.W), np.float32)
    tot = np.zeros(4)
    for st, lay in zip(strips, lays):
        ds = P.ccrd.DeviceStrip(cfg, st, im.arm_w, im.up_w, im.syn_w, image_rows=im.image[:, st.r0:st.r1])
        ds.lat.copy_(ccdist.pack_window(full_lat, off, lay))
        r = ds.forward()
        torch.cuda.synchronize()
        tot += r.cpu().numpy()
        xh[:, st.r0:st.r1] = ds.xhat.cpu().numpy()
        del ds
    return tot, xh


def _run_full(cfg, im):
    import paper_2403_11651_b200 as P
    b = P.DeviceBatch(cfg, [im])
    r = b.forward()
    torch.cuda.synchronize()
    return r.cpu().numpy()[0], b.xhat[0].cpu().numpy()


@pytest.mark.parametrize("H,W,L,ch,res,taps,nctx,world", STRIP_CASES)
def test_strips_bit_identical_to_full(H, W, L, ch, res, taps, nctx, world):
    cfg = strip_cfg(H, W, L, ch, res, taps, nctx)
    im = workload.make_image(cfg, 31, filter_kind="lanczos2" if taps == 8 else "random")
    full, xf = _run_full(cfg, im)
    for g in sorted({1, 2, world}):
        tot, xs = _run_strips(cfg, im, g)
        np.testing.assert_array_equal(xs, xf)
        np.testing.assert_allclose(tot, full, rtol=1e-7)
    ref = oracle.rd_forward_image(cfg, im, want_xhat=True)
    assert np.abs(xs - ref["x_hat"]).max() <= 1e-5
    for k, key in enumerate(["rate_bits", "sse", "mse", "cost"]):
        assert abs(tot[k] - ref[key]) <= 1e-4 * abs(ref[key]), key


@pytest.mark.parametrize("name,world", [("ref", 7), ("low", 4)])
def test_strips_paper_shapes(name, world):
    cfg = workload.CONFIGS[name]
    im = workload.make_image(cfg, 3, filter_kind="lanczos2")
    full, xf = _run_full(cfg, im)
    tot, xs = _run_strips(cfg, im, world)
    np.testing.assert_array_equal(xs, xf)
    np.testing.assert_allclose(tot, full, rtol=1e-7)


@pytest.mark.timeout(900)
def test_strips_8k_world8_vs_full_and_oracle():
    """BASELINE.json configs[4] at full size, 8 strips."""
    cfg = workload.CONFIGS["8k"]
    im = workload.make_image(cfg, 0)
    full, xf = _run_full(cfg, im)
    tot, xs = _run_strips(cfg, im, 8)
    np.testing.assert_array_equal(xs, xf)
    np.testing.assert_allclose(tot, full, rtol=1e-7)
    del xf
    oracle.set_threads(oracle.get_threads())
    ref = oracle.rd_forward_image(cfg, im, want_xhat=True)
    assert np.abs(xs - ref["x_hat"]).max() <= 1e-5
    for k, key in enumerate(["rate_bits", "sse", "mse", "cost"]):
        assert abs(tot[k] - ref[key]) <= 1e-4 * abs(ref[key]), key


def test_strip_window_too_small_is_rejected():
    import paper_2403_11651_b200 as P
    cfg = workload.CONFIGS["tiny"]
    d = P.desc_from_config(cfg)
    st = P.cc_strip_window(d, 32, 64)
    st.lo[1] += 1
    with pytest.raises(P.CcError):
        P.cc_workspace_bytes_strip(d, st) or P.cc_rd_forward_strip(d, st, P.CcImageIO(), 0, 0, 0)


def test_strips_u8_rows_bit_identical_to_full_u8():
    """8-bit image rows (desc.image_u8) through the strip entry point: the
    stitched x_hat and the summed shares equal the full 8-bit image's."""
    import paper_2403_11651_b200 as P
    from paper_2403_11651_b200 import dist as ccdist
    cfg = workload.CONFIGS["ref"].replace(H=150, W=222)
    im = workload.make_image(cfg, 33)
    im.image = workload.quantize_image_u8(im.image)
    b = P.DeviceBatch(cfg, [im], image_u8=True)
    full = b.forward().cpu().numpy()[0]
    xf = b.xhat[0].cpu().numpy()
    u8 = workload.to_u8(im.image)
    d = P.desc_from_config(cfg)
    strips, lays = ccdist.strip_layouts(d, 3)
    off = _full_off(cfg)
    full_lat = torch.from_numpy(im.latents).cuda()
    xh = np.zeros((3, cfg.H, cfg.W), np.float32)
    tot = np.zeros(4)
    for st, lay in zip(strips, lays):
        ds = P.ccrd.DeviceStrip(cfg, st, im.arm_w, im.up_w, im.syn_w, image_rows=u8[:, st.r0:st.r1])
        assert ds.desc.image_u8 == 1
        ds.lat.copy_(ccdist.pack_window(full_lat, off, lay))
        tot += ds.forward().cpu().numpy()
        xh[:, st.r0:st.r1] = ds.xhat.cpu().numpy()
    np.testing.assert_array_equal(xh, xf)
    np.testing.assert_allclose(tot, full, rtol=1e-7)
