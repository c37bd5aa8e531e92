"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by
element on the same seeded inputs.

Tolerances (north_star):
  * x_hat: 1e-5 absolute per pixel;
  * total rate bits and MSE: 1e-4 relative (expected ~1e-7);
  * per-latent bits: 1e-3 absolute (fast-intrinsic Laplace; expected ~1e-5);
    mu: 1e-5 absolute + 1e-5 relative;
  * dense upsampled tensor: per level 1e-5 relative to the level's max |value|.
"""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _P():
    import paper_2403_11651_b200 as P
    return P


@pytest.fixture(autouse=True, params=["tc", "ffma2", "tc+synmma", "tc+syntma"])
def arm_path(request):
    """Every parity case runs on both ARM paths (include/ccrd.h
    cc_set_arm_path): the tensor-core kernel (the default for the shapes it is
    compiled for; the others fall back to FFMA2) and the FFMA2 kernel; and
    once more with the synthesis 1x1 layer 0 on warp MMAs (cc_set_synth_path
    CC_SYN_MMA, opt-in; the shapes and entries it does not cover run FFMA2),
    and once with the TMA-staged persistent synthesis (CC_SYN_TMA; shapes and
    buffers it does not cover run the per-tile FFMA2 kernel)."""
    P = _P()
    arm = P.CC_ARM_FFMA2 if request.param == "ffma2" else P.CC_ARM_TC
    syn = (P.CC_SYN_MMA if request.param.endswith("synmma") else
           P.CC_SYN_TMA if request.param.endswith("syntma") else P.CC_SYN_FFMA2)
    with P.arm_path(arm), P.synth_path(syn):
        yield request.param


def run_forward(cfg, images, with_xhat=True):
    P = _P()
    b = P.DeviceBatch(cfg, images, with_xhat=with_xhat)
    res = b.forward()
    torch.cuda.synchronize()
    out = res.cpu().numpy()
    xh = [t.cpu().numpy() for t in b.xhat] if with_xhat else None
    return out, xh


def check_image(cfg, im, res_row, xh, tol_px=1e-5):
    ref = oracle.rd_forward_image(cfg, im, want_xhat=True)
    assert abs(res_row[0] - ref["rate_bits"]) <= 1e-4 * ref["rate_bits"], (res_row[0], ref["rate_bits"])
    assert abs(res_row[2] - ref["mse"]) <= 1e-4 * ref["mse"], (res_row[2], ref["mse"])
    assert abs(res_row[1] - ref["sse"]) <= 1e-4 * ref["sse"]
    assert abs(res_row[3] - ref["cost"]) <= 1e-4 * ref["cost"]
    if xh is not None:
        err = np.abs(xh.astype(np.float64) - ref["x_hat"]).max()
        assert err <= tol_px, f"max |x_hat - oracle| = {err}"
    return ref


@pytest.mark.parametrize("name", ["tiny", "low", "ref"])
@pytest.mark.parametrize("filt", ["random", "lanczos2"])
def test_rd_forward_configs(name, filt):
    cfg = workload.CONFIGS[name]
    im = workload.make_image(cfg, 100, filter_kind=filt)
    out, xh = run_forward(cfg, [im])
    check_image(cfg, im, out[0], xh[0])


@pytest.mark.parametrize("H,W,L,res,taps", [
    (37, 53, 5, 1, 8), (37, 53, 5, 1, 4), (33, 97, 4, 1, 8), (65, 129, 4, 3, 8), (64, 64, 4, 0, 8),
    (1, 1, 1, 1, 8), (3, 300, 2, 1, 8), (300, 3, 2, 1, 8), (5, 5, 2, 1, 8), (31, 63, 3, 1, 8),
    (100, 256, 3, 1, 8), (100, 256, 5, 1, 8),  # interior tiles: TMA staging with 1 and 3 S_1 planes
])
def test_rd_forward_odd_shapes(H, W, L, res, taps):
    cfg = workload.CONFIGS["tiny"].replace(H=H, W=W, L=L, syn_widths=(L, 8, 3), syn_n_res=res, up_taps=taps)
    im = workload.make_image(cfg, 7, filter_kind="lanczos2" if taps == 8 else "random")
    out, xh = run_forward(cfg, [im])
    check_image(cfg, im, out[0], xh[0])


def test_table1_shapes():
    """Table 1 ARM / synthesis widths (separable TConv reading) on a ragged size."""
    base = workload.CONFIGS["ref"]
    for key, a in workload.TABLE1.items():
        aw = a["arm"]
        cfg = base.replace(H=71, W=133, n_ctx=aw[0], arm_widths=aw, syn_widths=a["syn"],
                           syn_n_res=a["syn_n_res"], up_taps=a["up_kernel"])
        im = workload.make_image(cfg, key)
        out, xh = run_forward(cfg, [im])
        check_image(cfg, im, out[0], xh[0])


def test_batch_has_per_image_weights():
    cfg = workload.CONFIGS["ref"].replace(H=96, W=160)
    ims = workload.make_batch(cfg, [11, 12, 13])
    out, xh = run_forward(cfg, ims)
    for i, im in enumerate(ims):
        check_image(cfg, im, out[i], xh[i])
    assert len({round(r, 6) for r in out[:, 0]}) == 3


def test_arm_stage_per_latent():
    P = _P()
    for name, H, W in [("tiny", 64, 64), ("ref", 70, 101), ("low", 53, 37)]:
        cfg = workload.CONFIGS[name].replace(H=H, W=W)
        im = workload.make_image(cfg, 5)
        d = P.desc_from_config(cfg)
        lat = torch.from_numpy(im.latents).cuda()
        n = im.latents.size
        mu, sc, bits = (torch.zeros(n, device="cuda") for _ in range(3))
        rate = torch.zeros(1, dtype=torch.float64, device="cuda")
        ws_b = P.cc_workspace_bytes(d, 1)
        ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
        P.cc_arm_rate(d, lat.data_ptr(), im.arm_w, rate.data_ptr(), mu.data_ptr(), sc.data_ptr(),
                      bits.data_ptr(), ws.data_ptr(), ws_b, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        R, mu_o, b_o, bits_o, _ = oracle.rate(oracle.model(cfg), im.latents, im.arm_w, per_latent=True)
        np.testing.assert_allclose(mu.cpu().numpy(), mu_o, rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(sc.cpu().numpy(), b_o, rtol=1e-5, atol=0)
        np.testing.assert_allclose(bits.cpu().numpy(), bits_o, rtol=0, atol=1e-3)
        assert abs(rate.item() - R) <= 1e-5 * R


def test_arm_stage_logscale_clamps_and_floor():
    """Push the log-scale output past both clamps and latents far into the
    tails (probability floor): per-latent bits still match."""
    P = _P()
    cfg = workload.CONFIGS["tiny"].replace(lat_scale=6.0, lat_clip=60)
    im = workload.make_image(cfg, 9)
    for bias_s in (12.0, -12.0, 3.0):
        aw = im.arm_w.copy()
        aw[-1] = bias_s
        d = P.desc_from_config(cfg)
        lat = torch.from_numpy(im.latents).cuda()
        n = im.latents.size
        bits = torch.zeros(n, device="cuda")
        rate = torch.zeros(1, dtype=torch.float64, device="cuda")
        ws_b = P.cc_workspace_bytes(d, 1)
        ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
        P.cc_arm_rate(d, lat.data_ptr(), aw, rate.data_ptr(), 0, 0, bits.data_ptr(), ws.data_ptr(), ws_b, 0)
        torch.cuda.synchronize()
        R, _, _, bits_o, _ = oracle.rate(oracle.model(cfg), im.latents, aw, per_latent=True)
        np.testing.assert_allclose(bits.cpu().numpy(), bits_o, rtol=0, atol=1e-3)
        assert abs(rate.item() - R) <= 1e-5 * R


@pytest.mark.parametrize("filt", ["random", "lanczos2"])
def test_upsample_stage_per_level(filt):
    P = _P()
    for name, H, W in [("tiny", 64, 64), ("ref", 75, 141), ("ref", 128, 64)]:
        cfg = workload.CONFIGS[name].replace(H=H, W=W)
        im = workload.make_image(cfg, 21, filter_kind=filt)
        d = P.desc_from_config(cfg)
        lat = torch.from_numpy(im.latents).cuda()
        dense = torch.zeros((cfg.L, H, W), device="cuda")
        ws_b = P.cc_workspace_bytes(d, 1)
        ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
        P.cc_upsample(d, lat.data_ptr(), im.up_w, dense.data_ptr(), ws.data_ptr(), ws_b)
        torch.cuda.synchronize()
        ref, _ = oracle.upsample(oracle.model(cfg), im.latents, im.up_w)
        got = dense.cpu().numpy().astype(np.float64)
        for l in range(cfg.L):
            scale = max(np.abs(ref[l]).max(), 1e-30)
            err = np.abs(got[l] - ref[l]).max() / scale
            assert err <= 1e-5, f"level {l}: rel err {err}"


def test_synthesize_stage_from_dense():
    P = _P()
    cfg = workload.CONFIGS["ref"].replace(H=77, W=130)
    im = workload.make_image(cfg, 31)
    m = oracle.model(cfg)
    dense_o, _ = oracle.upsample(m, im.latents, im.up_w)
    dense32 = dense_o.astype(np.float32)
    xh_o, h1_o, _ = oracle.synthesis(m, dense32.astype(np.float64), im.syn_w)
    d = P.desc_from_config(cfg)
    dense = torch.from_numpy(dense32).cuda()
    img = torch.from_numpy(im.image).cuda()
    xh = torch.zeros((3, 77, 130), device="cuda")
    h1 = torch.zeros((3, 77, 130), device="cuda")
    sse = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws_b = P.cc_workspace_bytes(d, 1)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    P.cc_synthesize(d, dense.data_ptr(), im.syn_w, img.data_ptr(), xh.data_ptr(), sse.data_ptr(), h1.data_ptr(),
                    ws.data_ptr(), ws_b)
    torch.cuda.synchronize()
    np.testing.assert_allclose(h1.cpu().numpy(), h1_o, rtol=0, atol=1e-5)
    np.testing.assert_allclose(xh.cpu().numpy(), xh_o, rtol=0, atol=1e-5)
    sse_o = ((im.image.astype(np.float64) - xh_o) ** 2).sum()
    assert abs(sse.item() - sse_o) <= 1e-5 * sse_o


def test_deterministic_and_host_path_match():
    """Bitwise determinism, and the host-buffer (end-to-end) path -- three
    streams, three slots of four images reused from the 13th image on -- gives the
    same numbers bit for bit."""
    P = _P()
    cfg = workload.CONFIGS["ref"].replace(H=200, W=300)
    n = 14
    ims = workload.make_batch(cfg, list(range(41, 41 + n)))
    a, xa = run_forward(cfg, ims)
    b, xb = run_forward(cfg, ims)
    np.testing.assert_array_equal(a, b)
    for u, v in zip(xa, xb):
        np.testing.assert_array_equal(u, v)
    d = P.desc_from_config(cfg)
    lat = [torch.from_numpy(im.latents).pin_memory() for im in ims]
    img = [torch.from_numpy(im.image).pin_memory() for im in ims]
    xh = [torch.full_like(t, -7.0).pin_memory() for t in img]
    io = [P.CcImageIO(lat[i].data_ptr(), ims[i].arm_w.ctypes.data, ims[i].up_w.ctypes.data,
                      ims[i].syn_w.ctypes.data, img[i].data_ptr(), xh[i].data_ptr()) for i in range(n)]
    ws_b = P.cc_workspace_bytes_host(d, n)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    res = np.zeros((n, 4))
    for _ in range(2):
        P.cc_rd_forward_host(d, io, res, ws.data_ptr(), ws_b, torch.cuda.current_stream().cuda_stream)
        np.testing.assert_array_equal(res, a)
        for i in range(n):
            np.testing.assert_array_equal(xh[i].numpy(), xa[i])


@pytest.mark.slow
def test_full_size_2k_batch():
    """BASELINE.json configs[3] image size, two images through the same
    cc_rd_forward call bench.py times (all outputs vs the oracle)."""
    cfg = workload.CONFIGS["batched2k"]
    ims = workload.make_batch(cfg, [workload.image_seed(0, 0), workload.image_seed(0, 1)])
    oracle.set_threads(max(1, min(32, __import__("os").cpu_count() or 1)))
    out, xh = run_forward(cfg, ims)
    for i, im in enumerate(ims):
        check_image(cfg, im, out[i], xh[i])


@pytest.mark.slow
def test_full_size_8k_sampled_rows():
    """BASELINE.json configs[4] size: per-latent bits on sampled rows of every
    level (oracle evaluated row by row) and the total rate / MSE invariants."""
    P = _P()
    cfg = workload.CONFIGS["8k"]
    im = workload.make_image(cfg, 8)
    d = P.desc_from_config(cfg)
    lat = torch.from_numpy(im.latents).cuda()
    n = im.latents.size
    bits = torch.zeros(n, device="cuda")
    rate = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws_b = P.cc_workspace_bytes(d, 1)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    P.cc_arm_rate(d, lat.data_ptr(), im.arm_w, rate.data_ptr(), 0, 0, bits.data_ptr(), ws.data_ptr(), ws_b, 0)
    torch.cuda.synchronize()
    bits_np = bits.cpu().numpy()
    m = oracle.model(cfg)
    dims = cfg.level_dims()
    off = 0
    rng = np.random.default_rng(0)
    for l, (h, w) in enumerate(dims):
        for r in sorted(set([0, 1, 2, h - 1] + list(rng.integers(0, h, 3)))):
            _, ob = oracle.rate_rows(m, im.latents, im.arm_w, l, r, r + 1)
            np.testing.assert_allclose(bits_np[off + r * w: off + (r + 1) * w], ob[0], rtol=0, atol=1e-3)
        off += h * w
    # total rate = fp64 sum of the per-latent bits the kernel produced
    assert abs(rate.item() - bits_np.astype(np.float64).sum()) <= 1e-6 * rate.item()


def _quantised(ims):
    for im in ims:
        im.image = workload.quantize_image_u8(im.image)
    return ims


@pytest.mark.parametrize("name", ["low", "ref"])
def test_u8_images_match_fp32_and_oracle(name):
    """desc.image_u8 = 1: the kernels read 8-bit planes, x = v / 255 (IEEE fp32
    division).  On images whose values are 8-bit levels, the results equal
    the fp32-image path bit for bit (the same x values), and the oracle fed
    x = float32(v) / 255."""
    P = _P()
    cfg = workload.CONFIGS[name].replace(H=123, W=201)
    ims = _quantised(workload.make_batch(cfg, [61, 62]))
    a, xa = run_forward(cfg, ims)
    b = P.DeviceBatch(cfg, ims, with_xhat=True, image_u8=True)
    assert b.img[0].dtype == torch.uint8
    res = b.forward()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(res.cpu().numpy(), a)
    for u, v in zip(b.xhat, xa):
        np.testing.assert_array_equal(u.cpu().numpy(), v)
    for k, im in enumerate(ims):
        check_image(cfg, im, res.cpu().numpy()[k], None)


def test_u8_host_path_results_only():
    """The end-to-end host path with 8-bit images and no x_hat read-back (what
    bench.py's e2e times): same results as the device path, bit for bit."""
    P = _P()
    cfg = workload.CONFIGS["ref"].replace(H=200, W=300)
    n = 14
    ims = _quantised(workload.make_batch(cfg, list(range(71, 71 + n))))
    a, _ = run_forward(cfg, ims, with_xhat=False)
    d = P.desc_from_config(cfg)
    d.image_u8 = 1
    lat = [torch.from_numpy(im.latents).pin_memory() for im in ims]
    img = [torch.from_numpy(workload.to_u8(im.image)).pin_memory() for im in ims]
    io = [P.CcImageIO(lat[i].data_ptr(), ims[i].arm_w.ctypes.data, ims[i].up_w.ctypes.data,
                      ims[i].syn_w.ctypes.data, img[i].data_ptr(), None) for i in range(n)]
    ws_b = P.cc_workspace_bytes_host(d, n)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    res = np.zeros((n, 4))
    for _ in range(2):
        P.cc_rd_forward_host(d, io, res, ws.data_ptr(), ws_b, torch.cuda.current_stream().cuda_stream)
        np.testing.assert_array_equal(res, a)


def test_i8_latents_host_path():
    """latents_i8 (host path): int8 latent uploads widened on the device give
    the device path's results bit for bit; device entry points refuse the flag."""
    P = _P()
    cfg = workload.CONFIGS["ref"].replace(H=150, W=222)
    n = 3
    ims = _quantised(workload.make_batch(cfg, list(range(81, 81 + n))))
    assert max(np.abs(im.latents).max() for im in ims) <= 127
    a, _ = run_forward(cfg, ims, with_xhat=False)
    d = P.desc_from_config(cfg)
    d.image_u8 = 1
    d.latents_i8 = 1
    lat = [torch.from_numpy(im.latents.astype(np.int8)).pin_memory() for im in ims]
    img = [torch.from_numpy(workload.to_u8(im.image)).pin_memory() for im in ims]
    io = [P.CcImageIO(lat[i].data_ptr(), ims[i].arm_w.ctypes.data, ims[i].up_w.ctypes.data,
                      ims[i].syn_w.ctypes.data, img[i].data_ptr(), None) for i in range(n)]
    ws_b = P.cc_workspace_bytes_host(d, n)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    res = np.zeros((n, 4))
    P.cc_rd_forward_host(d, io, res, ws.data_ptr(), ws_b, torch.cuda.current_stream().cuda_stream)
    np.testing.assert_array_equal(res, a)
    b = P.DeviceBatch(cfg, ims, with_xhat=False)
    b.desc.latents_i8 = 1
    with pytest.raises(P.CcError) as e:
        b.forward()
    assert e.value.code == P.ccrd.CC_ENOTSUP


def test_u8_training_refused():
    P = _P()
    d = P.desc_from_config(workload.CONFIGS["ref"].replace(H=24, W=40))
    d.image_u8 = 1
    with pytest.raises(P.CcError) as e:
        P.cc_train_step(d, 8, 8, 8, 8, 8, None, 8, 8, 8, 1 << 30)
    assert e.value.code == P.ccrd.CC_ENOTSUP


@pytest.mark.parametrize("name,H,W,u8", [
    ("ref", 512, 768, False), ("ref", 333, 1024, True), ("low", 300, 512, False), ("ref", 1365, 2048, True),
    ("ref", 200, 304, False), ("ref", 70, 128, False), ("tiny", 200, 256, False), ("tiny", 160, 512, True),
])
def test_synth_tma_bit_identical_to_ldg(arm_path, name, H, W, u8):
    """CC_SYN_TMA (interior tiles staged by TMA, border tiles by clamped LDG;
    one CTA per tile, or with CCRD_SYN_CLU=1 vertical tile pairs in 2-CTA
    clusters that exchange their shared halo rows through distributed shared
    memory) computes every pixel exactly as the per-tile LDG kernel
    does, so x_hat and every result are bit-identical to CC_SYN_FFMA2 -- on
    shapes with many interior tiles, odd and even tile-row counts (a ghost
    CTA in the last pair), a ragged last tile row, 8-bit targets, and
    W = 304 / 128 (narrow: few or no interior tiles)."""
    if arm_path != "tc":
        pytest.skip("one ARM path suffices: the comparison is between synthesis paths")
    P = _P()
    cfg = workload.CONFIGS[name].replace(H=H, W=W)
    ims = workload.make_batch(cfg, [5, 6])
    if u8:
        ims = _quantised(ims)

    def fwd():
        bt = P.DeviceBatch(cfg, ims, with_xhat=True, image_u8=u8)
        r = bt.forward()
        torch.cuda.synchronize()
        return r.cpu().numpy(), [t.cpu().numpy() for t in bt.xhat]

    with P.synth_path(P.CC_SYN_FFMA2):
        a, xa = fwd()
    with P.synth_path(P.CC_SYN_TMA):
        b, xb = fwd()  # one CTA per tile (the default)
        os.environ["CCRD_SYN_CLU"] = "1"
        try:
            c, xc = fwd()  # vertical tile pairs in 2-CTA clusters (opt-in)
        finally:
            del os.environ["CCRD_SYN_CLU"]
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a, c)
    for u, v, w in zip(xa, xb, xc):
        np.testing.assert_array_equal(u, v)
        np.testing.assert_array_equal(u, w)
    if H * W <= 512 * 768:
        check_image(cfg, ims[0], b[0], xb[0])


def test_synth_tma_bit_identical_random_shapes(arm_path):
    """Seeded sweep of shapes for the TMA-staged synthesis: widths that are
    multiples of 16 (the TMA path's alignment) and not, heights with every
    residue of the 32-row tile, configs with 1 / 2 residual layers and L = 3..7;
    x_hat and results bit-identical to the per-tile LDG kernel."""
    if arm_path != "tc":
        pytest.skip("one ARM path suffices: the comparison is between synthesis paths")
    P = _P()
    rng = np.random.default_rng(2403)
    for trial in range(12):
        name = ["ref", "low", "tiny"][trial % 3]
        W = int(rng.integers(4, 40)) * 16 + (0 if trial % 4 else int(rng.integers(1, 15)))
        H = int(rng.integers(70, 400))
        L = {"ref": 7, "low": 7, "tiny": int(rng.integers(3, 5))}[name]
        cfg = workload.CONFIGS[name].replace(H=H, W=W, L=L, syn_widths=(L,) + tuple(workload.CONFIGS[name].syn_widths[1:]))
        ims = workload.make_batch(cfg, [trial])

        def fwd():
            bt = P.DeviceBatch(cfg, ims, with_xhat=True)
            r = bt.forward()
            torch.cuda.synchronize()
            return r.cpu().numpy(), bt.xhat[0].cpu().numpy()

        with P.synth_path(P.CC_SYN_FFMA2):
            a, xa = fwd()
        with P.synth_path(P.CC_SYN_TMA):
            b, xb = fwd()
        np.testing.assert_array_equal(a, b, err_msg=f"{name} {H}x{W} L={L}")
        np.testing.assert_array_equal(xa, xb, err_msg=f"{name} {H}x{W} L={L}")
