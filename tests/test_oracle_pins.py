"""Pins of the fp64 oracle against what the paper and the mathematics fix
(closed forms, printed values, library special cases, invariants).

Every test here is CPU-only.  Each pin is chosen so that a plausible mistake in
the oracle (dropped term, wrong sign or index, transposed operand) fails it.
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import workload

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------- dims
def test_dims_spec_examples():
    # 512x768 L=7 -> (8,12) at the coarsest; 5x5 L=2 -> (3,3)
    cfg = workload.CONFIGS["ref"]
    d = oracle.level_dims(oracle.model(cfg))
    assert d[0] == (512, 768) and d[-1] == (8, 12)
    d = oracle.level_dims(oracle.model(cfg.replace(H=5, W=5, L=2)))
    assert d == [(5, 5), (3, 3)]
    # ceil chain at the 2K and 8K sizes
    d = oracle.level_dims(oracle.model(workload.CONFIGS["batched2k"]))
    assert d == [(1365, 2048), (683, 1024), (342, 512), (171, 256), (86, 128), (43, 64), (22, 32)]
    assert sum(h * w for h, w in d) == 3728256
    d = oracle.level_dims(oracle.model(workload.CONFIGS["8k"]))
    assert d[-1] == (68, 120)


# ------------------------------------------------------------------------ Laplace
def test_laplace_printed_values():
    g = gold("laplace.json")
    assert oracle.laplace_prob(0, 0, 1) == pytest.approx(g["p0_mu0_b1"], abs=1e-15)
    assert oracle.laplace_bits(0, 0, 1) == pytest.approx(g["bits0_mu0_b1"], abs=1e-12)
    for k in range(1, g["first_floored_k_b1"]):
        want = g["bits_k_mu0_b1_slope"] * k + g["bits_k_mu0_b1_intercept"]
        assert oracle.laplace_bits(k, 0, 1) == pytest.approx(want, abs=1e-9)
        assert oracle.laplace_bits(-k, 0, 1) == pytest.approx(want, abs=1e-9)
    for k in range(g["first_floored_k_b1"], 40):
        assert oracle.laplace_bits(k, 0, 1) == g["floor_bits"]


def test_laplace_closed_form_random():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        mu = rng.uniform(-5, 5)
        b = math.exp(rng.uniform(math.log(1e-3), math.log(256)))
        y = float(rng.integers(-20, 21))
        a = abs(y - mu)
        if a >= 0.5:
            p = math.exp(-a / b) * math.sinh(1 / (2 * b))
        else:
            p = 1 - math.exp(-1 / (2 * b)) * math.cosh(a / b)
        got = oracle.laplace_prob(y, mu, b)
        assert got == pytest.approx(p, rel=1e-9, abs=1e-15)


def test_laplace_vs_torch_cdf():
    rng = np.random.default_rng(2)
    mu = torch.tensor(rng.uniform(-3, 3, 200), dtype=torch.float64)
    b = torch.tensor(np.exp(rng.uniform(-2, 3, 200)), dtype=torch.float64)
    y = torch.tensor(rng.integers(-8, 9, 200), dtype=torch.float64)
    d = torch.distributions.Laplace(mu, b)
    p = (d.cdf(y + 0.5) - d.cdf(y - 0.5)).numpy()
    got = np.array([oracle.laplace_prob(float(yy), float(m), float(bb)) for yy, m, bb in zip(y, mu, b)])
    np.testing.assert_allclose(got, p, rtol=1e-9, atol=1e-14)


def test_laplace_normalised_and_symmetric():
    # telescoping: sum_y F(y+1/2) - F(y-1/2) = 1
    for mu, b in [(0.0, 1.0), (0.3, 0.01), (-2.7, 5.0), (1.49, 40.0)]:
        s = sum(oracle.laplace_prob(y, mu, b) for y in range(-4000, 4001))
        assert s == pytest.approx(1.0, abs=1e-12)
    # symmetry P(y | 0, b) = P(-y | 0, b)
    for b in (0.2, 1.0, 7.0):
        for y in range(0, 12):
            assert oracle.laplace_prob(y, 0, b) == pytest.approx(oracle.laplace_prob(-y, 0, b), rel=1e-12)
    # floor: bits never exceed -log2(2^-16)
    assert oracle.laplace_bits(100, 0, 0.001) == 16.0


# ------------------------------------------------------------------------ context
def test_context_hand_examples():
    g = gold("context_3x3.json")
    cfg = workload.CONFIGS["tiny"]          # C = 8
    m = oracle.model(cfg)
    grid = np.array(g["grid"], np.int16)
    for case in g["cases"]:
        got = oracle.context(m, grid, *case["pos"])
        np.testing.assert_array_equal(got, case["ctx"])


def test_context_constant_grid():
    cfg = workload.CONFIGS["ref"]           # C = 16, needs rows i-2..i, cols j-3..j+3
    m = oracle.model(cfg)
    grid = np.full((9, 11), 5, np.int16)
    np.testing.assert_array_equal(oracle.context(m, grid, 4, 5), np.full(16, 5.0))


def test_rate_causality():
    """perturbing the latent at q never changes bits at any position
    earlier in raster order (and never touches another grid)."""
    cfg = workload.CONFIGS["tiny"].replace(H=12, W=14, L=2)
    im = workload.make_image(cfg, 3)
    m = oracle.model(cfg)
    _, _, _, bits0, _ = oracle.rate(m, im.latents, im.arm_w, per_latent=True)
    dims = cfg.level_dims()
    n0 = dims[0][0] * dims[0][1]
    rng = np.random.default_rng(0)
    for q in rng.choice(n0, 20, replace=False):
        lat = im.latents.copy()
        lat[q] += 3
        _, _, _, bits1, _ = oracle.rate(m, lat, im.arm_w, per_latent=True)
        np.testing.assert_array_equal(bits1[:q], bits0[:q])
        np.testing.assert_array_equal(bits1[n0:], bits0[n0:])
        # and some later position does change (the context is actually used)
        assert np.any(bits1[q:n0] != bits0[q:n0])


# ---------------------------------------------------------------------------- ARM
def _arm_blob(widths, Ws, bs):
    parts = []
    for W, b in zip(Ws, bs):
        parts += [np.asarray(W, np.float32).ravel(), np.asarray(b, np.float32).ravel()]
    return np.concatenate(parts)


def test_arm_zero_weights_mu0_b1():
    # all-zero weights -> mu = 0, b = exp(0) = 1
    cfg = workload.CONFIGS["ref"]
    m = oracle.model(cfg)
    mu, b = oracle.arm_mlp(m, np.arange(16.0), np.zeros(cfg.n_arm_w, np.float32))
    assert mu == 0.0 and b == 1.0


def test_arm_dot_product_example():
    # Linear 3->1, weights (1,2,3), input (1,1,1) -> 6 (last layer: no ReLU)
    cfg = workload.CONFIGS["tiny"].replace(n_ctx=3, arm_widths=(3, 2))
    m = oracle.model(cfg, arm_residual=(0,))
    blob = _arm_blob(None, [[[1, 2, 3], [0, 0, 0]]], [[0, 0]])
    mu, b = oracle.arm_mlp(m, [1, 1, 1], blob)
    assert mu == 6.0 and b == 1.0
    # negative pre-activation is NOT rectified on the last layer
    mu, _ = oracle.arm_mlp(m, [-1, -1, -1], blob)
    assert mu == -6.0


def test_arm_logscale_clamp():
    cfg = workload.CONFIGS["tiny"].replace(n_ctx=1, arm_widths=(1, 2))
    m = oracle.model(cfg, arm_residual=(0,))
    for s, want in [(10.0, 256.0), (-10.0, 1e-3), (0.5, math.exp(0.5))]:
        _, b = oracle.arm_mlp(m, [0.0], _arm_blob(None, [[[0], [0]]], [[0, s]]))
        assert b == pytest.approx(want, rel=1e-6)


def test_arm_residual_and_relu_order():
    # reading #8: z = ReLU(W z + b + z).  With W = 0, b = 0: z1 = ReLU(ctx).
    cfg = workload.CONFIGS["tiny"].replace(n_ctx=2, arm_widths=(2, 2, 2))
    m = oracle.model(cfg, arm_residual=(1, 0))
    blob = _arm_blob(None, [np.zeros((2, 2)), np.eye(2)], [[0, 0], [0, 0]])
    mu, b = oracle.arm_mlp(m, [-1.5, 0.7], blob)
    assert mu == 0.0 and b == pytest.approx(math.exp(0.7))
    # ReLU applies to the SUM (not x + ReLU(Wx)): W = I, b = 0, ctx = (-1, 0.5) -> ReLU(2x)
    blob = _arm_blob(None, [np.eye(2), np.eye(2)], [[0, 0], [0, 0]])
    mu, b = oracle.arm_mlp(m, [-1.0, 0.5], blob)
    assert mu == 0.0 and b == pytest.approx(math.exp(1.0))


def test_arm_vs_torch_linear():
    cfg = workload.CONFIGS["ref"]
    m = oracle.model(cfg)
    rng = np.random.default_rng(5)
    blob = rng.normal(0, 0.3, cfg.n_arm_w).astype(np.float32)
    layers, p = [], 0
    for k in range(len(cfg.arm_widths) - 1):
        i, o = cfg.arm_widths[k], cfg.arm_widths[k + 1]
        lin = torch.nn.Linear(i, o).double()
        with torch.no_grad():
            lin.weight.copy_(torch.from_numpy(blob[p:p + i * o].reshape(o, i).astype(np.float64)))
            lin.bias.copy_(torch.from_numpy(blob[p + i * o:p + i * o + o].astype(np.float64)))
        layers.append(lin)
        p += i * o + o
    for _ in range(50):
        ctx = rng.integers(-6, 7, 16).astype(np.float64)
        z = torch.from_numpy(ctx)
        z = torch.relu(layers[0](z))                 # 16 -> 24 (not residual)
        z = torch.relu(layers[1](z) + z)             # 24 -> 24 "LinR"
        z = layers[2](z)                             # 24 -> 2, last: no ReLU
        mu_t, s_t = z[0].item(), min(max(z[1].item(), math.log(1e-3)), math.log(256))
        mu, b = oracle.arm_mlp(m, ctx, blob)
        assert mu == pytest.approx(mu_t, rel=1e-12, abs=1e-12)
        assert b == pytest.approx(math.exp(s_t), rel=1e-12)


# --------------------------------------------------------------------------- rate
def _const_arm(cfg, mu, logb):
    blob = np.zeros(cfg.n_arm_w, np.float32)
    blob[-2] = mu
    blob[-1] = logb
    return blob


def test_rate_closed_form_constant_latents():
    g = gold("rate_constant.json")
    cfg = workload.CONFIGS["tiny"]
    m = oracle.model(cfg)
    n = cfg.n_latents
    assert n == 5440
    R, macs = oracle.rate(m, np.zeros(n, np.int16), _const_arm(cfg, 0, 0))
    assert R == pytest.approx(g["tiny_zero_latents_bits"], rel=1e-12)
    R, _ = oracle.rate(m, np.full(n, 2, np.int16), _const_arm(cfg, 0, 0))
    assert R == pytest.approx(g["tiny_all2_latents_bits"], rel=1e-12)
    # R >= 0 always, on random inputs too
    im = workload.make_image(cfg, 0)
    R, _ = oracle.rate(m, im.latents, im.arm_w)
    assert R > 0
    # general (mu, b): R = N * bits(c | mu, b)
    mu, b = 0.3, 2.5
    R, _ = oracle.rate(m, np.full(n, -1, np.int16), _const_arm(cfg, mu, math.log(b)))
    p = math.exp(-1.3 / b) * math.sinh(1 / (2 * b))
    assert R == pytest.approx(-n * math.log2(p), rel=1e-6)   # fp32 storage of log b


# -------------------------------------------------------------------- upsampling
def _torch_upsample_chain(lat_grid, k, dims_chain, K):
    """Reference: per x2 step, replicate pad E = K/4 then F.conv_transpose2d with
    the 2-D outer-product kernel k (x) k, stride 2, padding K/2 - 1 + 2E, crop."""
    x = torch.from_numpy(lat_grid.astype(np.float64))[None, None]
    kk = torch.from_numpy(np.outer(k, k).astype(np.float64))[None, None]
    E = K // 4
    for (h, w) in dims_chain:
        xp = F.pad(x, (E, E, E, E), mode="replicate")
        y = F.conv_transpose2d(xp, kk, stride=2, padding=K // 2 - 1 + 2 * E)
        x = y[:, :, :h, :w]
    return x[0, 0].numpy()


@pytest.mark.parametrize("K,H,W,L", [(8, 37, 53, 5), (4, 37, 53, 5), (8, 64, 64, 4), (8, 33, 17, 4)])
def test_upsample_vs_torch_conv_transpose(K, H, W, L):
    cfg = workload.CONFIGS["tiny"].replace(H=H, W=W, L=L, up_taps=K, syn_widths=(L, 8, 3))
    im = workload.make_image(cfg, 11)
    k = np.random.default_rng(3).normal(0, 0.5, K).astype(np.float32)   # asymmetric: pins orientation
    m = oracle.model(cfg)
    dense, _ = oracle.upsample(m, im.latents, k)
    dims = cfg.level_dims()
    np.testing.assert_array_equal(dense[0], im.level(cfg, 0))
    for l in range(1, L):
        ref = _torch_upsample_chain(im.level(cfg, l), k.astype(np.float64), dims[l - 1::-1], K)
        np.testing.assert_allclose(dense[l], ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K", [8, 4])
def test_upsample_bilinear_special_case(K):
    """With k = [0,0,1/4,3/4,3/4,1/4,0,0] (K=8) or [1/4,3/4,3/4,1/4] (K=4) each
    step is textbook bilinear x2 (torch F.interpolate, align_corners=False)."""
    cfg = workload.CONFIGS["tiny"].replace(H=64, W=96, L=4, up_taps=K)
    im = workload.make_image(cfg, 12, filter_kind="bilinear")
    dense, _ = oracle.upsample(oracle.model(cfg), im.latents, im.up_w)
    for l in range(1, 4):
        x = torch.from_numpy(im.level(cfg, l).astype(np.float64))[None, None]
        for _ in range(l):
            x = F.interpolate(x, scale_factor=2, mode="bilinear", align_corners=False)
        np.testing.assert_allclose(dense[l], x[0, 0].numpy(), rtol=0, atol=1e-12)


def test_upsample_preserves_constants():
    # a normalised filter maps a constant grid to the same constant
    cfg = workload.CONFIGS["tiny"].replace(H=45, W=71, L=6, syn_widths=(6, 8, 3))
    lat = np.full(cfg.n_latents, 7, np.int16)
    dense, _ = oracle.upsample(oracle.model(cfg), lat, workload.LANCZOS2_8)
    np.testing.assert_allclose(dense, 7.0, rtol=0, atol=1e-5)   # taps stored fp32


def test_upsample_L1_identity():
    # L = 1 -> the single grid, untouched
    cfg = workload.CONFIGS["tiny"].replace(L=1, syn_widths=(1, 8, 3))
    im = workload.make_image(cfg, 4)
    dense, macs = oracle.upsample(oracle.model(cfg), im.latents, im.up_w)
    np.testing.assert_array_equal(dense[0], im.latents.reshape(64, 64))
    assert macs.up == 0


def test_upsample_linear_in_filter_scatter_brute_force():
    """Independent brute force: a single impulse latent at level 1 scatters
    k[a] k[b] into out[2i + a - (K/2-1)][2j + b - (K/2-1)] away from borders."""
    cfg = workload.CONFIGS["tiny"].replace(H=32, W=32, L=2, syn_widths=(2, 8, 3))
    k = np.arange(1, 9, dtype=np.float32) / 10
    lat = np.zeros(cfg.n_latents, np.int16)
    i0, j0 = 7, 9
    lat[32 * 32 + i0 * 16 + j0] = 1
    dense, _ = oracle.upsample(oracle.model(cfg), lat, k)
    want = np.zeros((32, 32))
    for a in range(8):
        for b in range(8):
            want[2 * i0 + a - 3, 2 * j0 + b - 3] += k[a] * k[b]
    np.testing.assert_allclose(dense[1], want, rtol=0, atol=1e-7)


# --------------------------------------------------------------------- synthesis
def _torch_synthesis(cfg, dense, syn_w):
    x = torch.from_numpy(dense)[None]
    p = 0
    sw = syn_w.astype(np.float64)
    n1 = len(cfg.syn_widths) - 1
    for k in range(n1):
        i, o = cfg.syn_widths[k], cfg.syn_widths[k + 1]
        A = torch.from_numpy(sw[p:p + i * o].reshape(o, i, 1, 1))
        a = torch.from_numpy(sw[p + i * o:p + i * o + o])
        x = F.conv2d(x, A, a)
        if not (k == n1 - 1 and cfg.syn_n_res == 0):
            x = torch.relu(x)
        p += i * o + o
    for r in range(cfg.syn_n_res):
        G = torch.from_numpy(sw[p:p + 81].reshape(3, 3, 3, 3))
        g = torch.from_numpy(sw[p + 81:p + 84])
        x = x + F.conv2d(F.pad(x, (1, 1, 1, 1), mode="replicate"), G, g)
        if r < cfg.syn_n_res - 1:
            x = torch.relu(x)
        p += 84
    return x[0].numpy()


@pytest.mark.parametrize("name", ["tiny", "low", "ref"])
def test_synthesis_vs_torch_conv(name):
    cfg = workload.CONFIGS[name].replace(H=23, W=31)
    rng = np.random.default_rng(9)
    dense = rng.normal(0, 1, (cfg.L, 23, 31))
    syn_w = rng.normal(0, 0.3, cfg.n_syn_w).astype(np.float32)
    xh, _, macs = oracle.synthesis(oracle.model(cfg), dense, syn_w)
    np.testing.assert_allclose(xh, _torch_synthesis(cfg, dense, syn_w), rtol=1e-12, atol=1e-12)


def test_synthesis_zero_weights_constant_output():
    """All synthesis weights zero, biases kept -> x_hat is the per-channel
    constant ReLU(ReLU(a1) + g0) + g1 (2 residual layers)."""
    cfg = workload.CONFIGS["ref"].replace(H=16, W=20)
    rng = np.random.default_rng(10)
    syn_w = np.zeros(cfg.n_syn_w, np.float32)
    a1 = rng.normal(0, 1, 3).astype(np.float32)
    g0 = rng.normal(0, 1, 3).astype(np.float32)
    g1 = rng.normal(0, 1, 3).astype(np.float32)
    o1 = 7 * 40 + 40 + 40 * 3
    syn_w[o1:o1 + 3] = a1
    syn_w[o1 + 3 + 81:o1 + 3 + 84] = g0
    syn_w[o1 + 3 + 84 + 81:o1 + 3 + 168] = g1
    dense = rng.normal(0, 1, (7, 16, 20))
    xh, _, _ = oracle.synthesis(oracle.model(cfg), dense, syn_w)
    c = np.maximum(np.maximum(a1.astype(np.float64), 0) + g0, 0) + g1
    np.testing.assert_allclose(xh, np.broadcast_to(c[:, None, None], xh.shape), rtol=0, atol=1e-15)


def test_synthesis_identity_passthrough():
    """SPEC.md:316 engineered identity: 1x1 layers select dense channels 0..2
    (inputs >= 0 so the ReLUs pass them), zero residual weights and biases ->
    x_hat = those channels."""
    cfg = workload.CONFIGS["low"].replace(H=10, W=13)
    syn_w = np.zeros(cfg.n_syn_w, np.float32)
    A0 = np.zeros((16, 7), np.float32)
    A0[0, 0] = A0[1, 1] = A0[2, 2] = 1
    A1 = np.zeros((3, 16), np.float32)
    A1[0, 0] = A1[1, 1] = A1[2, 2] = 1
    syn_w[:112] = A0.ravel()
    syn_w[128:128 + 48] = A1.ravel()
    dense = np.abs(np.random.default_rng(1).normal(0, 1, (7, 10, 13)))
    xh, _, _ = oracle.synthesis(oracle.model(cfg), dense, syn_w)
    np.testing.assert_allclose(xh, dense[:3], rtol=0, atol=0)


# -------------------------------------------------------------------- MSE / cost
def test_cost_closed_form_zero_network():
    cfg = workload.CONFIGS["tiny"]
    im = workload.make_image(cfg, 6)
    syn_w = np.zeros(cfg.n_syn_w, np.float32)
    # tiny: 4->8->3 then ONE residual (last, no ReLU): x_hat = ReLU(a1) + g0
    a1 = np.array([0.2, -0.3, 0.6], np.float32)
    g0 = np.array([0.1, 0.25, -0.2], np.float32)
    o1 = 4 * 8 + 8 + 8 * 3
    syn_w[o1:o1 + 3] = a1
    syn_w[o1 + 3 + 81:o1 + 3 + 84] = g0
    c = np.maximum(a1.astype(np.float64), 0) + g0
    m = oracle.model(cfg)
    r = oracle.rd_forward(m, im.latents, im.arm_w, im.up_w, syn_w, im.image)
    x = im.image.astype(np.float64)
    mse = np.mean([np.mean((x[ch] - c[ch]) ** 2) for ch in range(3)])
    assert r["mse"] == pytest.approx(mse, rel=1e-12)
    assert r["sse"] == pytest.approx(mse * 3 * 64 * 64, rel=1e-12)
    R, _ = oracle.rate(m, im.latents, im.arm_w)
    assert r["rate_bits"] == pytest.approx(R, rel=1e-15)
    assert r["cost"] == pytest.approx(mse + cfg.lam * R / 4096, rel=1e-12)
    m.lam = 0.0
    r0 = oracle.rd_forward(m, im.latents, im.arm_w, im.up_w, syn_w, im.image)
    assert r0["cost"] == r0["mse"]


# ---------------------------------------------------------------------- MACs
def closed_form_macs(cfg, H, W):
    """MAC closed form from layer widths (SURVEY.md §8c 'MAC counts')."""
    dims = cfg.replace(H=H, W=W).level_dims()
    nlat = sum(h * w for h, w in dims)
    aw = cfg.arm_widths
    arm = sum(aw[k] * aw[k + 1] for k in range(len(aw) - 1)) * nlat
    up = sum((cfg.up_taps // 2) * (dims[j + 1][0] * dims[j][1] + dims[j][0] * dims[j][1])
             for l in range(1, cfg.L) for j in range(l))
    sw = cfg.syn_widths
    syn = (sum(sw[k] * sw[k + 1] for k in range(len(sw) - 1)) + 81 * cfg.syn_n_res) * H * W
    return arm, up, syn


@pytest.mark.parametrize("name,H,W", [("tiny", 64, 64), ("low", 67, 93), ("ref", 40, 57)])
def test_mac_counters_equal_closed_form(name, H, W):
    cfg = workload.CONFIGS[name].replace(H=H, W=W)
    im = workload.make_image(cfg, 2)
    r = oracle.rd_forward(oracle.model(cfg), im.latents, im.arm_w, im.up_w, im.syn_w, im.image)
    arm, up, syn = closed_form_macs(cfg, H, W)
    assert r["macs"] == dict(arm=arm, up=up, syn=syn)


def test_table1_params_and_macs():
    """Table 1: params exact (bias on every ARM / synthesis
    layer, none on the TConv: reading #10); MAC/pixel within 1% with the 2-D
    TConv-K accounting (K^2/4 MAC per produced sample) at 512x768, L = 7."""
    g = gold("table1.json")
    H, W, L = 512, 768, 7
    dims = [(-(-H // (1 << l)), -(-W // (1 << l))) for l in range(L)]
    nlat = sum(h * w for h, w in dims)
    for key, arch in workload.TABLE1.items():
        row = g["rows"][str(key)]
        aw, sw, R, K = arch["arm"], arch["syn"], arch["syn_n_res"], arch["up_kernel"]
        arm_p = sum(aw[k] * aw[k + 1] + aw[k + 1] for k in range(len(aw) - 1))
        syn_p = sum(sw[k] * sw[k + 1] + sw[k + 1] for k in range(len(sw) - 1)) + R * 84
        assert arm_p + K * K + syn_p == row["params"]
        arm_m = sum(aw[k] * aw[k + 1] for k in range(len(aw) - 1)) * nlat / (H * W)
        up_m = sum(K * K / 4 * dims[j][0] * dims[j][1] for l in range(1, L) for j in range(l)) / (H * W)
        syn_m = sum(sw[k] * sw[k + 1] for k in range(len(sw) - 1)) + 81 * R
        tot = arm_m + up_m + syn_m
        assert abs(tot - row["mac_per_pixel"]) / row["mac_per_pixel"] < 0.01
        assert arm_m / tot <= g["arm_share_max"]["value"]


# -------------------------------------------- Table 1 2-D TConv (NEXT-1)
def _torch_upsample_chain_2d(lat_grid, k2, dims_chain, K):
    """Reference: per x2 step, replicate pad E = K/4 then F.conv_transpose2d with
    the (non-separable) K x K kernel, stride 2, padding K/2 - 1 + 2E, crop."""
    x = torch.from_numpy(lat_grid.astype(np.float64))[None, None]
    kk = torch.from_numpy(k2.astype(np.float64))[None, None]
    E = K // 4
    for (h, w) in dims_chain:
        xp = F.pad(x, (E, E, E, E), mode="replicate")
        y = F.conv_transpose2d(xp, kk, stride=2, padding=K // 2 - 1 + 2 * E)
        x = y[:, :, :h, :w]
    return x[0, 0].numpy()


@pytest.mark.parametrize("K,H,W,L", [(8, 37, 53, 5), (4, 37, 53, 5), (8, 33, 17, 4), (4, 64, 64, 3)])
def test_upsample_2d_vs_torch_conv_transpose(K, H, W, L):
    """Table 1 TConv-K as a true 2-D kernel: random, asymmetric and
    non-separable (rank K), so orientation and indexing on both axes are pinned."""
    cfg = workload.CONFIGS["tiny"].replace(H=H, W=W, L=L, up_taps=K, up_2d=True, syn_widths=(L, 8, 3))
    im = workload.make_image(cfg, 13)
    k2 = np.random.default_rng(4).normal(0, 0.5, (K, K)).astype(np.float32)
    assert np.linalg.matrix_rank(k2.astype(np.float64)) == K
    dense, _ = oracle.upsample(oracle.model(cfg), im.latents, k2.ravel())
    dims = cfg.level_dims()
    np.testing.assert_array_equal(dense[0], im.level(cfg, 0))
    for l in range(1, L):
        ref = _torch_upsample_chain_2d(im.level(cfg, l), k2, dims[l - 1::-1], K)
        np.testing.assert_allclose(dense[l], ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K", [8, 4])
def test_upsample_2d_separable_kernel_equals_separable_path(K):
    """k2 = k (x) k through the 2-D scatter == the separable two-pass path (two
    independent code paths of the oracle; fp64 rounding only)."""
    base = workload.CONFIGS["tiny"].replace(H=41, W=58, L=5, up_taps=K, syn_widths=(5, 8, 3))
    im = workload.make_image(base, 14)
    # taps in multiples of 1/8: k (x) k is exact in fp32, so only the fp64
    # summation order differs between the two paths
    k = (np.random.default_rng(5).integers(-8, 9, K) / 8.0).astype(np.float32)
    d1, m1 = oracle.upsample(oracle.model(base), im.latents, k)
    k2 = np.outer(k, k).astype(np.float32)
    d2, m2 = oracle.upsample(oracle.model(base.replace(up_2d=True)), im.latents, k2.ravel())
    np.testing.assert_allclose(d2, d1, rtol=1e-12, atol=1e-9)


def test_upsample_2d_normalised_preserves_constants():
    cfg = workload.CONFIGS["t2300"].replace(H=45, W=71, L=6, syn_widths=(6, 40, 3))
    im = workload.make_image(cfg, 15, filter_kind="normalised2d")
    for ra in (0, 1):
        for sb in (0, 1):
            assert abs(im.up_w.reshape(8, 8)[ra::2, sb::2].sum() - 1.0) < 1e-6
    lat = np.full(cfg.n_latents, -5, np.int16)
    dense, _ = oracle.upsample(oracle.model(cfg), lat, im.up_w)
    np.testing.assert_allclose(dense, -5.0, rtol=0, atol=1e-4)


@pytest.mark.parametrize("name", ["t300", "t545", "t1079", "t2300"])
def test_table1_configs_oracle_macs_match_table(name):
    """The instrumented oracle on the Table 1 architectures (2-D TConv) counts
    (K/2)^2 MAC per produced sample and lands within 1 % of the paper's printed
    MAC/pixel (300 / 545 / 1079 / 2300)."""
    cfg = workload.CONFIGS[name]
    g = gold("table1.json")["rows"][name[1:]]
    im = workload.make_image(cfg, 16)
    r = oracle.rd_forward_image(cfg, im)
    dims = cfg.level_dims()
    K = cfg.up_taps
    up = sum((K // 2) ** 2 * dims[j][0] * dims[j][1] for l in range(1, cfg.L) for j in range(l))
    assert r["macs"]["up"] == up
    tot = sum(r["macs"].values()) / (cfg.H * cfg.W)
    assert abs(tot - g["mac_per_pixel"]) / g["mac_per_pixel"] < 0.01


# ---------------------------------------------------- decoder output (NEXT-3)
def test_decode_u8_closed_forms():
    """clamp to [0,1] then 255 x rounded half to even."""
    cfg = workload.CONFIGS["tiny"].replace(H=1, W=8)
    m = oracle.model(cfg)
    xh = np.zeros((3, 1, 8))
    xh[0, 0] = [-0.3, 0.0, 1 / 255, 128 / 255, 1.0, 1.7, 0.5 / 255, 1.5 / 255]
    xh[1, 0] = np.linspace(0, 1, 8)
    xh[2, 0] = 254.5 / 255
    out = oracle.decode_u8(m, xh)
    assert out.shape == (1, 8, 3)
    assert list(out[0, :, 0]) == [0, 0, 1, 128, 255, 255, 0, 2]   # clamps; ties to even
    assert list(out[0, :, 1]) == [int(np.rint(255 * v)) for v in np.linspace(0, 1, 8)]
    assert np.all(out[0, :, 2] == 254)                            # 254.5 -> even
    # monotone in x_hat
    xs = np.sort(np.random.default_rng(0).uniform(-0.2, 1.2, 8 * 3)).reshape(3, 1, 8)
    o = oracle.decode_u8(m, xs).transpose(2, 0, 1).ravel()
    assert np.all(np.diff(o.astype(int)) >= 0)
