"""Pins of the training-iteration oracle (oracle/cctrain.c, NEXT-2) -- CPU.

What fixes it independently of its own backward code:
  * its forward at u = 0 and integer y IS the RD oracle's forward (Eq. 1);
  * central finite differences of its fp64 forward agree with its analytic
    gradient for coordinates of every parameter group (latents at every level,
    each ARM layer's weights and biases, the upsampling taps -- separable and
    2-D --, each synthesis layer);
  * lambda = 0 removes the rate: the ARM gradient is exactly 0;
  * L = 1 has no upsampling: the tap gradient is exactly 0;
  * the Adam step equals torch.optim.Adam (library routine) on the same gradient;
  * a few iterations with a small step decrease the cost (descent sanity,
    SPEC.md:484).
"""
import numpy as np
import pytest
import torch

import oracle
import workload


def small_cfg(name="ref", **kw):
    base = workload.CONFIGS[name]
    d = dict(H=14, W=22, L=4, syn_widths=(4, 8, 3), syn_n_res=2)
    d.update(kw)
    if "L" in kw and "syn_widths" not in kw:
        d["syn_widths"] = (kw["L"], 8, 3)
    return base.replace(**d)


def setup(cfg, seed=1, filt="random"):
    im = workload.make_image(cfg, seed, filter_kind=filt)
    rng = np.random.default_rng(seed + 100)
    y = (im.latents + rng.uniform(-0.45, 0.45, im.latents.size)).astype(np.float32)  # continuous latents
    u = workload.gen_noise(rng, im.latents.size)
    par = oracle.pack_params(y, im.arm_w, im.up_w, im.syn_w)
    return im, par, u


def groups(cfg):
    """(name, start, stop) of the parameter groups in the packed layout."""
    n_lat = cfg.n_latents
    out = []
    dims = cfg.level_dims()
    off = 0
    for l, (h, w) in enumerate(dims):
        out.append((f"y{l}", off, off + h * w))
        off += h * w
    aw = cfg.arm_widths
    for k in range(len(aw) - 1):
        out.append((f"arm_W{k}", off, off + aw[k] * aw[k + 1]))
        off += aw[k] * aw[k + 1]
        out.append((f"arm_b{k}", off, off + aw[k + 1]))
        off += aw[k + 1]
    out.append(("up", off, off + cfg.n_up_w))
    off += cfg.n_up_w
    sw = cfg.syn_widths
    for k in range(len(sw) - 1):
        out.append((f"syn_A{k}", off, off + sw[k] * sw[k + 1]))
        off += sw[k] * sw[k + 1]
        out.append((f"syn_a{k}", off, off + sw[k + 1]))
        off += sw[k + 1]
    for r in range(cfg.syn_n_res):
        out.append((f"res{r}_G", off, off + 81))
        out.append((f"res{r}_g", off + 81, off + 84))
        off += 84
    assert off == n_lat + cfg.n_arm_w + cfg.n_up_w + cfg.n_syn_w
    return out


def test_forward_is_the_rd_oracle_at_zero_noise():
    cfg = small_cfg()
    im = workload.make_image(cfg, 3)
    par = oracle.pack_params(im.latents.astype(np.float32), im.arm_w, im.up_w, im.syn_w)
    out, _ = oracle.train_grad(oracle.model(cfg), par, np.zeros(cfg.n_latents, np.float32), im.image)
    ref = oracle.rd_forward_image(cfg, im)
    np.testing.assert_allclose(out, [ref["rate_bits"], ref["sse"], ref["mse"], ref["cost"]], rtol=1e-12)


@pytest.mark.parametrize("name,kw,filt", [
    ("ref", {}, "random"),
    ("ref", dict(L=5, H=19, W=13, syn_widths=(5, 8, 3), syn_n_res=1), "lanczos2"),
    ("low", dict(L=3, syn_widths=(3, 8, 3), syn_n_res=2), "random"),
    ("t300", dict(L=4, H=16, W=20, syn_widths=(4, 8, 3), syn_n_res=1), "normalised2d"),
])
def test_gradient_vs_central_finite_differences(name, kw, filt):
    cfg = small_cfg(name, **kw).replace(lam=0.05)   # rate term well represented
    im, par, u = setup(cfg, filt=filt)
    m = oracle.model(cfg)
    _, g = oracle.train_grad(m, par, u, im.image)
    rng = np.random.default_rng(7)
    checked = 0
    for gname, a, b in groups(cfg):
        for idx in rng.choice(np.arange(a, b), size=min(3, b - a), replace=False):
            p1, p2 = par.copy(), par.copy()
            eps = 1e-5 * max(1.0, abs(float(par[idx])))  # small: no ReLU kink crossed
            p1[idx] = np.float32(par[idx] + eps)
            p2[idx] = np.float32(par[idx] - eps)
            j1 = oracle.train_grad(m, p1, u, im.image)[0][3]
            j2 = oracle.train_grad(m, p2, u, im.image)[0][3]
            fd = (j1 - j2) / (float(p1[idx]) - float(p2[idx]))
            scale = max(abs(fd), abs(g[idx]), 1e-3 * np.abs(g[a:b]).max(), 1e-9)
            assert abs(fd - g[idx]) <= 2e-3 * scale, (gname, idx, fd, g[idx])
            checked += 1
    assert checked >= 3 * 8


def test_lambda_zero_removes_the_rate_gradient():
    cfg = small_cfg().replace(lam=0.0)
    im, par, u = setup(cfg)
    out, g = oracle.train_grad(oracle.model(cfg), par, u, im.image)
    n_lat = cfg.n_latents
    assert np.all(g[n_lat:n_lat + cfg.n_arm_w] == 0.0)
    assert out[3] == out[2]


def test_single_level_has_no_upsampling_gradient():
    cfg = small_cfg(L=1, syn_widths=(1, 8, 3), syn_n_res=1)
    im, par, u = setup(cfg)
    _, g = oracle.train_grad(oracle.model(cfg), par, u, im.image)
    a = cfg.n_latents + cfg.n_arm_w
    assert np.all(g[a:a + cfg.n_up_w] == 0.0)


def test_adam_step_equals_torch_adam():
    rng = np.random.default_rng(0)
    n = 257
    p = rng.normal(0, 1, n).astype(np.float32)
    m1, m2 = np.zeros(n), np.zeros(n)
    tp = torch.nn.Parameter(torch.from_numpy(p.astype(np.float64)))
    opt = torch.optim.Adam([tp], lr=1e-2, betas=(0.9, 0.999), eps=1e-8)
    for t in range(1, 4):
        g = rng.normal(0, 1, n)
        oracle.adam_step(p, g, m1, m2, 1e-2, 0.9, 0.999, 1e-8, t)
        tp.grad = torch.from_numpy(g)
        opt.step()
        np.testing.assert_allclose(p, tp.detach().numpy(), rtol=2e-6, atol=2e-7)  # p is stored fp32
        tp.data = torch.from_numpy(p.astype(np.float64))


def test_descent_sanity():
    cfg = small_cfg().replace(H=24, W=32)
    im, par, u = setup(cfg)
    m = oracle.model(cfg)
    m1, m2 = np.zeros(par.size), np.zeros(par.size)
    costs = []
    for t in range(1, 16):
        out, g = oracle.train_grad(m, par, np.zeros_like(u), im.image)
        costs.append(out[3])
        oracle.adam_step(par, g, m1, m2, 3e-3, 0.9, 0.999, 1e-8, t)
    assert costs[-1] < 0.9 * costs[0]
