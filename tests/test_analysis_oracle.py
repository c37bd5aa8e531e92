"""Pins of the N-O analysis-transform oracle (oracle/ccanalysis.c, NEXT-4).

* every step against torch's library ops in fp64 (depth-wise conv2d with
  groups = C and zero padding, 1x1 conv2d, avg_pool2d with ceil_mode and
  count_include_pad=False, relu), composed in the readings' order;
* zero weights -> all-zero pyramid;
* grid dims == the decoder's ceil dims (reading A6);
* MAC count: the instrumented oracle == the closed form, and at 512x768 it is
  within 10 % of the paper's printed "160 kMAC per pixel".
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import workload


def torch_analysis(acfg, image, w):
    C = acfg.C
    t = torch.from_numpy(w.astype(np.float64))
    off = [0]

    def take(n, shape):
        v = t[off[0]: off[0] + n].reshape(shape)
        off[0] += n
        return v

    x = torch.from_numpy(image.astype(np.float64))[None]
    x = F.conv2d(x, take(C * 3, (C, 3, 1, 1)), take(C, (C,)))
    lat = []
    for l in range(acfg.L):
        for b in range(acfg.blocks):
            down = l > 0 and b == 0
            k = take(C * 49, (C, 1, 7, 7))
            kb = take(C, (C,))
            W1 = take(4 * C * C, (4 * C, C, 1, 1))
            b1 = take(4 * C, (4 * C,))
            W2 = take(4 * C * C, (C, 4 * C, 1, 1))
            b2 = take(C, (C,))
            y = F.conv2d(x, k, kb, stride=2 if down else 1, padding=3, groups=C)
            y = F.conv2d(F.relu(F.conv2d(y, W1, b1)), W2, b2)
            if down:
                Wid = take(C * C, (C, C, 1, 1))
                bid = take(C, (C,))
                idn = F.avg_pool2d(x, 2, 2, ceil_mode=True, count_include_pad=False)
                y = y + F.conv2d(idn, Wid, bid)
            else:
                y = y + x
            x = y
        lat.append(F.conv2d(x, take(C, (1, C, 1, 1)), take(1, (1,)))[0, 0].numpy().ravel())
    assert off[0] == w.size
    return np.concatenate(lat)


def closed_form_macs(acfg):
    C, tot = acfg.C, 3 * acfg.C * acfg.H * acfg.W
    for l in range(acfg.L):
        h, w = -(-acfg.H // (1 << l)), -(-acfg.W // (1 << l))
        tot += acfg.blocks * (C * 49 + 8 * C * C) * h * w + (C * C * h * w if l > 0 else 0) + C * h * w
    return tot


@pytest.mark.parametrize("kw", [dict(), dict(H=19, W=30, L=5, C=4, blocks=1), dict(H=2, W=3, L=2, C=8, blocks=3)])
def test_analysis_vs_torch(kw):
    acfg = workload.ANALYSIS["no_tiny"].replace(**kw)
    image, w = workload.make_analysis_input(acfg, 3)
    got, macs = oracle.analysis_forward(acfg, image, w)
    np.testing.assert_allclose(got, torch_analysis(acfg, image, w), rtol=1e-10, atol=1e-12)
    assert macs == closed_form_macs(acfg)
    assert np.abs(got).max() > 1e-3


def test_analysis_zero_weights_zero_latents():
    acfg = workload.ANALYSIS["no_tiny"]
    image, w = workload.make_analysis_input(acfg, 4)
    got, _ = oracle.analysis_forward(acfg, image, np.zeros_like(w))
    assert np.all(got == 0.0)


def test_analysis_grid_dims_and_paper_complexity():
    acfg = workload.ANALYSIS["no_kodak"]
    cfg = workload.CONFIGS["ref"]
    assert sum(h * w for h, w in cfg.level_dims()) == sum(
        -(-acfg.H // (1 << l)) * -(-acfg.W // (1 << l)) for l in range(acfg.L))
    kmac = closed_form_macs(acfg) / (acfg.H * acfg.W) / 1e3
    assert abs(kmac - 160.0) / 160.0 < 0.10, kmac
