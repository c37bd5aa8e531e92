"""Pins of the oracle's autoregressive decode (oracle.arm_decode, NEXT-3;
PAPER.md:101-105, 341-365): the decoder recovers the latents one by one in
raster order, the ARM conditioning each on already decoded neighbours; the
entropy decoder (out of scope) is played by the true latents, revealed once
their (mu, b) exist.

What pins it to something other than itself:
  * causality ("conditioned on previously decoded" values):
    with the causal template no context ever reads an undecoded latent, the
    decoded latents equal the encoded ones, and every latent's (mu, b, bits)
    equals the encoder's all-at-once ARM (oracle.rate per latent) exactly --
    a dropped / misplaced context or a wrong reveal order breaks the equality;
  * a non-causal template (a right neighbour, dy = 0, dx = +1) is detected
    (status -1): the decode order really is enforced;
  * zero network: mu = 0, b = exp(0) = 1 for every latent, bits = the
    closed-form Laplace(0, 1) bin mass (telescoping).
"""
import math

import numpy as np
import pytest

import oracle
import workload


@pytest.mark.parametrize("name", ["tiny", "low", "t1079"])
def test_decode_equals_encoder_per_latent(name):
    cfg = workload.CONFIGS[name].replace(H=23, W=37)
    im = workload.make_image(cfg, 5)
    m = oracle.model(cfg)
    st, dec, mu, b, bits, rate = oracle.arm_decode(m, im.latents, im.arm_w)
    assert st == 0
    np.testing.assert_array_equal(dec, im.latents)
    R, mu_e, b_e, bits_e, _ = oracle.rate(m, im.latents, im.arm_w, per_latent=True)
    np.testing.assert_array_equal(mu, mu_e)
    np.testing.assert_array_equal(b, b_e)
    np.testing.assert_array_equal(bits, bits_e)
    assert rate == pytest.approx(R, rel=1e-12)


def test_non_causal_template_is_detected():
    cfg = workload.CONFIGS["tiny"].replace(H=9, W=11)
    im = workload.make_image(cfg, 6)
    m = oracle.model(cfg)
    m.ctx_dx[0] = 1          # first context: the right neighbour (dy = 0, dx = +1)
    m.ctx_dy[0] = 0
    st, *_ = oracle.arm_decode(m, im.latents, im.arm_w)
    assert st == -1


def test_zero_network_closed_form():
    cfg = workload.CONFIGS["tiny"].replace(H=8, W=12)
    im = workload.make_image(cfg, 7)
    m = oracle.model(cfg)
    st, dec, mu, b, bits, rate = oracle.arm_decode(m, im.latents, np.zeros_like(im.arm_w))
    assert st == 0
    assert np.all(mu == 0.0) and np.all(b == 1.0)

    def ref_bits(y):
        cdf = lambda t: 0.5 * math.exp(t) if t < 0 else 1.0 - 0.5 * math.exp(-t)
        return -math.log2(max(cdf(y + 0.5) - cdf(y - 0.5), 2.0 ** -16))
    np.testing.assert_allclose(bits, [ref_bits(float(y)) for y in im.latents], rtol=1e-12)
