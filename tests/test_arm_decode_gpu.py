"""GPU parity of the wavefront ARM decode (cc_arm_decode, NEXT-3).

* decoded latents == the encoded ones (exact);
* per-latent (mu, scale, bits) bit-identical to the encoder's cc_arm_rate
  (same arithmetic, arm_math.cuh; the wavefront order cannot change a latent's
  value when every context is decoded before it);
* no poison read (no context read of a not-yet-decoded latent);
* vs the oracle's raster decode (oracle.arm_decode): bits within the encoder's
  1e-3-bit per-latent tolerance, rate 1e-5 relative;
* a too-small skew (test hook CCRD_DEC_SKEW) MUST produce poison reads and
  different outputs -- the harness detects schedule errors;
* several images in one call (each with its own ARM), every Table 1 ARM.
"""
import os

import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def run_decode(cfg, ims, skew=None):
    import paper_2403_11651_b200 as P
    d = P.desc_from_config(cfg)
    lat = [torch.from_numpy(im.latents).cuda() for im in ims]
    dec = [torch.full_like(t, -32768) for t in lat]
    n = lat[0].numel()
    mu = [torch.zeros(n, device="cuda") for _ in ims]
    sc = [torch.zeros(n, device="cuda") for _ in ims]
    bits = [torch.zeros(n, device="cuda") for _ in ims]
    rate = torch.zeros(len(ims), dtype=torch.float64, device="cuda")
    poison = torch.zeros(1, dtype=torch.int32, device="cuda")
    io = [P.CcImageIO(lat[i].data_ptr(), ims[i].arm_w.ctypes.data, 0, 0, 0, 0) for i in range(len(ims))]
    wsb = P.cc_arm_decode_workspace_bytes(d, len(ims))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    old = os.environ.get("CCRD_DEC_SKEW")
    if skew is not None:
        os.environ["CCRD_DEC_SKEW"] = str(skew)
    try:
        P.cc_arm_decode(d, io, [t.data_ptr() for t in dec], rate.data_ptr(), [t.data_ptr() for t in mu],
                        [t.data_ptr() for t in sc], [t.data_ptr() for t in bits], poison.data_ptr(), ws.data_ptr(),
                        wsb, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    finally:
        if skew is not None:
            if old is None:
                del os.environ["CCRD_DEC_SKEW"]
            else:
                os.environ["CCRD_DEC_SKEW"] = old
    return ([t.cpu().numpy() for t in dec], rate.cpu().numpy(), [t.cpu().numpy() for t in mu],
            [t.cpu().numpy() for t in sc], [t.cpu().numpy() for t in bits], int(poison.item()))


def encoder_arm(cfg, im):
    import paper_2403_11651_b200 as P
    d = P.desc_from_config(cfg)
    lat = torch.from_numpy(im.latents).cuda()
    n = lat.numel()
    mu, sc, bits = (torch.zeros(n, device="cuda") for _ in range(3))
    rate = torch.zeros(1, dtype=torch.float64, device="cuda")
    wsb = P.cc_workspace_bytes(d, 1)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    # the decoder shares the FFMA2 encoder's arithmetic (arm_math.cuh): compare
    # against that path (the tensor-core path agrees within the tolerances of
    # test_arm_tc_gpu.py, not bit for bit)
    with P.arm_path(P.CC_ARM_FFMA2):
        P.cc_arm_rate(d, lat.data_ptr(), im.arm_w, rate.data_ptr(), mu.data_ptr(), sc.data_ptr(), bits.data_ptr(),
                      ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return mu.cpu().numpy(), sc.cpu().numpy(), bits.cpu().numpy(), float(rate.item())


@pytest.mark.parametrize("name,H,W", [("ref", 37, 61), ("low", 64, 96), ("tiny", 5, 7), ("t300", 41, 29),
                                      ("t545", 33, 47), ("t1079", 29, 35), ("t2300", 31, 40)])
def test_decode_bit_identical_to_encoder(name, H, W):
    cfg = workload.CONFIGS[name].replace(H=H, W=W)
    ims = [workload.make_image(cfg, 200 + k) for k in range(3)]
    dec, rate, mu, sc, bits, poison = run_decode(cfg, ims)
    assert poison == 0
    for k, im in enumerate(ims):
        np.testing.assert_array_equal(dec[k], im.latents)
        mu_e, sc_e, bits_e, rate_e = encoder_arm(cfg, im)
        np.testing.assert_array_equal(mu[k], mu_e)
        np.testing.assert_array_equal(sc[k], sc_e)
        np.testing.assert_array_equal(bits[k], bits_e)
        assert rate[k] == pytest.approx(rate_e, rel=1e-6)


def test_decode_vs_oracle_raster_decode():
    cfg = workload.CONFIGS["ref"].replace(H=48, W=80)
    im = workload.make_image(cfg, 210)
    dec, rate, mu, sc, bits, poison = run_decode(cfg, [im])
    st, dec_o, mu_o, b_o, bits_o, rate_o = oracle.arm_decode(oracle.model(cfg), im.latents, im.arm_w)
    assert st == 0 and poison == 0
    np.testing.assert_array_equal(dec[0], dec_o)
    assert np.abs(bits[0] - bits_o).max() <= 1e-3
    assert rate[0] == pytest.approx(rate_o, rel=1e-5)


def test_too_small_skew_is_detected():
    cfg = workload.CONFIGS["ref"].replace(H=32, W=48)
    im = workload.make_image(cfg, 211)
    good = run_decode(cfg, [im])
    bad = run_decode(cfg, [im], skew=1)   # the 16-context template needs a = 4
    assert good[5] == 0 and bad[5] > 0
    assert not np.array_equal(good[4][0], bad[4][0])


def test_too_small_skew_is_detected_on_every_row_and_column():
    """Ring rows are reused every RR rows and ring columns every 32 columns;
    with the poison counter the kernel re-poisons a ring row when its row
    starts and keeps the 8 slots ahead of the wavefront poisoned, so the
    premature reads of a too-small skew are counted on rows past RR and
    columns past 32 too: the count grows in proportion to the grid."""
    def count(H, W):
        cfg = workload.CONFIGS["ref"].replace(H=H, W=W)
        im = workload.make_image(cfg, 213)
        return run_decode(cfg, [im], skew=1)[5]
    base = count(64, 48)            # a = 1: RR = 64 ring rows for w = 48
    assert base > 0
    assert count(256, 48) > 3 * base     # 4x the rows, 3/4 of them past RR
    assert count(64, 192) > 3 * base     # 4x the columns, 7/8 of them past 32


@pytest.mark.timeout(600)
def test_decode_full_2k_image():
    """BASELINE.json configs[3] size (1365 x 2048): bit-identical to the encoder."""
    cfg = workload.CONFIGS["batched2k"]
    im = workload.make_image(cfg, 212)
    dec, rate, mu, sc, bits, poison = run_decode(cfg, [im])
    assert poison == 0
    np.testing.assert_array_equal(dec[0], im.latents)
    mu_e, sc_e, bits_e, rate_e = encoder_arm(cfg, im)
    np.testing.assert_array_equal(bits[0], bits_e)
    np.testing.assert_array_equal(mu[0], mu_e)
