"""Table 1 exact architectures (NEXT-1): ARMs with C = 8 /
16 / 24 context, the non-separable 2-D TConv-4 / TConv-8 upsampling, and the
synthesis widths.  CPU: the library's closed-form MAC count equals the
oracle's instrumented counters.  GPU: CUDA path vs the fp64 oracle on the
Kodak-sized configs and ragged shapes (north_star tolerances), per-level dense
parity of the 2-D upsampling stage, and the strip entry refusing 2-D."""
import numpy as np
import pytest

import oracle
import workload

TABLE1 = ["t300", "t545", "t1079", "t2300"]


@pytest.mark.parametrize("name", TABLE1)
def test_library_mac_closed_form_equals_oracle_counters(name):
    from paper_2403_11651_b200 import ccrd
    cfg = workload.CONFIGS[name].replace(H=61, W=93)
    im = workload.make_image(cfg, 3)
    r = oracle.rd_forward_image(cfg, im)
    m = ccrd.cc_mac_per_pixel(ccrd.desc_from_config(cfg))
    assert (m.arm_macs, m.up_macs, m.syn_macs) == (r["macs"]["arm"], r["macs"]["up"], r["macs"]["syn"])


def _run(cfg, im):
    import torch
    import paper_2403_11651_b200 as P
    b = P.DeviceBatch(cfg, [im])
    res = b.forward()
    torch.cuda.synchronize()
    return res.cpu().numpy()[0], b.xhat[0].cpu().numpy()


def _check(cfg, im):
    got, xh = _run(cfg, im)
    ref = oracle.rd_forward_image(cfg, im, want_xhat=True)
    assert np.abs(xh - ref["x_hat"]).max() <= 1e-5
    for k, key in enumerate(["rate_bits", "sse", "mse", "cost"]):
        assert abs(got[k] - ref[key]) <= 1e-4 * abs(ref[key]), key


@pytest.mark.gpu
@pytest.mark.parametrize("name", TABLE1)
@pytest.mark.parametrize("filt", ["random", "normalised2d"])
def test_table1_rd_forward_vs_oracle(name, filt):
    cfg = workload.CONFIGS[name]
    _check(cfg, workload.make_image(cfg, 21, filter_kind=filt))


@pytest.mark.gpu
@pytest.mark.parametrize("name,H,W,L", [("t2300", 37, 53, 7), ("t300", 70, 45, 7), ("t545", 33, 97, 7),
                                        ("t1079", 9, 5, 7), ("t2300", 5, 300, 7), ("t300", 130, 67, 7)])
def test_table1_ragged_shapes(name, H, W, L):
    cfg = workload.CONFIGS[name]
    cfg = cfg.replace(H=H, W=W, L=L, syn_widths=(L,) + cfg.syn_widths[1:])
    from paper_2403_11651_b200 import ccrd
    if ccrd.cc_validate(ccrd.desc_from_config(cfg)) == ccrd.CC_ENOTSUP:
        pytest.skip("synthesis shape not compiled")
    _check(cfg, workload.make_image(cfg, 22, filter_kind="normalised2d"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["t2300", "t300"])
def test_table1_upsample_stage_per_level(name):
    """Dense tensor of the 2-D upsampling (cc_upsample) per level, relative to
    the level's max |value| (pixel parity cannot see coarse levels)."""
    import torch
    import paper_2403_11651_b200 as P
    cfg = workload.CONFIGS[name].replace(H=96, W=136)
    im = workload.make_image(cfg, 23, filter_kind="normalised2d")
    d = P.desc_from_config(cfg)
    lat = torch.from_numpy(im.latents).cuda()
    dense = torch.zeros((cfg.L, cfg.H, cfg.W), device="cuda")
    ws_b = P.cc_workspace_bytes(d, 1)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    P.cc_upsample(d, lat.data_ptr(), im.up_w, dense.data_ptr(), ws.data_ptr(), ws_b,
                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref, _ = oracle.upsample(oracle.model(cfg), im.latents, im.up_w)
    got = dense.cpu().numpy()
    for l in range(cfg.L):
        scale = max(1e-30, np.abs(ref[l]).max())
        assert np.abs(got[l] - ref[l]).max() <= 1e-5 * scale, l


@pytest.mark.gpu
def test_strips_refuse_2d():
    import paper_2403_11651_b200 as P
    d = P.desc_from_config(workload.CONFIGS["t300"])
    with pytest.raises(P.CcError) as e:
        P.cc_strip_window(d, 0, 64)
        st = P.cc_strip_window(d, 0, 64)
        P.cc_rd_forward_strip(d, st, P.CcImageIO(), 0, 0, 0)
    assert e.value.code in (P.ccrd.CC_ENOTSUP, P.ccrd.CC_EINVAL)
