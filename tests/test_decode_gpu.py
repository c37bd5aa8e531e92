"""Decoder output stage (NEXT-3; cc_decode): latents -> upsampling -> synthesis
-> clamp to [0,1] -> 8-bit RGB, vs the oracle (decode_u8 of the fp64 x_hat).

Both sides round 255 clamp(x_hat) to nearest, ties to even (reading N3); the
CUDA x_hat is fp32 (within 1e-5 of the oracle's), so a pixel may differ by one
code only where 255 x_hat lies within 255 x 1e-5 of a rounding boundary:
everywhere else the bytes are identical (checked), and nowhere by more than 1."""
import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def gpu_decode(cfg, im):
    import paper_2403_11651_b200 as P
    d = P.desc_from_config(cfg)
    lat = torch.from_numpy(im.latents).cuda()
    out = torch.zeros((cfg.H, cfg.W, 3), dtype=torch.uint8, device="cuda")
    ws_b = P.cc_workspace_bytes(d, 1)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    P.cc_decode(d, lat.data_ptr(), im.up_w, im.syn_w, out.data_ptr(), ws.data_ptr(), ws_b,
                torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("name,kw,filt", [
    ("tiny", {}, "lanczos2"), ("ref", {}, "lanczos2"), ("ref", dict(H=37, W=53), "random"),
    ("t2300", {}, "normalised2d"), ("t300", dict(H=70, W=45), "normalised2d"), ("low", dict(H=5, W=300), "lanczos2"),
])
def test_decode_vs_oracle(name, kw, filt):
    cfg = workload.CONFIGS[name].replace(**kw)
    im = workload.make_image(cfg, 12, filter_kind=filt)
    got = gpu_decode(cfg, im)
    want, xh = oracle.decode_image(cfg, im)
    diff = np.abs(got.astype(int) - want.astype(int))
    assert diff.max() <= 1
    v = 255.0 * np.clip(xh, 0.0, 1.0).transpose(1, 2, 0)        # [H][W][3]
    near_tie = np.abs(v - np.floor(v) - 0.5) < 255 * 2e-5
    assert np.all(diff[~near_tie] == 0)
    assert 0 < np.count_nonzero(want) and np.count_nonzero(want != 255) > 0   # not a degenerate image
