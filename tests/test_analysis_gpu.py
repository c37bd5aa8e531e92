"""GPU parity of the N-O analysis transform (cc_analysis_forward, NEXT-4)
against the fp64 oracle (oracle/ccanalysis.c, pinned in
test_analysis_oracle.py), per latent grid, relative to the grid's max |value|:
  * fp32 GEMMs: 1e-4 (fp32 sums of <= 4C = 256 terms through 3L = 21
    residual blocks; measured ~1e-6);
  * TF32 tensor-core GEMMs: 3e-2 (TF32 keeps 10 mantissa bits: ~2^-11
    relative per product, accumulating over the 21 blocks; measured below).
"""
import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def gpu_analysis(acfg, image, w, tf32):
    import paper_2403_11651_b200 as P
    ad = P.analysis_desc(acfg, tf32)
    n_lat = sum(-(-acfg.H // (1 << l)) * -(-acfg.W // (1 << l)) for l in range(acfg.L))
    img = torch.from_numpy(image).cuda()
    wt = torch.from_numpy(w).cuda()
    lat = torch.zeros(n_lat, device="cuda")
    ws_b = P.cc_analysis_workspace_bytes(ad)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    P.cc_analysis_forward(ad, img.data_ptr(), wt.data_ptr(), lat.data_ptr(), ws.data_ptr(), ws_b,
                          torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return lat.cpu().numpy().astype(np.float64)


def check(acfg, got, ref, tol):
    off = 0
    worst = 0.0
    for l in range(acfg.L):
        n = -(-acfg.H // (1 << l)) * -(-acfg.W // (1 << l))
        scale = np.abs(ref[off:off + n]).max()
        err = np.abs(got[off:off + n] - ref[off:off + n]).max() / scale
        worst = max(worst, err)
        assert err <= tol, (l, err)
        off += n
    return worst


@pytest.mark.parametrize("name,kw", [("no_tiny", {}), ("no_kodak", dict(H=96, W=136)), ("no_kodak", dict(H=37, W=70)),
                                     ("no_tiny", dict(H=5, W=3, L=3))])
@pytest.mark.parametrize("tf32", [False, True])
def test_analysis_vs_oracle(name, kw, tf32):
    acfg = workload.ANALYSIS[name].replace(**kw)
    image, w = workload.make_analysis_input(acfg, 9)
    ref, _ = oracle.analysis_forward(acfg, image, w)
    got = gpu_analysis(acfg, image, w, tf32)
    check(acfg, got, ref, 3e-2 if tf32 else 1e-4)


@pytest.mark.timeout(900)
def test_analysis_full_kodak_size_vs_oracle():
    acfg = workload.ANALYSIS["no_kodak"]
    image, w = workload.make_analysis_input(acfg, 10)
    ref, _ = oracle.analysis_forward(acfg, image, w)
    check(acfg, gpu_analysis(acfg, image, w, False), ref, 1e-4)
    check(acfg, gpu_analysis(acfg, image, w, True), ref, 3e-2)
