"""GPU parity of the N-O analysis transform (cc_analysis_forward, NEXT-4)
against the fp64 oracle (oracle/ccanalysis.c, pinned in
test_analysis_oracle.py), per latent grid, relative to the grid's max |value|:
  * fp32 GEMMs: 1e-4 (fp32 sums of <= 4C = 256 terms through 3L = 21
    residual blocks; measured ~1e-6);
  * TF32 (mode 1: fused tcgen05 block kernel for C = 64; mode 2: cuBLASLt
    TF32 GEMMs) and FP16 operands (mode 3, same 10-bit mantissa): 3e-2 (TF32 keeps 10 mantissa bits: ~2^-11 relative per
    product, accumulating over the 21 blocks; measured below).
"""
import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def gpu_analysis(acfg, image, w, tf32):
    """image [3][H][W] -> latents [n_lat], or a batch [N][3][H][W] -> [N][n_lat] (one call)."""
    import paper_2403_11651_b200 as P
    n = image.shape[0] if image.ndim == 4 else 1
    ad = P.analysis_desc(acfg, tf32, n)
    n_lat = sum(-(-acfg.H // (1 << l)) * -(-acfg.W // (1 << l)) for l in range(acfg.L))
    img = torch.from_numpy(np.ascontiguousarray(image)).cuda()
    wt = torch.from_numpy(w).cuda()
    lat = torch.zeros((n, n_lat) if image.ndim == 4 else n_lat, device="cuda")
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
                                     ("no_tiny", dict(H=5, W=3, L=3)),
                                     # fused kernel: ragged 4 x 32 tiles, 1-pixel grids, a level whose only
                                     # block is the downsampling one (it also carries the merge)
                                     ("no_kodak", dict(H=9, W=33, L=5, blocks=1)),
                                     ("no_kodak", dict(H=70, W=37, L=6, blocks=2))])
@pytest.mark.parametrize("tf32", [0, 1, 2, 3])
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
    errs = [check(acfg, gpu_analysis(acfg, image, w, 0), ref, 1e-4)]
    for mode in (1, 2, 3):
        errs.append(check(acfg, gpu_analysis(acfg, image, w, mode), ref, 3e-2))
    print("analysis full-size max per-grid relative error (fp32, fused TF32, cuBLASLt TF32, fused FP16):", errs)


@pytest.mark.parametrize("tf32", [0, 1, 2, 3])
def test_analysis_batch_equals_single_image_calls(tf32):
    """N images in one call (the fused kernels tile all of them in one launch):
    each image's latents equal its single-image call bit for bit, and match
    the oracle.  Ragged 4 x 32 tiles (H = 45, W = 70)."""
    acfg = workload.ANALYSIS["no_kodak"].replace(H=45, W=70, L=5)
    ins = [workload.make_analysis_input(acfg, 30 + k) for k in range(3)]
    w = ins[0][1]
    batch = np.stack([i for i, _ in ins])
    got = gpu_analysis(acfg, batch, w, tf32)
    for k in range(3):
        single = gpu_analysis(acfg, batch[k], w, tf32)
        np.testing.assert_array_equal(got[k], single.astype(np.float32).astype(np.float64))
        ref, _ = oracle.analysis_forward(acfg, batch[k], w)
        check(acfg, got[k], ref, 3e-2 if tf32 else 1e-4)
