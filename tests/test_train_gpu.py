"""GPU parity of the training iteration (cc_train_step, NEXT-2) against the
fp64 training oracle (oracle/cctrain.c, pinned in test_train_oracle.py).

Tolerances (fp32 GPU vs fp64 oracle, training):
  * cost components of the forward: 1e-5 relative;
  * gradient, per parameter group (latents of each level, each ARM layer's
    weights / biases, taps, each synthesis layer): max |g - g_oracle| <=
    2e-3 x max |g_oracle| of the group (fp32 chains through up to 8 layers and
    sums over 10^5-10^6 terms; measured far below);
  * Adam: the GPU update from its own gradient == the oracle's Adam applied to
    that gradient, to fp32 rounding.
"""
import numpy as np
import pytest

import oracle
import workload
from test_train_oracle import groups

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def make_state(cfg, seed, filt="random"):
    im = workload.make_image(cfg, seed, filter_kind=filt)
    rng = np.random.default_rng(seed + 1000)
    y = workload.gen_continuous_latents(rng, im.latents)
    u = workload.gen_noise(rng, im.latents.size)
    return im, y, u


def gpu_grad(cfg, im, y, u):
    import paper_2403_11651_b200 as P
    tr = P.DeviceTrainer(cfg, y, im.arm_w, im.up_w, im.syn_w, im.image)
    res = tr.step(noise=u, update=False)
    torch.cuda.synchronize()
    return tr, res.cpu().numpy(), tr.grad.cpu().numpy().astype(np.float64)


def check_grad(cfg, g, g_ref):
    for name, a, b in groups(cfg):
        scale = np.abs(g_ref[a:b]).max()
        if scale == 0.0:
            assert np.abs(g[a:b]).max() == 0.0, name
            continue
        err = np.abs(g[a:b] - g_ref[a:b]).max()
        assert err <= 2e-3 * scale, (name, err, scale)


CASES = [
    ("ref", dict(H=40, W=56), "lanczos2"),
    ("ref", dict(H=37, W=61), "random"),
    ("low", dict(H=33, W=47), "lanczos2"),
    ("t1079", dict(H=29, W=35, up_2d=False, up_taps=8), "lanczos2"),   # [16,16,16,2] ARM, [7,16,3]+2
]


@pytest.mark.parametrize("name,kw,filt", CASES)
def test_train_gradient_vs_oracle(name, kw, filt):
    cfg = workload.CONFIGS[name].replace(**kw).replace(lam=0.02)
    im, y, u = make_state(cfg, 5, filt)
    _, res, g = gpu_grad(cfg, im, y, u)
    out, g_ref = oracle.train_grad(oracle.model(cfg), oracle.pack_params(y, im.arm_w, im.up_w, im.syn_w), u,
                                   im.image)
    np.testing.assert_allclose(res, out, rtol=1e-5)
    check_grad(cfg, g, g_ref)


def test_train_adam_update_matches_oracle_adam():
    import paper_2403_11651_b200 as P
    cfg = workload.CONFIGS["ref"].replace(H=40, W=56)
    im, y, u = make_state(cfg, 6, "lanczos2")
    tr = P.DeviceTrainer(cfg, y, im.arm_w, im.up_w, im.syn_w, im.image)
    p0 = tr.params.cpu().numpy().copy()
    m1, m2 = np.zeros(p0.size), np.zeros(p0.size)
    for t in range(1, 4):
        tr.step(noise=u, lr=1e-2)
        torch.cuda.synchronize()
        g = tr.grad.cpu().numpy().astype(np.float64)
        oracle.adam_step(p0, g, m1, m2, 1e-2, 0.9, 0.999, 1e-8, t)
        np.testing.assert_allclose(tr.params.cpu().numpy(), p0, rtol=1e-5, atol=1e-6)
        p0 = tr.params.cpu().numpy().copy()   # continue from the GPU's fp32 state


def test_train_descent():
    import paper_2403_11651_b200 as P
    cfg = workload.CONFIGS["ref"].replace(H=64, W=96)
    im, y, u = make_state(cfg, 7, "lanczos2")
    tr = P.DeviceTrainer(cfg, y, im.arm_w, im.up_w, im.syn_w, im.image)
    rng = np.random.default_rng(3)
    costs = []
    for _ in range(60):
        r = tr.step(noise=workload.gen_noise(rng, y.size), lr=5e-3)
        costs.append(float(r[3].item()))
    assert np.mean(costs[-10:]) < 0.8 * np.mean(costs[:5]), costs[:3] + costs[-3:]


@pytest.mark.timeout(900)
def test_train_gradient_full_size_ref_vs_oracle():
    """BASELINE.json configs[2] (512x768, the size the paper's encoding times
    are for) -- the configuration bench.py --train times."""
    cfg = workload.CONFIGS["ref"]
    im, y, u = make_state(cfg, 8, "random")
    _, res, g = gpu_grad(cfg, im, y, u)
    out, g_ref = oracle.train_grad(oracle.model(cfg), oracle.pack_params(y, im.arm_w, im.up_w, im.syn_w), u,
                                   im.image)
    np.testing.assert_allclose(res, out, rtol=1e-5)
    check_grad(cfg, g, g_ref)


def test_train_refuses_2d():
    import paper_2403_11651_b200 as P
    assert P.cc_train_workspace_bytes(P.desc_from_config(workload.CONFIGS["t2300"])) == 0


def test_train_concurrent_streams_bit_identical():
    """Several trainers stepping concurrently on their own streams (the
    multi-image training mode bench.py --train --images N times) give exactly
    the parameters each reaches alone: the per-stream constant weight banks
    (train.cu acquire_bank) keep one image's weights from leaking into
    another's kernels -- including with more streams than banks."""
    import paper_2403_11651_b200 as P
    cfg = workload.CONFIGS["ref"].replace(H=96, W=128)
    K, steps = 5, 4
    states = [make_state(cfg, 40 + k) for k in range(K)]

    def trainers():
        out = []
        for im, y, u in states:
            tr = P.DeviceTrainer(cfg, y, im.arm_w, im.up_w, im.syn_w, im.image)
            tr.noise.copy_(torch.as_tensor(u))
            out.append(tr)
        torch.cuda.synchronize()
        return out

    alone = trainers()
    for tr in alone:
        for _ in range(steps):
            tr.step(lr=1e-3)
    torch.cuda.synchronize()
    conc = trainers()
    streams = [torch.cuda.Stream() for _ in range(K)]
    for _ in range(steps):
        for tr, st in zip(conc, streams):
            tr.step(lr=1e-3, stream_ptr=st.cuda_stream)
    torch.cuda.synchronize()
    for a, c in zip(alone, conc):
        assert torch.equal(a.params, c.params)
        assert torch.equal(a.result, c.result)


def test_train_concurrent_host_threads_bit_identical():
    """Trainers stepping from SEVERAL HOST THREADS at once, each on its own
    stream, more threads than constant banks (6 > 4): a bank is held from the
    start of a call to the end of its enqueue (train.cu acquire_bank /
    release_bank), so no thread's weight copy can land in a bank another
    thread's kernels are still reading.  Every image ends bit-identical to
    its own serial run."""
    import threading
    import paper_2403_11651_b200 as P
    cfg = workload.CONFIGS["ref"].replace(H=64, W=96)
    K, steps = 6, 6
    states = [make_state(cfg, 70 + k) for k in range(K)]

    def trainers():
        out = []
        for im, y, u in states:
            tr = P.DeviceTrainer(cfg, y, im.arm_w, im.up_w, im.syn_w, im.image)
            tr.noise.copy_(torch.as_tensor(u))
            out.append(tr)
        torch.cuda.synchronize()
        return out

    alone = trainers()
    for tr in alone:
        for _ in range(steps):
            tr.step(lr=1e-3)
    torch.cuda.synchronize()
    conc = trainers()
    streams = [torch.cuda.Stream() for _ in range(K)]
    errors = []
    start = threading.Barrier(K)

    def run(tr, st):
        try:
            start.wait()
            for _ in range(steps):
                tr.step(lr=1e-3, stream_ptr=st.cuda_stream)
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=run, args=(tr, st)) for tr, st in zip(conc, streams)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    torch.cuda.synchronize()
    for a, c in zip(alone, conc):
        assert torch.equal(a.params, c.params)
        assert torch.equal(a.result, c.result)
