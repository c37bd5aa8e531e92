"""Single-image strip partition (BASELINE.json configs[4]) --
host logic on CPU.

* strip_rows / owned latent rows partition the image and every grid exactly;
* the window cc_strip_window computes (receptive field of the forward) is
  SUFFICIENT, pinned against the fp64 oracle (not against the CUDA path):
  scrambling every latent outside a strip's window leaves the oracle's x_hat
  on the strip's rows and its per-latent bits on the strip's owned latents
  bit-identical; and it is TIGHT at level 0 (scrambling the window's first row
  changes the strip's output), so the rule is not vacuous;
* the halo exchange (grouped send / recv, gloo world size 2 and 3) fills every
  rank's window buffer exactly with the rows its neighbours own.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle
import workload
from paper_2403_11651_b200 import ccrd
from paper_2403_11651_b200 import dist as ccdist


def _full_off(cfg):
    dims = cfg.level_dims()
    return [sum(h * w for h, w in dims[:l]) for l in range(cfg.L)]


@pytest.mark.parametrize("H,world", [(4320, 8), (4320, 2), (1365, 4), (37, 3), (64, 5), (9, 4), (2, 1)])
def test_strip_rows_partition(H, world):
    strips = ccdist.strip_rows(H, world)
    assert strips[0][0] == 0 and strips[-1][1] == H and len(strips) == world
    for (a, b), (c, _) in zip(strips, strips[1:]):
        assert b == c
    assert all(r0 % 2 == 0 and r1 > r0 for r0, r1 in strips)


@pytest.mark.parametrize("name,world", [("8k", 8), ("8k", 3), ("ref", 5), ("tiny", 4)])
def test_owned_latent_rows_partition_every_grid(name, world):
    cfg = workload.CONFIGS[name]
    d = ccrd.desc_from_config(cfg)
    strips, lays = ccdist.strip_layouts(d, world)
    for l, (h, w) in enumerate(cfg.level_dims()):
        rows = []
        for st in strips:
            rows += list(range(st.own_lo[l], st.own_hi[l]))
            assert 0 <= st.lo[l] <= st.own_lo[l] or st.own_hi[l] == st.own_lo[l]
            assert st.hi[l] <= h
        assert rows == list(range(h)), l
    assert sum(lay.n for lay in lays) >= cfg.n_latents


def test_strip_window_rejects_bad_rows():
    d = ccrd.desc_from_config(workload.CONFIGS["tiny"])
    for r0, r1 in [(1, 10), (10, 10), (0, 65), (-2, 4)]:
        with pytest.raises(ccrd.CcError):
            ccrd.cc_strip_window(d, r0, r1)


def _oracle_outputs(cfg, im, latents):
    m = oracle.model(cfg)
    r = oracle.rd_forward(m, latents, im.arm_w, im.up_w, im.syn_w, im.image, want_xhat=True)
    _, _, _, bits, _ = oracle.rate(m, latents, im.arm_w, per_latent=True)
    return r["x_hat"], bits


# compiled shapes (the windows are also run on the GPU in test_strips_gpu.py)
STRIP_CASES = [
    (70, 45, 7, 40, 2, 8, 16, 3),
    (61, 33, 7, 16, 2, 4, 8, 2),
    (96, 40, 4, 8, 3, 8, 8, 4),
    (50, 22, 5, 8, 1, 8, 8, 5),
]


def strip_cfg(H, W, L, ch, res, taps, nctx):
    arm = (16, 24, 24, 2) if nctx == 16 else (8, 8, 8, 2)
    return workload.CONFIGS["ref"].replace(H=H, W=W, L=L, n_ctx=nctx, arm_widths=arm, syn_widths=(L, ch, 3),
                                           syn_n_res=res, up_taps=taps)


@pytest.mark.parametrize("H,W,L,ch,res,taps,nctx,world", STRIP_CASES)
def test_window_sufficient_and_tight_vs_oracle(H, W, L, ch, res, taps, nctx, world):
    cfg = strip_cfg(H, W, L, ch, res, taps, nctx)
    im = workload.make_image(cfg, 31, filter_kind="lanczos2" if taps == 8 else "random")
    d = ccrd.desc_from_config(cfg)
    xh0, bits0 = _oracle_outputs(cfg, im, im.latents)
    off = _full_off(cfg)
    dims = cfg.level_dims()
    rng = np.random.default_rng(5)
    strips, _ = ccdist.strip_layouts(d, world)
    for st in strips:
        lat = im.latents.copy()
        for l, (h, w) in enumerate(dims):   # scramble everything outside the window
            g = lat[off[l]: off[l] + h * w].reshape(h, w)
            for rows in (slice(0, st.lo[l]), slice(st.hi[l], h)):
                g[rows] = rng.integers(-16, 17, g[rows].shape)
        xh, bits = _oracle_outputs(cfg, im, lat)
        np.testing.assert_array_equal(xh[:, st.r0:st.r1], xh0[:, st.r0:st.r1])
        for l, (h, w) in enumerate(dims):
            a, b = off[l] + st.own_lo[l] * w, off[l] + st.own_hi[l] * w
            np.testing.assert_array_equal(bits[a:b], bits0[a:b])
        if st.lo[0] > 0:   # tightness at level 0: the window's first row matters
            lat = im.latents.copy()
            lat[off[0] + st.lo[0] * W: off[0] + (st.lo[0] + 1) * W] += 5
            xh, _ = _oracle_outputs(cfg, im, lat)
            assert np.abs(xh[:, st.r0:st.r1] - xh0[:, st.r0:st.r1]).max() > 0


def test_pack_window_matches_rows():
    cfg = workload.CONFIGS["tiny"].replace(H=50, W=30)
    d = ccrd.desc_from_config(cfg)
    im = workload.make_image(cfg, 2)
    off = _full_off(cfg)
    _, lays = ccdist.strip_layouts(d, 3)
    for lay in lays:
        buf = ccdist.pack_window(im.latents, off, lay)
        for l in range(cfg.L):
            g = im.level(cfg, l)
            s, e = lay.rows(l, lay.lo[l], lay.hi[l])
            np.testing.assert_array_equal(buf[s:e].reshape(-1, lay.w[l]), g[lay.lo[l]:lay.hi[l]])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _halo_worker(rank, world, port, cfg_kw, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = workload.CONFIGS["ref"].replace(**cfg_kw)
    d = ccrd.desc_from_config(cfg)
    im = workload.make_image(cfg, 77)
    _, lays = ccdist.strip_layouts(d, world)
    full = torch.from_numpy(im.latents)
    buf = ccdist.pack_window(full, _full_off(cfg), lays[rank], owned_only=True, fill=-999)
    got = ccdist.exchange_halos(buf, lays, rank)
    np.save(os.path.join(out_dir, f"buf{rank}.npy"), buf.numpy())
    np.save(os.path.join(out_dir, f"n{rank}.npy"), np.array([got]))
    tdist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,cfg_kw", [(2, dict(H=96, W=80)), (3, dict(H=140, W=64))])
def test_gloo_halo_exchange(tmp_path, world, cfg_kw):
    mp.spawn(_halo_worker, args=(world, _free_port(), cfg_kw, str(tmp_path)), nprocs=world, join=True)
    cfg = workload.CONFIGS["ref"].replace(**cfg_kw)
    d = ccrd.desc_from_config(cfg)
    im = workload.make_image(cfg, 77)
    _, lays = ccdist.strip_layouts(d, world)
    for rank in range(world):
        want = ccdist.pack_window(im.latents, _full_off(cfg), lays[rank])
        got = np.load(tmp_path / f"buf{rank}.npy")
        np.testing.assert_array_equal(got, want)
        halo = sum((lays[rank].hi[l] - lays[rank].lo[l] - (lays[rank].own_hi[l] - lays[rank].own_lo[l]))
                   * lays[rank].w[l] for l in range(cfg.L))
        assert np.load(tmp_path / f"n{rank}.npy")[0] == 2 * halo
