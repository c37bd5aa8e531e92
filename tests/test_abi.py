"""CPU-only checks of the C ABI: the library loads, exports every function
include/ccrd.h declares, validates descriptors with the documented error codes,
and its MAC closed form matches the oracle's instrumented counters.  No compute
call runs here (there is no GPU); compute entries must fail loudly (CC_ECUDA)
rather than fall back to the CPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
import paper_2403_11651_b200 as P
import workload
from paper_2403_11651_b200 import ccrd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ccrd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cc_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    L = P.load()
    names = header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n
    assert sorted(ccrd.EXPORTS) == names


def test_struct_layout_matches_header():
    # offsets the header implies (natural alignment, x86-64)
    assert C.sizeof(ccrd.CcRdResult) == 32
    assert C.sizeof(ccrd.CcImageIO) == 48
    assert ccrd.CcModelDesc.lam.offset % 8 == 0
    assert C.sizeof(ccrd.CcMacBreakdown) == 64


@pytest.mark.parametrize("name", list(workload.CONFIGS))
def test_configs_validate(name):
    d = P.desc_from_config(workload.CONFIGS[name])
    assert P.cc_validate(d) == 0
    assert P.cc_workspace_bytes(d, 2) > 0


def test_validation_error_codes():
    cfg = workload.CONFIGS["ref"]
    bad = P.desc_from_config(cfg)
    bad.ctx_dy[3], bad.ctx_dx[3] = 0, 1          # non-causal (dy = 0, dx > 0)
    assert P.cc_validate(bad) == ccrd.CC_EINVAL
    bad = P.desc_from_config(cfg)
    bad.ctx_dy[3], bad.ctx_dx[3] = bad.ctx_dy[4], bad.ctx_dx[4]   # duplicate
    assert P.cc_validate(bad) == ccrd.CC_EINVAL
    bad = P.desc_from_config(cfg)
    bad.arm_residual_mask = 1                     # 16 -> 24 cannot be residual
    assert P.cc_validate(bad) == ccrd.CC_EINVAL
    bad = P.desc_from_config(cfg)
    bad.arm_residual_mask = 1 << 2                # last layer residual
    assert P.cc_validate(bad) == ccrd.CC_EINVAL
    bad = P.desc_from_config(cfg)
    bad.up_taps = 6
    assert P.cc_validate(bad) == ccrd.CC_ENOTSUP
    bad = P.desc_from_config(cfg)
    bad.syn_widths[1] = 12                        # valid per the paper, not compiled
    assert P.cc_validate(bad) == ccrd.CC_ENOTSUP
    bad = P.desc_from_config(cfg)
    bad.H = 0
    assert P.cc_validate(bad) == ccrd.CC_EINVAL
    bad = P.desc_from_config(cfg)
    bad.L = 13
    assert P.cc_validate(bad) == ccrd.CC_EINVAL
    bad = P.desc_from_config(cfg)
    bad.syn_widths[0] = 6                         # != L
    assert P.cc_validate(bad) == ccrd.CC_EINVAL
    bad = P.desc_from_config(cfg)
    bad.p_floor = 0.0
    assert P.cc_validate(bad) == ccrd.CC_EINVAL
    assert P.cc_workspace_bytes(bad, 1) == 0
    with pytest.raises(ccrd.CcError) as e:
        P.cc_mac_per_pixel(bad)
    assert "p_floor" in str(e.value)


def test_workspace_and_device_errors_without_gpu():
    cfg = workload.CONFIGS["tiny"]
    d = P.desc_from_config(cfg)
    im = workload.make_image(cfg, 0)
    io = [P.CcImageIO(1, im.arm_w.ctypes.data, im.up_w.ctypes.data, im.syn_w.ctypes.data, 0, 0)]
    with pytest.raises(ccrd.CcError) as e:
        P.cc_rd_forward(d, io, 8, 8, 1)               # workspace too small
    assert e.value.code == ccrd.CC_EWORKSPACE
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        ws = P.cc_workspace_bytes(d, 1)
        with pytest.raises(ccrd.CcError) as e:
            P.cc_rd_forward(d, io, 8, 8, ws)          # no device: loud failure, no CPU fallback
        assert e.value.code == ccrd.CC_ECUDA


@pytest.mark.parametrize("name,H,W", [("tiny", 64, 64), ("low", 67, 93), ("ref", 40, 57),
                                      ("batched2k", 1365, 2048)])
def test_mac_closed_form_matches_oracle_counters(name, H, W):
    cfg = workload.CONFIGS[name].replace(H=H, W=W)
    m = P.cc_mac_per_pixel(P.desc_from_config(cfg))
    if H * W > 100000:
        # counters of the rate stage and upsampling only (cheap), synthesis by width arithmetic
        om = oracle.model(cfg)
        im_lat = np.zeros(cfg.n_latents, np.int16)
        _, macs = oracle.rate(om, im_lat, np.zeros(cfg.n_arm_w, np.float32))
        _, umacs = oracle.upsample(om, im_lat, np.zeros(cfg.up_taps, np.float32))
        assert (m.arm_macs, m.up_macs) == (macs.arm, umacs.up)
        return
    im = workload.make_image(cfg, 1)
    r = oracle.rd_forward(oracle.model(cfg), im.latents, im.arm_w, im.up_w, im.syn_w, im.image)
    assert (m.arm_macs, m.up_macs, m.syn_macs) == (r["macs"]["arm"], r["macs"]["up"], r["macs"]["syn"])
    assert m.n_latents == cfg.n_latents


def test_reference_config_mac_per_pixel():
    # Ref 512x768 -> 1951.3 MAC/px; batched 2K -> 1951.7
    assert P.cc_mac_per_pixel(P.desc_from_config(workload.CONFIGS["ref"])).total == pytest.approx(1951.25, abs=0.01)
    assert P.cc_mac_per_pixel(P.desc_from_config(workload.CONFIGS["batched2k"])).total == pytest.approx(1951.68,
                                                                                                      abs=0.01)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_up_2d_validation_and_table1_configs():
    for name in ("t300", "t545", "t1079", "t2300"):
        assert P.cc_validate(P.desc_from_config(workload.CONFIGS[name])) == 0, name
    d = P.desc_from_config(workload.CONFIGS["t300"])
    d.up_2d = 2
    assert P.cc_validate(d) == ccrd.CC_EINVAL


def test_training_entry_errors_without_gpu():
    cfg = workload.CONFIGS["ref"].replace(H=24, W=40)
    d = P.desc_from_config(cfg)
    n = P.cc_train_param_count(d)
    assert n == cfg.n_latents + cfg.n_arm_w + cfg.n_up_w + cfg.n_syn_w
    ws = P.cc_train_workspace_bytes(d)
    assert ws > 0
    with pytest.raises(ccrd.CcError) as e:           # workspace too small
        P.cc_train_step(d, 8, 8, 8, 8, 8, P.CcAdam(1e-3, 0.9, 0.999, 1e-8, 1), 8, 8, 8, 16)
    assert e.value.code == ccrd.CC_EWORKSPACE
    with pytest.raises(ccrd.CcError) as e:           # Adam step 0
        P.cc_train_step(d, 8, 8, 8, 8, 8, P.CcAdam(1e-3, 0.9, 0.999, 1e-8, 0), 8, 8, 8, ws)
    assert e.value.code == ccrd.CC_EINVAL
    big = P.desc_from_config(cfg.replace(H=32768, W=65536))  # H W = 2^31: 32-bit plane offsets
    assert P.cc_validate(big) == 0 and P.cc_train_workspace_bytes(big) == 0
    with pytest.raises(ccrd.CcError) as e:
        P.cc_train_step(big, 8, 8, 8, 8, 8, None, 8, 8, 8, 1 << 30)
    assert e.value.code == ccrd.CC_ENOTSUP
    d2 = P.desc_from_config(workload.CONFIGS["t2300"])     # 2-D TConv: not compiled for training
    assert P.cc_train_workspace_bytes(d2) == 0
    with pytest.raises(ccrd.CcError) as e:
        P.cc_train_step(d2, 8, 8, 8, 8, 8, None, 8, 8, 8, 1 << 30)
    assert e.value.code == ccrd.CC_ENOTSUP
    if not _has_gpu():
        with pytest.raises(ccrd.CcError) as e:       # no device: loud failure
            P.cc_train_step(d, 8, 8, 8, 8, 8, None, 8, 8, 8, ws)
        assert e.value.code == ccrd.CC_ECUDA


def test_strip_entry_errors_without_gpu():
    cfg = workload.CONFIGS["ref"]
    d = P.desc_from_config(cfg)
    st = P.cc_strip_window(d, 100, 300)
    ws = P.cc_workspace_bytes_strip(d, st)
    assert ws > 0 and P.cc_strip_latent_count(d, st) > 0
    im = workload.make_image(cfg, 0)
    io = P.CcImageIO(1, im.arm_w.ctypes.data, im.up_w.ctypes.data, im.syn_w.ctypes.data, 0, 0)
    with pytest.raises(ccrd.CcError) as e:
        P.cc_rd_forward_strip(d, st, io, 8, 8, 16)
    assert e.value.code == ccrd.CC_EWORKSPACE
    if not _has_gpu():
        with pytest.raises(ccrd.CcError) as e:
            P.cc_rd_forward_strip(d, st, io, 8, 8, ws)
        assert e.value.code == ccrd.CC_ECUDA


def test_analysis_entry_errors_without_gpu():
    acfg = workload.ANALYSIS["no_kodak"]
    ad = P.analysis_desc(acfg, 1, 4)
    assert P.cc_analysis_param_count(ad) == acfg.n_params           # 787,719 (A1-A7)
    ws4 = P.cc_analysis_workspace_bytes(ad)
    ws1 = P.cc_analysis_workspace_bytes(P.analysis_desc(acfg, 1, 1))
    assert ws4 >= 4 * 2 * acfg.H * acfg.W * acfg.C * 4 and ws1 < ws4   # x / y for the whole batch
    # the unfused modes also hold one image's 4C expansion and the cuBLASLt workspace
    assert P.cc_analysis_workspace_bytes(P.analysis_desc(acfg, 2, 1)) > ws1
    for bad in (dict(N=0), dict(tf32=4), dict(C=6), dict(L=0), dict(blocks=0), dict(H=0)):
        d = P.analysis_desc(acfg, 1, 1)
        for k, v in bad.items():
            setattr(d, k, v)
        assert P.cc_analysis_workspace_bytes(d) == 0, bad
        with pytest.raises(ccrd.CcError):
            P.cc_analysis_param_count(d)
    with pytest.raises(ccrd.CcError) as e:                             # workspace too small
        P.cc_analysis_forward(ad, 8, 8, 8, 8, 16, 0)
    assert e.value.code == ccrd.CC_EWORKSPACE
    if not _has_gpu():
        with pytest.raises(ccrd.CcError) as e:                         # no device: loud failure
            P.cc_analysis_forward(ad, 8, 8, 8, 8, ws4, 0)
        assert e.value.code == ccrd.CC_ECUDA


def test_image_u8_validation():
    d = P.desc_from_config(workload.CONFIGS["ref"])
    assert d.image_u8 == 0 and P.cc_validate(d) == 0
    d.image_u8 = 1
    assert P.cc_validate(d) == 0
    # the host path stages fp32-sized image slots either way
    assert P.cc_workspace_bytes_host(d, 2) == P.cc_workspace_bytes_host(P.desc_from_config(workload.CONFIGS["ref"]), 2)
    d.image_u8 = 2
    assert P.cc_validate(d) == ccrd.CC_EINVAL
    d.image_u8 = 0
    d.latents_i8 = 1                       # valid (host path), slot grows by the int8 upload area
    assert P.cc_validate(d) == 0
    assert P.cc_workspace_bytes_host(d, 2) > P.cc_workspace_bytes_host(P.desc_from_config(workload.CONFIGS["ref"]), 2)
    d.latents_i8 = 3
    assert P.cc_validate(d) == ccrd.CC_EINVAL


def test_u8_image_helpers():
    x = np.array([[0.0, 0.5, 1.0, 0.25, 0.998]], np.float32)
    v = workload.to_u8(x)
    np.testing.assert_array_equal(v, [[0, 128, 255, 64, 254]])
    q = workload.from_u8(v)
    assert q.dtype == np.float32
    np.testing.assert_array_equal(workload.to_u8(q), v)          # round trip exact
    np.testing.assert_array_equal(q, v.astype(np.float32) / np.float32(255))


def test_arm_decode_entry_errors_without_gpu():
    cfg = workload.CONFIGS["ref"].replace(H=24, W=40)
    d = P.desc_from_config(cfg)
    wsb = P.cc_arm_decode_workspace_bytes(d, 3)
    assert wsb >= 3 * cfg.L * 8
    d8 = P.desc_from_config(cfg)
    d8.latents_i8 = 1                      # host-path transfer format: refused by device entries
    assert P.cc_arm_decode_workspace_bytes(d8, 3) == 0
    im = workload.make_image(cfg, 1)
    io = [P.CcImageIO(8, im.arm_w.ctypes.data, 0, 0, 0, 0)]
    with pytest.raises(ccrd.CcError) as e:          # workspace too small
        P.cc_arm_decode(d, io, [8], 8, ws_ptr=8, ws_bytes=1)
    assert e.value.code == ccrd.CC_EWORKSPACE
    if not _has_gpu():
        with pytest.raises(ccrd.CcError) as e:      # no device: loud failure
            P.cc_arm_decode(d, io, [8], 8, ws_ptr=8, ws_bytes=wsb)
        assert e.value.code == ccrd.CC_ECUDA


def test_arm_path_selection_without_gpu():
    """cc_set_arm_path / cc_arm_path_for (include/ccrd.h): host-only; the
    tensor-core path covers the [16,24,24,2], [16,16,16,2] and [24,24,24,2]
    ARMs, every other shape runs FFMA2 whatever is asked."""
    old = P.cc_get_arm_path()
    try:
        with pytest.raises(ccrd.CcError) as e:
            P.cc_set_arm_path(7)
        assert e.value.code == ccrd.CC_EINVAL
        ref = P.desc_from_config(workload.CONFIGS["ref"])
        low = P.desc_from_config(workload.CONFIGS["low"])
        t2300 = P.desc_from_config(workload.CONFIGS["t2300"])
        P.cc_set_arm_path(P.CC_ARM_AUTO)
        assert P.cc_get_arm_path() == P.CC_ARM_AUTO
        assert P.cc_arm_path_for(ref) == P.CC_ARM_TC           # AUTO: where the tensor cores measured faster
        assert P.cc_arm_path_for(t2300) == P.CC_ARM_FFMA2 and P.cc_arm_path_for(low) == P.CC_ARM_FFMA2
        P.cc_set_arm_path(P.CC_ARM_FFMA2)
        assert P.cc_arm_path_for(ref) == P.CC_ARM_FFMA2
        ws_ffma2 = P.cc_workspace_bytes(ref, 3)
        P.cc_set_arm_path(P.CC_ARM_TC)
        assert P.cc_arm_path_for(ref) == P.CC_ARM_TC and P.cc_arm_path_for(low) == P.CC_ARM_FFMA2
        assert P.cc_arm_path_for(t2300) == P.CC_ARM_TC
        assert P.cc_workspace_bytes(ref, 3) == ws_ffma2      # the layout does not depend on the path
    finally:
        P.cc_set_arm_path(old)


def test_synth_path_selection_without_gpu():
    """cc_set_synth_path / cc_get_synth_path (include/ccrd.h): host-only
    switch, CC_EINVAL for unknown values, AUTO by default."""
    old = P.cc_get_synth_path()
    try:
        with pytest.raises(ccrd.CcError) as e:
            P.cc_set_synth_path(5)
        assert e.value.code == ccrd.CC_EINVAL
        for path in (P.CC_SYN_MMA, P.CC_SYN_FFMA2, P.CC_SYN_AUTO):
            P.cc_set_synth_path(path)
            assert P.cc_get_synth_path() == path
        ref = P.desc_from_config(workload.CONFIGS["ref"])
        ws = P.cc_workspace_bytes(ref, 3)
        P.cc_set_synth_path(P.CC_SYN_MMA)
        assert P.cc_workspace_bytes(ref, 3) == ws            # the layout does not depend on the path
    finally:
        P.cc_set_synth_path(old)
