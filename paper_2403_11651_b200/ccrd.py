"""Thin ctypes binding of libccrd.so (include/ccrd.h) -- argument marshalling
only.  Every step of the RD forward runs in the library's CUDA kernels; there
is no Python or CPU fallback: if the library cannot be loaded, or no CUDA
device is present, calls raise.

Functions keep the C names (cc_rd_forward, cc_arm_rate, ...).  Device buffers
are passed as raw pointers (ints); ``torch`` is only used by the convenience
helpers at the bottom for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

from . import build as _build

CC_MAX_LEVELS = 12
CC_MAX_CTX = 32
CC_MAX_LAYERS = 8

CC_OK, CC_EINVAL, CC_ENOTSUP, CC_EWORKSPACE, CC_ECUDA, CC_ENONFINITE = 0, -1, -2, -3, -4, -5


class CcModelDesc(C.Structure):
    _fields_ = [
        ("H", C.c_int32), ("W", C.c_int32), ("L", C.c_int32),
        ("n_ctx", C.c_int32),
        ("ctx_dy", C.c_int8 * CC_MAX_CTX), ("ctx_dx", C.c_int8 * CC_MAX_CTX),
        ("arm_n_layers", C.c_int32), ("arm_widths", C.c_int32 * (CC_MAX_LAYERS + 1)),
        ("arm_residual_mask", C.c_uint32),
        ("up_taps", C.c_int32), ("up_2d", C.c_int32),
        ("syn_n_1x1", C.c_int32), ("syn_widths", C.c_int32 * (CC_MAX_LAYERS + 1)),
        ("syn_n_res", C.c_int32),
        ("logscale_min", C.c_float), ("logscale_max", C.c_float),
        ("p_floor", C.c_float),
        ("lam", C.c_double),
        ("image_u8", C.c_int32),
        ("latents_i8", C.c_int32),
    ]


class CcRdResult(C.Structure):
    _fields_ = [("rate_bits", C.c_double), ("sse", C.c_double), ("mse", C.c_double), ("cost", C.c_double)]


class CcImageIO(C.Structure):
    _fields_ = [("latents", C.c_void_p), ("arm_w", C.c_void_p), ("up_w", C.c_void_p),
                ("syn_w", C.c_void_p), ("image", C.c_void_p), ("x_hat", C.c_void_p)]


class CcMacBreakdown(C.Structure):
    _fields_ = [("arm", C.c_double), ("up", C.c_double), ("syn", C.c_double), ("total", C.c_double),
                ("arm_macs", C.c_int64), ("up_macs", C.c_int64), ("syn_macs", C.c_int64),
                ("n_latents", C.c_int64)]


class CcStrip(C.Structure):
    """include/ccrd.h cc_strip: owned pixel rows [r0, r1), owned latent rows
    [own_lo[l], own_hi[l]) and the latent-buffer window [lo[l], hi[l])."""
    _fields_ = [("r0", C.c_int32), ("r1", C.c_int32),
                ("own_lo", C.c_int32 * CC_MAX_LEVELS), ("own_hi", C.c_int32 * CC_MAX_LEVELS),
                ("lo", C.c_int32 * CC_MAX_LEVELS), ("hi", C.c_int32 * CC_MAX_LEVELS)]


class CcAdam(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("t", C.c_int32)]


class CcAnalysisDesc(C.Structure):
    _fields_ = [("H", C.c_int32), ("W", C.c_int32), ("L", C.c_int32), ("C", C.c_int32), ("blocks", C.c_int32),
                ("tf32", C.c_int32), ("N", C.c_int32)]


class CcProfileSummary(C.Structure):
    _fields_ = [("arm_ms", C.c_double), ("syn_ms", C.c_double), ("reduce_ms", C.c_double), ("pyr_ms", C.c_double),
                ("arm_launches", C.c_int64), ("syn_launches", C.c_int64), ("reduce_launches", C.c_int64),
                ("pyr_launches", C.c_int64)]


# Symbols include/ccrd.h declares (checked by tests/test_abi.py).
EXPORTS = ["cc_workspace_bytes", "cc_rd_forward", "cc_workspace_bytes_host", "cc_rd_forward_host",
           "cc_arm_rate", "cc_upsample", "cc_synthesize", "cc_mac_per_pixel", "cc_validate",
           "cc_strerror", "cc_last_error", "cc_version", "cc_last_launch_count",
           "cc_profile_begin", "cc_profile_end", "cc_strip_window", "cc_strip_latent_count",
           "cc_workspace_bytes_strip", "cc_rd_forward_strip", "cc_train_param_count",
           "cc_train_workspace_bytes", "cc_train_step", "cc_decode", "cc_analysis_param_count",
           "cc_analysis_workspace_bytes", "cc_analysis_forward", "cc_arm_decode_workspace_bytes", "cc_arm_decode",
           "cc_set_arm_path", "cc_get_arm_path", "cc_arm_path_for", "cc_set_synth_path", "cc_get_synth_path"]

# ARM rate paths and synthesis 1x1 paths (include/ccrd.h)
CC_ARM_AUTO, CC_ARM_FFMA2, CC_ARM_TC = 0, 1, 2
CC_SYN_AUTO, CC_SYN_FFMA2, CC_SYN_MMA, CC_SYN_TMA = 0, 1, 2, 3

_lib = None


def lib_path() -> str:
    return _build.LIB


def load(rebuild_if_stale: bool = True) -> C.CDLL:
    """Load libccrd.so (building it in-tree with nvcc if missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    alt = os.environ.get("CCRD_LIB")  # experiment variant built by tools/ (same ABI)
    if alt:
        rebuild_if_stale = False
        try:
            _build.build()
        except FileNotFoundError:
            pass  # no nvcc: fall through to loading what exists
    if not os.path.exists(alt or _build.LIB):
        raise ImportError(f"libccrd.so not built ({_build.LIB}); run paper_2403_11651_b200/build.py")
    L = C.CDLL(alt or _build.LIB)
    P, V, S = C.POINTER, C.c_void_p, C.c_size_t
    D = P(CcModelDesc)
    L.cc_workspace_bytes.restype = S
    L.cc_workspace_bytes.argtypes = [D, C.c_int32]
    L.cc_workspace_bytes_host.restype = S
    L.cc_workspace_bytes_host.argtypes = [D, C.c_int32]
    L.cc_rd_forward.restype = C.c_int
    L.cc_rd_forward.argtypes = [D, P(CcImageIO), C.c_int32, V, V, S, V]
    L.cc_rd_forward_host.restype = C.c_int
    L.cc_rd_forward_host.argtypes = [D, P(CcImageIO), C.c_int32, V, V, S, V]
    L.cc_arm_rate.restype = C.c_int
    L.cc_arm_rate.argtypes = [D, V, V, V, V, V, V, V, S, V]
    L.cc_arm_decode_workspace_bytes.restype = S
    L.cc_arm_decode_workspace_bytes.argtypes = [D, C.c_int32]
    L.cc_arm_decode.restype = C.c_int
    L.cc_arm_decode.argtypes = [D, V, C.c_int32, V, V, V, V, V, V, V, S, V]
    L.cc_upsample.restype = C.c_int
    L.cc_upsample.argtypes = [D, V, V, V, V, S, V]
    L.cc_synthesize.restype = C.c_int
    L.cc_synthesize.argtypes = [D, V, V, V, V, V, V, V, S, V]
    L.cc_mac_per_pixel.restype = C.c_double
    L.cc_mac_per_pixel.argtypes = [D, P(CcMacBreakdown)]
    L.cc_validate.restype = C.c_int
    L.cc_validate.argtypes = [D]
    L.cc_strerror.restype = C.c_char_p
    L.cc_strerror.argtypes = [C.c_int]
    L.cc_last_error.restype = C.c_char_p
    L.cc_version.restype = C.c_char_p
    L.cc_last_launch_count.restype = C.c_int64
    L.cc_profile_begin.restype = C.c_int
    L.cc_profile_end.restype = C.c_int
    L.cc_profile_end.argtypes = [P(CcProfileSummary)]
    L.cc_strip_window.restype = C.c_int
    L.cc_strip_window.argtypes = [D, C.c_int32, C.c_int32, P(CcStrip)]
    L.cc_strip_latent_count.restype = C.c_int64
    L.cc_strip_latent_count.argtypes = [D, P(CcStrip)]
    L.cc_workspace_bytes_strip.restype = S
    L.cc_workspace_bytes_strip.argtypes = [D, P(CcStrip)]
    L.cc_rd_forward_strip.restype = C.c_int
    L.cc_rd_forward_strip.argtypes = [D, P(CcStrip), P(CcImageIO), V, V, S, V]
    L.cc_train_param_count.restype = C.c_int64
    L.cc_train_param_count.argtypes = [D]
    L.cc_train_workspace_bytes.restype = S
    L.cc_train_workspace_bytes.argtypes = [D]
    A = P(CcAnalysisDesc)
    L.cc_analysis_param_count.restype = C.c_int64
    L.cc_analysis_param_count.argtypes = [A]
    L.cc_analysis_workspace_bytes.restype = S
    L.cc_analysis_workspace_bytes.argtypes = [A]
    L.cc_analysis_forward.restype = C.c_int
    L.cc_analysis_forward.argtypes = [A, V, V, V, V, S, V]
    L.cc_decode.restype = C.c_int
    L.cc_decode.argtypes = [D, V, V, V, V, V, S, V]
    L.cc_train_step.restype = C.c_int
    L.cc_train_step.argtypes = [D, V, V, V, V, V, P(CcAdam), V, V, V, S, V]
    L.cc_set_arm_path.restype = C.c_int
    L.cc_set_arm_path.argtypes = [C.c_int32]
    L.cc_get_arm_path.restype = C.c_int32
    L.cc_arm_path_for.restype = C.c_int32
    L.cc_arm_path_for.argtypes = [D]
    L.cc_set_synth_path.restype = C.c_int
    L.cc_set_synth_path.argtypes = [C.c_int32]
    L.cc_get_synth_path.restype = C.c_int32
    _lib = L
    return L


class CcError(RuntimeError):
    def __init__(self, code: int, where: str):
        L = load()
        super().__init__(f"{where}: {L.cc_strerror(code).decode()} ({code}): {L.cc_last_error().decode()}")
        self.code = code


def _check(rc: int, where: str):
    if rc != CC_OK:
        raise CcError(rc, where)


# ------------------------------------------------------------------ descriptor
def make_desc(H, W, L, ctx, arm_widths, arm_residual, up_taps, syn_widths, syn_n_res,
              logscale_min, logscale_max, p_floor, lam, up_2d=False) -> CcModelDesc:
    d = CcModelDesc()
    d.H, d.W, d.L = H, W, L
    d.n_ctx = len(ctx)
    for c, (dy, dx) in enumerate(ctx):
        d.ctx_dy[c] = dy
        d.ctx_dx[c] = dx
    d.arm_n_layers = len(arm_widths) - 1
    for k, v in enumerate(arm_widths):
        d.arm_widths[k] = v
    d.arm_residual_mask = sum(1 << k for k, r in enumerate(arm_residual) if r)
    d.up_taps = up_taps
    d.up_2d = int(bool(up_2d))
    d.syn_n_1x1 = len(syn_widths) - 1
    for k, v in enumerate(syn_widths):
        d.syn_widths[k] = v
    d.syn_n_res = syn_n_res
    d.logscale_min, d.logscale_max, d.p_floor = logscale_min, logscale_max, p_floor
    d.lam = lam
    return d


def desc_from_config(cfg, H: Optional[int] = None, W: Optional[int] = None) -> CcModelDesc:
    """Descriptor from a workload.Config (the shared, arithmetic-free config)."""
    return make_desc(cfg.H if H is None else H, cfg.W if W is None else W, cfg.L, cfg.ctx,
                     cfg.arm_widths, cfg.arm_residual, cfg.up_taps, cfg.syn_widths, cfg.syn_n_res,
                     cfg.logscale_min, cfg.logscale_max, cfg.p_floor, cfg.lam,
                     up_2d=getattr(cfg, "up_2d", False))


# ------------------------------------------------------------------ raw calls
def cc_workspace_bytes(desc: CcModelDesc, n_img: int) -> int:
    return load().cc_workspace_bytes(C.byref(desc), n_img)


def cc_workspace_bytes_host(desc: CcModelDesc, n_img: int) -> int:
    return load().cc_workspace_bytes_host(C.byref(desc), n_img)


def cc_validate(desc: CcModelDesc) -> int:
    return load().cc_validate(C.byref(desc))


def cc_mac_per_pixel(desc: CcModelDesc) -> CcMacBreakdown:
    out = CcMacBreakdown()
    v = load().cc_mac_per_pixel(C.byref(desc), C.byref(out))
    if v < 0:
        raise CcError(cc_validate(desc), "cc_mac_per_pixel")
    return out


def cc_rd_forward(desc, io: Sequence[CcImageIO], results_ptr: int, ws_ptr: int, ws_bytes: int,
                  stream_ptr: int = 0) -> None:
    arr = (CcImageIO * len(io))(*io)
    _check(load().cc_rd_forward(C.byref(desc), arr, len(io), results_ptr, ws_ptr, ws_bytes, stream_ptr),
           "cc_rd_forward")


def cc_rd_forward_host(desc, io: Sequence[CcImageIO], results: np.ndarray, ws_ptr: int, ws_bytes: int,
                       stream_ptr: int = 0) -> None:
    assert results.dtype == np.float64 and results.size >= 4 * len(io) and results.flags.c_contiguous
    arr = (CcImageIO * len(io))(*io)
    _check(load().cc_rd_forward_host(C.byref(desc), arr, len(io), results.ctypes.data, ws_ptr, ws_bytes,
                                     stream_ptr), "cc_rd_forward_host")


def cc_arm_rate(desc, latents_ptr, arm_w: np.ndarray, rate_ptr, mu_ptr, scale_ptr, bits_ptr, ws_ptr, ws_bytes,
                stream_ptr=0) -> None:
    aw = np.ascontiguousarray(arm_w, np.float32)
    _check(load().cc_arm_rate(C.byref(desc), latents_ptr, aw.ctypes.data, rate_ptr, mu_ptr, scale_ptr, bits_ptr,
                              ws_ptr, ws_bytes, stream_ptr), "cc_arm_rate")


def cc_arm_decode_workspace_bytes(desc, n_img: int) -> int:
    return load().cc_arm_decode_workspace_bytes(C.byref(desc), n_img)


def cc_arm_decode(desc, io: Sequence["CcImageIO"], decoded_ptrs, rate_ptr, mu_ptrs=None, scale_ptrs=None,
                  bits_ptrs=None, poison_ptr=0, ws_ptr=0, ws_bytes=0, stream_ptr=0) -> None:
    """NEXT-3 wavefront ARM decode of len(io) images (include/ccrd.h): io[i].latents
    (device) play the entropy decoder, io[i].arm_w host blobs; *_ptrs: lists of
    device pointers (or None)."""
    n = len(io)
    arr = (CcImageIO * n)(*io)
    vp = C.c_void_p * n

    def ptrs(lst):
        return vp(*lst) if lst is not None else None
    _check(load().cc_arm_decode(C.byref(desc), arr, n, ptrs(decoded_ptrs), rate_ptr, ptrs(mu_ptrs),
                                ptrs(scale_ptrs), ptrs(bits_ptrs), poison_ptr or None, ws_ptr, ws_bytes, stream_ptr),
           "cc_arm_decode")


def cc_upsample(desc, latents_ptr, up_w: np.ndarray, dense_ptr, ws_ptr=0, ws_bytes=0, stream_ptr=0) -> None:
    uw = np.ascontiguousarray(up_w, np.float32)
    _check(load().cc_upsample(C.byref(desc), latents_ptr, uw.ctypes.data, dense_ptr, ws_ptr, ws_bytes, stream_ptr),
           "cc_upsample")


def cc_synthesize(desc, dense_ptr, syn_w: np.ndarray, image_ptr, x_hat_ptr, sse_ptr, h1_ptr, ws_ptr, ws_bytes,
                  stream_ptr=0) -> None:
    sw = np.ascontiguousarray(syn_w, np.float32)
    _check(load().cc_synthesize(C.byref(desc), dense_ptr, sw.ctypes.data, image_ptr, x_hat_ptr, sse_ptr, h1_ptr,
                                ws_ptr, ws_bytes, stream_ptr), "cc_synthesize")


def cc_strip_window(desc, r0: int, r1: int) -> CcStrip:
    st = CcStrip()
    _check(load().cc_strip_window(C.byref(desc), r0, r1, C.byref(st)), "cc_strip_window")
    return st


def cc_strip_latent_count(desc, strip: CcStrip) -> int:
    n = load().cc_strip_latent_count(C.byref(desc), C.byref(strip))
    if n < 0:
        raise CcError(CC_EINVAL, "cc_strip_latent_count")
    return n


def cc_workspace_bytes_strip(desc, strip: CcStrip) -> int:
    return load().cc_workspace_bytes_strip(C.byref(desc), C.byref(strip))


def cc_rd_forward_strip(desc, strip: CcStrip, io: CcImageIO, result_ptr: int, ws_ptr: int, ws_bytes: int,
                        stream_ptr: int = 0) -> None:
    _check(load().cc_rd_forward_strip(C.byref(desc), C.byref(strip), C.byref(io), result_ptr, ws_ptr, ws_bytes,
                                      stream_ptr), "cc_rd_forward_strip")


def cc_decode(desc, latents_ptr, up_w: np.ndarray, syn_w: np.ndarray, out_ptr, ws_ptr, ws_bytes, stream_ptr=0):
    uw = np.ascontiguousarray(up_w, np.float32)
    sw = np.ascontiguousarray(syn_w, np.float32)
    _check(load().cc_decode(C.byref(desc), latents_ptr, uw.ctypes.data, sw.ctypes.data, out_ptr, ws_ptr, ws_bytes,
                            stream_ptr), "cc_decode")


def analysis_desc(acfg, tf32=0, n=1) -> CcAnalysisDesc:
    """tf32: 0 fp32 | 1 (or True) TF32, fused tensor-core blocks | 2 TF32 cuBLASLt unfused |
    3 fused with FP16 operands + TMA-staged depth-wise (stride-1 blocks);
    n: images per call (one shared network)."""
    return CcAnalysisDesc(acfg.H, acfg.W, acfg.L, acfg.C, acfg.blocks, int(tf32), int(n))


def cc_analysis_param_count(ad: CcAnalysisDesc) -> int:
    n = load().cc_analysis_param_count(C.byref(ad))
    if n < 0:
        raise CcError(CC_EINVAL, "cc_analysis_param_count")
    return n


def cc_analysis_workspace_bytes(ad: CcAnalysisDesc) -> int:
    return load().cc_analysis_workspace_bytes(C.byref(ad))


def cc_analysis_forward(ad: CcAnalysisDesc, image_ptr, weights_ptr, latents_ptr, ws_ptr, ws_bytes, stream_ptr=0):
    _check(load().cc_analysis_forward(C.byref(ad), image_ptr, weights_ptr, latents_ptr, ws_ptr, ws_bytes, stream_ptr),
           "cc_analysis_forward")


def cc_train_param_count(desc) -> int:
    n = load().cc_train_param_count(C.byref(desc))
    if n < 0:
        raise CcError(cc_validate(desc), "cc_train_param_count")
    return n


def cc_train_workspace_bytes(desc) -> int:
    return load().cc_train_workspace_bytes(C.byref(desc))


def cc_train_step(desc, params_ptr, noise_ptr, image_ptr, m_ptr, v_ptr, opt: Optional[CcAdam], result_ptr, grad_ptr,
                  ws_ptr, ws_bytes, stream_ptr=0) -> None:
    _check(load().cc_train_step(C.byref(desc), params_ptr, noise_ptr, image_ptr, m_ptr, v_ptr,
                                C.byref(opt) if opt is not None else None, result_ptr, grad_ptr, ws_ptr, ws_bytes,
                                stream_ptr), "cc_train_step")


def cc_last_launch_count() -> int:
    return load().cc_last_launch_count()


def cc_set_arm_path(path: int) -> None:
    _check(load().cc_set_arm_path(path), "cc_set_arm_path")


def cc_get_arm_path() -> int:
    return load().cc_get_arm_path()


def cc_arm_path_for(desc) -> int:
    return load().cc_arm_path_for(C.byref(desc))


def cc_set_synth_path(path: int) -> None:
    _check(load().cc_set_synth_path(path), "cc_set_synth_path")


def cc_get_synth_path() -> int:
    return load().cc_get_synth_path()


class synth_path:
    """Context manager: run a block with a given synthesis 1x1 path, then restore."""

    def __init__(self, path: int):
        self.path, self.old = path, None

    def __enter__(self):
        self.old = cc_get_synth_path()
        cc_set_synth_path(self.path)
        return self

    def __exit__(self, *exc):
        cc_set_synth_path(self.old)
        return False


class arm_path:
    """Context manager: run a block with a given ARM path, then restore."""

    def __init__(self, path: int):
        self.path, self.old = path, None

    def __enter__(self):
        self.old = cc_get_arm_path()
        cc_set_arm_path(self.path)
        return self

    def __exit__(self, *exc):
        cc_set_arm_path(self.old)
        return False


def cc_profile_begin() -> None:
    _check(load().cc_profile_begin(), "cc_profile_begin")


def cc_profile_end() -> CcProfileSummary:
    out = CcProfileSummary()
    _check(load().cc_profile_end(C.byref(out)), "cc_profile_end")
    return out


def cc_version() -> str:
    return load().cc_version().decode()


# ------------------------------------------------------------- torch helpers
class DeviceBatch:
    """Device-resident inputs of n images (torch tensors for memory only) and
    the host weight blobs, laid out for cc_rd_forward."""

    def __init__(self, cfg, images: List, device="cuda", with_xhat=True, image_u8=False):
        """image_u8: images go to the device as uint8 planes (desc.image_u8 = 1,
        x = v / 255); im.image must then hold 8-bit levels (workload.to_u8)."""
        import torch

        def to_u8(x):  # storage format: v = rint(255 x)
            return np.clip(np.rint(np.asarray(x, np.float64) * 255.0), 0, 255).astype(np.uint8)
        self.cfg = cfg
        self.desc = desc_from_config(cfg)
        self.desc.image_u8 = int(bool(image_u8))
        self.n = len(images)
        self.lat = [torch.from_numpy(im.latents).to(device) for im in images]
        self.img = [torch.from_numpy(to_u8(im.image) if image_u8 else im.image).to(device) for im in images]
        self.xhat = [torch.empty(im.image.shape, dtype=torch.float32, device=device) for im in images] \
            if with_xhat else None
        self.arm_w = [np.ascontiguousarray(im.arm_w, np.float32) for im in images]
        self.up_w = [np.ascontiguousarray(im.up_w, np.float32) for im in images]
        self.syn_w = [np.ascontiguousarray(im.syn_w, np.float32) for im in images]
        self.ws_bytes = cc_workspace_bytes(self.desc, self.n)
        if self.ws_bytes == 0:
            raise CcError(cc_validate(self.desc), "cc_workspace_bytes")
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)
        self.results = torch.zeros((self.n, 4), dtype=torch.float64, device=device)
        self.io = [CcImageIO(self.lat[i].data_ptr(), self.arm_w[i].ctypes.data, self.up_w[i].ctypes.data,
                             self.syn_w[i].ctypes.data, self.img[i].data_ptr(),
                             self.xhat[i].data_ptr() if with_xhat else None) for i in range(self.n)]

    def forward(self, stream_ptr: Optional[int] = None):
        import torch
        s = torch.cuda.current_stream().cuda_stream if stream_ptr is None else stream_ptr
        cc_rd_forward(self.desc, self.io, self.results.data_ptr(), self.ws.data_ptr(), self.ws_bytes, s)
        return self.results


class DeviceStrip:
    """One strip of one image on the device (include/ccrd.h "strips"): the
    latent window buffer, the strip's image rows, its x_hat rows, workspace and
    the device result slot.  ``lat`` is filled by the caller (owned rows from
    the bitstream, halo rows by dist.exchange_halos)."""

    def __init__(self, cfg, strip: "CcStrip", arm_w, up_w, syn_w, image_rows=None, device="cuda",
                 with_xhat=True):
        import torch
        self.cfg = cfg
        self.desc = desc_from_config(cfg)
        self.strip = strip
        n = cc_strip_latent_count(self.desc, strip)
        self.lat = torch.zeros(n, dtype=torch.int16, device=device)
        rows = strip.r1 - strip.r0
        self.img = None if image_rows is None else torch.as_tensor(image_rows).to(device).contiguous()
        if self.img is not None:
            assert tuple(self.img.shape) == (3, rows, cfg.W), self.img.shape
            self.desc.image_u8 = int(self.img.dtype == torch.uint8)   # 8-bit rows: x = v / 255
        self.xhat = torch.empty((3, rows, cfg.W), dtype=torch.float32, device=device) if with_xhat else None
        self.arm_w = np.ascontiguousarray(arm_w, np.float32)
        self.up_w = np.ascontiguousarray(up_w, np.float32)
        self.syn_w = np.ascontiguousarray(syn_w, np.float32)
        self.ws_bytes = cc_workspace_bytes_strip(self.desc, strip)
        if self.ws_bytes == 0:
            raise CcError(CC_EINVAL, "cc_workspace_bytes_strip")
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)
        self.result = torch.zeros(4, dtype=torch.float64, device=device)
        self.io = CcImageIO(self.lat.data_ptr(), self.arm_w.ctypes.data, self.up_w.ctypes.data,
                            self.syn_w.ctypes.data, self.img.data_ptr() if self.img is not None else None,
                            self.xhat.data_ptr() if with_xhat else None)

    def forward(self, stream_ptr: Optional[int] = None):
        import torch
        s = torch.cuda.current_stream().cuda_stream if stream_ptr is None else stream_ptr
        cc_rd_forward_strip(self.desc, self.strip, self.io, self.result.data_ptr(), self.ws.data_ptr(),
                            self.ws_bytes, s)
        return self.result


class DeviceTrainer:
    """Device state of one image's encoder training (NEXT-2): the parameter
    vector [y | arm_w | up_w | syn_w], Adam moments, gradient, image, workspace."""

    def __init__(self, cfg, y, arm_w, up_w, syn_w, image, device="cuda"):
        import torch
        self.cfg = cfg
        self.desc = desc_from_config(cfg)
        self.n = cc_train_param_count(self.desc)
        par = np.concatenate([np.asarray(y, np.float32).ravel(), np.asarray(arm_w, np.float32).ravel(),
                              np.asarray(up_w, np.float32).ravel(), np.asarray(syn_w, np.float32).ravel()])
        assert par.size == self.n, (par.size, self.n)
        self.params = torch.from_numpy(par).to(device)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.grad = torch.zeros_like(self.params)
        self.image = torch.as_tensor(np.ascontiguousarray(image, np.float32)).to(device)
        self.noise = torch.zeros(int(np.asarray(y).size), dtype=torch.float32, device=device)
        self.result = torch.zeros(4, dtype=torch.float64, device=device)
        self.ws_bytes = cc_train_workspace_bytes(self.desc)
        if self.ws_bytes == 0:
            raise CcError(CC_ENOTSUP, "cc_train_workspace_bytes")
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)
        self.t = 0

    def step(self, noise=None, lr=1e-2, betas=(0.9, 0.999), eps=1e-8, update=True, stream_ptr=None):
        import torch
        if noise is not None:
            self.noise.copy_(torch.as_tensor(noise))
        s = torch.cuda.current_stream().cuda_stream if stream_ptr is None else stream_ptr
        opt = None
        if update:
            self.t += 1
            opt = CcAdam(lr, betas[0], betas[1], eps, self.t)
        cc_train_step(self.desc, self.params.data_ptr(), self.noise.data_ptr(), self.image.data_ptr(),
                      self.m.data_ptr(), self.v.data_ptr(), opt, self.result.data_ptr(), self.grad.data_ptr(),
                      self.ws.data_ptr(), self.ws_bytes, s)
        return self.result
