"""ctypes wrapper of the fp64 CPU oracle (oracle/ccoracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py -- never by the product
package ``paper_2403_11651_b200``.  It shares no code with the CUDA path; the
only thing both sides use is ``workload`` (seeded inputs, no method arithmetic).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ccoracle.c")
_SRC_TRAIN = os.path.join(_HERE, "cctrain.c")  # NEXT-2: one training iteration
_SRC_ANALYSIS = os.path.join(_HERE, "ccanalysis.c")  # NEXT-4: N-O analysis transform
_LIB = os.path.join(_HERE, "libccoracle.so")

MAX_LAYERS = 8


class OrcModel(C.Structure):
    _fields_ = [
        ("H", C.c_int32), ("W", C.c_int32), ("L", C.c_int32),
        ("n_ctx", C.c_int32), ("ctx_dy", C.c_int32 * 32), ("ctx_dx", C.c_int32 * 32),
        ("arm_n_layers", C.c_int32), ("arm_widths", C.c_int32 * (MAX_LAYERS + 1)),
        ("arm_residual", C.c_int32 * MAX_LAYERS),
        ("up_taps", C.c_int32), ("up_2d", C.c_int32),
        ("syn_n_1x1", C.c_int32), ("syn_widths", C.c_int32 * (MAX_LAYERS + 1)),
        ("syn_n_res", C.c_int32),
        ("logscale_min", C.c_double), ("logscale_max", C.c_double),
        ("p_floor", C.c_double), ("lam", C.c_double),
    ]


class OrcAnalysis(C.Structure):
    _fields_ = [("H", C.c_int32), ("W", C.c_int32), ("L", C.c_int32), ("C", C.c_int32), ("blocks", C.c_int32)]


class OrcAdam(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("t", C.c_int32)]


class OrcMacs(C.Structure):
    _fields_ = [("arm", C.c_int64), ("up", C.c_int64), ("syn", C.c_int64)]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C99 + OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(_SRC_TRAIN), os.path.getmtime(_SRC_ANALYSIS),
            os.path.getmtime(os.path.join(_HERE, "ccoracle.h"))):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC, _SRC_TRAIN, _SRC_ANALYSIS, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.POINTER
        L.orc_level_dims.restype = C.c_int64
        L.orc_level_dims.argtypes = [P(OrcModel), P(C.c_int32), P(C.c_int32)]
        L.orc_laplace_prob.restype = C.c_double
        L.orc_laplace_prob.argtypes = [C.c_double] * 3
        L.orc_laplace_bits.restype = C.c_double
        L.orc_laplace_bits.argtypes = [C.c_double] * 4
        L.orc_arm_mlp.restype = None
        L.orc_arm_mlp.argtypes = [P(OrcModel), C.c_void_p, C.c_void_p, P(C.c_double), P(C.c_double),
                                  P(C.c_int64)]
        L.orc_context.restype = None
        L.orc_context.argtypes = [P(OrcModel), C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_void_p]
        L.orc_rate.restype = C.c_double
        L.orc_rate.argtypes = [P(OrcModel), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               P(OrcMacs)]
        L.orc_rate_rows.restype = C.c_double
        L.orc_rate_rows.argtypes = [P(OrcModel), C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_void_p]
        L.orc_upsample.restype = None
        L.orc_upsample.argtypes = [P(OrcModel), C.c_void_p, C.c_void_p, C.c_void_p, P(OrcMacs)]
        L.orc_synthesis.restype = None
        L.orc_synthesis.argtypes = [P(OrcModel), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, P(OrcMacs)]
        L.orc_rd_forward.restype = C.c_int
        L.orc_rd_forward.argtypes = [P(OrcModel)] + [C.c_void_p] * 8 + [P(OrcMacs)]
        L.orc_analysis_param_count.restype = C.c_int64
        L.orc_analysis_param_count.argtypes = [P(OrcAnalysis)]
        L.orc_analysis_forward.restype = C.c_int
        L.orc_analysis_forward.argtypes = [P(OrcAnalysis), C.c_void_p, C.c_void_p, C.c_void_p, P(C.c_int64)]
        L.orc_decode_u8.restype = None
        L.orc_decode_u8.argtypes = [P(OrcModel), C.c_void_p, C.c_void_p]
        L.orc_arm_decode.restype = C.c_int
        L.orc_arm_decode.argtypes = [P(OrcModel), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, P(C.c_double)]
        L.orc_train_param_count.restype = C.c_int64
        L.orc_train_param_count.argtypes = [P(OrcModel)]
        L.orc_train_grad.restype = C.c_int
        L.orc_train_grad.argtypes = [P(OrcModel)] + [C.c_void_p] * 5
        L.orc_adam_step.restype = None
        L.orc_adam_step.argtypes = [C.c_int64] + [C.c_void_p] * 4 + [P(OrcAdam)]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return lib().orc_get_threads()


def model(cfg, H=None, W=None, arm_residual=None) -> OrcModel:
    """Build the oracle's model record from a workload.Config."""
    m = OrcModel()
    m.H = cfg.H if H is None else H
    m.W = cfg.W if W is None else W
    m.L = cfg.L
    m.n_ctx = cfg.n_ctx
    for c, (dy, dx) in enumerate(cfg.ctx):
        m.ctx_dy[c] = dy
        m.ctx_dx[c] = dx
    aw = cfg.arm_widths
    m.arm_n_layers = len(aw) - 1
    for k, v in enumerate(aw):
        m.arm_widths[k] = v
    res = cfg.arm_residual if arm_residual is None else arm_residual
    for k, v in enumerate(res):
        m.arm_residual[k] = v
    m.up_taps = cfg.up_taps
    m.up_2d = int(getattr(cfg, "up_2d", False))
    sw = cfg.syn_widths
    m.syn_n_1x1 = len(sw) - 1
    for k, v in enumerate(sw):
        m.syn_widths[k] = v
    m.syn_n_res = cfg.syn_n_res
    m.logscale_min = cfg.logscale_min
    m.logscale_max = cfg.logscale_max
    m.p_floor = cfg.p_floor
    m.lam = cfg.lam
    return m


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def level_dims(m: OrcModel):
    h = (C.c_int32 * 12)()
    w = (C.c_int32 * 12)()
    lib().orc_level_dims(C.byref(m), h, w)
    return [(h[l], w[l]) for l in range(m.L)]


def laplace_prob(y, mu, b):
    return lib().orc_laplace_prob(float(y), float(mu), float(b))


def laplace_bits(y, mu, b, p_floor=2.0 ** -16):
    return lib().orc_laplace_bits(float(y), float(mu), float(b), float(p_floor))


def context(m: OrcModel, grid: np.ndarray, i: int, j: int) -> np.ndarray:
    g = _c(grid, np.int16)
    out = np.zeros(m.n_ctx, np.float64)
    lib().orc_context(C.byref(m), _p(g), g.shape[0], g.shape[1], i, j, _p(out))
    return out


def arm_mlp(m: OrcModel, ctx, arm_w):
    ctx = _c(ctx, np.float64)
    aw = _c(arm_w, np.float32)
    mu, b, macs = C.c_double(), C.c_double(), C.c_int64(0)
    lib().orc_arm_mlp(C.byref(m), _p(ctx), _p(aw), C.byref(mu), C.byref(b), C.byref(macs))
    return mu.value, b.value


def rate(m: OrcModel, latents, arm_w, per_latent=False):
    """Returns R (bits) [, mu, b, bits arrays packed like the latents], macs."""
    lat = _c(latents, np.int16)
    aw = _c(arm_w, np.float32)
    macs = OrcMacs()
    if per_latent:
        n = lat.size
        mu, b, bits = (np.zeros(n) for _ in range(3))
        R = lib().orc_rate(C.byref(m), _p(lat), _p(aw), _p(mu), _p(b), _p(bits), C.byref(macs))
        return R, mu, b, bits, macs
    R = lib().orc_rate(C.byref(m), _p(lat), _p(aw), None, None, None, C.byref(macs))
    return R, macs


def rate_rows(m: OrcModel, latents, arm_w, level, r0, r1):
    lat = _c(latents, np.int16)
    aw = _c(arm_w, np.float32)
    w = level_dims(m)[level][1]
    bits = np.zeros((r1 - r0) * w)
    R = lib().orc_rate_rows(C.byref(m), _p(lat), _p(aw), level, r0, r1, _p(bits))
    return R, bits.reshape(r1 - r0, w)


def upsample(m: OrcModel, latents, up_w):
    lat = _c(latents, np.int16)
    uw = _c(up_w, np.float32)
    dense = np.zeros((m.L, m.H, m.W))
    macs = OrcMacs()
    lib().orc_upsample(C.byref(m), _p(lat), _p(uw), _p(dense), C.byref(macs))
    return dense, macs


def synthesis(m: OrcModel, dense, syn_w):
    d = _c(dense, np.float64)
    sw = _c(syn_w, np.float32)
    xh = np.zeros((3, m.H, m.W))
    h1 = np.zeros((3, m.H, m.W))
    macs = OrcMacs()
    lib().orc_synthesis(C.byref(m), _p(d), _p(sw), _p(xh), _p(h1), C.byref(macs))
    return xh, h1, macs


def rd_forward(m: OrcModel, latents, arm_w, up_w, syn_w, image, want_xhat=False, want_dense=False):
    """Returns dict(rate_bits, sse, mse, cost, macs[, x_hat, dense])."""
    lat = _c(latents, np.int16)
    aw, uw, sw = (_c(a, np.float32) for a in (arm_w, up_w, syn_w))
    img = _c(image, np.float32)
    out = np.zeros(4)
    xh = np.zeros((3, m.H, m.W)) if want_xhat else None
    dn = np.zeros((m.L, m.H, m.W)) if want_dense else None
    macs = OrcMacs()
    rc = lib().orc_rd_forward(C.byref(m), _p(lat), _p(aw), _p(uw), _p(sw), _p(img), _p(out),
                              _p(xh) if xh is not None else None, _p(dn) if dn is not None else None,
                              C.byref(macs))
    if rc != 0:
        raise ValueError(f"orc_rd_forward rc={rc}")
    r = dict(rate_bits=out[0], sse=out[1], mse=out[2], cost=out[3],
             macs=dict(arm=macs.arm, up=macs.up, syn=macs.syn))
    if want_xhat:
        r["x_hat"] = xh
    if want_dense:
        r["dense"] = dn
    return r


def rd_forward_image(cfg, im, **kw):
    """Convenience: run on a workload.Image."""
    return rd_forward(model(cfg), im.latents, im.arm_w, im.up_w, im.syn_w, im.image, **kw)


def time_rd_forward(cfg, im, threads: int):
    """Wall-clock one oracle RD forward (bench.py cpu_baseline leg)."""
    set_threads(threads)
    t0 = time.perf_counter()
    r = rd_forward_image(cfg, im)
    return time.perf_counter() - t0, r


# ------------------------------------------------------------ training (NEXT-2)
def train_param_count(m: OrcModel) -> int:
    return lib().orc_train_param_count(C.byref(m))


def pack_params(latents_float, arm_w, up_w, syn_w) -> np.ndarray:
    """[y | arm_w | up_w | syn_w] fp32 (the documented parameter layout)."""
    return np.concatenate([np.asarray(latents_float, np.float32).ravel(), np.asarray(arm_w, np.float32).ravel(),
                           np.asarray(up_w, np.float32).ravel(), np.asarray(syn_w, np.float32).ravel()])


def train_grad(m: OrcModel, params, noise, image):
    """(out[4] = rate_bits, sse, mse, cost), gradient (fp64, parameter layout)."""
    par = _c(params, np.float32)
    nz = _c(noise, np.float32)
    img = _c(image, np.float32)
    out = np.zeros(4)
    grad = np.zeros(train_param_count(m))
    rc = lib().orc_train_grad(C.byref(m), _p(par), _p(nz), _p(img), _p(out), _p(grad))
    if rc != 0:
        raise ValueError(f"orc_train_grad rc={rc}")
    return out, grad


def adam_step(params: np.ndarray, grad, mom1: np.ndarray, mom2: np.ndarray, lr, beta1, beta2, eps, t):
    """In place on params (fp32), mom1 / mom2 (fp64)."""
    assert params.dtype == np.float32 and mom1.dtype == np.float64 and mom2.dtype == np.float64
    g = _c(grad, np.float64)
    lib().orc_adam_step(params.size, _p(params), _p(g), _p(mom1), _p(mom2),
                        C.byref(OrcAdam(lr, beta1, beta2, eps, t)))


def decode_u8(m: OrcModel, x_hat) -> np.ndarray:
    """Decoder output (NEXT-3): interleaved 8-bit RGB [H][W][3] of clamp(x_hat)."""
    xh = _c(x_hat, np.float64)
    out = np.zeros((m.H, m.W, 3), np.uint8)
    lib().orc_decode_u8(C.byref(m), _p(xh), _p(out))
    return out


def arm_decode(m: OrcModel, truth, arm_w):
    """NEXT-3: raster-order autoregressive decode (the entropy decoder played by
    `truth`).  Returns (status, decoded int16, mu, b, bits, rate); status -1 if
    a context read an undecoded latent."""
    t = _c(truth, np.int16)
    aw = _c(arm_w, np.float32)
    n = t.size
    dec = np.full(n, -32768, np.int16)
    mu, b, bits = (np.zeros(n) for _ in range(3))
    rate = C.c_double(0.0)
    st = lib().orc_arm_decode(C.byref(m), _p(t), _p(aw), _p(dec), _p(mu), _p(b), _p(bits), C.byref(rate))
    return st, dec, mu, b, bits, rate.value


def decode_image(cfg, im):
    """Oracle decode of a workload image: RD forward's x_hat -> 8-bit RGB."""
    r = rd_forward_image(cfg, im, want_xhat=True)
    return decode_u8(model(cfg), r["x_hat"]), r["x_hat"]


# -------------------------------------------------- N-O analysis (NEXT-4)
def analysis_model(acfg) -> OrcAnalysis:
    return OrcAnalysis(acfg.H, acfg.W, acfg.L, acfg.C, acfg.blocks)


def analysis_forward(acfg, image, weights):
    """Continuous latents (fp64, packed level after level) and the MAC count."""
    m = analysis_model(acfg)
    n_lat = sum(-(-acfg.H // (1 << l)) * -(-acfg.W // (1 << l)) for l in range(acfg.L))
    out = np.zeros(n_lat)
    macs = C.c_int64(0)
    img = _c(image, np.float32)
    w = _c(weights, np.float32)
    assert w.size == lib().orc_analysis_param_count(C.byref(m))
    rc = lib().orc_analysis_forward(C.byref(m), _p(img), _p(w), _p(out), C.byref(macs))
    if rc != 0:
        raise ValueError(f"orc_analysis_forward rc={rc}")
    return out, macs.value
