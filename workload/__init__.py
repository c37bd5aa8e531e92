"""Seeded synthetic workloads for the Cool-chic RD forward (shared by the oracle
side and the CUDA side; holds NONE of the method's arithmetic).

What lives here: the named configurations of BASELINE.json ``configs`` (layer
widths, sizes, value distributions), the context-template master list
(reading #4 of DESIGN.md), and numpy generators that draw, from a
seed, the integer latent pyramid, the fp32 decoder parameters and the RGB image.
Nothing here evaluates the ARM, the upsampling, the synthesis or the RD cost --
the oracle (``oracle/``) and the CUDA library (``paper_2403_11651_b200``) each
do that on their own.

Input recipe:
  * ``SeedSequence(seed).spawn(3)`` gives the image / latent / weight streams.
  * image: per channel, clip(0.5 + 0.5 * sum_s a_s c_{s,ch} sin(2pi(fx_s j/W +
    fy_s i/H) + phi_{s,ch}) / sum_s a_s + N(0, 0.02), 0, 1), 8 sinusoids,
    a_s ~ U(0,1), c ~ U(0.5,1), f ~ U(-16,16) cycles/image, phi ~ U(0, 2pi)
    (BASELINE.json configs[0]: "seeded sum of 8 random-frequency sinusoids plus
    N(0,0.02) noise, clipped").  The paper's Kodak / CLIC images are not in the
    container; these stand in for their shapes only.
  * latents: grid l has ceil(H/2^l) x ceil(W/2^l) entries, drawn
    i.i.d. Laplace(0, scale) (numpy scale parametrisation), rounded half-even,
    clipped to +-clip, stored int16, packed level after level, row-major.
  * weights: every ARM / synthesis weight and bias and every upsampling tap
    ~ N(0, 0.1) (standard deviation 0.1), fp32, drawn in blob order.  A
    ``filter_kind="lanczos2"`` variant replaces the 8 upsampling taps by the
    per-phase-normalised Lanczos-2 filter so every level carries O(1) signal
    (SURVEY.md §8c parity input (b)).
"""
from __future__ import annotations

import dataclasses
from concurrent.futures import ThreadPoolExecutor
from typing import List, Optional

import numpy as np

# nearest-causal-first master list of (dy, dx) context offsets.
# The paper's Fig. 2 (which would show the template) is missing from PAPER.md
# (PAPER.md:84-89); reading #4 adopts the first C entries of this list.
MASTER_CTX = [
    (0, -1), (0, -2), (-1, 0), (-1, -1), (-1, 1), (-1, -2), (-1, 2), (0, -3),
    (-2, 0), (-2, -1), (-2, 1), (-1, -3), (-1, 3), (-2, -2), (-2, 2), (-2, -3),
    (-2, 3), (-3, 0), (-3, -1), (-3, 1), (-3, -2), (-3, 2), (0, -4), (-1, -4),
]

# Per-phase-normalised Lanczos-2 8-tap filter (SURVEY.md §8c parity input (b)):
# each polyphase half (odd taps / even taps) sums to 1.
LANCZOS2_8 = np.array([-0.017726664, -0.083880068, 0.233000189, 0.868606543,
                       0.868606543, 0.233000189, -0.083880068, -0.017726664],
                      dtype=np.float32)


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration (architecture + input distribution)."""
    name: str
    H: int
    W: int
    L: int
    n_ctx: int
    arm_widths: tuple          # (n_ctx, hidden..., 2)      Table 1 ARM column
    syn_widths: tuple          # (L, C_h..., 3)             Table 1 synthesis 1x1 layers
    syn_n_res: int             # residual 3x3 3->3 layers   Table 1 "3-3-ConvR-3"
    up_taps: int = 8           # shared separable k (x) k   BASELINE.json configs[0]
    up_2d: bool = False        # Table 1 non-separable K x K TConv (NEXT-1): up_w has K*K taps
    lat_scale: float = 1.0
    lat_clip: int = 16
    lam: float = 1e-3
    n_img: int = 1
    logscale_min: float = float(np.log(1e-3))   # SPEC.md:223 (reading #2)
    logscale_max: float = float(np.log(256.0))
    p_floor: float = 2.0 ** -16                  # BASELINE.json configs[0] (reading #3)

    @property
    def ctx(self):
        return MASTER_CTX[: self.n_ctx]

    @property
    def arm_residual(self):
        """Reading #7: layer k is residual (Table 1 "LinR") iff in == out and k is
        not the module's last layer."""
        w = self.arm_widths
        n = len(w) - 1
        return tuple(int(w[k] == w[k + 1] and k < n - 1) for k in range(n))

    def level_dims(self):
        """ceil(H/2^l) x ceil(W/2^l) -- sizes only, used to shape
        the generated latent arrays."""
        return [(-(-self.H // (1 << l)), -(-self.W // (1 << l))) for l in range(self.L)]

    @property
    def n_latents(self):
        return sum(h * w for h, w in self.level_dims())

    @property
    def n_arm_w(self):
        w = self.arm_widths
        return sum(w[k] * w[k + 1] + w[k + 1] for k in range(len(w) - 1))

    @property
    def n_up_w(self):
        return self.up_taps * self.up_taps if self.up_2d else self.up_taps

    @property
    def n_syn_w(self):
        w = self.syn_widths
        return (sum(w[k] * w[k + 1] + w[k + 1] for k in range(len(w) - 1))
                + self.syn_n_res * (81 + 3))

    def replace(self, **kw):
        return dataclasses.replace(self, **kw)


# BASELINE.json "configs" (indices in comments).
CONFIGS = {
    # [0] Tiny
    "tiny": Config("tiny", 64, 64, 4, 8, (8, 8, 8, 2), (4, 8, 3), 1,
                   lat_scale=1.5, lat_clip=8),
    # [1] Low-complexity (~300 MAC/pixel by name; 559.3 by its explicit widths)
    "low": Config("low", 512, 768, 7, 8, (8, 8, 8, 2), (7, 16, 3), 2),
    # [2] Reference complexity (~2000 MAC/pixel)
    "ref": Config("ref", 512, 768, 7, 16, (16, 24, 24, 2), (7, 40, 3), 2),
    # [3] Batched 2K: 64 images of 1365x2048 at the ~2000 config
    "batched2k": Config("batched2k", 1365, 2048, 7, 16, (16, 24, 24, 2), (7, 40, 3), 2,
                        n_img=64),
    # [4] Single large image 4320x7680 at the ~2000 config
    "8k": Config("8k", 4320, 7680, 7, 16, (16, 24, 24, 2), (7, 40, 3), 2),
}

# Table 1 exact architectures (NEXT-1): ARM with C = width
# of its first layer, 2-D non-separable TConv-K upsampling, synthesis widths.
TABLE1 = {
    300: dict(arm=(8, 8, 2), up_kernel=4, syn=(7, 8, 3), syn_n_res=1),
    545: dict(arm=(8, 8, 8, 2), up_kernel=4, syn=(7, 16, 3), syn_n_res=2),
    1079: dict(arm=(16, 16, 16, 2), up_kernel=4, syn=(7, 16, 3), syn_n_res=2),
    2300: dict(arm=(24, 24, 24, 2), up_kernel=8, syn=(7, 40, 3), syn_n_res=2),
}

# ... as workload configs on Kodak-sized synthetic images (512 x 768, L = 7;
# PAPER.md:347 "768 x 512"), the value distributions of configs[1]/[2].
for _k, _a in TABLE1.items():
    CONFIGS[f"t{_k}"] = Config(f"t{_k}", 512, 768, 7, _a["arm"][0], _a["arm"], _a["syn"], _a["syn_n_res"],
                               up_taps=_a["up_kernel"], up_2d=True)


@dataclasses.dataclass
class Image:
    """One image's inputs: packed latents, fp32 blobs, planar RGB fp32 image."""
    latents: np.ndarray      # int16 [N_lat], levels 0..L-1 packed row-major
    arm_w: np.ndarray        # fp32 blob, per layer W[out][in] then b[out]
    up_w: np.ndarray         # fp32 [taps]
    syn_w: np.ndarray        # fp32 blob: 1x1 A[out][in], a[out]; then per res 3x3 G[co][ci][ky][kx], g[co]
    image: np.ndarray        # fp32 [3, H, W] in [0, 1]
    seed: int = 0

    def level(self, cfg: Config, l: int) -> np.ndarray:
        dims = cfg.level_dims()
        off = sum(h * w for h, w in dims[:l])
        h, w = dims[l]
        return self.latents[off: off + h * w].reshape(h, w)


def _streams(seed: int):
    ss = np.random.SeedSequence(seed)
    return [np.random.default_rng(s) for s in ss.spawn(3)]


def gen_image(rng: np.random.Generator, H: int, W: int) -> np.ndarray:
    """Seeded sum of 8 random-frequency sinusoids + N(0, 0.02) noise, clipped to
    [0, 1] (BASELINE.json configs[0]).  Evaluated with the angle-sum identity so
    large images generate quickly; fp32 output, planar [3, H, W]."""
    S = 8
    a = rng.uniform(0.0, 1.0, S)
    c = rng.uniform(0.5, 1.0, (S, 3))
    fx = rng.uniform(-16.0, 16.0, S)
    fy = rng.uniform(-16.0, 16.0, S)
    phi = rng.uniform(0.0, 2 * np.pi, (S, 3))
    jj = np.arange(W, dtype=np.float64) / W
    ii = np.arange(H, dtype=np.float64) / H
    out = np.empty((3, H, W), dtype=np.float32)
    for ch in range(3):
        acc = np.zeros((H, W), dtype=np.float64)
        for s in range(S):
            ax = 2 * np.pi * fx[s] * jj + phi[s, ch]        # [W]
            by = 2 * np.pi * fy[s] * ii                     # [H]
            # sin(ax + by) = sin(ax)cos(by) + cos(ax)sin(by)
            acc += (a[s] * c[s, ch]) * (np.outer(np.cos(by), np.sin(ax)) + np.outer(np.sin(by), np.cos(ax)))
        val = 0.5 + 0.5 * acc / a.sum() + rng.normal(0.0, 0.02, (H, W))
        out[ch] = np.clip(val, 0.0, 1.0).astype(np.float32)
    return out


def to_u8(img: np.ndarray) -> np.ndarray:
    """8-bit planes of an image in [0, 1] (the paper's sources are 8-bit RGB):
    v = rint(255 x), clipped.  A storage format, not method arithmetic."""
    return np.clip(np.rint(np.asarray(img, np.float64) * 255.0), 0, 255).astype(np.uint8)


def from_u8(v: np.ndarray) -> np.ndarray:
    """x = v / 255 in fp32 (IEEE division) -- the value the kernels read for
    desc.image_u8 = 1; the oracle is fed this image."""
    return np.asarray(v, np.uint8).astype(np.float32) / np.float32(255.0)


def quantize_image_u8(img: np.ndarray) -> np.ndarray:
    """An fp32 image whose values are exactly representable as 8-bit levels."""
    return from_u8(to_u8(img))


def gen_latents(rng: np.random.Generator, cfg: Config) -> np.ndarray:
    """i.i.d. rounded Laplace(0, lat_scale) clipped to +-lat_clip, int16, packed
    level by level (BASELINE.json configs[0]/[1]; reading #20)."""
    parts = []
    for h, w in cfg.level_dims():
        v = np.rint(rng.laplace(0.0, cfg.lat_scale, (h, w)))
        parts.append(np.clip(v, -cfg.lat_clip, cfg.lat_clip).astype(np.int16).ravel())
    return np.concatenate(parts)


def gen_weights(rng: np.random.Generator, cfg: Config, filter_kind: str = "random"):
    """fp32 blobs drawn N(0, 0.1) in blob order: ARM, upsampling taps, synthesis."""
    arm_w = rng.normal(0.0, 0.1, cfg.n_arm_w).astype(np.float32)
    up_w = rng.normal(0.0, 0.1, cfg.n_up_w).astype(np.float32)
    syn_w = rng.normal(0.0, 0.1, cfg.n_syn_w).astype(np.float32)
    if filter_kind == "lanczos2":
        if cfg.up_taps != 8:
            raise ValueError("lanczos2 filter is 8 taps")
        up_w = LANCZOS2_8.copy()
    elif filter_kind == "bilinear":
        up_w = (np.array([0, 0, .25, .75, .75, .25, 0, 0], np.float32) if cfg.up_taps == 8
                else np.array([.25, .75, .75, .25], np.float32))
    elif filter_kind == "normalised2d":
        # a NON-separable K x K kernel whose four polyphase components
        # (rows a = 2t+1-r, columns b = 2u+1-s) each sum to 1, so every level
        # carries O(1) signal: bilinear (x) bilinear plus seeded noise,
        # renormalised per phase
        k1 = (np.array([0, 0, .25, .75, .75, .25, 0, 0]) if cfg.up_taps == 8 else np.array([.25, .75, .75, .25]))
        k2 = np.outer(k1, k1) + rng.normal(0.0, 0.05, (cfg.up_taps, cfg.up_taps))
        for ra in (0, 1):
            for sb in (0, 1):
                k2[ra::2, sb::2] /= k2[ra::2, sb::2].sum()
        up_w = k2.astype(np.float32).ravel()
    elif filter_kind != "random":
        raise ValueError(filter_kind)
    if cfg.up_2d and filter_kind in ("lanczos2", "bilinear"):
        up_w = np.outer(up_w, up_w).astype(np.float32).ravel()  # separable special case k (x) k
    if filter_kind == "normalised2d" and not cfg.up_2d:
        raise ValueError("normalised2d needs up_2d")
    return arm_w, up_w, syn_w


def gen_noise(rng: np.random.Generator, n: int) -> np.ndarray:
    """Training-proxy noise u ~ U(-1/2, 1/2) (reading T1),
    fp32: the random numbers of the training iteration are INPUT data."""
    return rng.uniform(-0.5, 0.5, n).astype(np.float32)


def gen_continuous_latents(rng: np.random.Generator, latents_int: np.ndarray) -> np.ndarray:
    """A training state's continuous latents y: the integer draw plus a seeded
    offset in (-1/2, 1/2) (fp32)."""
    return (latents_int.astype(np.float64) + rng.uniform(-0.49, 0.49, latents_int.size)).astype(np.float32)


def make_image(cfg: Config, seed: int, filter_kind: str = "random") -> Image:
    r_img, r_lat, r_w = _streams(seed)
    img = gen_image(r_img, cfg.H, cfg.W)
    lat = gen_latents(r_lat, cfg)
    arm_w, up_w, syn_w = gen_weights(r_w, cfg, filter_kind)
    return Image(lat, arm_w, up_w, syn_w, img, seed)


def make_batch(cfg: Config, seeds: List[int], filter_kind: str = "random",
               threads: Optional[int] = None) -> List[Image]:
    """Generate several images in parallel (numpy releases the GIL)."""
    if len(seeds) <= 1:
        return [make_image(cfg, s, filter_kind) for s in seeds]
    with ThreadPoolExecutor(max_workers=threads or min(16, len(seeds))) as ex:
        return list(ex.map(lambda s: make_image(cfg, s, filter_kind), seeds))


def image_seed(base: int, index: int) -> int:
    """Per-image seed: SeedSequence(base + image_index)."""
    return base + index


# ------------------------------------------------ N-O analysis (NEXT-4)
@dataclasses.dataclass(frozen=True)
class AnalysisConfig:
    """N-O Cool-chic analysis transform (readings A1-A7 of
    DESIGN.md): L grids, C features, `blocks` ConvNeXt-style blocks per level."""
    name: str
    H: int
    W: int
    L: int = 7
    C: int = 64
    blocks: int = 3

    def replace(self, **kw):
        return dataclasses.replace(self, **kw)

    @property
    def n_params(self):
        C = self.C
        blk = C * 49 + C + 4 * C * C + 4 * C + 4 * C * C + C
        n = C * 3 + C
        for l in range(self.L):
            n += self.blocks * blk + (C * C + C if l > 0 else 0) + C + 1
        return n


ANALYSIS = {
    "no_tiny": AnalysisConfig("no_tiny", 37, 53, L=4, C=8, blocks=2),
    "no_kodak": AnalysisConfig("no_kodak", 512, 768),
    "no_2k": AnalysisConfig("no_2k", 1365, 2048),
}


def gen_analysis_weights(rng: np.random.Generator, acfg: AnalysisConfig) -> np.ndarray:
    """Seeded fp32 blob in the oracle's order, variance-preserving scales (the
    paper's weights are trained; these only keep 3L residual blocks bounded):
    dw ~ N(0, 1/7), W1 ~ N(0, 1/sqrt(C)), W2 ~ N(0, 0.3/sqrt(4C)), identity and
    stem ~ N(0, 1/sqrt(fan_in)), merge ~ N(0, 1/sqrt(C)), biases ~ N(0, 0.02)."""
    C = acfg.C
    parts = [rng.normal(0, 1 / np.sqrt(3), C * 3), rng.normal(0, 0.02, C)]
    for l in range(acfg.L):
        for b in range(acfg.blocks):
            parts += [rng.normal(0, 1 / 7, C * 49), rng.normal(0, 0.02, C),
                      rng.normal(0, 1 / np.sqrt(C), 4 * C * C), rng.normal(0, 0.02, 4 * C),
                      rng.normal(0, 0.3 / np.sqrt(4 * C), 4 * C * C), rng.normal(0, 0.02, C)]
            if l > 0 and b == 0:
                parts += [rng.normal(0, 1 / np.sqrt(C), C * C), rng.normal(0, 0.02, C)]
        parts += [rng.normal(0, 1 / np.sqrt(C), C), rng.normal(0, 0.02, 1)]
    w = np.concatenate(parts).astype(np.float32)
    assert w.size == acfg.n_params
    return w


def make_analysis_input(acfg: AnalysisConfig, seed: int):
    """(image [3][H][W] fp32 -- the sinusoid recipe of configs[0] --, weights)."""
    r_img, _, r_w = _streams(seed)
    return gen_image(r_img, acfg.H, acfg.W), gen_analysis_weights(r_w, acfg)
