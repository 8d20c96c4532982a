"""numpy restatement of the BASELINE.json cube generator (csrc/synth.cu).

TEST / BENCH INFRASTRUCTURE ONLY (see oracle/__init__.py).  The device
generator ``ut_synth_cube`` writes every sample of a cube from a counter hash
of (seed, pixel, band); this module produces the same samples on the host,
bit for bit, for any set of pixels:

* the reference arm of ``bench.py`` (``--impl reference``) builds its bounded
  sample (the training pixels plus a block of rows) here, so that arm never
  maps the repo's CUDA library;
* ``tests/test_gpu_synth.py`` checks device == host bit for bit.

Bit equality holds because synth.cu performs every floating-point step as one
binary32 IEEE operation with round-to-nearest (``__fadd_rn`` / ``__fmul_rn`` /
``__fdiv_rn`` / ``__fsqrt_rn``, no contraction into FMA) and this module
performs the same operations, in the same order, on numpy float32 arrays; the
constants are the same binary32 bit patterns (hex literals there,
``float.fromhex`` here), and the uniforms are small integers times 2^-24
(exact).  The scene (class means, Cholesky factors, shapes, training points)
comes from ``paper_1612_06457_b200.synthetic.make_scene`` (host numpy).
"""

from __future__ import annotations

import numpy as np

F = np.float32
_U64 = np.uint64


def _h(s: str) -> np.float32:
    return F(float.fromhex(s))


# binary32 constants of synth.cu (synth_log / synth_sincos_q)
SQRT_HALF = _h("0x1.6a09e6p-1")
LN2 = _h("0x1.62e43p-1")
LOG_P = [_h("0x1.c71c72p-3"), _h("0x1.24924ap-2"), _h("0x1.99999ap-2"), _h("0x1.555556p-1")]
PI_2 = _h("0x1.921fb6p+0")
SIN_P = [_h("-0x1.612462p-33"), _h("0x1.ae6456p-26"), _h("-0x1.71de3ap-19"),
         _h("0x1.a01a02p-13"), _h("-0x1.111112p-7"), _h("0x1.555556p-3")]
COS_P = [_h("-0x1.93974ap-37"), _h("0x1.1eed8ep-29"), _h("-0x1.27e4fcp-22"),
         _h("0x1.a01a02p-16"), _h("-0x1.6c16c2p-10"), _h("0x1.555556p-5"), F(-0.5)]
TWO_M24 = F(2.0 ** -24)
MAX_BANDS = 32


def device_seed(cfg_seed: int) -> int:
    """The 64-bit generator seed synthetic.generate passes to ut_synth_cube."""
    return (int(cfg_seed) * 0x9E3779B1 + 17) & 0xFFFFFFFFFFFFFFFF


def splitmix64(z: np.ndarray) -> np.ndarray:
    """synth.cu splitmix64 on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = z + _U64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
    return z ^ (z >> _U64(31))


def synth_log(u: np.ndarray) -> np.ndarray:
    """synth.cu synth_log, u in (0, 1] float32."""
    bits = u.view(np.int32)
    e = ((bits >> 23) & 0xFF) - 126
    m = ((bits & 0x007FFFFF) | (126 << 23)).astype(np.int32).view(F)
    low = m < SQRT_HALF
    m = np.where(low, m * F(2.0), m)
    e = np.where(low, e - 1, e)
    f = m + F(-1.0)
    s = f / (f + F(2.0))
    s2 = s * s
    p = LOG_P[0]
    for c in LOG_P[1:]:
        p = c + s2 * p
    lnm = F(2.0) * s + s * (s2 * p)
    return e.astype(F) * LN2 + lnm


def synth_sincos_q(a: np.ndarray):
    """synth.cu synth_sincos_q: sin, cos of a pi/2, a in [0, 1)."""
    x = a * PI_2
    x2 = x * x
    ps = np.full_like(x, SIN_P[0])
    for c in SIN_P[1:]:
        ps = c + x2 * ps
    s = x + -(x * (x2 * ps))
    pc = np.full_like(x, COS_P[0])
    for c in COS_P[1:]:
        pc = c + x2 * pc
    c = F(1.0) + x2 * pc
    return s, c


def normal_pair(h: np.ndarray):
    """synth.cu synth_normal_pair: two normals per 64-bit hash."""
    u1 = (_U64(2) * (h >> _U64(41)) + _U64(1)).astype(F) * TWO_M24
    u2 = (h & _U64(0xFFFFFF)).astype(F) * TWO_M24
    r = np.sqrt(F(-2.0) * synth_log(u1))
    t = u2 * F(4.0)
    q = np.floor(t)
    s, c = synth_sincos_q(t - q)
    qi = q.astype(np.int64) & 3
    sn = np.select([qi == 0, qi == 1, qi == 2], [s, c, -s], -c)
    cs = np.select([qi == 0, qi == 1, qi == 2], [c, -s, -c], s)
    return r * cs, r * sn


def class_at(shapes: np.ndarray, ys, xs) -> np.ndarray:
    """synth.cu class_at: last shape containing the pixel wins, else class 0."""
    ys = np.asarray(ys, dtype=np.int64)
    xs = np.asarray(xs, dtype=np.int64)
    out = np.zeros(np.broadcast(ys, xs).shape, dtype=np.int32)
    for kind, cls, a, b, c, d in np.asarray(shapes, dtype=np.int64).tolist():
        if kind == 0:
            inside = (ys >= a) & (xs >= b) & (ys < c) & (xs < d)
        else:
            dy, dx = ys - a, xs - b
            inside = (dy * d) ** 2 + (dx * c) ** 2 <= (c * d) ** 2
        out[inside] = cls
    return out


def _cast(v: np.ndarray, dtype) -> np.ndarray:
    dtype = np.dtype(dtype)
    if dtype == np.float32:
        return v
    if dtype == np.float64 or dtype == np.float16:
        return v.astype(dtype)
    if dtype == np.uint16:
        return np.floor(F(4095.0) * v + F(0.5)).astype(np.uint16)
    if dtype == np.uint8:
        return np.floor(F(255.0) * v + F(0.5)).astype(np.uint8)
    raise ValueError(f"unsupported sample type {dtype}")


def pixels(scene, ys, xs, dtype=None) -> np.ndarray:
    """(B, n) samples of the scene's cube at global pixels (ys[i], xs[i])."""
    cfg = scene.cfg
    b = cfg.bands
    ys = np.asarray(ys, dtype=np.int64).ravel()
    xs = np.asarray(xs, dtype=np.int64).ravel()
    n = ys.size
    gpix = ys.astype(_U64) * _U64(cfg.width) + xs.astype(_U64)
    seed = _U64(device_seed(cfg.seed))
    z = np.empty((MAX_BANDS, n), dtype=F)
    with np.errstate(over="ignore"):
        base = gpix * _U64(0x100000001B3)
        for q in range(0, MAX_BANDS, 2):
            z[q], z[q + 1] = normal_pair(splitmix64(seed ^ (base + _U64(q))))
    cls = class_at(scene.shapes, ys, xs)
    mu = scene.means.astype(F)
    L = scene.chol.astype(F)
    out = np.empty((b, n), dtype=F)
    for c in np.unique(cls).tolist():
        sel = np.flatnonzero(cls == c)
        zc = z[:, sel] if sel.size != n else z
        v = np.empty(sel.size, dtype=F)
        tmp = np.empty(sel.size, dtype=F)
        for band in range(b):
            v.fill(mu[c, band])
            for q in range(band + 1):   # v = v + L[b, q] z[q], one rounding each
                np.multiply(zc[q], L[c, band, q], out=tmp)
                np.add(v, tmp, out=v)
            np.clip(v, F(0.0), F(1.0), out=v)
            out[band, sel] = v
    return _cast(out, dtype if dtype is not None else _np_dtype(cfg))


def _np_dtype(cfg):
    name = str(cfg.dtype).replace("torch.", "")
    return np.dtype(name)


def _rows_block(args):
    scene, a, b_, dt = args
    w = scene.cfg.width
    yy, xx = np.meshgrid(np.arange(a, b_), np.arange(w), indexing="ij")
    return pixels(scene, yy, xx, dt).reshape(scene.cfg.bands, b_ - a, w)


def rows(scene, r0: int, r1: int, procs: int = 1, dtype=None) -> np.ndarray:
    """(B, r1 - r0, W) block of the scene's cube.  ``procs`` > 1 splits the rows
    over forked worker processes (numpy's many small float32 operations keep
    threads serialized on the GIL); only call it that way from a process that
    has not initialised CUDA."""
    cfg = scene.cfg
    dt = dtype if dtype is not None else _np_dtype(cfg)
    out = np.empty((cfg.bands, r1 - r0, cfg.width), dtype=dt)
    step = 4
    spans = [(a, min(a + step, r1)) for a in range(r0, r1, step)]
    if procs <= 1:
        for a, b_ in spans:
            out[:, a - r0:b_ - r0] = _rows_block((scene, a, b_, dt))
        return out
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    with ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("fork")) as pool:
        for (a, b_), blk in zip(spans, pool.map(_rows_block,
                                                [(scene, a, b_, dt) for a, b_ in spans],
                                                chunksize=4)):
            out[:, a - r0:b_ - r0] = blk
    return out
