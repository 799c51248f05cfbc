"""Experiment artefacts of the paper's figures: radiance images,
the x5 difference image and the viridis hit-count heatmap.

Image I/O mirrors the reference's image.cpp byte for byte (write_pfm /
read_pfm / write_ppm / read_ppm, image.hpp:29-43): PFM little-endian with
scale -1.0 and rows bottom-to-top; binary PPM P6 maxval 255, input clamped to
[0, 1], optional 1/2.2 power before quantisation by lround(v * 255).
The heatmap maps the per-pixel average hits per sample through the canonical
256-entry viridis table over [0, 20] ("the color from black
to yellow in the viridis colormap represents 0 to 20 times"), written as a
linear PPM; the difference image is clamp(scale * |a - b|) (image_error,
tracer.hpp:72-80) written as a linear PPM.

Images are float32 arrays of shape (height, width, 3), row 0 at the top
(ImageF, image.hpp:11-21)."""
from __future__ import annotations

import json
import os
from typing import Union

import numpy as np

from ._native import ImageIoError

_HERE = os.path.dirname(os.path.abspath(__file__))
_MAX_DIM = 1 << 16


def _check_dims(width: int, height: int) -> None:
    # check_dims (image.cpp:13-18)
    if width <= 0 or height <= 0 or width > _MAX_DIM or height > _MAX_DIM:
        raise ImageIoError(f"image dimensions out of range: {width}x{height}")


def _as_image(img) -> np.ndarray:
    a = np.ascontiguousarray(img, np.float32)
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError(f"expected an (height, width, 3) image, got shape {a.shape}")
    return a


def write_pfm(path: str, img) -> None:
    """write_pfm (image.cpp:42-55)."""
    a = _as_image(img)
    h, w = a.shape[:2]
    _check_dims(w, h)
    try:
        with open(path, "wb") as f:
            f.write(f"PF\n{w} {h}\n-1.0\n".encode())
            f.write(a[::-1].astype("<f4").tobytes())
    except OSError as e:
        raise ImageIoError(f"cannot open for writing: {path}") from e


def _tokens(data: bytes, count: int):
    """The first `count` header tokens (whitespace-separated, '#' comments
    skipped, next_token in image.cpp:21-38) and the offset just past the
    single whitespace byte that ends the last one."""
    toks, i, n = [], 0, len(data)
    while len(toks) < count:
        while i < n:
            if data[i:i + 1] == b"#":
                while i < n and data[i:i + 1] != b"\n":
                    i += 1
            elif data[i:i + 1].isspace():
                i += 1
            else:
                break
        j = i
        while j < n and not data[j:j + 1].isspace():
            j += 1
        toks.append(data[i:j].decode(errors="replace"))
        i = j + 1  # next_token consumes the delimiter
    return toks, i


def read_pfm(path: str) -> np.ndarray:
    """read_pfm (image.cpp:57-76)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise ImageIoError(f"cannot open: {path}") from e
    (magic, ws, hs, ss), off = _tokens(data, 4)
    if magic != "PF":
        raise ImageIoError(f"not a color PFM file: {path}")
    w, h, scale = int(ws), int(hs), float(ss)
    _check_dims(w, h)
    if scale >= 0.0:
        raise ImageIoError(f"big-endian PFM not supported: {path}")
    need = w * h * 12
    if len(data) - off < need:
        raise ImageIoError(f"short read: {path}")
    a = np.frombuffer(data, "<f4", w * h * 3, off).reshape(h, w, 3)
    return np.ascontiguousarray(a[::-1]).astype(np.float32)


def write_ppm(path: str, img, gamma_encode: bool) -> None:
    """write_ppm (image.cpp:78-100): clamp, optional v^(1/2.2) in float,
    lround(v * 255)."""
    a = _as_image(img)
    h, w = a.shape[:2]
    _check_dims(w, h)
    v = np.fmin(np.fmax(a, np.float32(0.0)), np.float32(1.0))
    if gamma_encode:
        v = np.power(v, np.float32(1.0) / np.float32(2.2), dtype=np.float32)
    x = (v * np.float32(255.0)).astype(np.float32)          # the float product
    q = np.floor(x.astype(np.float64) + 0.5)                 # lround (x >= 0), exact in double
    try:
        with open(path, "wb") as f:
            f.write(f"P6\n{w} {h}\n255\n".encode())
            f.write(q.astype(np.uint8).tobytes())
    except OSError as e:
        raise ImageIoError(f"cannot open for writing: {path}") from e


def read_ppm(path: str) -> np.ndarray:
    """read_ppm (image.cpp:102-126): linear floats in [0, 1]."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise ImageIoError(f"cannot open: {path}") from e
    (magic, ws, hs, ms), off = _tokens(data, 4)
    if magic != "P6":
        raise ImageIoError(f"not a binary PPM file: {path}")
    w, h, maxval = int(ws), int(hs), int(ms)
    _check_dims(w, h)
    if maxval != 255:
        raise ImageIoError(f"unsupported PPM maxval: {maxval}")
    if len(data) - off < w * h * 3:
        raise ImageIoError(f"short read: {path}")
    b = np.frombuffer(data, np.uint8, w * h * 3, off).reshape(h, w, 3)
    return (b.astype(np.float32) / np.float32(255.0)).astype(np.float32)


# --------------------------------------------------------------------------
# viridis heatmap
# --------------------------------------------------------------------------

def _load_viridis() -> np.ndarray:
    with open(os.path.join(_HERE, "data", "viridis_u8.json")) as f:
        return np.asarray(json.load(f)["rgb"], np.float32) / np.float32(255.0)


VIRIDIS = _load_viridis()   # (256, 3) float32 in [0, 1]


def viridis(x) -> np.ndarray:
    """Canonical 256-entry viridis with linear interpolation; x clamped to
    [0, 1]. Returns (..., 3) float32."""
    t = np.clip(np.asarray(x, np.float64), 0.0, 1.0) * 255.0
    i0 = np.floor(t).astype(np.int64)
    i1 = np.minimum(i0 + 1, 255)
    f = (t - i0)[..., None]
    return (VIRIDIS[i0] * (1.0 - f) + VIRIDIS[i1] * f).astype(np.float32)


def heatmap(per_pixel_nodes_found, vmax: float = 20.0) -> np.ndarray:
    """Average cache hits per sample per pixel -> viridis over [0, vmax]."""
    v = np.asarray(per_pixel_nodes_found, np.float64)
    if v.ndim != 2:
        raise ValueError("per-pixel hit counts must be a (height, width) array")
    return viridis(v / vmax)


def write_heatmap(stats: Union[str, "object"], out_path: str, vmax: float = 20.0) -> np.ndarray:
    """cmd_heatmap: stats JSON text/path or a StatsFile
    -> linear PPM of the viridis heatmap. ValueError when the field is missing."""
    from . import parse_stats_json
    if isinstance(stats, str):
        text = stats
        if not stats.lstrip().startswith("{"):
            with open(stats) as f:
                text = f.read()
        stats = parse_stats_json(text)
    img = heatmap(np.asarray(stats.per_pixel_nodes_found).reshape(stats.height, stats.width), vmax)
    write_ppm(out_path, img, gamma_encode=False)
    return img


def write_diff(a, b, out_path: str, scale: float = 5.0):
    """cmd_diff: clamp(scale * |a - b|) as a linear PPM;
    returns image_error's DiffStats (mean_abs, max_abs, diff)."""
    from . import image_error
    d = image_error(a, b, scale)
    write_ppm(out_path, d.diff, gamma_encode=False)
    return d


def radiance_image(frame) -> np.ndarray:
    """FrameBuffers::radiance_image: accumulated radiance / samples, float32."""
    return frame.radiance_image()

