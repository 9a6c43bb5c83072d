"""Field renders and report figures (drop-in for
/root/reference/pkg/src/ptychokit/render.py).

``render`` writes the reference's 16-bit grayscale PNG of a field's magnitude
or phase with the JSON scaling sidecar (render.py:25-44), so ``load_render``
maps pixels back to physical values.  The report figures (error trace, scan
positions, registration benchmark) are drawn with matplotlib when it is
installed; without it (this image) they are rasterised directly with Pillow
-- the same files, simpler drawings.  Host-side reporting, not the hot path.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .errors import ParameterError

_U16_MAX = 65535


def _host(a) -> np.ndarray:
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(a)


def render(field, kind: str, path) -> Path:
    """render.py:25-44: 16-bit grayscale PNG plus a ``<path>.json`` scaling sidecar."""
    from PIL import Image
    f = _host(field)
    if kind == "magnitude":
        img = np.abs(f).astype(float)
        vmin, vmax = float(img.min()), float(img.max())
    elif kind == "phase":
        img = np.angle(f)
        vmin, vmax = -np.pi, np.pi
    else:
        raise ParameterError(f"kind must be 'magnitude' or 'phase', got {kind!r}")
    span = vmax - vmin
    scaled = (img - vmin) / span if span > 0 else np.zeros_like(img)
    png = np.round(scaled * _U16_MAX).astype(np.uint16)
    path = Path(path)
    Image.fromarray(png).save(path)
    sidecar = {"kind": kind, "vmin": vmin, "vmax": vmax, "levels": _U16_MAX, "shape": list(f.shape)}
    Path(str(path) + ".json").write_text(json.dumps(sidecar, indent=2))
    return path


def load_render(path):
    """render.py:47-53: pixels back to physical values via the sidecar."""
    from PIL import Image
    path = Path(path)
    sidecar = json.loads(Path(str(path) + ".json").read_text())
    png = np.asarray(Image.open(path), dtype=float)
    values = sidecar["vmin"] + png / sidecar["levels"] * (sidecar["vmax"] - sidecar["vmin"])
    return values, sidecar


# ---------------------------------------------------------------- figures --

def _mpl():
    try:
        import matplotlib
        matplotlib.use("Agg")
        import matplotlib.pyplot as plt
        return plt
    except ImportError:
        return None


class _Canvas:
    """Minimal raster plot (Pillow) used when matplotlib is absent."""

    def __init__(self, xs, ys, size=(640, 480), logy=False):
        from PIL import Image, ImageDraw
        self.img = Image.new("RGB", size, "white")
        self.draw = ImageDraw.Draw(self.img)
        self.w, self.h = size
        self.logy = logy
        xs = np.asarray(xs, float)
        ys = np.asarray(ys, float)
        if logy:
            ys = np.log10(np.maximum(ys, 1e-300))
        self.x0, self.x1 = (float(xs.min()), float(xs.max())) if xs.size else (0.0, 1.0)
        self.y0, self.y1 = (float(ys.min()), float(ys.max())) if ys.size else (0.0, 1.0)
        if self.x1 == self.x0:
            self.x1 = self.x0 + 1.0
        if self.y1 == self.y0:
            self.y1 = self.y0 + 1.0
        self.draw.rectangle([40, 20, self.w - 20, self.h - 40], outline="black")

    def _xy(self, x, y):
        if self.logy:
            y = np.log10(max(float(y), 1e-300))
        px = 40 + (float(x) - self.x0) / (self.x1 - self.x0) * (self.w - 60)
        py = self.h - 40 - (float(y) - self.y0) / (self.y1 - self.y0) * (self.h - 60)
        return px, py

    def line(self, xs, ys, color="blue"):
        pts = [self._xy(x, y) for x, y in zip(xs, ys)]
        if len(pts) > 1:
            self.draw.line(pts, fill=color, width=2)
        elif pts:
            self.points(xs, ys, color)

    def points(self, xs, ys, color="blue", r=2):
        for x, y in zip(xs, ys):
            px, py = self._xy(x, y)
            self.draw.ellipse([px - r, py - r, px + r, py + r], outline=color)

    def save(self, path):
        self.img.save(path)


def plot_error_trace(trace, path) -> Path:
    """render.py:56-66: normalised intensity error per iteration (log scale)."""
    path = Path(path)
    trace = [float(t) for t in trace]
    it = np.arange(1, len(trace) + 1)
    plt = _mpl()
    if plt is not None:
        fig, ax = plt.subplots(figsize=(6, 4))
        ax.semilogy(it, trace)
        ax.set_xlabel("iteration")
        ax.set_ylabel("normalized intensity error")
        fig.tight_layout()
        fig.savefig(path, dpi=120)
        plt.close(fig)
        return path
    c = _Canvas(it if len(it) else [0], trace if trace else [1.0], logy=True)
    c.line(it, trace)
    c.save(path)
    return path


def plot_positions(nominal, refined, path, truth=None) -> Path:
    """render.py:69-88: nominal, refined (and true) scan positions."""
    path = Path(path)
    nominal, refined = _host(nominal), _host(refined)
    truth = None if truth is None else _host(truth)
    plt = _mpl()
    if plt is not None:
        fig, ax = plt.subplots(figsize=(5, 5))
        ax.scatter(nominal[:, 0], nominal[:, 1], s=8, label="nominal")
        ax.scatter(refined[:, 0], refined[:, 1], s=8, label="refined")
        if truth is not None:
            ax.scatter(truth[:, 0], truth[:, 1], s=8, label="truth")
        ax.set_aspect("equal")
        ax.invert_yaxis()
        ax.legend()
        fig.tight_layout()
        fig.savefig(path, dpi=120)
        plt.close(fig)
        return path
    allp = np.concatenate([p for p in (nominal, refined, truth) if p is not None])
    c = _Canvas(allp[:, 0], -allp[:, 1], size=(520, 520))
    c.points(nominal[:, 0], -nominal[:, 1], "blue")
    c.points(refined[:, 0], -refined[:, 1], "red")
    if truth is not None:
        c.points(truth[:, 0], -truth[:, 1], "green")
    c.save(path)
    return path


def plot_benchmark(rows, path) -> Path:
    """render.py:91-105: seconds per registration vs upsampling factor."""
    path = Path(path)
    plt = _mpl()
    methods = sorted({r["method"] for r in rows})
    if plt is not None:
        fig, ax = plt.subplots(figsize=(6, 4))
        for m in methods:
            sel = [r for r in rows if r["method"] == m]
            ax.loglog([r["kappa"] for r in sel], [r["seconds"] for r in sel], "o-", label=m)
        ax.set_xlabel("upsampling factor")
        ax.set_ylabel("seconds")
        ax.legend()
        fig.tight_layout()
        fig.savefig(path, dpi=120)
        plt.close(fig)
        return path
    ks = [r["kappa"] for r in rows] or [1]
    ts = [r["seconds"] for r in rows] or [1.0]
    c = _Canvas(ks, ts, logy=True)
    for m, color in zip(methods, ("blue", "red", "green", "black")):
        sel = [r for r in rows if r["method"] == m]
        c.line([r["kappa"] for r in sel], [r["seconds"] for r in sel], color)
    c.save(path)
    return path
