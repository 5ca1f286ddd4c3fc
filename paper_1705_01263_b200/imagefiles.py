"""Framebuffer output: PFM (bit-exact float32 interchange) as in imagefiles.py:26-57."""

from __future__ import annotations

import numpy as np

__all__ = ["write_pfm", "read_pfm"]


def write_pfm(path, image: np.ndarray) -> None:
    """(H, W, 3) float image -> little-endian colour PFM, rows stored bottom-up (imagefiles.py:26-38)."""
    img = np.asarray(image, dtype=np.float32)
    if img.ndim == 2:
        img = np.repeat(img[:, :, None], 3, axis=2)
    if img.ndim != 3 or img.shape[2] != 3:
        raise ValueError("PFM writer expects an (H, W, 3) array")
    h, w = img.shape[:2]
    header = b"PF\n" + f"{w} {h}\n".encode("ascii") + b"-1.0\n"
    with open(path, "wb") as f:
        f.write(header)
        f.write(np.ascontiguousarray(img[::-1], dtype="<f4").tobytes())


def read_pfm(path) -> np.ndarray:
    """PFM -> (H, W, 3) float32 (imagefiles.py:41-57)."""
    with open(path, "rb") as f:
        kind = f.readline().strip()
        if kind not in (b"PF", b"Pf"):
            raise ValueError(f"{path}: not a PFM file")
        w, h = (int(x) for x in f.readline().split())
        scale = float(f.readline().strip())
        ch = 3 if kind == b"PF" else 1
        data = np.frombuffer(f.read(4 * w * h * ch), dtype="<f4" if scale < 0 else ">f4", count=w * h * ch)
    img = data.reshape(h, w, ch)
    if ch == 1:
        img = np.repeat(img, 3, axis=2)
    img = img[::-1]
    if abs(scale) != 1.0:
        img = img * abs(scale)
    return np.ascontiguousarray(img, dtype=np.float32)
