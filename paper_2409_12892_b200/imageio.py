"""Image interchange (ref: imageio.py:7-41).

PFM is the lossless float format the reference uses to hand images (ground
truth, renders) between tools: "PF" header, "W H", scale -1.0 (little-endian),
then float32 RGB rows stored bottom to top.  `write_pfm` produces the same
bytes as the reference's writer; `read_pfm` returns float64 like the
reference's reader (or a device tensor when `device` is given).  PNG previews
clamp to [0, 1] and quantise with round-half-up, as the reference does.

Images are (H, W, 3) numpy arrays or torch tensors (device tensors are copied
to the host first).
"""

from __future__ import annotations

import numpy as np
import torch


def _host(image) -> np.ndarray:
    if isinstance(image, torch.Tensor):
        image = image.detach().cpu().numpy()
    return np.asarray(image)


def write_pfm(path, image) -> None:
    """(H, W, 3) float image -> little-endian RGB PFM (ref: imageio.py:7-18)."""
    img = _host(image).astype(np.float32)
    if img.ndim != 3 or img.shape[2] != 3:
        raise ValueError(f"expected (H, W, 3) image, got shape {img.shape}")
    h, w = img.shape[:2]
    body = np.flipud(img).astype("<f4", copy=False)
    with open(path, "wb") as f:
        f.write(b"PF\n" + f"{w} {h}\n".encode("ascii") + b"-1.0\n")
        f.write(np.ascontiguousarray(body).tobytes())


def read_pfm(path, device=None):
    """RGB PFM -> (H, W, 3) float64 (ref: imageio.py:21-30); a torch tensor on
    `device` when one is given."""
    with open(path, "rb") as f:
        if f.readline().strip() != b"PF":
            raise ValueError(f"not a color PFM file: {path}")
        w, h = (int(t) for t in f.readline().split())
        scale = float(f.readline())
        raw = f.read(w * h * 3 * 4)
    arr = np.frombuffer(raw, dtype="<f4" if scale < 0 else ">f4").reshape(h, w, 3)
    out = np.flipud(arr).astype(np.float64)
    if device is not None:
        return torch.from_numpy(np.ascontiguousarray(out)).to(device)
    return out


def write_png(path, image) -> None:
    """8-bit PNG preview: clamp to [0, 1], x255, round half up (ref: imageio.py:33-36)."""
    from PIL import Image
    arr = np.clip(_host(image).astype(np.float64), 0.0, 1.0)
    Image.fromarray(np.floor(arr * 255.0 + 0.5).astype(np.uint8)).save(path)


def read_png(path) -> np.ndarray:
    """PNG -> (H, W, 3) float64 in [0, 1] (ref: imageio.py:39-41)."""
    from PIL import Image
    return np.asarray(Image.open(path).convert("RGB"), dtype=np.float64) / 255.0
