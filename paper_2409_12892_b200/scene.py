"""Scene, camera and parameter-vector types on the device.

Mirrors ref: scene.py (GaussianScene 137-217, ParamVector 52-76, Layout
44-46, sort_x / sort_x_inverse 79-92, flatten / unflatten 220-258,
scene_with_offset 261-265, Camera 272-304, JSON IO 420-472).  The scene is
held as ONE attribute-major float64 device vector x[a * G + g] -- the layout
every product writes -- so flatten() is free and the LM
update is a single axpy.
"""

from __future__ import annotations

import enum
import json
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .errors import LayoutError

GEOM_PARAMS = 11
POS_SLICE = slice(0, 3)
ROT_SLICE = slice(3, 7)
SCALE_SLICE = slice(7, 10)
OPACITY_INDEX = 10
SH_START = 11


def num_coefficients(degree: int) -> int:
    if degree not in (0, 1, 2, 3):
        raise ValueError(f"SH degree must be in 0..3, got {degree}")
    return (degree + 1) ** 2


def params_per_gaussian(sh_degree: int) -> int:
    return GEOM_PARAMS + 3 * num_coefficients(sh_degree)


def default_device():
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")


class Layout(enum.Enum):
    ATTRIBUTE_MAJOR = "attribute_major"
    GAUSSIAN_MAJOR = "gaussian_major"


@dataclass(frozen=True)
class ParamVector:
    """Flat parameter vector with an explicit layout tag (ref: scene.py:52-76).

    `values` is a 1-D device tensor (float32 or float64)."""

    values: torch.Tensor
    layout: Layout
    gaussian_count: int
    params_per_gaussian: int

    def __post_init__(self):
        expected = self.gaussian_count * self.params_per_gaussian
        if tuple(self.values.shape) != (expected,):
            raise ValueError(f"expected vector of length {expected}, got shape {tuple(self.values.shape)}")

    def __len__(self) -> int:
        return int(self.values.shape[0])

    def with_values(self, values: torch.Tensor) -> "ParamVector":
        return replace(self, values=values)

    def require_layout(self, layout: Layout) -> None:
        if self.layout is not layout:
            raise LayoutError(f"expected {layout.value} vector, got {self.layout.value}")

    def numpy(self) -> np.ndarray:
        return self.values.detach().double().cpu().numpy()


def _transpose(v: torch.Tensor, rows: int, cols: int) -> torch.Tensor:
    out = torch.empty_like(v)
    if v.is_cuda:
        fn = "slm_transpose_f64" if v.dtype == torch.float64 else "slm_transpose_f32"
        _lib.call(fn, _lib.ptr(v), _lib.ptr(out), rows, cols, _lib.stream_ptr())
    else:  # host-side layout change of a CPU tensor (not on the product path)
        out.copy_(v.view(rows, cols).t().reshape(-1))
    return out


def sort_x(v: ParamVector) -> ParamVector:
    """Attribute-major -> gaussian-major (sortX kernel)."""
    v.require_layout(Layout.ATTRIBUTE_MAJOR)
    g, p = v.gaussian_count, v.params_per_gaussian
    return ParamVector(_transpose(v.values.contiguous(), p, g), Layout.GAUSSIAN_MAJOR, g, p)


def sort_x_inverse(v: ParamVector) -> ParamVector:
    v.require_layout(Layout.GAUSSIAN_MAJOR)
    g, p = v.gaussian_count, v.params_per_gaussian
    return ParamVector(_transpose(v.values.contiguous(), g, p), Layout.ATTRIBUTE_MAJOR, g, p)


class GaussianScene:
    """Immutable scene: attribute-major float64 device vector + SH degree +
    background (ref: scene.py:137-217)."""

    def __init__(self, x: torch.Tensor, sh_degree: int, background=(0.0, 0.0, 0.0)):
        P = params_per_gaussian(sh_degree)
        if x.dim() != 1 or x.numel() % P != 0:
            raise ValueError(f"parameter vector length {x.numel()} is not a multiple of {P}")
        self.x = x if x.dtype == torch.float64 else x.double()
        self.sh_degree = int(sh_degree)
        self.background = np.asarray(background, dtype=np.float64).reshape(3)
        self._x32 = None

    @classmethod
    def from_arrays(cls, positions, rotations, log_scales, opacity_logits, sh_coeffs, sh_degree,
                    background=(0.0, 0.0, 0.0), device=None) -> "GaussianScene":
        pos = np.asarray(positions, np.float64)
        g = pos.shape[0]
        k = num_coefficients(sh_degree)
        shapes = {"positions": (pos, (g, 3)), "rotations": (np.asarray(rotations, np.float64), (g, 4)),
                  "log_scales": (np.asarray(log_scales, np.float64), (g, 3)),
                  "opacity_logits": (np.asarray(opacity_logits, np.float64), (g,)),
                  "sh_coeffs": (np.asarray(sh_coeffs, np.float64), (g, 3, k))}
        for name, (a, shp) in shapes.items():
            if a.shape != shp:
                raise ValueError(f"{name} must have shape {shp}, got {a.shape}")
        mat = np.concatenate([shapes["positions"][0].T, shapes["rotations"][0].T, shapes["log_scales"][0].T,
                              shapes["opacity_logits"][0][None, :], shapes["sh_coeffs"][0].reshape(g, 3 * k).T])
        x = torch.from_numpy(np.ascontiguousarray(mat).reshape(-1)).to(device or default_device())
        return cls(x, sh_degree, background)

    @classmethod
    def from_reference(cls, ref_scene, device=None) -> "GaussianScene":
        """Build from a reference-shaped object (fields positions, rotations, ...)."""
        return cls.from_arrays(ref_scene.positions, ref_scene.rotations, ref_scene.log_scales,
                               ref_scene.opacity_logits, ref_scene.sh_coeffs, ref_scene.sh_degree,
                               ref_scene.background, device)

    @property
    def num_gaussians(self) -> int:
        return self.x.numel() // self.params_per_gaussian

    @property
    def params_per_gaussian(self) -> int:
        return params_per_gaussian(self.sh_degree)

    @property
    def param_count(self) -> int:
        return self.x.numel()

    @property
    def device(self):
        return self.x.device

    def _rows(self, sl):
        return self.x.view(self.params_per_gaussian, self.num_gaussians)[sl]

    @property
    def positions(self):
        return self._rows(POS_SLICE).t()

    @property
    def rotations(self):
        return self._rows(ROT_SLICE).t()

    @property
    def log_scales(self):
        return self._rows(SCALE_SLICE).t()

    @property
    def opacity_logits(self):
        return self._rows(OPACITY_INDEX)

    @property
    def opacities(self):
        return torch.sigmoid(self.opacity_logits)

    @property
    def sh_coeffs(self):
        k = num_coefficients(self.sh_degree)
        return self._rows(slice(SH_START, None)).t().reshape(-1, 3, k)

    def x32(self) -> torch.Tensor:
        """float32 copy used by the product chain kernels (cached)."""
        if self._x32 is None:
            out = torch.empty(self.x.numel(), dtype=torch.float32, device=self.x.device)
            _lib.call("slm_f64_to_f32", _lib.ptr(self.x), _lib.ptr(out), out.numel(), _lib.stream_ptr())
            self._x32 = out
        return self._x32

    def is_finite(self) -> bool:
        return bool(torch.isfinite(self.x).all()) and bool(np.isfinite(self.background).all())

    def numpy_matrix(self) -> np.ndarray:
        """(G, P) host matrix in the reference attribute order."""
        return self.x.detach().cpu().numpy().reshape(self.params_per_gaussian, -1).T.copy()


def flatten(scene: GaussianScene, layout: Layout = Layout.ATTRIBUTE_MAJOR) -> ParamVector:
    """ref: scene.py:220-236."""
    g, p = scene.num_gaussians, scene.params_per_gaussian
    v = ParamVector(scene.x.clone(), Layout.ATTRIBUTE_MAJOR, g, p)
    return v if layout is Layout.ATTRIBUTE_MAJOR else sort_x(v)


def unflatten(v: ParamVector, sh_degree: int, background=(0.0, 0.0, 0.0)) -> GaussianScene:
    """ref: scene.py:239-258."""
    if v.params_per_gaussian != params_per_gaussian(sh_degree):
        raise ValueError(f"vector has {v.params_per_gaussian} params per Gaussian, degree {sh_degree} needs "
                         f"{params_per_gaussian(sh_degree)}")
    am = v if v.layout is Layout.ATTRIBUTE_MAJOR else sort_x_inverse(v)
    return GaussianScene(am.values.double().clone(), sh_degree, background)


def scene_with_offset(scene: GaussianScene, delta: ParamVector, gamma: float = 1.0) -> GaussianScene:
    """x + gamma * delta, delta attribute-major (ref: scene.py:261-265)."""
    delta.require_layout(Layout.ATTRIBUTE_MAJOR)
    d = delta.values
    out = torch.empty_like(scene.x)
    if d.dtype == torch.float32 and scene.x.is_cuda:
        _lib.call("slm_axpy_scene", _lib.ptr(scene.x), _lib.ptr(d.contiguous()), float(gamma), _lib.ptr(out),
                  out.numel(), _lib.stream_ptr())
    else:
        out = scene.x + gamma * d.double()
    return GaussianScene(out, scene.sh_degree, scene.background)


# ---------------------------------------------------------------------------
# Cameras
# ---------------------------------------------------------------------------

@dataclass(frozen=True, eq=False)
class Camera:
    """Pinhole camera, world-to-camera rotation + translation (ref: scene.py:272-304)."""

    rotation: np.ndarray
    translation: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        object.__setattr__(self, "rotation", np.asarray(self.rotation, np.float64).reshape(3, 3))
        object.__setattr__(self, "translation", np.asarray(self.translation, np.float64).reshape(3))
        if self.width < 1 or self.height < 1:
            raise ValueError("camera resolution must be at least 1x1")
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if self.width >= 65536 or self.height >= 32768:
            raise ValueError("resolution exceeds the 16/15-bit pixel coordinate packing")

    @property
    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation

    @property
    def num_pixels(self) -> int:
        return self.width * self.height

    @classmethod
    def from_reference(cls, c) -> "Camera":
        return cls(c.rotation, c.translation, c.fx, c.fy, c.cx, c.cy, c.width, c.height)

    def to_struct(self, pix_base: int = 0) -> _lib.SlmCamera:
        s = _lib.SlmCamera()
        for i, v in enumerate(self.rotation.reshape(-1)):
            s.R[i] = float(v)
        for i, v in enumerate(self.translation):
            s.t[i] = float(v)
        s.fx, s.fy, s.cx, s.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        for i, v in enumerate(self.center):
            s.C[i] = float(v)
        s.W, s.H, s.pix_base = int(self.width), int(self.height), int(pix_base)
        return s


def look_at_camera(eye, target, up, fx, fy, width, height) -> Camera:
    """ref: scene.py:307-319."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    rot = np.stack([right, down, fwd])
    return Camera(rotation=rot, translation=-rot @ eye, fx=fx, fy=fy, cx=width / 2.0, cy=height / 2.0,
                  width=width, height=height)


def cameras_struct_tensor(cameras, device) -> tuple[torch.Tensor, list[int]]:
    """Pack cameras into a device byte tensor of SlmCamera with subset-global
    pixel bases; returns (tensor, bases)."""
    import ctypes as C
    n = len(cameras)
    arr = (_lib.SlmCamera * n)()
    bases, base = [], 0
    for i, c in enumerate(cameras):
        arr[i] = c.to_struct(base)
        bases.append(base)
        base += c.num_pixels
    raw = bytes(C.string_at(C.addressof(arr), C.sizeof(arr)))
    t = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)
    return t, bases


# ---------------------------------------------------------------------------
# JSON interop with the reference formats (ref: scene.py:420-472)
# ---------------------------------------------------------------------------

def scene_to_json(scene: GaussianScene) -> str:
    m = scene.numpy_matrix()
    k = num_coefficients(scene.sh_degree)
    payload = {"sh_degree": scene.sh_degree, "background": scene.background.tolist(),
               "gaussians": [{"pos": r[0:3].tolist(), "rot": r[3:7].tolist(), "log_scale": r[7:10].tolist(),
                              "opacity_logit": float(r[10]), "sh": r[11:].reshape(3, k).tolist()} for r in m]}
    return json.dumps(payload, indent=1)


def scene_from_json(text: str, device=None) -> GaussianScene:
    p = json.loads(text)
    gs = p["gaussians"]
    if not gs:
        raise ValueError("scene must contain at least one Gaussian")
    sh = np.asarray([g["sh"] for g in gs], np.float64)
    deg = int(round(np.sqrt(sh.shape[2]))) - 1
    if deg != p["sh_degree"]:
        raise ValueError("sh_degree field does not match coefficient count")
    return GaussianScene.from_arrays([g["pos"] for g in gs], [g["rot"] for g in gs],
                                     [g["log_scale"] for g in gs], [g["opacity_logit"] for g in gs], sh, deg,
                                     p["background"], device)


def cameras_to_json(cameras) -> str:
    return json.dumps([{"world_to_camera": np.hstack([c.rotation, c.translation[:, None]]).tolist(),
                        "fx": c.fx, "fy": c.fy, "cx": c.cx, "cy": c.cy, "width": c.width, "height": c.height}
                       for c in cameras], indent=1)


def cameras_from_json(text: str) -> list[Camera]:
    out = []
    for c in json.loads(text):
        w2c = np.asarray(c["world_to_camera"], np.float64).reshape(3, 4)
        out.append(Camera(w2c[:, :3], w2c[:, 3], c["fx"], c["fy"], c["cx"], c["cy"], int(c["width"]),
                          int(c["height"])))
    return out
