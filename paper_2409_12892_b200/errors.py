"""Exception classes with the reference's names and bases.

ref: scene.py:48-49 (LayoutError), jacobian.py:42-43 (CacheOrderError),
residuals.py:35-36 (ImageSizeError); SPEC:395 (PCG non-SPD abort).
"""


class SplatLMError(RuntimeError):
    """Library / build problem (missing .so, ABI mismatch)."""


class LayoutError(ValueError):
    """A parameter vector arrived in the wrong layout."""


class CacheOrderError(ValueError):
    """A cache arrived in the wrong sort order for this product."""


class ImageSizeError(ValueError):
    """Two images that must match in shape do not."""


class NonSPDError(RuntimeError):
    """p^T g <= 0 inside PCG (loss of positive definiteness)."""
