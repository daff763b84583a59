"""Image container crossing the API boundary (fvr.imgio.Image,
/root/reference/pkg/src/fvr/imgio.py:21-55).  The file formats (FIM1, PNM)
live in formats.py."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Image:
    """Float intensity image on the [0, 255] scale; ``data`` is (H, W, C) f32."""

    width: int
    height: int
    channels: int
    data: np.ndarray = None

    def __post_init__(self):
        if self.channels not in (1, 3):
            raise ValueError("channels must be 1 or 3")
        shape = (self.height, self.width, self.channels)
        if self.data is None:
            self.data = np.zeros(shape, dtype=np.float32)
        else:
            self.data = np.ascontiguousarray(self.data, dtype=np.float32).reshape(shape)
        if not np.all(np.isfinite(self.data)) or np.any(self.data < 0):
            raise ValueError("image data must be finite and non-negative")

    @classmethod
    def from_array(cls, arr: np.ndarray) -> "Image":
        arr = np.asarray(arr)
        if arr.ndim == 2:
            arr = arr[:, :, None]
        h, w, c = arr.shape
        return cls(w, h, c, arr)

    def channel(self, c: int) -> "Image":
        return Image(self.width, self.height, 1, self.data[:, :, c : c + 1].copy())

    def to_rgb(self) -> "Image":
        if self.channels == 3:
            return self
        return Image(self.width, self.height, 3, np.repeat(self.data, 3, axis=2))
