"""Scene types of the drop-in boundary (mirror of potr/scene.py:28-93).

Only the in-memory types cross the boundary; PLY / camera-JSON ingestion is
host-side I/O outside the hot path and stays with the reference package.
Any object exposing the same attributes (e.g. the reference's own Splats and
Camera) is accepted wherever these are.
"""

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Splats:
    """Activated splat attributes (scene.py:42-61)."""

    positions: np.ndarray  # (N, 3) world units
    sh: np.ndarray         # (N, 3, 16) channel-major, coefficient 0 = DC
    opacities: np.ndarray  # (N,) in (0, 1)
    scales: np.ndarray     # (N, 3) per-axis stddev, > 0
    rotations: np.ndarray  # (N, 4) unit wxyz with w >= 0

    def __len__(self):
        return self.positions.shape[0]

    def subset(self, idx):
        return Splats(self.positions[idx], self.sh[idx], self.opacities[idx],
                      self.scales[idx], self.rotations[idx])

    def copy(self):
        return Splats(self.positions.copy(), self.sh.copy(), self.opacities.copy(),
                      self.scales.copy(), self.rotations.copy())


@dataclass
class Camera:
    """Pinhole camera (scene.py:64-77); rotation is world-to-camera."""

    eye: np.ndarray        # (3,)
    rotation: np.ndarray   # (3, 3) rows orthonormal, det +1
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    image: np.ndarray | None = None

    def pixel_count(self):
        return self.width * self.height


@dataclass
class Scene:
    splats: Splats
    cameras: list
    targets: list = field(default_factory=list)

    def freeze_targets(self, targets):
        """scene.py:86-93: install the reference renders read-only."""
        frozen = []
        for t in targets:
            t = np.ascontiguousarray(t, dtype=np.float64)
            t.flags.writeable = False
            frozen.append(t)
        self.targets = frozen
