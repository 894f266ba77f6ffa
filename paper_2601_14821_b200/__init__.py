"""B200-native POTR hot paths (arXiv 2601.14821): removal-effect scoring and
training-free SH recompute as sm_100a kernels behind the reference's Python
API.  See DESIGN.md.

    from paper_2601_14821_b200 import rasterizer, compaction
    stats = rasterizer.compute_delta_mse(splats, cameras, targets)

`install()` rebinds the reference package (potr) to these implementations.
"""

__version__ = "0.1.0"

from . import fixture, scene  # noqa: F401  (host-only modules, no torch needed)


def __getattr__(name):
    # device modules import torch lazily so `import paper_2601_14821_b200` stays cheap
    import importlib
    if name in ("rasterizer", "compaction", "pruning", "distributed", "device", "metrics",
                "install"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
