"""One C3 prune-score batch (8 views) after a warm-up batch: the launch set
`ncu` captures when profiling a single pipeline round.

    ncu --set full -k regex:<kernel> -s <skip> -c <count> python tools/prof_batch.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_14821_b200 import device as D, rasterizer as R  # noqa: E402
from paper_2601_14821_b200.fixture import config_scene  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
splats, cams = config_scene(cfg)
cams = cams[:16]
dev = D.current_device()
ds = D.DeviceSplats.from_host(splats, dev)
tg = R.render_targets_device(ds, cams[:8])
for _ in range(2):
    R.forward_stats_device(ds, cams[:8], tg)
torch.cuda.synchronize()
print("done")
