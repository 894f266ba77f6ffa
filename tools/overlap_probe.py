"""Where the end-to-end forward_stats time goes at C3 (upload overlap probe).

    python tools/overlap_probe.py [--config C3]

Prints wall times (ms) of: the SH upload alone (sync ring / async + wait),
the geometry upload, forward_stats from pageable arrays at several lookahead
depths, and the same pass on device-resident splats.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_14821_b200 import _native, device as D, rasterizer as R  # noqa: E402
from paper_2601_14821_b200.fixture import config_scene  # noqa: E402
from paper_2601_14821_b200.scene import Splats  # noqa: E402


def wall(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    args = ap.parse_args()
    splats, cams = config_scene(args.config)
    pert = splats.copy()
    pert.opacities = pert.opacities * 0.97
    dev = D.current_device()
    targets = []
    for t in R.render_targets(splats, cams):
        t.flags.writeable = False
        targets.append(t)
    host = Splats(*(np.array(getattr(pert, f), dtype=np.float64, copy=True)
                    for f in ("positions", "sh", "opacities", "scales", "rotations")))
    ctx = D.context()
    out = {}
    out["sh_sync_ring"] = wall(lambda: D.to_device(host.sh, dev))

    def async_sh():
        ds = D.DeviceSplats.from_host(host, dev, async_sh=True)
        ds.wait_upload()
    out["from_host_async_sh_plus_wait"] = wall(async_sh)
    out["from_host_sync"] = wall(lambda: D.DeviceSplats.from_host(host, dev))
    geo = Splats(host.positions, np.zeros((1, 3, 16)), host.opacities, host.scales,
                 host.rotations)
    out["geometry_upload"] = wall(lambda: [D.to_device(a, dev) for a in
                                           (geo.positions, geo.opacities, geo.scales,
                                            geo.rotations)])
    ds = D.DeviceSplats.from_host(host, dev)
    dt = D.targets_cache.get(targets, cams, dev)
    out["device_resident_pass"] = wall(lambda: R.forward_stats_device(ds, cams, dt))
    imp, _, dm, _ = R.forward_stats_device(ds, cams, dt)
    out["readback_importance_and_delta_mse"] = wall(lambda: (D.to_host(imp), D.to_host(dm)))
    for la in (1, 3, 6, 8):
        ctx.call("potr_set_option", _native.OPT_LOOKAHEAD, la)
        out[f"forward_stats_pageable_lookahead{la}"] = wall(
            lambda: R.forward_stats(host, cams, targets).delta_mse[0])
    ctx.call("potr_set_option", _native.OPT_LOOKAHEAD, 6)
    ctx.profile(True)
    R.forward_stats(host, cams, targets)
    prof = ctx.profile_read()
    ctx.profile(False)
    out["stage_ms_lookahead6"] = {k: round(v[0], 2) for k, v in prof.items() if v[0]}
    for k, v in out.items():
        print(k, v if isinstance(v, dict) else round(v, 2))


if __name__ == "__main__":
    main()
