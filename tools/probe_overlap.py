"""Probe: how much do two frames in flight on two streams overlap?

Two renderers (two contexts = two streams, the hierarchy uploaded into each)
render alternate frames of the C2 trajectory; device time of the whole batch
against the same frames on one stream.  Run under gpurun:
    PYTHONPATH=. python tools/probe_overlap.py
"""
import json
import time

import torch

import paper_2406_12080_b200 as hs
from paper_2406_12080_b200 import _native as N
from paper_2406_12080_b200 import scenes


def main():
    cfg = scenes.CONFIGS["c2"]
    h = scenes.hierarchy(cfg, threads=16)
    nr = 2
    rs = [hs.Renderer(0, exact=True) for _ in range(nr)]
    dhs = [r.upload(h, validate=False) for r in rs]
    L = N.lib()
    cams = [c.to_c() for c in scenes.trajectory(cfg, 70)]
    warm, timed = cams[:6], cams[6:66]
    for r, dh in zip(rs, dhs):
        for c in warm:
            hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, c, cfg.tau, r._cut, r._frame, None), r.ctx)
    streams = [torch.cuda.ExternalStream(r.stream_handle()) for r in rs]
    out = {}
    for mode in ("one", "two", "one", "two"):
        for r in rs:
            r.set_async(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        if mode == "two":
            streams[1].wait_event(e0)
        for i, c in enumerate(timed):
            k = (i % nr) if mode == "two" else 0
            r = rs[k]
            hs._check(L.hs_render_hierarchy(r.ctx, dhs[k].handle, c, cfg.tau, r._cut, r._frame, None), r.ctx)
        if mode == "two":
            ej = torch.cuda.Event()
            ej.record(streams[1])
            streams[0].wait_event(ej)
        e1.record(streams[0])
        e1.synchronize()
        for r in rs:
            r.synchronize()
            r.set_async(False)
        ms = e0.elapsed_time(e1)
        out[mode] = {"ms_per_frame": ms / len(timed), "fps": 1e3 * len(timed) / ms}
        print(mode, out[mode], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
