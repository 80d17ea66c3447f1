"""The reference's CPU path timed per BASELINE.md §2 (the oracle restatement,
oracle/hsplat_oracle.cpp, built like the reference's CMake Release: -O3, no
-march; fork-join parallel_for over the host cores, single-threaded stable
sort / duplicate / tile ranges, serial cut gather).  Test infrastructure: it
is the reported CPU baseline, never the product.

  python tools/cpu_baseline.py [--out profiles/r02_cpu_baseline.json] [--quick]

Runs: C1 all stages x 5 reps; C2 one view x 3 reps; C3 one view per tau; C4
frames 0-19 (10 cut-refresh pairs, bench_path cadence) extrapolated to 1000
frames (labelled as such).  C5 is not run (the oracle's 304 B/node AoS copy of
2e8 nodes plus the generator's host copy exceed what a CPU baseline should
hold).  Every number is in seconds per frame of StageTimes buckets
(render.hpp:24-31).
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STAGES = ("cut_expand", "weights", "preprocess", "duplicate", "tile_ranges", "alpha_blend")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_info(orc) -> dict:
    return {"cpu_model": cpu_model(), "nproc": os.cpu_count(), "threads_used": orc.thread_count(),
            "build": "oracle/hsplat_oracle.cpp, g++ -O3 -DNDEBUG, no -march (SSE2 scalar, no FMA), like the "
                     "reference's CMake Release defaults (proj/CMakeLists.txt:8-10)"}


def frame(orc, oh, cam, tau):
    t0 = time.perf_counter()
    f = orc.render_hierarchy(oh, cam, tau, keep_ctx=False)
    wall = time.perf_counter() - t0
    st = f.times()
    st["wall"] = wall
    sz = f.sizes()
    st["cut_entries"] = sz["ncut"]
    return st


def mean_of(rows):
    keys = rows[0].keys()
    return {k: sum(r[k] for r in rows) / len(rows) for k in keys}


def run(quick: bool) -> dict:
    from oracle import oracle as orc
    from paper_2406_12080_b200 import multi, scenes
    out = {"host": host_info(orc), "units": "seconds per frame (StageTimes buckets + wall)"}

    # C1: all stages, 5 reps of one view
    cfg = scenes.CONFIGS["c1"]
    oh = orc.OracleHierarchy(scenes.hierarchy(cfg))
    cam = scenes.camera(cfg, 100)
    frame(orc, oh, cam, cfg.tau)  # warm-up
    rows = [frame(orc, oh, cam, cfg.tau) for _ in range(5)]
    out["c1"] = {"workload": cfg.name, "reps": 5, "mean": mean_of(rows), "frames_per_s": 1.0 / mean_of(rows)["wall"]}
    del oh

    # C2 / C3 / C4 on the 10M-leaf hierarchy
    cfg = scenes.CONFIGS["c2"]
    t0 = time.perf_counter()
    h = scenes.hierarchy(cfg)
    oh = orc.OracleHierarchy(h)
    del h
    out["c2_setup_s"] = time.perf_counter() - t0
    cam = scenes.camera(cfg, 100)
    reps = 1 if quick else 3
    rows = [frame(orc, oh, cam, cfg.tau) for _ in range(reps)]
    out["c2"] = {"workload": cfg.name, "view": "trajectory frame 100", "reps": reps, "mean": mean_of(rows),
                 "frames_per_s": 1.0 / mean_of(rows)["wall"]}
    out["c3"] = {}
    for tau in ((3.0,) if quick else (0.0, 1.5, 3.0, 6.0, 12.0)):
        r = frame(orc, oh, cam, tau)
        out["c3"][str(tau)] = {"view": "trajectory frame 100", **r, "frames_per_s": 1.0 / r["wall"]}
    if not quick:
        # C4: bench_path cadence over frames 0-19, extrapolated to the 1000-frame trajectory
        cams = scenes.trajectory(cfg, 20, first=0)
        t0 = time.perf_counter()
        stats = orc.bench_path(oh, cams, cfg.tau)
        el = time.perf_counter() - t0
        out["c4"] = {"frames_measured": 20, "seconds_measured": el, "frames_per_s": 20 / el,
                     "extrapolated_1000_frames_s": el * 1000 / 20, "label": "extrapolated from frames 0-19",
                     "mean_rendered": float(stats[:, multi.STAT_FIELDS.index("rendered")].mean())}
    out["c5"] = "not run: 2e8-node hierarchy (58 GB of device SoA; the oracle's AoS copy is 61 GB)"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    res = run(a.quick)
    s = json.dumps(res, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
