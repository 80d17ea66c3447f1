"""Benchmark: frames/sec of per-view LOD cut + 3DGS forward render.

Metric (BASELINE.json): frames/sec at 1080p, tau = 3 px, 10M-leaf hierarchy;
cut+render ms/frame.  One step = one frame of the camera trajectory: k_select_cut
over all 20M nodes, fused interpolation/preprocess, duplication, radix sort,
tile ranges and alpha blend (BASELINE.json configs[1] = SURVEY.md config C2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun (one rank per GPU): the 1000-frame trajectory is
partitioned into contiguous per-rank blocks with the hierarchy replicated on
every GPU (weak scaling: K frames per rank); there is no data-path collective.
Timing: CUDA events on the renderer's stream, barrier + synchronize on both
sides, max over ranks.  --impl reference times the reference's CPU path (the
oracle restatement, oracle/hsplat_oracle.cpp) on this box's host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec at 1080p, tau=3px, 10M-leaf hierarchy; cut+render ms/frame"
UNIT = "frames/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# kernels behind each HBM-bound stage (for the per-stage ncu DRAM traffic)
STAGE_KERNELS = {"cut": ("k_select_cut", "k_cut_offsets", "k_cut_gather"), "preprocess": ("k_preprocess<1>",),
                 "duplicate+sort": ("k_tile_count", "k_tile_plan", "k_bucket", "k_bucket_huge", "k_tile_split",
                                    "k_tile_sort", "k_tile_finalize")}


def pipe_peaks():
    """FP32 / FP32x2 / FP64 / MUFU throughput measured on this GPU by tools/peaks (built by
    __graft_entry__.build()); the blend's roofline denominators."""
    exe = os.path.join(ROOT, "tools", "peaks")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
        return json.loads(out.strip().splitlines()[-1])
    except Exception:
        return None


def ncu_traffic():
    """Per-launch DRAM bytes per kernel from the newest committed ncu --set full capture
    (profiles/r*_traffic_v*.json, written by tools/ncu_traffic.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic_v*.json")),
                   key=lambda f: int(f.rsplit("_v", 1)[1].split(".")[0]))
    if not files:
        return {}, None
    with open(files[-1]) as f:
        d = json.load(f)
    return d.get("kernels", {}), os.path.relpath(files[-1], ROOT)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 7 for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def frames_for_rank(rank: int, world: int, steps: int, warmup: int):
    """Contiguous, even-length per-rank blocks of the trajectory."""
    per = steps + warmup
    per += per % 2
    return rank * per, per


def run_reference(args, cfg):
    """--impl reference: the reference's CPU path (oracle port) on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    from oracle import oracle as orc
    from paper_2406_12080_b200 import scenes

    h = scenes.hierarchy(cfg)
    oh = orc.OracleHierarchy(h)
    del h
    cores = orc.thread_count()
    cams = scenes.trajectory(cfg, args.warmup + args.steps, first=0)
    for cam in cams[: min(args.warmup, 1)]:
        orc.render_hierarchy(oh, cam, cfg.tau, keep_ctx=False)
    budget = args.reference_budget_s
    done, t0 = 0, time.perf_counter()
    for cam in cams[args.warmup:]:
        orc.render_hierarchy(oh, cam, cfg.tau, keep_ctx=False)
        done += 1
        if time.perf_counter() - t0 > budget:
            break
    el = time.perf_counter() - t0
    v = done / el
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": done,
        "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * el / done, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "leaves": cfg.leaves, "width": cfg.width, "height": cfg.height,
                   "tau": cfg.tau, "l2": "inputs larger than L2 (host run)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{done} frame(s) of the {cfg.name} trajectory (steps capped at "
                                   f"{budget:.0f} s of CPU time)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, h, frames: int = 2):
    from oracle import oracle as orc
    from paper_2406_12080_b200 import scenes
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from cpu_baseline import STAGES, host_info

    oh = orc.OracleHierarchy(h)
    cams = scenes.trajectory(cfg, frames, first=100)
    stages = dict.fromkeys(STAGES, 0.0)
    t0 = time.perf_counter()
    for cam in cams:
        f = orc.render_hierarchy(oh, cam, cfg.tau, keep_ctx=False)
        for k, v in f.times().items():
            stages[k] += v / frames
    el = time.perf_counter() - t0
    info = host_info(orc)
    full = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_cpu_baseline.json"))
    return {"value": frames / el, "unit": UNIT, "cores": orc.thread_count(), "kind": "port",
            "sample": f"{frames} frames (100..{99 + frames}) of the {cfg.name} trajectory, oracle "
                      f"render_hierarchy incl. select_cut + cut_render_splats + render_forward",
            "stages_s": stages, "cpu_model": info["cpu_model"], "nproc": info["nproc"], "build": info["build"],
            "full_plan": ("profiles/" + full[-1]) if full else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--mode", default="exact", choices=["exact", "fast"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tau-sweep", action="store_true")
    ap.add_argument("--no-inscene", action="store_true")
    ap.add_argument("--no-replay", action="store_true")
    ap.add_argument("--reference-budget-s", type=float, default=120.0)
    ap.add_argument("--lanes", type=int, default=2,
                    help="frame lanes (streams): consecutive frames on different lanes overlap on the device")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_2406_12080_b200 import scenes
    cfg = scenes.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_2406_12080_b200 as hs
    from paper_2406_12080_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    r = hs.Renderer(local, exact=(args.mode == "exact"))
    t0 = time.perf_counter()
    if cfg.name.startswith("c5"):
        # 16 chunks + skybox generated one at a time and consolidated on the device
        # (the 58 GB hierarchy never exists on the host)
        h = None
        dh = scenes.multichunk(r, cfg.leaves, sky=cfg.sky)
        gen_s, upload_s = time.perf_counter() - t0, 0.0
    else:
        # every rank builds its replica; split the host cores between the ranks
        h = scenes.hierarchy(cfg, threads=max(1, (os.cpu_count() or 1) // world))
        gen_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        dh = r.upload(h, validate=False)
        upload_s = time.perf_counter() - t0
    L = N.lib()
    first, count = frames_for_rank(rank, world, args.steps, args.warmup)
    cams = scenes.trajectory(cfg, count, first=first)
    ccams = [c.to_c() for c in cams]
    warm, timed = ccams[: args.warmup], ccams[args.warmup: args.warmup + args.steps]

    # frame lanes: frame object k (with its own cut object) binds to lane k at its first
    # render; frame i of the trajectory goes to object i % NL, so consecutive frames
    # overlap (one frame's latency-bound sort stages beside the next one's HBM-bound
    # cut and preprocess).  Every frame is still the full cut + render.
    NL = max(1, min(4, args.lanes))
    r.set_lanes(NL)
    lane_frames, lane_cuts = [r._frame], [r._cut]
    for _ in range(NL - 1):
        fr, cu = N.C.c_void_p(), N.C.c_void_p()
        hs._check(L.hs_frame_create(r.ctx, N.C.byref(fr)), r.ctx)
        hs._check(L.hs_cut_create(r.ctx, N.C.byref(cu)), r.ctx)
        lane_frames.append(fr)
        lane_cuts.append(cu)

    def render(c, tau, k, cut_only=False):
        if cut_only:  # reuse lane k's cut (bench_path's odd frames)
            hs._check(L.hs_render_cut(r.ctx, dh.handle, lane_cuts[k], c, lane_frames[k], None), r.ctx)
        else:
            hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, c, tau, lane_cuts[k], lane_frames[k], None), r.ctx)

    def wait_lanes():
        for fr in lane_frames:
            hs._check(L.hs_frame_wait(r.ctx, fr), r.ctx)  # fails if any timed frame overflowed

    # warm-up (synchronous: grows every lane's duplicate buffers to this trajectory's needs)
    for k in range(NL):
        for c in warm:
            render(c, cfg.tau, k)
    stream = torch.cuda.ExternalStream(r.stream_handle())

    # ---- timed region: K frames, async enqueue, CUDA events on the renderer stream
    r.set_async(True)
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    r.synchronize()
    sampler.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = L.hs_kernel_launch_count()
    e0.record(stream)
    for i, c in enumerate(timed):
        render(c, cfg.tau, i % NL)
    r.join()
    e1.record(stream)
    launches = L.hs_kernel_launch_count() - launches0
    e1.synchronize()
    r.synchronize()
    clocks = sampler.stop()
    barrier()
    wait_lanes()
    ms_local = e0.elapsed_time(e1)
    ms_total = max_over_ranks(ms_local)
    value = world * len(timed) / (ms_total / 1e3)

    # the same frames on one lane (frame after frame: the per-frame latency view)
    barrier()
    torch.cuda.synchronize()
    r.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for c in timed:
        render(c, cfg.tau, 0)
    e1.record(stream)
    e1.synchronize()
    barrier()
    wait_lanes()
    r.set_async(False)
    one_ms = max_over_ranks(e0.elapsed_time(e1))
    single_lane = {"value": world * len(timed) / (one_ms / 1e3), "unit": UNIT, "ms_per_step": one_ms / len(timed),
                   "what": "same frames, one lane: each frame starts after the previous one ends"}

    # ---- reference cadence (bench.hpp:70-84): cut refreshed on even frames, reused on odd ones
    r.set_async(True)
    barrier()
    torch.cuda.synchronize()
    r.synchronize()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for i, c in enumerate(timed):  # a refresh pair stays on one lane; pairs alternate lanes
        render(c, cfg.tau, (i // 2) % NL, cut_only=(i % 2 == 1))
    r.join()
    e3.record(stream)
    e3.synchronize()
    r.synchronize()
    barrier()
    wait_lanes()
    r.set_async(False)
    cad_ms = max_over_ranks(e2.elapsed_time(e3))
    cadence = {"value": world * len(timed) / (cad_ms / 1e3), "unit": UNIT, "ms_per_step": cad_ms / len(timed),
               "what": "bench_path cadence: select_cut on even frames only (bench.hpp:70-84), same frames"}

    # ---- BASELINE configs[2] (C3): the tau sweep on the same hierarchy and frames
    tau_sweep = {}
    if not args.no_tau_sweep:
        r.set_async(True)
        for tau in (0.0, 1.5, 3.0, 6.0, 12.0):
            sweep = timed[: min(len(timed), 20)]
            for k in range(NL):
                render(sweep[0], tau, k)
            r.set_async(False)
            wait_lanes()
            for k in range(NL):
                render(sweep[0], tau, k)
            r.set_async(True)
            barrier()
            r.synchronize()
            e4 = torch.cuda.Event(enable_timing=True)
            e5 = torch.cuda.Event(enable_timing=True)
            e4.record(stream)
            for i, c in enumerate(sweep):
                render(c, tau, i % NL)
            r.join()
            e5.record(stream)
            e5.synchronize()
            r.synchronize()
            wait_lanes()
            fi = N.hs_frame_info()
            hs._check(L.hs_frame_get_info(r.ctx, r._frame, fi), r.ctx)
            ms = max_over_ranks(e4.elapsed_time(e5)) / len(sweep)
            tau_sweep[str(tau)] = {"frames_per_s": world * 1e3 / ms, "ms_per_frame": ms,
                                   "cut_entries": int(fi.n_splats), "duplicates": int(fi.n_duplicates)}
        r.set_async(False)

    # ---- second C2 workload: SURVEY §8d's in-scene trajectory (6 m high, through the city)
    inscene = None
    if not args.no_inscene and not cfg.name.startswith("c5"):
        icams = [c.to_c() for c in scenes.trajectory_inscene(cfg, min(len(timed), 40) + 2, first=first)]
        for k in range(NL):  # synchronous: grows the duplicate buffers (screen-covering splats)
            render(icams[0], cfg.tau, k)
            render(icams[1], cfg.tau, k)
        r.set_async(True)
        barrier()
        r.synchronize()
        e6, e7 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e6.record(stream)
        for i, c in enumerate(icams[2:]):
            render(c, cfg.tau, i % NL)
        r.join()
        e7.record(stream)
        e7.synchronize()
        r.synchronize()
        wait_lanes()
        r.set_async(False)
        fi = N.hs_frame_info()
        hs._check(L.hs_frame_get_info(r.ctx, r._frame, fi), r.ctx)
        nfr = len(icams) - 2
        ims = max_over_ranks(e6.elapsed_time(e7)) / nfr
        inscene = {"frames_per_s": world * 1e3 / ims, "ms_per_frame": ims, "frames": nfr,
                   "cut_entries": int(fi.n_splats), "visible": int(fi.n_visible), "duplicates": int(fi.n_duplicates),
                   "rendered_count": int(fi.rendered_count),
                   "what": "scenes.trajectory_inscene: closed loop through the city at 6 m, 20 m look-ahead, "
                           "pitched down; splats beside the camera just in front of its image plane project to "
                           "screen-covering ellipses under the reference's projection and saturate every pixel"}

    # ---- the trajectory replay (multi.replay_trajectory, bench_path cadence) with the data plane:
    # per-frame images to rank 0 over NCCL (device tensors, overlapped with rendering) and one
    # all_gather of the per-frame stats; wall clock between barriers, max over ranks
    replay = None
    if not args.no_replay:
        from paper_2406_12080_b200 import multi
        per = min(len(timed), 40)
        per += per % 2
        rcams = scenes.trajectory(cfg, per * world, first=0)
        src = multi.GpuFrameSource(r, dh)
        sums = []

        def on_image(i, t):  # rank 0: the image landed; keep a device-side checksum per frame
            sums.append(t.view(torch.int32).sum(dtype=torch.int64))
        multi.replay_trajectory(src, rcams[: 2 * world], cfg.tau, gather_images=world > 1, on_image=on_image)
        sums.clear()
        barrier()
        torch.cuda.synchronize()
        r.synchronize()
        t0 = time.perf_counter()
        rstats = multi.replay_trajectory(src, rcams, cfg.tau, gather_images=world > 1, on_image=on_image)
        torch.cuda.synchronize()
        rep_s = max_over_ranks(time.perf_counter() - t0)
        replay = {"frames_per_s": len(rcams) / rep_s, "frames": len(rcams), "seconds": rep_s,
                  "images_gathered_to_rank0": len(sums) if world > 1 else 0,
                  "gather_bytes_per_frame": 20 * cfg.width * cfg.height if world > 1 else 0,
                  "mean_rendered": float(rstats[:, 0].mean()),
                  "what": "bench_path cadence (cut on even frames), synchronous frames, per-stage events; "
                          "N > 1: every frame's RenderOutput sent to rank 0 (batch_isend_irecv, double-buffered) "
                          "and the stats all_gathered"}
        src.tracker.close()

    # ---- stage breakdown + roofline inputs: the same frames twice, per-stage CUDA events as
    # timed above (no counters), then with the blend's work counters on (HS_OPT_STATS) for the
    # frames' work (the frames are deterministic: the same work both times)
    st = hs.StageTimes()
    breakdown = timed[: min(len(timed), 16)]
    for c in breakdown:
        s = N.hs_stage_times()
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, c, cfg.tau, r._cut, r._frame, s), r.ctx)
        st.add(s)
    r.set_stats(True)
    infos = []
    for c in breakdown:
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, c, cfg.tau, r._cut, r._frame, None), r.ctx)
        fi = N.hs_frame_info()
        hs._check(L.hs_frame_get_info(r.ctx, r._frame, fi), r.ctx)
        infos.append(fi)
    r.set_stats(False)
    nf = len(infos)
    stage_ms = {k: 1e3 * getattr(st, k) / nf for k in ("cut_expand", "weights", "preprocess", "duplicate",
                                                      "tile_ranges", "alpha_blend")}
    mean = lambda k: sum(getattr(fi, k) for fi in infos) / nf  # noqa: E731
    C_, V_, D_, Ct = mean("n_splats"), mean("n_visible"), mean("n_duplicates"), mean("n_transition")
    NE, NC, NEt = mean("n_eval"), mean("n_contrib"), mean("n_eval_t")
    NX, NP = mean("n_exp"), mean("n_pow")
    nodes = dh.n
    W, H = cfg.width, cfg.height
    tiles = infos[0].tiles_x * infos[0].tiles_y
    pk, pk_kind = peaks()
    hbm = pk.get("hbm_gbs", 6450.9)
    # algorithmic bytes per frame: SURVEY.md §8(d) (DESIGN.md §7 restates them)
    P = -(-(max(1, (tiles - 1).bit_length()) + 31) // 8)  # passes of one (tile | depth) 64-bit key sort
    bytes_cut = 32 * nodes + 12 * C_
    bytes_pre = C_ * (8 + 236 + 4 + 64 + 4) + Ct * (236 + 4)
    bytes_scan = 8 * C_
    bytes_dup = V_ * (4 + 8 + 4) + 12 * D_
    bytes_sort = 8 * D_ + P * 24 * D_
    bytes_ranges = 8 * D_ + 8 * tiles

    def gbs(b, ms):
        return b / (ms * 1e6) if ms else None
    stages = {
        "cut": {"ms": stage_ms["cut_expand"], "bound": "hbm", "bytes": bytes_cut,
                "gbs": gbs(bytes_cut, stage_ms["cut_expand"]), "formula": "32 N + 12 C"},
        "preprocess": {"ms": stage_ms["preprocess"], "bound": "hbm", "bytes": bytes_pre,
                       "gbs": gbs(bytes_pre, stage_ms["preprocess"]), "formula": "316 C + 240 C_t"},
        # the tile ranges (tile_start) come out of the same kernels (k_tile_plan), so their
        # bytes are counted with this stage and its time
        "duplicate+sort": {"ms": stage_ms["duplicate"] + stage_ms["tile_ranges"], "bound": "hbm",
                           "bytes": bytes_scan + bytes_dup + bytes_sort + bytes_ranges,
                           "gbs": gbs(bytes_scan + bytes_dup + bytes_sort + bytes_ranges,
                                      stage_ms["duplicate"] + stage_ms["tile_ranges"]),
                           "formula": f"scan 8 C + duplicate (16 V + 12 D) + sort (8 D + {P} x 24 D) "
                                      "+ tile ranges (8 D + 8 tiles)"},
        "alpha_blend": {"ms": stage_ms["alpha_blend"], "bound": "fp32"},
    }
    # blend: SURVEY.md §8(d) ops per (pixel, entry) evaluation, N_eval counted on the device as
    # the evaluations each pixel executes up to and including its break entry (entries the reach
    # masks skip are not counted); exact mode adds the FP64 libm replicas per live pair
    sm_mhz = clocks.get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
    props = torch.cuda.get_device_properties(local)
    pp = pipe_peaks()
    fp32_nominal = props.multi_processor_count * 128 * 2 * sm_mhz * 1e6 / 1e12
    if pp:
        fp32_peak = max(pp["fp32_tflops"], pp["fp32x2_tflops"])
        fp32_src = f"measured (tools/peaks: FFMA {pp['fp32_tflops']:.1f}, FFMA2 {pp['fp32x2_tflops']:.1f} TFLOP/s)"
    else:
        fp32_peak, fp32_src = fp32_nominal, f"nominal {props.multi_processor_count} SMs x 128 x 2 x {sm_mhz:.0f} MHz"
    blend_s = stage_ms["alpha_blend"] * 1e-3
    fp32_ops = 20 * NE + 10 * NEt
    exact = args.mode == "exact"
    fp64_flops = (14 * NX + 27 * NP) if exact else 0.0   # expf / powf replicas: 6 + 9 DFMA, 2 + 9 DMUL/DADD
    mufu_ops = 0.0 if exact else NX + 2 * NP             # ex2; lg2 + ex2
    blend_tf = fp32_ops / blend_s / 1e12
    traffic, traffic_src = ncu_traffic()

    def tget(name):  # ncu names carry template arguments: k_blend<0, 0>
        for k, v in traffic.items():
            if k == name or k.startswith(name + "<") or k.startswith(name.rstrip(">") + ","):
                return v
        return {}
    blend_key = "k_blend<0" if args.mode == "exact" else "k_blend<1"
    roofline = {"bound": "fp32", "kernel": "k_blend", "achieved": blend_tf, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": blend_tf / fp32_peak,
                "traffic": tget(blend_key).get("dram_bytes"),
                "traffic_source": traffic_src,
                "formula": "FP32 ops = 20 N_eval + 10 N_eval,t (SURVEY.md §8d); N_eval = executed evaluations "
                           "up to and including each pixel's break",
                "n_eval": NE, "n_eval_t": NEt, "n_exp": NX, "n_pow": NP,
                "fp64": {"achieved_tflops": fp64_flops / blend_s / 1e12,
                         "peak_tflops": pp["fp64_tflops"] if pp else None,
                         "frac": (fp64_flops / blend_s / 1e12 / pp["fp64_tflops"]) if (pp and exact) else None,
                         "formula": "14 flops per expf replica + 27 per powf replica (FMA = 2)"} if exact else None,
                "mufu": {"achieved_tops": mufu_ops / blend_s / 1e12,
                         "peak_tops": pp["mufu_ex2_tops"] if pp else None} if not exact else None,
                # what bounds it (same ncu capture): instruction issue, not DRAM or one math pipe
                "ncu_pct_of_peak": tget(blend_key).get("pct_of_peak"),
                "algorithmic_bytes": 8 * D_ + 64 * D_ + 20 * W * H,
                "peak_source": fp32_src, "pipe_peaks": pp,
                "hbm_stages": {k: {"gbs": v.get("gbs"), "frac": (v["gbs"] / hbm) if v.get("gbs") else None,
                                   "bytes": v.get("bytes"), "formula": v.get("formula"),
                                   "traffic": sum(tget(kk).get("dram_bytes", 0.0)
                                                  for kk in STAGE_KERNELS.get(k, ())) or None}
                               for k, v in stages.items() if v.get("bound") == "hbm"},
                "hbm_peak_gbs": hbm, "hbm_peak_source": pk_kind}

    # ---- end to end through the public API: camera in (host struct -> kernel parameters),
    # the whole RenderOutput (colour, inverse depth, transmittance) out to pinned host
    # memory every frame.  NF frame objects in a ring: frame i's read-back (copy stream)
    # overlaps the kernels of frames i+1.., and a frame object is re-rendered only after
    # its previous read-back landed.
    # 2 x NL frame objects (each with its own cut), bound round-robin to the lanes
    NF = 2 * NL
    f32 = N.C.POINTER(N.C.c_float)
    frames = lane_frames + [N.C.c_void_p() for _ in range(NF - NL)]
    fcuts = lane_cuts + [N.C.c_void_p() for _ in range(NF - NL)]
    for fr, cu in zip(frames[NL:], fcuts[NL:]):
        hs._check(L.hs_frame_create(r.ctx, N.C.byref(fr)), r.ctx)
        hs._check(L.hs_cut_create(r.ctx, N.C.byref(cu)), r.ctx)
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, timed[0], cfg.tau, cu, fr, None), r.ctx)
    pinned = [torch.empty(5 * W * H, dtype=torch.float32, pin_memory=True) for _ in range(NF)]
    outs = [(N.C.cast(p.data_ptr(), f32), N.C.cast(p.data_ptr() + 12 * W * H, f32),
             N.C.cast(p.data_ptr() + 16 * W * H, f32)) for p in pinned]
    e2e_cams = [c.to_c() for c in cams[args.warmup: args.warmup + args.steps]]  # host camera structs
    rc = N.C.c_int32()
    r.set_async(True)
    barrier()
    torch.cuda.synchronize()
    r.synchronize()
    t0 = time.perf_counter()
    for i, c in enumerate(e2e_cams):
        fi = i % NF
        if i >= NF:
            hs._check(L.hs_frame_download_wait(r.ctx, frames[fi], N.C.byref(rc)), r.ctx)
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, c, cfg.tau, fcuts[fi], frames[fi], None), r.ctx)
        hs._check(L.hs_frame_download_async(r.ctx, frames[fi], *outs[fi]), r.ctx)
    for i in range(max(0, len(timed) - NF), len(timed)):
        hs._check(L.hs_frame_download_wait(r.ctx, frames[i % NF], N.C.byref(rc)), r.ctx)
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    r.set_async(False)
    for fr in frames:
        hs._check(L.hs_frame_wait(r.ctx, fr), r.ctx)
    for fr, cu in zip(frames[1:], fcuts[1:]):
        L.hs_frame_destroy(fr)
        L.hs_cut_destroy(cu)
    e2e = {"value": world * len(timed) / e2e_s, "unit": UNIT, "h2d_bytes_per_step": N.C.sizeof(N.hs_camera),
           "d2h_bytes_per_step": 20 * W * H + N.C.sizeof(N.hs_frame_info),
           "pipelining": f"{NF} frame objects on {NL} lanes; read-back of frame i on a copy stream overlaps "
                         "frames i+1.."}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and h is not None:
        cpu = cpu_baseline(cfg, h)
    elif h is None:
        cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
               "sample": "not run: the oracle's 304 B/node AoS copy of 2e8 nodes exceeds host RAM"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": len(timed),
            "warmup": args.warmup, "ms_per_step": ms_total / len(timed), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "leaves": cfg.leaves, "nodes": nodes, "width": W, "height": H,
                       "tau": cfg.tau, "blend_mode": args.mode, "frames": f"trajectory frames {first}.. per rank",
                       "parallelism": f"view-parallel x{world} (hierarchy replicated)", "frame_lanes": NL,
                       "l2": f"inputs larger than L2 (hierarchy {nodes * 288 / 1e9:.1f} GB resident; no flush needed)"},
            "roofline": roofline,
            "stages_ms": stage_ms,
            "stages": stages,
            "per_frame": {"cut_entries": C_, "transitioning": Ct, "visible": V_, "duplicates": D_, "n_eval": NE,
                          "n_eval_t": NEt, "n_contrib": NC, "n_exp": NX, "n_pow": NP},
            "single_lane": single_lane,
            "reference_cadence": cadence,
            "tau_sweep": tau_sweep,
            "inscene": inscene,
            "replay": replay,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "setup_s": {"generate": gen_s, "upload": upload_s},
        }
        print(json.dumps(line), flush=True)
    r.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
