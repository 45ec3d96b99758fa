"""Benchmark: 1080p novel-view frames/s (reconstruct + render) on B200.

Workload (BASELINE.json configs[1]): 8 synthetic
input views (2x4 rig, 0.3 m span), full_scale_config (Table 6 schedule),
encoder images 576x960, render images 1920x1080, 1080p target view,
random-init weights (init_param_store seed 3), synthetic plane scene
(make_scene seed 21). One step = one frame: lvs::forward + render_target.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lvsg|reference]

N > 1 runs under torchrun, one rank per GPU; rank r renders its own target
viewpoint (config 5 grid) of the same input views, resident on every GPU --
the path partitions by target, so there is no data-path collective (weak
scaling; paper_2411_16680_b200/shard.py). Timing is the max over ranks;
rank 0 prints one JSON line.

`value` is device-timed (CUDA events on the launching stream) with inputs
resident in HBM; `e2e` goes through the host C ABI (lvsg_forward_render)
with pinned host buffers and both copies inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "1080p novel-view frames/sec (reconstruct+render), ms/frame, HBM GB/s vs peak"
CPU_SAMPLE_DIV = 4  # the bounded CPU sample: config-2 schedule at 1/4 extents


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------
# algorithmic work per frame, from the plan
# ---------------------------------------------------------------------------

def frame_work(cfg, He, We, Hr, Wr):
    from paper_2411_16680_b200 import plan_forward
    from paper_2411_16680_b200.config import ModelConfig  # noqa: F401
    plan = plan_forward(cfg, He, We)
    M, C = cfg.views, cfg.channels
    Ca = 3 if cfg.direct_rgb else C
    conv = 2 * 27 * C * He * We * M
    h, w = He, We
    for _ in range(cfg.pyramid_levels):
        conv += 4 * 2 * 9 * C * C * h * w * M
        h //= 2
        w //= 2
    attn = 0
    gather_texel_views = 0
    from paper_2411_16680_b200.lvs import plan_forward as _pf  # noqa: F401
    for s, sp in enumerate(plan.steps):
        cin = 2 * C if s == 0 else 2 * C + Ca + 1
        conv += 2 * 9 * cin * C * sp.feat_h * sp.feat_w * M
        conv += 4 * 2 * 9 * C * C * sp.feat_h * sp.feat_w * M
        P = sp.layers * sp.height * sp.width
        gather_texel_views += P * M
        toks = [t.strip() for t in cfg.steps[s].blocks.split(",")]
        for t in toks:
            if t.startswith("A"):
                h_ = int(t[1:])
                attn += P * (4 * h_ * C * C + 4 * M * h_ * C)
            elif t == "C":
                conv += 2 * 2 * 9 * C * C * sp.height * sp.width * sp.layers
    last = plan.steps[-1]
    Pf = last.layers * last.height * last.width
    attn += Pf * (2 * C * C + 2 * M * C)  # blend head
    # conv3x3 algorithmic HBM bytes: every conv reads its input channels once
    # and writes its output once; the residual conv also reads the residual
    # (conv_residual / conv_mlp_residual: conv1 2N, conv2 3N for N = one
    # 32-channel map); the last encoder conv of a level also writes the pool
    N = lambda px: px * C * 4  # noqa: E731
    conv_bytes = M * He * We * 3 * 4 + N(M * He * We)  # stem
    h, w = He, We
    for _ in range(cfg.pyramid_levels):
        conv_bytes += 2 * 5 * N(M * h * w) + N(M * (h // 2) * (w // 2))
        h //= 2
        w //= 2
    for s, sp in enumerate(plan.steps):
        px = M * sp.feat_h * sp.feat_w
        cin = 2 * C if s == 0 else 2 * C + Ca + 1
        conv_bytes += px * cin * 4 + N(px) + 2 * 5 * N(px)  # update_cnn stem + 2 pairs
        nC = sum(1 for t in cfg.steps[s].blocks.split(",") if t.strip() == "C")
        conv_bytes += nC * 5 * N(sp.layers * sp.height * sp.width)
    Ho, Wo = plan.out_height, plan.out_width
    # fused Stage 3 + 4: LDM pre-activation maps + M input images + output
    render_bytes = Pf * (2 + M) * 4 + M * Hr * Wr * 3 * 4 + Ho * Wo * 3 * 4
    gather_bytes = 0
    for s, sp in enumerate(plan.steps):
        gather_bytes += M * sp.feat_h * sp.feat_w * C * 4 + sp.layers * sp.height * sp.width * (4 + M * C * 4)
    return {"conv_flops": conv, "conv_bytes": conv_bytes, "attn_flops": attn,
            "render_bytes": render_bytes,
            "gather_bytes": gather_bytes, "out_hw": (Ho, Wo),
            "final_texel_views": last.layers * Ho * Wo * M}


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref): the bounded sample
# ---------------------------------------------------------------------------

_ref_state = {}


def _ref_worker_init():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from bindings import Reference
    from paper_2411_16680_b200.workloads import config2
    c = config2(div=CPU_SAMPLE_DIV)
    _ref_state.update(ref=Reference(), case=c, w=c.flat())


def _ref_worker_frame(_):
    r, c, w = _ref_state["ref"], _ref_state["case"], _ref_state["w"]
    t = time.perf_counter()
    r.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target, w)
    return time.perf_counter() - t


def cpu_sample_desc():
    d = CPU_SAMPLE_DIV
    return (f"config-2 schedule at 1/{d} extents (8 views, encoder {576 // d}x{960 // d}, render "
            f"{1080 // d}x{1920 // d}, 1/{d * d} of every per-texel stage); one sample = "
            f"1/{d * d} frame, fps scaled accordingly")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def calibration():
    """The 1/16-frame sample against one full config-2 frame of the reference
    timed on a B200 host (profiles/ref_fullframe.py -> profiles/r2/)."""
    p = os.path.join(ROOT, "profiles", "r2", "ref_fullframe.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return {"full_frame_s": d.get("full_frame_s"),
            "sample_x16_s": d.get("sample_extrapolated_frame_s"),
            "full_over_extrapolated": d.get("full_over_extrapolated"),
            "cpu_model": d.get("cpu_model"), "source": "profiles/r2/ref_fullframe.json"}


def cpu_baseline_single():
    """oracle/_ref (the reference built from its sources) on one host core."""
    from bindings import REF_SO
    if not os.path.exists(REF_SO):
        return None
    _ref_worker_init()
    secs = _ref_worker_frame(0)
    frames = 1.0 / (CPU_SAMPLE_DIV ** 2)
    return {"value": frames / secs, "unit": "frames/s", "cores": 1, "kind": "reference",
            "sample": cpu_sample_desc(), "sample_seconds": secs, "cpu_model": cpu_model(),
            "host_cores": os.cpu_count(), "calibration": calibration()}


def reference_arm(args):
    """--impl reference: the reference CPU path on all usable host cores, as
    P concurrent single-threaded processes (the reference is single-threaded,
    SURVEY.md §8(d)); each step runs one bounded sample per process."""
    import multiprocessing as mp
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from bindings import REF_SO
    base = {"metric": METRIC, "unit": "frames/s", "impl": "reference", "n_gpus": args.gpus,
            "higher_is_better": True}
    if not os.path.exists(REF_SO):
        print(json.dumps(dict(base, unavailable="oracle/_ref/libref.so not built")))
        return
    cores = os.cpu_count() or 1
    try:
        mem_gb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
    except Exception:
        mem_gb = 64.0
    procs = max(1, min(cores, int(mem_gb // 4.0), args.ref_procs or 10 ** 9))
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_ref_worker_init) as pool:
        for _ in range(args.warmup):
            pool.map(_ref_worker_frame, range(procs))
        t0 = time.perf_counter()
        per = []
        for _ in range(args.steps):
            per += pool.map(_ref_worker_frame, range(procs))
        wall = time.perf_counter() - t0
    frames = args.steps * procs / (CPU_SAMPLE_DIV ** 2)
    fps = frames / wall
    out = dict(base, value=fps, steps=args.steps, warmup=args.warmup,
               ms_per_step=1000.0 * wall / args.steps, scaling="weak", vs_baseline=None,
               dtype="f32", data="synthetic",
               config={"workload": "config2 (8 views, full_scale_config, 576x960 -> 1080p)",
                       "sample": cpu_sample_desc(), "processes": procs},
               cpu_baseline={"value": fps, "unit": "frames/s", "cores": procs, "kind": "reference",
                             "sample": cpu_sample_desc(),
                             "mean_sample_seconds": statistics.mean(per),
                             "cpu_model": cpu_model(), "host_cores": cores,
                             "calibration": calibration()},
               e2e={"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0})
    print(json.dumps(out))


# ---------------------------------------------------------------------------
# the lvsg arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lvsg", choices=["lvsg", "reference"])
    ap.add_argument("--config", default="config2", choices=["config2", "config3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--ref-procs", type=int, default=0)
    ap.add_argument("--shard-encoder", action="store_true",
                    help="view-sharded encode + pyramid all-gather even at N=1 (default at N>1)")
    ap.add_argument("--mode", default="targets", choices=["targets", "frames", "rows"],
                    help="N > 1 partition (SURVEY.md §8(e)): targets = one target viewpoint per "
                         "rank (config-5 grid) with a view-sharded encoder; frames = the config-4 "
                         "video dealt round-robin (frame r + k N on rank r, no exchange); rows = one "
                         "target split into output row bands (replicated solve, band render, NCCL "
                         "all-gather of the bands)")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="N>1 pyramid exchange: stores fused into the encoder epilogue over "
                         "CUDA IPC (falls back to nccl if any rank cannot map its peers) or "
                         "an NCCL all-gather per level")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    import torch.distributed as dist
    import paper_2411_16680_b200 as q
    from paper_2411_16680_b200 import shard
    from paper_2411_16680_b200 import workloads as wl

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # targets: each rank its own target viewpoint (config 5 grid) when sharded;
    # frames: rank r holds frames r and r + N of the config-4 video (device
    # resident, alternated step by step); rows: every rank the same target
    mode = args.mode if world > 1 or args.mode != "targets" else "targets"
    frames = []
    if mode == "frames":
        frames = [wl.config4_frame((rank + k * world) % 30) for k in range(2)]
        case = frames[0]
    elif mode == "rows":
        case = wl.config2() if args.config == "config2" else wl.config3()
    else:
        center = shard.target_center(rank, world)
        case = (wl.config2(target_center=center) if args.config == "config2"
                else wl.config3())
    cfg = case.cfg
    M = cfg.views
    model = q.Model(cfg, device=local)
    model.init_weights(case.seed)
    enc = torch.from_numpy(case.enc_images).to(dev)
    ren = torch.from_numpy(case.ren_images).to(dev)
    fr_dev = [(torch.from_numpy(f.enc_images).to(dev), torch.from_numpy(f.ren_images).to(dev))
              for f in frames]
    plan = q.plan_forward(cfg, enc.shape[1], enc.shape[2])
    Ho, Wo = plan.out_height, plan.out_width
    rgb = torch.empty((Ho, Wo, 3), dtype=torch.float32, device=dev)
    # rows: this rank's band of the output, gathered into rgb every step
    band_rows = Ho // world if mode == "rows" else Ho
    if mode == "rows" and Ho % world:
        raise SystemExit(f"--mode rows needs the {Ho} output rows divisible by {world}")
    r0, r1 = rank * band_rows, (rank + 1) * band_rows
    band = torch.empty((band_rows, Wo, 3), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    # one dedicated stream carries the frames, the L2 flushes and the timing
    # events (the library enqueues every kernel of the frame on it)
    stream = torch.cuda.Stream(device=dev)

    He, We = enc.shape[1], enc.shape[2]
    K = cfg.pyramid_levels
    # N > 1: the encoder is view-sharded -- rank r encodes views
    # view_range(r) of the frame and the pyramid levels are all-gathered over
    # NVLink (NCCL, on the frame stream) -- then every rank reconstructs and
    # renders its own target from the full pyramid
    sharded = (world > 1 and mode == "targets") or args.shard_encoder
    v0, v1 = shard.view_range(rank, world, M)
    levels = []

    # N > 1 exchange: fused into the encoder (each rank's pooled levels stored
    # straight into every peer's pyramid over NVLink, then a one-element NCCL
    # all-reduce as the stream-ordered barrier) or an NCCL all-gather
    exchange = "nccl"
    barrier_t = None
    if sharded and world > 1 and args.exchange == "fused":
        ok = 1
        try:
            mine = model.pyramid_export((He, We))
            handles = [None] * world
            dist.all_gather_object(handles, mine)
            model.pyramid_import([h for r, h in enumerate(handles) if r != rank])
        except Exception as e:  # reported; every rank then uses the all-gather
            print(f"rank {rank}: fused pyramid exchange unavailable ({e})", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            exchange = "fused"
            barrier_t = torch.zeros(1, dtype=torch.int32, device=dev)
        else:
            model.pyramid_import([])

    def exchange_levels():
        if exchange == "fused":
            dist.all_reduce(barrier_t)  # every rank's encoder (and its peer stores) done
        else:
            for lv in levels:
                shard.allgather_views(lv, M)

    nstep = [0]

    def step():
        if mode == "frames":
            f = frames[nstep[0] % len(frames)]
            e, r = fr_dev[nstep[0] % len(frames)]
            nstep[0] += 1
            model.forward_render_device(e, f.enc_cams, r, f.ren_cams, f.target, rgb, stream)
            return
        if mode == "rows":
            model.forward_render_device(enc, case.enc_cams, ren, case.ren_cams, case.target, band,
                                        stream, rows=(r0, r1))
            if world > 1:
                dist.all_gather_into_tensor(rgb, band)  # the band gather (NCCL, frame stream)
            else:
                rgb.copy_(band)
            return
        if not sharded:
            model.forward_render_device(enc, case.enc_cams, ren, case.ren_cams, case.target, rgb,
                                        stream)
            return
        if exchange == "fused":
            dist.all_reduce(barrier_t)  # no rank still reads the pyramid the encode overwrites
        model.encode_device(enc, v0, v1, stream)
        exchange_levels()
        model.forward_render_device(None, case.enc_cams, ren, case.ren_cams, case.target, rgb,
                                    stream, enc_hw=(He, We))

    # warm-up (the first also sizes the arena); the last one is profiled per
    # stage with CUDA events (never inside the timed region). N > 1 profiles
    # the full single-GPU frame so the stage table means the same at every N.
    with torch.cuda.stream(stream):
        if sharded:
            model.encode_device(enc, 0, M, stream)
            levels = [model.pyramid_level(k) for k in range(K)]
        for i in range(args.warmup):
            if i == args.warmup - 1:
                model.profile(True)
                model.forward_render_device(enc, case.enc_cams, ren, case.ren_cams, case.target,
                                            rgb, stream)
                torch.cuda.synchronize()
                stages = model.profile_read()
                model.profile(False)
            step()
            torch.cuda.synchronize()
        if sharded:
            model.encode_device(enc, v0, v1, stream)
            n_enc = model.last_launch_count()
            model.forward_render_device(None, case.enc_cams, ren, case.ren_cams, case.target, rgb,
                                        stream, enc_hw=(He, We))
            launches_per_step = n_enc + model.last_launch_count()
        else:
            step()
            launches_per_step = model.last_launch_count()
        torch.cuda.synchronize()

    # timed region: K frames, per-frame CUDA events, L2 flushed between frames
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks, torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    ms_max = shard.max_over_ranks(ms, dev)
    ms_per_step = ms_max / args.steps
    # frames / targets: every rank completes a frame per step; rows: the ranks
    # complete one frame together per step
    units = 1 if mode == "rows" else world
    fps = shard.aggregate_fps(units, args.steps, ms_max / 1000.0)

    # e2e through the host C ABI: pinned host inputs, H2D + forward + render +
    # D2H of the frame, every step
    e2e = None
    if not args.no_e2e:
        enc_h = torch.from_numpy(case.enc_images).pin_memory()
        ren_h = torch.from_numpy(case.ren_images).pin_memory()
        out_h = torch.empty((Ho, Wo, 3), dtype=torch.float32).pin_memory()
        e_np, r_np, o_np = enc_h.numpy(), ren_h.numpy(), out_h.numpy()
        outs = [o_np, torch.empty_like(out_h).pin_memory().numpy()]
        pending = []
        nsub = [0]

        host_frames = [(torch.from_numpy(f.enc_images).pin_memory().numpy(),
                        torch.from_numpy(f.ren_images).pin_memory().numpy(), f) for f in frames]

        # rows / view-sharded targets: the same two-frames-in-flight pipeline
        # as lvsg_submit_frame, built from the device entry points -- frame
        # k+1's uploads (own stream) run under frame k's solve, frame k's
        # read-back (own stream) under frame k+1's; two device slots of the
        # uploaded images and of the frame, released by a host wait on the
        # read-back of frame k-1 before frame k+1 is enqueued
        piped = mode == "rows" or sharded
        if piped:
            h2d_s = torch.cuda.Stream(device=dev)
            d2h_s = torch.cuda.Stream(device=dev)
            enc_d = [enc, torch.empty_like(enc)]
            ren_d = [ren, torch.empty_like(ren)]
            rgb_d = [rgb, torch.empty_like(rgb)]
            outs_t = [out_h, torch.empty_like(out_h).pin_memory()]
            up_ev = [torch.cuda.Event(), torch.cuda.Event()]
            done_ev = [torch.cuda.Event(), torch.cuda.Event()]
            slot_busy = [False, False]

        def piped_step():
            s = nsub[0] % 2
            nsub[0] += 1
            if slot_busy[s]:
                done_ev[s].synchronize()  # frame k-1 (this slot) read back: slot free
            with torch.cuda.stream(h2d_s):
                if mode == "rows":
                    enc_d[s].copy_(enc_h, non_blocking=True)
                else:
                    enc_d[s][v0:v1].copy_(enc_h[v0:v1], non_blocking=True)
                ren_d[s].copy_(ren_h, non_blocking=True)
                up_ev[s].record(h2d_s)
            with torch.cuda.stream(stream):
                stream.wait_event(up_ev[s])
                if mode == "rows":
                    model.forward_render_device(enc_d[s], case.enc_cams, ren_d[s], case.ren_cams,
                                                case.target, band, stream, rows=(r0, r1))
                    if world > 1:
                        dist.all_gather_into_tensor(rgb_d[s], band)
                    else:
                        rgb_d[s].copy_(band)
                else:
                    if exchange == "fused":
                        dist.all_reduce(barrier_t)  # no rank still reads the pyramid
                    model.encode_device(enc_d[s], v0, v1, stream)
                    exchange_levels()
                    model.forward_render_device(None, case.enc_cams, ren_d[s], case.ren_cams,
                                                case.target, rgb_d[s], stream, enc_hw=(He, We))
                d2h_s.wait_stream(stream)
            with torch.cuda.stream(d2h_s):
                if rank == 0 or mode != "rows":
                    outs_t[s].copy_(rgb_d[s], non_blocking=True)
                done_ev[s].record(d2h_s)
            slot_busy[s] = True

        def piped_drain():
            for s in range(2):
                if slot_busy[s]:
                    done_ev[s].synchronize()
                    slot_busy[s] = False

        def e2e_step():
            if piped:
                piped_step()
                return
            if mode == "frames":
                # pipelined host frames, this rank's share of the video
                if len(pending) == 2:
                    model.wait_frame(pending.pop(0))
                e_h, r_h, f = host_frames[nsub[0] % len(host_frames)]
                pending.append(model.submit_frame(e_h, f.enc_cams, r_h, f.ren_cams, f.target,
                                                  outs[nsub[0] % 2]))
                nsub[0] += 1
                return
            # pipelined host frames (lvsg_submit_frame / lvsg_wait_frame): at
            # most two in flight, so frame k+1's uploads run under frame k
            if len(pending) == 2:
                model.wait_frame(pending.pop(0))
            pending.append(model.submit_frame(e_np, case.enc_cams, r_np, case.ren_cams,
                                              case.target, outs[nsub[0] % 2]))
            nsub[0] += 1

        for _ in range(3):  # warm-up: both frame slots allocate their buffers
            e2e_step()
        while pending:
            model.wait_frame(pending.pop(0))
        if piped:
            piped_drain()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
            if os.environ.get("LVSG_BENCH_DEBUG"):
                print(f"e2e step {time.perf_counter() - t0:.4f}", file=sys.stderr)
        while pending:
            model.wait_frame(pending.pop(0))
        if piped:
            piped_drain()
        sec = shard.max_over_ranks(time.perf_counter() - t0, dev)
        h2d = (enc_h[v0:v1].numel() if sharded else enc_h.numel()) * 4 + ren_h.numel() * 4
        d2h = out_h.numel() * 4 if (rank == 0 or mode != "rows") else 0
        e2e = {"value": shard.aggregate_fps(units, args.e2e_steps, sec), "unit": "frames/s",
               "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps,
               "path": ("lvsg_submit_frame / lvsg_wait_frame (host C ABI, pinned buffers, "
                        "two frames in flight)" if not piped
                        else "pinned host views -> device (every rank, upload stream) -> "
                        "lvsg_forward_render_rows_device (this rank's band) -> NCCL all-gather "
                        "of the bands -> rank 0 reads the frame back (read-back stream); two "
                        "frames in flight" if mode == "rows" else
                        "pinned host views (own encoder share + render views, upload stream) "
                        "-> lvsg_encode_device -> pyramid exchange -> "
                        "lvsg_forward_render_device (resident pyramid) -> pinned frame "
                        "(read-back stream); two frames in flight")}
        if not sharded and mode == "targets":
            # input-side decimation variant: only the
            # 1080p views are uploaded; the encoder input is their device
            # resize to 576 x 960 (a different encoder input than the
            # analytic 576 x 960 views above, so reported beside, not as, e2e)
            def dec_step():
                if len(pending) == 2:
                    model.wait_frame(pending.pop(0))
                pending.append(model.submit_frame_decimated(r_np, case.ren_cams, case.target,
                                                            (He, We), outs[nsub[0] % 2]))
                nsub[0] += 1
            for _ in range(3):
                dec_step()
            while pending:
                model.wait_frame(pending.pop(0))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                dec_step()
            while pending:
                model.wait_frame(pending.pop(0))
            sec = time.perf_counter() - t0
            e2e["decimated"] = {"value": args.e2e_steps / sec, "unit": "frames/s",
                                "h2d_bytes_per_step": int(ren_h.numel() * 4),
                                "d2h_bytes_per_step": int(out_h.numel() * 4),
                                "path": "lvsg_submit_frame_decimated / lvsg_wait_frame (1080p "
                                        "views only; device resize to the encoder extents)"}

    if rank == 0:
        peaks = load_peaks()
        work = frame_work(cfg, enc.shape[1], enc.shape[2], ren.shape[1], ren.shape[2])
        stage_rows = {}
        for k, (sms, n) in stages.items():
            stage_rows[k] = {"ms": round(sms, 4), "launches": n}
        if "conv" in stages:
            sec = stages["conv"][0] / 1e3
            ach = work["conv_flops"] / sec / 1e12
            stage_rows["conv"].update(gbs=round(work["conv_bytes"] / sec / 1e9, 1),
                                      frac_hbm=round(work["conv_bytes"] / sec / 1e9 / peaks["hbm_gbs"], 4),
                                      tflops=round(ach, 2),
                                      frac_bf16_peak=round(ach / peaks["bf16_tflops"], 4))
        if "attention" in stages:
            ach = work["attn_flops"] / (stages["attention"][0] / 1e3) / 1e12
            stage_rows["attention"].update(tflops=round(ach, 2))
        if "render" in stages:
            gbs = work["render_bytes"] / (stages["render"][0] / 1e3) / 1e9
            stage_rows["render"].update(gbs=round(gbs, 1), frac_hbm=round(gbs / peaks["hbm_gbs"], 4))
        dom = max(stages.items(), key=lambda kv: kv[1][0])[0] if stages else None
        # DRAM bytes measured by ncu for the same command (profiles/r2/traffic.json,
        # made by profiles/traffic_summary.py from a dram__bytes launch list)
        traffic = {}
        for tj in (os.path.join(ROOT, "profiles", "r2", "traffic.json"),
                   os.path.join(ROOT, "profiles", "r1", "traffic.json")):
            if os.path.exists(tj):
                traffic = json.load(open(tj))
                break
        if dom == "conv":
            # the conv family is HBM-bound at C = 32 fp32 activations (~55
            # FLOP/B against a bf16 ridge of ~250): roofline in bytes
            sec = stages["conv"][0] / 1e3
            gbs = work["conv_bytes"] / sec / 1e9
            tfl = work["conv_flops"] / sec / 1e12
            tc = traffic.get("conv3x3", {})
            roof = {"bound": "hbm",
                    "kernel": "conv3x3_tc_kernel (all conv3x3 launches of a frame)",
                    "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": gbs / peaks["hbm_gbs"],
                    "traffic": tc.get("dram_bytes_per_frame"),
                    "traffic_note": (f"ncu dram__bytes_read+write summed over the frame's "
                                     f"{tc.get('launches')} conv launches ({tc.get('source')}) "
                                     f"vs {work['conv_bytes'] / 1e9:.2f} GB algorithmic"
                                     if tc else None),
                    "per_unit": (f"{work['conv_bytes'] / 1e9:.2f} GB algorithmic per frame (each "
                                 "conv reads its inputs and residual once and writes its output "
                                 f"once); {work['conv_flops'] / 1e9:.1f} GFLOP"),
                    "peak_source": peaks["source"] + ", HBM copy bandwidth",
                    "tensor": {"achieved_tflops": tfl, "peak_tflops": peaks["bf16_tflops"],
                               "frac": tfl / peaks["bf16_tflops"],
                               "note": "fp32 conv FLOPs run as a 3-term fp16 split (3 tensor "
                                       "MACs per fp32 MAC): the split's ceiling is peak/3"}}
        elif dom == "render":
            gbs = work["render_bytes"] / (stages["render"][0] / 1e3) / 1e9
            roof = {"bound": "hbm", "kernel": "render_fused_kernel", "achieved": gbs,
                    "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"],
                    "traffic": None, "peak_source": peaks["source"]}
        else:
            roof = {"bound": "hbm", "kernel": dom, "achieved": None, "peak": peaks["hbm_gbs"],
                    "unit": "GB/s", "frac": None, "traffic": None}
        if "frame_dram_bytes" in traffic:
            # whole-frame DRAM traffic (ncu, every launch of one frame) over the
            # device-timed frame
            fb = traffic["frame_dram_bytes"]
            roof["frame_dram"] = {"bytes": fb, "gbs": fb / (ms_per_step / 1e3) / 1e9,
                                  "frac": fb / (ms_per_step / 1e3) / 1e9 / peaks["hbm_gbs"],
                                  "source": traffic.get("source")}
        roof["stages"] = stage_rows
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            try:
                cpu = cpu_baseline_single()
            except Exception as e:  # reported, never fatal
                cpu = {"value": None, "error": str(e)}
        if mode == "frames":
            per_gpu = (f"config-4 video frames {rank}, {rank}+{world}, ... (2 resident frames "
                       "per rank, alternated), full forward + render each")
            par = f"frame-sharded x{world}, no data-path collective" if world > 1 else "single GPU"
        elif mode == "rows":
            per_gpu = (f"one target: the replicated solve + output rows "
                       f"[{r0}, {r1}) of {Ho}")
            par = (f"row-band x{world}: replicated solve, band render, NCCL all-gather of the "
                   "bands every frame" if world > 1 else "single GPU")
        else:
            per_gpu = ("one target viewpoint per rank (config-5 grid), "
                       f"{v1 - v0} of {M} encoder views per rank") if world > 1 else "1 target"
            par = (f"target-sharded x{world}; encoder view-sharded, pyramid "
                   + ("exchange fused into the encoder epilogue (CUDA IPC stores over NVLink + "
                      "NCCL one-element barrier)" if exchange == "fused" else
                      "all-gathered per level with NCCL") + " per frame") \
                if world > 1 else "single GPU"
        out = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if mode == "rows" else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (make_scene seed 21 plane scene, init_param_store seed 3 weights)",
            "config": {"workload": f"{args.config}: {M} views, full_scale_config, encoder "
                                   f"{enc.shape[1]}x{enc.shape[2]}, render {ren.shape[1]}x"
                                   f"{ren.shape[2]}, output {Ho}x{Wo}"
                                   + (" (config-4 video frames)" if mode == "frames" else ""),
                       "mode": mode, "per_gpu": per_gpu,
                       "l2": "flushed (256 MB write) between timed frames",
                       "parallelism": par},
            "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "roofline": roof, "cpu_baseline": cpu, "clocks": clocks.summary(),
        }
        print(json.dumps(out))
    torch.cuda.synchronize()
    model.close()  # release the context before torch tears CUDA down
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
