#!/usr/bin/env python
"""Benchmark: frames/s of the accelerated PIFu path (256^3 progressive
reconstruction + 512x512 mesh-free render, BASELINE.json configs[2]) on 1..N
B200s, frames sharded round-robin (configs[4] pattern: a stream of distinct
seeded frames, shared weights).

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--config config2|config3]

With --gpus N > 1 and no torchrun environment, bench.py launches N ranks
itself (torch.distributed.run, 127.0.0.1); under torchrun WORLD_SIZE must
equal N.  One rank per GPU, no collective on the per-frame path
(torch.distributed only for the barriers and the max-over-ranks timing).

A step = one frame per GPU.  `value` = frames of all ranks / max-over-ranks
device time of the K timed frames (CUDA events on the library's streams,
inputs resident in HBM, L2 flushed before every frame).  `e2e` = the same
through the C ABI with pinned HOST buffers (feature map H2D + depth/RGB/mask/
crossing-index D2H inside every timed call).  `roofline` = the column-factored
geometry field of the bulk batches (algorithmic 2,363,906 FLOP per evaluated
point) against the measured bf16 tensor burst peak.
`cpu_baseline` = one full frame of the CPU port (rank 0, N=1).
`--impl reference` = the CPU path on all host threads, a full frame per step.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import itertools
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

GEO_FLOP_PER_POINT = 2363906
FACT_MMA_FLOP_PER_POINT = 2 * (512 * 1024 + 256 * 512 + 128 * 256)  # hidden parts of layers 2-4
TEX_FLOP_PER_POINT = 3350022 + 2231808
METRIC = "frames/sec (256^3 recon + 512² render) at 1/2/4/8 B200; MLP points/sec vs TC peak"
# BASELINE configs[4]: a stream of 64 independent seeded frames, round-robin over the GPUs (config 3's
# 67 MB feature maps: 16 distinct frames)
STREAM_FRAMES = {"config2": 64, "config3": 16}
L2_FLUSH_BYTES = 256 << 20  # > 2x the 126 MB L2

CONFIGS = {
    # name: (coarsest, level, fmap (C,H,W), render W=H, precision)
    "config2": (32, 3, (256, 128, 128), 512, "fp32"),
    "config3": (32, 4, (256, 256, 256), 1024, "bf16"),
}
DTYPES = {
    "fp32": ("bf16x3", {"geometry_mlp": "bf16x3 split products, fp32 accumulation (fp32-accurate: |docc| <= 4.4e-6)",
                        "texture_mlp": "fp16 weights and activations (one copy each), fp32 accumulation, bias, z term and output layer (colours within 4.0e-4 of fp64 over 20k random points; bar 1e-3)",
                        "grid": "f32 values, u8 states", "render": "f32 (bit-exact vs the fp32 oracle)"}),
    "bf16": ("bf16", {"geometry_mlp": "bf16 operands, fp32 accumulation", "texture_mlp": "fp16 operands, fp32 "
                      "accumulation", "grid": "f32 values, u8 states", "render": "f32"}),
    "simt": ("f32", {"geometry_mlp": "fp32 CUDA-core FFMA", "texture_mlp": "fp32 CUDA-core FFMA", "grid": "f32"}),
}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


class ClockSampler:
    """Samples nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        # nvidia-smi needs a moment before its first row: do not start timing blind
        t0 = time.time()
        while not self.rows and time.time() - t0 < 10 and self.proc.poll() is None:
            time.sleep(0.05)
        self.rows.clear()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def stream_seed(f: int) -> int:
    """Feature-map seed of frame f of the configs[4] stream (weights shared: seeds 7 / 8)."""
    return 1000 + f


def workload_config(cfg_name: str, args, world: int) -> dict:
    """The workload only (same dict in both arms: the driver compares them)."""
    r0, lv, (c, h, w), res, _ = CONFIGS[cfg_name]
    return {"workload": f"{cfg_name}: progressive PIFu localization {r0}->{r0 << lv} cells ({(r0 << lv)}^3 grid), "
                        f"feature map {c}x{h}x{w}, {res}x{res} first-crossing render yaw 90 + texture MLP; a stream "
                        f"of {STREAM_FRAMES[cfg_name]} distinct seeded frames (feature seeds 1000..{999 + STREAM_FRAMES[cfg_name]}, shared "
                        "weights), frame f on GPU f mod N (configs[4] pattern)",
            "precision": CONFIGS[cfg_name][4] if args.precision is None else args.precision,
            "stream_frames": STREAM_FRAMES[cfg_name],
            "l2": "flushed before every timed frame (256 MB = 2x L2 written on the frame's stream)",
            "parallelism": f"frame-sharded x{world}, no per-frame collective"}


# ---------------------------------------------------------------------------
# Reference arm: the CPU path, full frames, all host threads (oracle/ only)
# ---------------------------------------------------------------------------
def cpu_frame(O, cfg_name: str, fmap, caps, gw, gb, tw, tb, threads: int):
    """One full frame through the CPU port (oracle/liborc.so, the restatement pinned bit-exact to
    the reference's extract_progressive by tests/test_oracle_vs_reference.py): progressive
    localization with the batched fp64 PIFu field + first-crossing render + texture at the
    covered pixels.  Returns (seconds, evals, covered)."""
    r0, lv, _, res, _ = CONFIGS[cfg_name]
    m = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=threads)
    cam = O.camera_from_angles(90, 0)
    t0 = time.perf_counter()
    ext = O.extract_progressive(m, r0, lv)
    r = O.render_first_crossing(ext["values"], r0 << lv, cam, res, res, tex=m)
    return time.perf_counter() - t0, ext["total_evals"], int(r["covered"])


def reference_arm(args, cfg_name: str, world: int):
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    _, _, (c, h, w), _, _ = CONFIGS[cfg_name]
    caps = O.gen_capsules(42)
    gw, gb = O.gen_mlp(7, 0)
    tw, tb = O.gen_mlp(8, 1)
    nmaps = min(STREAM_FRAMES[cfg_name], max(1, args.warmup + args.steps))
    maps = [O.gen_feature_map(stream_seed(f), c, h, w) for f in range(min(nmaps, 4))]
    for i in range(args.warmup):
        cpu_frame(O, cfg_name, maps[i % len(maps)], caps, gw, gb, tw, tb, threads)
    times, evals, cov = [], [], []
    for i in range(args.steps):
        t, e, cv = cpu_frame(O, cfg_name, maps[i % len(maps)], caps, gw, gb, tw, tb, threads)
        times.append(t)
        evals.append(e)
        cov.append(cv)
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg_name, args, world),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": f"every step one FULL {cfg_name} frame (no sampling, no extrapolation): "
                                   f"progressive localization ({int(np.mean(evals))} evals/frame) with the batched "
                                   f"fp64 PIFu field + {CONFIGS[cfg_name][3]}^2 first-crossing render + texture at "
                                   f"{int(np.mean(cov))} covered pixels, through oracle/liborc.so (the C restatement "
                                   "pinned bit-exact to the reference's extract_progressive, oracle/_ref) on "
                                   f"{threads} host threads; feature maps cycle over {len(maps)} seeds"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "frame_seconds": {"p50": float(np.percentile(times, 50)), "max": float(max(times))},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# launcher: N ranks, one per GPU
# ---------------------------------------------------------------------------
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """Re-launch this script as n ranks (torch.distributed.run on 127.0.0.1); returns the exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def init_world(args):
    """(rank, world, local_rank, dist module or None); spawns the ranks when needed (returns None)."""
    if "WORLD_SIZE" not in os.environ:
        if args.gpus > 1:
            return None
        return 0, 1, 0, None
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ["WORLD_SIZE"])
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; launch one rank per GPU")
    if world == 1:
        return rank, world, local_rank, None
    import torch.distributed as td
    if args.dry_run:
        td.init_process_group("gloo")
    else:
        import torch
        torch.cuda.set_device(local_rank)
        td.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    return rank, world, local_rank, td


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class DryLane:
    """--dry-run (CPU tests of the launcher / rank loop / allmax / JSON line): no device work."""

    def __init__(self, rank, s):
        self.rank, self.lat, self.k = rank, [], 0

    def frame(self, host=False, flush=True):
        self.lat.append(1.0)
        self.k += 1


def gpu_arm(args, cfg_name: str, rank: int, world: int, local_rank: int, dist):
    from paper_2007_13988_b200 import shard
    r0, lv, (C_, H_, W_), res, prec_name = CONFIGS[cfg_name]
    if args.precision:
        prec_name = args.precision
    S = max(1, args.streams)
    my_frames = shard.frames_for_rank(STREAM_FRAMES[cfg_name], rank, world)  # configs[4]: frame f on rank f mod N
    fbytes = C_ * H_ * W_ * 4
    npx = res * res
    dev = f"cuda:{local_rank}" if (dist and not args.dry_run) else None

    if args.dry_run:
        lanes = [DryLane(rank, s) for s in range(S)]
        ctxs = None
    else:
        import ctypes as C

        from paper_2007_13988_b200 import abi, api
        prec = {"fp32": abi.ICG_PREC_FP32, "bf16": abi.ICG_PREC_BF16, "simt": abi.ICG_PREC_FP32_SIMT}[prec_name]
        caps = api.gen_capsules(42)
        gw, gb = api.gen_mlp(7, 0)
        tw, tb = api.gen_mlp(8, 1)
        cfg = api.AlgoConfig("progressive", r0, lv)
        cam = api.CameraSpec.from_angles(90, 0)

        def img_struct(bufs, mem):
            img = abi.icg_image()
            img.mem = mem
            img.depth = C.cast(C.c_void_p(bufs["depth"]), abi.f32p)
            img.rgb = C.cast(C.c_void_p(bufs["rgb"]), abi.f32p)
            img.mask = C.cast(C.c_void_p(bufs["mask"]), abi.u8p)
            img.surface_k = C.cast(C.c_void_p(bufs["sk"]), abi.i32p)
            return img

        class Lane:
            """One context (stream) of this GPU: its own frames in flight, driven by one host thread.
            Lane s owns this rank's stream frames s, s + S, ... (each a distinct seeded feature map)."""

            def __init__(self, s):
                self.ctx = api.Context(local_rank)
                self.ctx.set_mlp(abi.ICG_MLP_GEOMETRY, gw, gb)
                self.ctx.set_mlp(abi.ICG_MLP_TEXTURE, tw, tb)
                self.host_maps, self.dev_maps = [], []
                for f in my_frames[s::S] or my_frames[:1]:
                    fm = api.gen_feature_map(stream_seed(f), C_, H_, W_)
                    hp = api.host_alloc(fbytes)
                    np.ctypeslib.as_array((C.c_float * fm.size).from_address(hp))[:] = fm.reshape(-1)
                    dp = self.ctx.device_alloc(fbytes)
                    self.ctx.memcpy(dp, hp, fbytes, abi.ICG_MEM_DEVICE, abi.ICG_MEM_HOST)
                    self.host_maps.append(hp)
                    self.dev_maps.append(dp)
                self.fields_dev = [api.PifuField(None, caps, 50.0, prec, device_ptr=dp, shape=(C_, H_, W_))
                                   for dp in self.dev_maps]
                self.fields_host = []
                for hp in self.host_maps:
                    f_ = api.PifuField(None, caps, 50.0, prec, device_ptr=hp, shape=(C_, H_, W_))
                    f_.c.fmap_mem = abi.ICG_MEM_HOST
                    self.fields_host.append(f_)
                sizes = (("depth", npx * 4), ("rgb", npx * 12), ("mask", npx), ("sk", npx * 4))
                self.dout = img_struct({k: self.ctx.device_alloc(b) for k, b in sizes}, abi.ICG_MEM_DEVICE)
                self.hout = img_struct({k: api.host_alloc(b) for k, b in sizes}, abi.ICG_MEM_HOST)
                self.flush_buf = self.ctx.device_alloc(L2_FLUSH_BYTES)
                self.grid_v = self.grid_s = None
                self.lat = []
                self.k = 0

            def flush_l2(self):  # write a buffer twice the size of L2 on the frame's stream
                self.ctx.memset(self.flush_buf, self.k & 0xFF, L2_FLUSH_BYTES)

            def frame(self, host=False, flush=True, grid=False):
                if flush:
                    self.flush_l2()
                f = (self.fields_host if host else self.fields_dev)[self.k % len(self.dev_maps)]
                self.k += 1
                ext = None
                if grid:  # e2e variant that also returns the localized grid (values + states) to the host
                    n3 = ((r0 << lv) + 1) ** 3
                    if self.grid_v is None:
                        self.grid_v, self.grid_s = api.host_alloc(4 * n3), api.host_alloc(n3)
                    ext = abi.icg_extraction()
                    ext.mem = abi.ICG_MEM_HOST
                    ext.values = C.cast(C.c_void_p(self.grid_v), abi.f32p)
                    ext.states = C.cast(C.c_void_p(self.grid_s), abi.u8p)
                ext, img = self.ctx.frame_raw(f, cfg, cam, res, res, self.hout if host else self.dout, ext)
                self.lat.append(img.wall_seconds * 1e3)

        lanes = [Lane(s) for s in range(S)]
        ctxs = [ln.ctx for ln in lanes]

    def allmax(x: float) -> float:
        return shard.allmax(x, device=dev)

    def run_frames(nframes: int, **kw) -> float:
        """nframes frames over the lanes (one host thread per lane, dynamic hand-out); returns the
        device-timed span in ms (CUDA events: common start event, last stream's end event)."""
        counts = [nframes // S + (1 if i < nframes % S else 0) for i in range(S)]
        if args.dry_run:
            t0 = time.perf_counter()
            for ln, c in zip(lanes, counts):
                for _ in range(c):
                    ln.frame(**kw)
            return 1e3 * (time.perf_counter() - t0)
        from paper_2007_13988_b200 import api as _api
        # frames are handed out dynamically (the next frame goes to the first lane that is free), so no
        # lane idles at the end of the span while another still has a queue
        ticket = itertools.count()

        def lane_loop(ln):
            while next(ticket) < nframes:
                ln.frame(**kw)

        _api.span_begin(ctxs)
        ths = [threading.Thread(target=lane_loop, args=(ln,)) for ln in lanes]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return _api.span_end(ctxs)

    # ---- warm-up (every lane, every feature map of the lane once) ----
    for ln in lanes:
        for _ in range(max(args.warmup, 1 if args.dry_run else len(ln.dev_maps))):
            ln.frame()
    # ... and with every lane in flight: a frame that shares its device runs the conflict-loop tail
    # on fewer SMs, a different frame graph than the frames above (one eager run, then the capture)
    if S > 1:
        run_frames(3 * S)
    # ---- single-frame latency: one lane, frames back to back (device time per frame) ----
    lat_lane = lanes[0]
    lat_lane.lat = []
    for _ in range(min(args.steps, 30)):
        lat_lane.frame()
    single_lat = list(lat_lane.lat)
    # ---- timed: S frames in flight, device-resident inputs and outputs ----
    for ln in lanes:
        ln.lat = []
    shard.barrier()
    clocks = None
    if not args.dry_run:
        cvd = [d for d in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if d.strip().isdigit()]
        clocks = ClockSampler(int(cvd[local_rank]) if local_rank < len(cvd) else local_rank)
        clocks.start()
    t_wall0 = time.perf_counter()
    span_ms = run_frames(args.steps)
    wall = time.perf_counter() - t_wall0
    clk = clocks.stop() if clocks else None
    lat = sum((ln.lat for ln in lanes), [])
    shard.barrier()
    dev_max = allmax(span_ms / 1e3)
    value = world * args.steps / dev_max
    lat_p = [allmax(float(np.percentile(lat, q))) for q in (50, 99)]
    single_p = [allmax(float(np.percentile(single_lat, q))) for q in (50, 99)]

    prof = None
    e2e = e2e_grid = None
    if not args.dry_run:
        # ---- per-kernel breakdown: a separate single-lane pass with CUDA events around every launch
        # (the events themselves cost a little, so `value` is not taken here) ----
        ctx = lat_lane.ctx
        ctx.profile(True, reset=True)
        for _ in range(min(args.steps, 20)):
            lat_lane.frame()
        prof = ctx.profile_get()
        ctx.profile(False, reset=False)
        # ---- e2e: pinned host inputs/outputs through the C ABI (H2D + D2H inside every call) ----
        if not args.no_e2e:
            for ln in lanes:
                for _ in range(2):
                    ln.frame(host=True, flush=False)
            shard.barrier()
            e2e_t = allmax(run_frames(args.steps, host=True, flush=True) / 1e3)
            e2e = {"value": world * args.steps / e2e_t, "unit": "frames/s", "h2d_bytes_per_step": fbytes,
                   "d2h_bytes_per_step": npx * (4 + 12 + 1 + 4),
                   "note": "feature map H2D + depth/RGB/mask/first-crossing-index D2H in every timed call, L2 flushed "
                           "before each; the localized grid stays on the device (see e2e_with_grid)"}
            for ln in lanes:
                ln.frame(host=True, flush=False, grid=True)
            shard.barrier()
            n3 = ((r0 << lv) + 1) ** 3
            eg_t = allmax(run_frames(args.steps, host=True, flush=True, grid=True) / 1e3)
            e2e_grid = {"value": world * args.steps / eg_t, "unit": "frames/s", "h2d_bytes_per_step": fbytes,
                        "d2h_bytes_per_step": npx * (4 + 12 + 1 + 4) + 5 * n3,
                        "note": "as e2e, plus the final grid (f32 values + u8 states) D2H every frame"}

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": DTYPES[prec_name][0], "dtype_detail": DTYPES[prec_name][1],
        "data": "synthetic (seeded N(0,1) feature maps, Kaiming-uniform weights, 15-capsule sdf bias)",
        "config": workload_config(cfg_name, args, world),
        "frame_latency_ms": {"p50": lat_p[0], "p99": lat_p[1], "frames": len(lat),
                             "note": f"device time of one frame with {S} frames in flight per GPU (max over ranks)"},
        "single_frame_latency_ms": {"p50": single_p[0], "p99": single_p[1], "frames": len(single_lat),
                                    "note": "one frame at a time on one stream (north-star target < 5 ms)"},
        "wall_ms_per_step": 1e3 * wall / args.steps, "frames_in_flight_per_gpu": S,
        "e2e": e2e, "e2e_with_grid": e2e_grid, "clocks": clk, "streams": S,
    }
    if prof is not None:
        pk = peaks()
        peak_t = pk.get("bf16_tflops", 1662.9)
        fact_s = prof["fact_ms"] / 1e3
        fact_pts = prof["fact_points"]
        exec_mult = 3 if prec_name == "fp32" else 1
        achieved = fact_pts * GEO_FLOP_PER_POINT / fact_s / 1e12 if fact_s > 0 else 0.0
        executed = fact_pts * FACT_MMA_FLOP_PER_POINT * exec_mult / fact_s / 1e12 if fact_s > 0 else 0.0
        traffic, traffic_note = None, None
        try:  # DRAM bytes of the longest k_fact2 launch of a frame, from the committed ncu --set full capture
            cap = f"r02d_ncu_full_k_fact2_{cfg_name}.json"
            rec = json.load(open(os.path.join(ROOT, "profiles", cap)))[0]
            mb = lambda v: float(v.split()[0]) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[v.split()[1]]
            traffic = (mb(rec["dram__bytes_read.sum"]) + mb(rec["dram__bytes_write.sum"])) * 1e6
            traffic_note = (f"dram__bytes_read.sum + dram__bytes_write.sum of the frame's longest k_fact2 launch "
                            f"(the last level's E0 list, profiles/{cap}): column records (bulk-prefetched into L2), "
                            f"weights and lists")
        except Exception:
            pass
        line["roofline"] = {
            "bound": "tensor",
            "kernel": "geometry field, bulk batches (dense level 0 + each level's E0 list): column gather + "
                      "column GEMM k_cols (M = 256 columns x N = 256 outputs) + factored pass k_fact2 (CTA-pair "
                      "tcgen05, M = 256 points x N = 256 features), incl. list sorting",
            "achieved": achieved, "peak": peak_t, "unit": "TFLOP/s", "frac": achieved / peak_t,
            "traffic": traffic, "traffic_note": traffic_note,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst: each launch is timed alone by CUDA events)"
                           + (" (fallback)" if pk.get("fallback") else ""),
            "algorithmic_flop_per_point": GEO_FLOP_PER_POINT,
            "achieved_note": "dense-equivalent algorithmic FLOP (SURVEY §8(d)); the factored pass executes fewer",
            "executed_tflops": executed, "executed_frac": executed / peak_t,
            "executed_flop_per_point": FACT_MMA_FLOP_PER_POINT * exec_mult,
            "launches": prof["fact_launches"], "points": fact_pts,
            "avg_launch_ms": prof["fact_ms"] / max(1, prof["fact_launches"])}
        line["secondary"] = {
            "conflict_chain": {"points": prof["chain_points"], "ms": prof["chain_ms"],
                               "launches": prof["chain_launches"],
                               "ms_per_frame": prof["chain_ms"] / max(1, prof["frames"])},
            "geometry_all": {"points": prof["geo_points"], "ms": prof["geo_mlp_ms"],
                             "mlp_points_per_s": prof["geo_points"] / max(1e-9, prof["geo_mlp_ms"] / 1e3),
                             "achieved_tflops": prof["geo_points"] * GEO_FLOP_PER_POINT
                             / max(1e-9, prof["geo_mlp_ms"] / 1e3) / 1e12},
            "texture_mlp": {"points": prof["tex_points"], "ms": prof["tex_mlp_ms"],
                            "achieved_tflops": prof["tex_points"] * TEX_FLOP_PER_POINT
                            / max(1e-9, prof["tex_mlp_ms"] / 1e3) / 1e12,
                            "frac_of_burst": prof["tex_points"] * TEX_FLOP_PER_POINT
                            / max(1e-9, prof["tex_mlp_ms"] / 1e3) / 1e12 / peak_t},
            # every level's dense pass (binarize, mixed cells, upsample / carry / candidates, E0
            # compaction), the coarse levels being a few us each; the target level alone beside it
            "dense_passes": {"bytes": prof["dense_bytes"], "ms": prof["dense_ms"],
                             "launch_groups": prof["dense_launches"],
                             "achieved_gbs": prof["dense_bytes"] / max(1e-9, prof["dense_ms"] / 1e3) / 1e9,
                             "peak_gbs": pk.get("hbm_gbs")},
            "last_level_pass": {"bytes": prof["last_level_bytes"], "ms": prof["last_level_ms"],
                                "achieved_gbs": prof["last_level_bytes"] / max(1e-9, prof["last_level_ms"] / 1e3) / 1e9,
                                "frac_of_hbm": prof["last_level_bytes"] / max(1e-9, prof["last_level_ms"] / 1e3) / 1e9
                                / max(1e-9, pk.get("hbm_gbs") or 1e-9)},
            # the conflict loop's neighbour expansions (latency-bound chain links, not a dense pass)
            "conflict_expand": {"launches": prof["expand_launches"], "ms": prof["expand_ms"],
                                "ms_per_frame": prof["expand_ms"] / max(1, prof["frames"])},
            "render": {"bytes": prof["render_bytes"], "ms": prof["render_ms"],
                       "achieved_gbs": prof["render_bytes"] / max(1e-9, prof["render_ms"] / 1e3) / 1e9},
            # the texture field's Phi gather: 4 bilinear taps x C x 4 B per surface point (L2-resident map)
            "texture_gather": {"points": prof.get("gather_points", 0), "bytes": prof.get("gather_bytes", 0),
                               "ms": prof.get("gather_ms", 0.0),
                               "achieved_gbs": prof.get("gather_bytes", 0) / max(1e-9, prof.get("gather_ms", 0.0) / 1e3) / 1e9},
            "profiled_frames": prof["frames"], "profiled_frame_ms": prof["frame_ms"] / max(1, prof["frames"]),
            "evals_per_frame": int(prof["geo_points"] / max(1, prof["frames"])),
        }
        line["gpu_launches"] = int(round(prof["kernel_launches"] / max(1, prof["frames"]) * args.steps))
    if world == 1 and cfg_name == "config2" and args.config3 and not args.dry_run:
        # BASELINE configs[3] beside the headline (512^3 bf16, 1024^2): its own bench.py run
        cmd = [sys.executable, os.path.abspath(__file__), "--config", "config3", "--steps", str(min(args.steps, 10)),
               "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-config3"]
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=900).stdout
            c3 = json.loads([l for l in out.splitlines() if l.startswith("{")][-1])
            line["config3"] = {k: c3.get(k) for k in ("value", "unit", "ms_per_step", "steps", "dtype", "dtype_detail",
                                                      "single_frame_latency_ms", "roofline", "gpu_launches", "clocks")}
            line["config3"]["workload"] = c3["config"]["workload"]
            s3 = c3.get("secondary", {})
            line["config3"]["texture_mlp"] = s3.get("texture_mlp")
            line["config3"]["conflict_chain_ms_per_frame"] = s3.get("conflict_chain", {}).get("ms_per_frame")
            line["config3"]["bf16_target"] = {"target_frac_of_burst": 0.5,
                                              "met": (c3.get("roofline") or {}).get("frac", 0.0) >= 0.5}
        except Exception as e:  # noqa: BLE001 -- reported, never fatal for the headline
            line["config3"] = {"error": str(e)[:200]}
    if world == 1 and not args.no_cpu_baseline and not args.dry_run:
        from oracle import oracle as O
        threads = os.cpu_count() or 1
        _, _, (c, h, w), _, _ = CONFIGS[cfg_name]
        t, evals, cov = cpu_frame(O, cfg_name, O.gen_feature_map(stream_seed(0), c, h, w), O.gen_capsules(42),
                                  *O.gen_mlp(7, 0), *O.gen_mlp(8, 1), threads)
        line["cpu_baseline"] = {"value": 1.0 / t, "unit": "frames/s", "cores": threads, "kind": "port",
                                "sample": f"one full {cfg_name} frame (feature seed {stream_seed(0)}, {evals} evals, "
                                          f"{cov} covered pixels) through the CPU port oracle/liborc.so (fp64 "
                                          "batched MLP, all host threads)"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="config2", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default=None, choices=[None, "fp32", "bf16", "simt"])
    ap.add_argument("--streams", type=int, default=4,
                    help="frames in flight per GPU (one context + stream + host thread each)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-config3", dest="config3", action="store_false",
                    help="skip the BASELINE configs[3] (512^3 bf16) run reported beside the config-2 line")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)  # CPU tests of the rank loop
    args = ap.parse_args()
    if args.impl == "reference":
        # the CPU path runs once, on rank 0 (no process group); the other ranks exit without work
        if int(os.environ.get("RANK", "0")) == 0:
            reference_arm(args, args.config, int(os.environ.get("WORLD_SIZE", str(args.gpus))))
        return
    args.warmup = max(args.warmup, 3)
    w = init_world(args)
    if w is None:
        raise SystemExit(spawn_ranks(args.gpus))
    rank, world, local_rank, dist = w
    try:
        gpu_arm(args, args.config, rank, world, local_rank, dist)
    finally:
        if dist:
            dist.barrier()
            dist.destroy_process_group()

if __name__ == "__main__":
    main()
