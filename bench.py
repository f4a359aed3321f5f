#!/usr/bin/env python
"""Benchmark: frames/s of the accelerated PIFu path (256^3 progressive
reconstruction + 512x512 mesh-free render, BASELINE.json configs[2]) on 1..N
B200s, frames sharded round-robin (configs[4] pattern).

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

A step = one frame per GPU.  `value` = frames of all ranks / max-over-ranks
device time of the K timed frames (CUDA events on the library's stream, inputs
resident in HBM, L2 flushed between frames).  `e2e` = the same through the
C-ABI with pinned HOST buffers (feature map H2D + depth/RGB/mask D2H inside the
timed call), host wall clock.  `roofline` = the fused geometry-MLP kernel
(algorithmic 2,363,906 FLOP per evaluated point) against the measured bf16
tensor peak.  `cpu_baseline` = the CPU port timed on this host (rank 0, N=1).
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

import numpy as np  # noqa: E402

GEO_FLOP_PER_POINT = 2363906
FACT_MMA_FLOP_PER_POINT = 2 * (512 * 1024 + 256 * 512 + 128 * 256)  # hidden parts of layers 2-4
TEX_FLOP_PER_POINT = 3350022 + 2231808
METRIC = "frames/sec (256^3 recon + 512² render) at 1/2/4/8 B200; MLP points/sec vs TC peak"

CONFIGS = {
    # name: (coarsest, level, fmap (C,H,W), render W=H, precision)
    "config2": (32, 3, (256, 128, 128), 512, "fp32"),
    "config3": (32, 4, (256, 256, 256), 1024, "bf16"),
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


def make_inputs(cfg_name: str):
    from paper_2007_13988_b200 import api
    caps = api.gen_capsules(42)
    gw, gb = api.gen_mlp(7, 0)
    tw, tb = api.gen_mlp(8, 1)
    return caps, gw, gb, tw, tb


def fmap_seed(rank: int, i: int) -> int:
    return 1000 + 8192 * rank + i


# ---------------------------------------------------------------------------
# CPU legs (oracle port / reference)
# ---------------------------------------------------------------------------
def cpu_port_frame(cfg_name: str, threads: int):
    """One full frame through the CPU port (oracle/liborc.so): progressive
    localization + first-crossing render + texture.  Returns seconds."""
    from oracle import oracle as O
    from paper_2007_13988_b200 import api
    r0, lv, (c, h, w), res, _ = CONFIGS[cfg_name]
    caps, gw, gb, tw, tb = make_inputs(cfg_name)
    fmap = api.gen_feature_map(fmap_seed(0, 0), c, h, w)
    m = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=threads)
    cam = O.camera_from_angles(90, 0)
    t0 = time.perf_counter()
    ext = O.extract_progressive(m, r0, lv)
    O.render_first_crossing(ext["values"], r0 << lv, cam, res, res, tex=m)
    return time.perf_counter() - t0, ext["total_evals"]


def reference_arm(args, cfg_name: str):
    """Reference arm: the reference's own operators from oracle/_ref (the
    unmodified headers): extract_progressive's full control flow driven through
    a FieldOracle (replaying the frame's occupancies), plus the per-point PIFu
    FieldOracle evaluation cost measured on a 1/64 stride sample of the frame's
    evaluated nodes and surface points through FieldOracle::occupancy_batch /
    texture_batch with all host threads, scaled by 64."""
    from oracle import oracle as O
    from paper_2007_13988_b200 import api
    threads = os.cpu_count() or 1
    r0, lv, (c, h, w), res, _ = CONFIGS[cfg_name]
    caps, gw, gb, tw, tb = make_inputs(cfg_name)
    fmap = api.gen_feature_map(fmap_seed(0, 0), c, h, w)
    m = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=threads)
    cells = r0 << lv
    # the frame's occupancies (computed once, untimed, by the CPU port)
    ext = O.extract_progressive(m, r0, lv)
    cam = O.camera_from_angles(90, 0)
    rnd = O.render_first_crossing(ext["values"], cells, cam, res, res, want_points=True)
    n = cells + 1
    ev = np.flatnonzero(ext["states"] == 2)
    i, j, k = ev % n, (ev // n) % n, ev // (n * n)
    nodes = np.stack([-1 + 2 * i / cells, -1 + 2 * j / cells, 1 - 2 * k / cells], 1)
    spts = rnd["surface_pts"][rnd["mask"] == 1]
    stride = 64
    node_sample, surf_sample = nodes[::stride], spts[::stride]
    rp = O.Replay(ext["values"], ext["states"], cells)

    def step():
        t0 = time.perf_counter()
        r = O.ref_extract(rp.pt_fn, rp.user, r0, lv, workers=threads)  # reference control flow, full frame
        t1 = time.perf_counter()
        O.ref_occupancy_batch(m.pt_fn, m.user, node_sample, workers=threads)
        t2 = time.perf_counter()
        O.render_first_crossing(ext["values"], cells, cam, res, res)
        t3 = time.perf_counter()
        O.ref_texture_batch(m.pt_fn, m.pt_tex_fn, m.user, surf_sample, workers=threads)
        t4 = time.perf_counter()
        assert r["total_evals"] == len(ev)
        return (t1 - t0) + (t3 - t2) + stride * ((t2 - t1) + (t4 - t3))

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg_name, args),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "reference",
                         "sample": f"reference extract_progressive control flow over the full frame "
                                   f"({len(ev)} evals, replayed occupancies) + FieldOracle PIFu evaluation of a "
                                   f"1/{stride} stride sample of those nodes ({len(node_sample)}) and of the "
                                   f"{len(spts)} surface points, scaled x{stride}"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg_name: str, args) -> dict:
    r0, lv, (c, h, w), res, prec = CONFIGS[cfg_name]
    return {"workload": f"{cfg_name}: progressive PIFu localization {r0}->{r0 << lv} cells ({(r0 << lv)}^3 grid), "
                        f"feature map {c}x{h}x{w}, {res}x{res} first-crossing render yaw 90 + texture MLP; "
                        "frames sharded round-robin over GPUs (configs[4] pattern)",
            "precision": prec if args.precision is None else args.precision,
            "frames_in_flight_per_gpu": args.streams,
            "feature_maps_per_stream": args.frames, "l2": "flushed before every frame (320 MB device copy on "
                                                          "the frame's stream); inputs cycle over distinct feature maps",
            "parallelism": f"frame-sharded x{args.gpus}, no per-frame collective"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="config2", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default=None, choices=[None, "fp32", "bf16", "simt"])
    ap.add_argument("--frames", type=int, default=4, help="distinct device-resident feature maps per stream")
    ap.add_argument("--l2", default="flush", choices=["flush", "cycle"],
                    help="flush: 320 MB device copy before every frame; cycle: no flush, the distinct "
                         "feature maps cycled over (streams x frames x 16.8 MB) exceed the 126 MB L2")
    ap.add_argument("--streams", type=int, default=4,
                    help="frames in flight per GPU (one context + stream + host thread each)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg_name = args.config

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, cfg_name)
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as td
        torch.cuda.set_device(local_rank)
        td.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = td

    from paper_2007_13988_b200 import abi, api
    r0, lv, (C_, H_, W_), res, prec_name = CONFIGS[cfg_name]
    if args.precision:
        prec_name = args.precision
    prec = {"fp32": abi.ICG_PREC_FP32, "bf16": abi.ICG_PREC_BF16, "simt": abi.ICG_PREC_FP32_SIMT}[prec_name]
    caps, gw, gb, tw, tb = make_inputs(cfg_name)
    S = max(1, args.streams)
    cfg = api.AlgoConfig("progressive", r0, lv)
    cam = api.CameraSpec.from_angles(90, 0)
    fbytes = C_ * H_ * W_ * 4
    npx = res * res
    import ctypes as C

    def img_struct(bufs, mem):
        img = abi.icg_image()
        img.mem = mem
        img.depth = C.cast(C.c_void_p(bufs["depth"]), abi.f32p)
        img.rgb = C.cast(C.c_void_p(bufs["rgb"]), abi.f32p)
        img.mask = C.cast(C.c_void_p(bufs["mask"]), abi.u8p)
        img.surface_k = C.cast(C.c_void_p(bufs["sk"]), abi.i32p)
        return img

    class Lane:
        """One context (stream) of this GPU: its own frames in flight, driven by one host thread."""

        def __init__(self, s):
            self.ctx = api.Context(local_rank)
            self.ctx.set_mlp(abi.ICG_MLP_GEOMETRY, gw, gb)
            self.ctx.set_mlp(abi.ICG_MLP_TEXTURE, tw, tb)
            self.host_maps, self.dev_maps = [], []
            for i in range(args.frames):
                fm = api.gen_feature_map(fmap_seed(rank, s * args.frames + i), C_, H_, W_)
                hp = api.host_alloc(fbytes)
                np.ctypeslib.as_array((np.ctypeslib.ctypes.c_float * fm.size).from_address(hp))[:] = fm.reshape(-1)
                dp = self.ctx.device_alloc(fbytes)
                self.ctx.memcpy(dp, hp, fbytes, abi.ICG_MEM_DEVICE, abi.ICG_MEM_HOST)
                self.host_maps.append(hp)
                self.dev_maps.append(dp)
            self.fields_dev = [api.PifuField(None, caps, 50.0, prec, device_ptr=dp, shape=(C_, H_, W_))
                               for dp in self.dev_maps]
            self.fields_host = []
            for hp in self.host_maps:
                f = api.PifuField(None, caps, 50.0, prec, device_ptr=hp, shape=(C_, H_, W_))
                f.c.fmap_mem = abi.ICG_MEM_HOST
                self.fields_host.append(f)
            sizes = (("depth", npx * 4), ("rgb", npx * 12), ("mask", npx), ("sk", npx * 4))
            self.dout = img_struct({k: self.ctx.device_alloc(b) for k, b in sizes}, abi.ICG_MEM_DEVICE)
            self.hout = img_struct({k: api.host_alloc(b) for k, b in sizes}, abi.ICG_MEM_HOST)
            self.flush_a = self.ctx.device_alloc(320 << 20)
            self.flush_b = self.ctx.device_alloc(320 << 20)
            self.lat = []
            self.k = 0

        def flush_l2(self):
            self.ctx.memcpy(self.flush_b, self.flush_a, 320 << 20, abi.ICG_MEM_DEVICE, abi.ICG_MEM_DEVICE)

        def frame(self, host=False, flush=True):
            if flush and args.l2 == "flush":
                self.flush_l2()
            f = (self.fields_host if host else self.fields_dev)[self.k % args.frames]
            self.k += 1
            ext, img = self.ctx.frame_raw(f, cfg, cam, res, res, self.hout if host else self.dout)
            self.lat.append(img.wall_seconds * 1e3)

    lanes = [Lane(s) for s in range(S)]
    ctxs = [ln.ctx for ln in lanes]
    from paper_2007_13988_b200 import shard

    def barrier():
        shard.barrier()

    def allmax(x: float) -> float:
        return shard.allmax(x, device=f"cuda:{local_rank}" if dist else None)

    def run_frames(nframes: int, host: bool) -> float:
        """nframes frames round-robin over the lanes (one host thread per lane); returns the
        device-timed span (CUDA events: common start event, last stream's end event), ms."""
        counts = [nframes // S + (1 if i < nframes % S else 0) for i in range(S)]
        api.span_begin(ctxs)
        ths = [threading.Thread(target=lambda ln=ln, c=c: [ln.frame(host) for _ in range(c)])
               for ln, c in zip(lanes, counts)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return api.span_end(ctxs)

    # ---- warm-up (every lane) ----
    for ln in lanes:
        for _ in range(args.warmup):
            ln.frame()
    # ---- single-frame latency: one lane, frames back to back (device time per frame) ----
    lat_lane = lanes[0]
    lat_lane.lat = []
    for _ in range(min(args.steps, 30)):
        lat_lane.frame()
    single_lat = list(lat_lane.lat)
    # ---- timed: S frames in flight, device-resident inputs and outputs ----
    for ln in lanes:
        ln.lat = []
    barrier()
    cvd = [d for d in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if d.strip().isdigit()]
    clocks = ClockSampler(int(cvd[local_rank]) if local_rank < len(cvd) else local_rank)
    clocks.start()
    t_wall0 = time.perf_counter()
    span_ms = run_frames(args.steps, host=False)
    wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    lat = sum((ln.lat for ln in lanes), [])
    barrier()
    dev_max = allmax(span_ms / 1e3)
    value = world * args.steps / dev_max

    # ---- per-kernel breakdown: a separate single-lane pass with CUDA events around every launch
    # (the events themselves cost a little, so `value` is not taken here) ----
    ctx = lat_lane.ctx
    ctx.profile(True, reset=True)
    for _ in range(min(args.steps, 20)):
        lat_lane.frame()
    prof = ctx.profile_get()
    ctx.profile(False, reset=False)

    # ---- e2e: pinned host inputs/outputs through the C ABI (H2D + D2H inside every call) ----
    e2e = None
    if not args.no_e2e:
        for ln in lanes:
            for _ in range(2):
                ln.frame(host=True, flush=False)
        barrier()
        e2e_ms = run_frames(args.steps, host=True)
        e2e_t = allmax(e2e_ms / 1e3)
        e2e = {"value": world * args.steps / e2e_t, "unit": "frames/s", "h2d_bytes_per_step": fbytes,
               "d2h_bytes_per_step": npx * (4 + 12 + 1 + 4)}

    # ---- roofline of the dominant kernel: the column-factored geometry field on the bulk batches ----
    pk = peaks()
    peak_t = pk.get("bf16_tflops_sustained", 1385.7)
    fact_s = prof["fact_ms"] / 1e3
    fact_pts = prof["fact_points"]
    # algorithmic (dense-equivalent) work per evaluated point; executed MMA work of
    # the factored pass: layers 2-4 hidden parts (688,128 MAC/point) x3 for bf16x3
    exec_mult = 3 if prec_name == "fp32" else 1
    achieved = fact_pts * GEO_FLOP_PER_POINT / fact_s / 1e12 if fact_s > 0 else 0.0
    executed = fact_pts * FACT_MMA_FLOP_PER_POINT * exec_mult / fact_s / 1e12 if fact_s > 0 else 0.0
    traffic, traffic_note = None, None
    try:  # DRAM bytes of the factored pass's level-3 launch, from the committed ncu --set full capture
        rec = json.load(open(os.path.join(ROOT, "profiles", "r01e_ncu_full_fact2_L3.json")))[0]
        mb = lambda v: float(v.split()[0]) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[v.split()[1]]
        traffic = (mb(rec["dram__bytes_read.sum"]) + mb(rec["dram__bytes_write.sum"])) * 1e6
        traffic_note = ("dram__bytes_read.sum + dram__bytes_write.sum of the level-3 k_fact2 launch (280 k points, "
                        "profiles/r01e_ncu_full_fact2_L3.json): weights, column records and lists, L2-resident at 92 %")
    except Exception:
        pass
    roofline = {"bound": "tensor",
                "kernel": "geometry field, bulk batches (dense level 0 + each level's E0 list): column pass "
                          "k_mlp_pair<COLS> + factored pass k_fact2 (CTA-pair tcgen05, M = 256 points x N = 256 "
                          "features), incl. list sorting",
                "achieved": achieved, "peak": peak_t, "unit": "TFLOP/s", "frac": achieved / peak_t,
                "traffic": traffic, "traffic_note": traffic_note,
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained" + (" (fallback)" if pk.get("fallback") else ""),
                "algorithmic_flop_per_point": GEO_FLOP_PER_POINT,
                "achieved_note": "dense-equivalent algorithmic FLOP (SURVEY §8(d)); the factored pass executes fewer",
                "executed_tflops": executed, "executed_frac": executed / peak_t,
                "executed_flop_per_point": FACT_MMA_FLOP_PER_POINT * exec_mult,
                "launches": prof["fact_launches"], "points": fact_pts,
                "avg_launch_ms": prof["fact_ms"] / max(1, prof["fact_launches"])}
    secondary = {
        "conflict_chain": {"points": prof["chain_points"], "ms": prof["chain_ms"], "launches": prof["chain_launches"]},
        "geometry_all": {"points": prof["geo_points"], "ms": prof["geo_mlp_ms"],
                         "mlp_points_per_s": prof["geo_points"] / max(1e-9, prof["geo_mlp_ms"] / 1e3),
                         "achieved_tflops": prof["geo_points"] * GEO_FLOP_PER_POINT / max(1e-9, prof["geo_mlp_ms"] / 1e3) / 1e12},
        "texture_mlp": {"points": prof["tex_points"], "ms": prof["tex_mlp_ms"],
                        "achieved_tflops": prof["tex_points"] * TEX_FLOP_PER_POINT / max(1e-9, prof["tex_mlp_ms"] / 1e3) / 1e12},
        "dense_passes": {"bytes": prof["dense_bytes"], "ms": prof["dense_ms"],
                         "achieved_gbs": prof["dense_bytes"] / max(1e-9, prof["dense_ms"] / 1e3) / 1e9,
                         "peak_gbs": pk.get("hbm_gbs")},
        "render": {"bytes": prof["render_bytes"], "ms": prof["render_ms"],
                   "achieved_gbs": prof["render_bytes"] / max(1e-9, prof["render_ms"] / 1e3) / 1e9},
        "profiled_frames": prof["frames"], "profiled_frame_ms": prof["frame_ms"] / max(1, prof["frames"]),
    }

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        t, evals = cpu_port_frame(cfg_name, threads)
        cpu_baseline = {"value": 1.0 / t, "unit": "frames/s", "cores": threads, "kind": "port",
                        "sample": f"one full {cfg_name} frame (feature seed {fmap_seed(0, 0)}, {evals} evals) through "
                                  "the CPU port oracle/liborc.so (fp64 batched MLP, all host threads)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dev_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16x3 (fp32-accurate)" if prec_name == "fp32" else prec_name,
            "data": "synthetic (seeded N(0,1) feature maps, Kaiming-uniform weights, 15-capsule sdf bias)",
            "config": dict(workload_config(cfg_name, args), wall_ms_per_step=1e3 * wall / args.steps,
                           frame_latency_ms={"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
                                             "note": f"device time of one frame with {S} frames in flight"},
                           single_frame_latency_ms={"p50": float(np.percentile(single_lat, 50)),
                                                    "p99": float(np.percentile(single_lat, 99)),
                                                    "note": "one frame at a time on one stream"},
                           evals_per_frame=int(prof["geo_points"] / max(1, prof["frames"]))),
            "e2e": e2e, "roofline": roofline, "secondary": secondary, "cpu_baseline": cpu_baseline,
            "gpu_launches": int(round(prof["kernel_launches"] / max(1, prof["frames"]) * args.steps)), "clocks": clk,
            "streams": S,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
