"""Throughput with S contexts (streams) on one GPU, one host thread each (dev experiment)."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2007_13988_b200 import abi, api
import ctypes as C
S = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
caps = api.gen_capsules(42)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
ctxs, fields, imgs = [], [], []
for s in range(S):
    ctx = api.Context(0); ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
    fm = api.gen_feature_map(1000 + s)
    fields.append(api.PifuField(fm, caps, 50.0, abi.ICG_PREC_FP32))
    npx = 512 * 512
    bufs = {k: ctx.device_alloc(b) for k, b in (("depth", npx * 4), ("rgb", npx * 12), ("mask", npx), ("sk", npx * 4))}
    img = abi.icg_image(); img.mem = abi.ICG_MEM_DEVICE
    img.depth = C.cast(C.c_void_p(bufs["depth"]), abi.f32p); img.rgb = C.cast(C.c_void_p(bufs["rgb"]), abi.f32p)
    img.mask = C.cast(C.c_void_p(bufs["mask"]), abi.u8p); img.surface_k = C.cast(C.c_void_p(bufs["sk"]), abi.i32p)
    ctxs.append(ctx); imgs.append(img)
cfg = api.AlgoConfig("progressive", 32, 3); cam = api.CameraSpec.from_angles(90, 0)
for s in range(S):
    for _ in range(3): ctxs[s].frame_raw(fields[s], cfg, cam, 512, 512, imgs[s])
lat = [[] for _ in range(S)]
def run(s):
    for i in range(N // S):
        ext, img = ctxs[s].frame_raw(fields[s], cfg, cam, 512, 512, imgs[s])
        lat[s].append(img.wall_seconds * 1e3)
t0 = time.perf_counter()
th = [threading.Thread(target=run, args=(s,)) for s in range(S)]
[t.start() for t in th]; [t.join() for t in th]
dt = time.perf_counter() - t0
print(f"S={S} frames={N // S * S} wall {dt*1e3:.1f} ms -> {N // S * S / dt:.1f} frames/s, per-frame device ms p50 {np.median(sum(lat, [])):.2f}")
