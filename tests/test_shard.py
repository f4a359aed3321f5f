"""Frame sharding over ranks (configs[4] pattern) on CPU: world_size 2, gloo.

Each rank extracts its round-robin share of frames with the CPU oracle (the
checker, standing in for the per-GPU `api.Context`), rank 0 gathers the
per-frame summaries; they must equal a single-process run frame by frame, and
the max-over-ranks timing reduction must see both ranks.
"""
import hashlib
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2007_13988_b200 import shard  # noqa: E402

N_FRAMES = 5


def frame_summary(i: int) -> dict:
    from oracle import oracle as O
    caps = O.gen_capsules(100 + i)
    fld = O.Analytic(caps, 0.02)
    r = O.extract_progressive(fld, 8, 2)
    return {"frame": i, "evals": r["evals_per_level"], "total": r["total_evals"],
            "bin_sha": hashlib.sha256(r["binarized"].tobytes()).hexdigest()}


def _worker(rank, world, port, out_path):
    import torch.distributed as td
    td.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        res = shard.run_sharded(N_FRAMES, frame_summary, rank, world)
        t = shard.allmax(float(rank + 1))
        s = shard.allsum(len(shard.frames_for_rank(N_FRAMES, rank, world)))
        shard.barrier()
        if rank == 0:
            import json
            json.dump({"res": res, "max": t, "sum": s}, open(out_path, "w"))
        else:
            assert res is None
    finally:
        td.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_frames_for_rank_partition():
    for world in (1, 2, 3, 8):
        seen = sorted(i for r in range(world) for i in shard.frames_for_rank(17, r, world))
        assert seen == list(range(17))
    assert shard.frames_for_rank(5, 1, 2) == [1, 3]
    with pytest.raises(ValueError):
        shard.frames_for_rank(5, 2, 2)


def test_sharded_extraction_gloo_world2(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "rank0.json")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    import json
    got = json.load(open(out))
    single = [frame_summary(i) for i in range(N_FRAMES)]
    assert got["res"] == single
    assert got["max"] == 2.0 and got["sum"] == N_FRAMES
