"""Host logic of the N > 1 bench path, on CPU with the gloo backend
(world_size 2): the max-over-ranks timing reduction, the partition of the
configs[4] batch over the ranks (every scene exactly once, rank-seeded
targets), rank-0-only output of the reference arm, and the self-spawn of
`bench.py --gpus N` without torchrun. The device path has no collective
(independent scenes per rank), so this is all the
multi-process logic there is."""
import json
import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench

    D = bench.Dist(device="cpu")
    # rank r reports (r + 1) ms for the device loop and (10 - r) ms end to end
    mx = D.max([rank + 1.0, 10.0 - rank])
    lo, hi = bench.partition(64, D.world, D.rank)
    sums = [float(np.abs(bench.batch_scene(i)[1]).sum()) for i in (lo, hi - 1)]

    class A:
        gpus, steps, warmup, scene = world, 1, 0, "reef"

    ref = bench.run_reference(A) if rank != 0 else "rank0"
    D.barrier()
    D.close()
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"max": mx, "lo": lo, "hi": hi, "vsums": sums, "ref": ref}, f)


def test_two_rank_gloo_host_logic(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    r = [json.load(open(tmp_path / f"r{i}.json")) for i in range(world)]
    assert r[0]["max"] == r[1]["max"] == [2.0, 10.0]
    # configs[4]: 64 scenes, contiguous halves, every scene exactly once
    assert (r[0]["lo"], r[0]["hi"], r[1]["lo"], r[1]["hi"]) == (0, 32, 32, 64)
    # independent scenes: rank-seeded tightening velocities differ
    assert len({*r[0]["vsums"], *r[1]["vsums"]}) == 4
    # the reference arm prints on rank 0 only
    assert r[1]["ref"] is None


def test_partition_covers_every_scene():
    sys.path.insert(0, ROOT)
    import bench

    for world in (1, 2, 3, 4, 8):
        owned = [i for r in range(world) for i in range(*bench.partition(64, world, r))]
        assert owned == list(range(64))


def test_spawn_command(monkeypatch):
    """--gpus N without WORLD_SIZE re-launches itself under torch.distributed.run."""
    sys.path.insert(0, ROOT)
    import bench

    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])

    class A:
        gpus = 4

    bench.spawn(A)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
