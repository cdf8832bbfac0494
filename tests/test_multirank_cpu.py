"""Host logic of the N > 1 bench path, on CPU with the gloo backend
(world_size 2): per-rank independent scenes, the max-over-ranks timing
reduction and the whole-job rate, and rank-0-only output of the reference arm.
The device path has no collective (independent scenes per rank, DESIGN.md
"Multi-GPU"), so this is all the multi-process logic there is."""
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
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r reports (r + 1) ms for the device loop and (10 - r) ms end to end
    mx = bench.max_over_ranks([rank + 1.0, 10.0 - rank], dist, "cpu")
    sc = bench.make_scene("reef", rank)

    class A:
        gpus, steps, warmup, scene = world, 2, 3, "reef"

    ref = bench.run_reference(A) if rank != 0 else "rank0"
    dist.barrier()
    dist.destroy_process_group()
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"max": mx, "nv": int(sc.nv), "ntri": int(len(sc.triangles)),
                   "ysum": float(np.abs(sc.y).sum()), "ref": ref}, f)


def test_two_rank_gloo_host_logic(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    r = [json.load(open(tmp_path / f"r{i}.json")) for i in range(world)]
    assert r[0]["max"] == r[1]["max"] == [2.0, 10.0]
    # independent, same-sized scenes (rank-seeded target)
    assert r[0]["nv"] == r[1]["nv"] and r[0]["ntri"] == r[1]["ntri"]
    assert r[0]["ysum"] != r[1]["ysum"]  # rank-seeded squeeze phase of the target
    # the reference arm prints on rank 0 only
    assert r[1]["ref"] is None


def test_whole_job_rate():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.whole_job_rate(1, 10, 1000.0) == 10.0
    assert bench.whole_job_rate(4, 10, 2000.0) == 20.0
