"""GPU experiment: S concurrent contexts (threads, own streams, 1/S of the grid each) stepping
independent reef-knot frames; frames/s vs S."""
import sys, threading, time
import numpy as np
sys.path.insert(0, ".")
import bench
from paper_2211_04045_b200 import capi

N = 16
scenes = [bench.batch_scene(i) for i in range(N)]
base = scenes[0][0]


def worker(share, idx, out, reps):
    ctx = capi.Context(0)
    ctx.set_grid_share(share)
    mesh = capi.Mesh.from_scene(ctx, base)
    dyn = capi.Dynamics(ctx, mesh, base.x)
    for i in idx[:1]:  # warm-up
        capi.step(ctx, mesh, dyn, scenes[i][0].x, scenes[i][1], delta=5e-4)
    out["ready"] += 1
    while out["ready"] < share:
        time.sleep(0.001)
    t = time.time()
    steps = 0
    for _ in range(reps):
        for i in idx:
            x, v, st = capi.step(ctx, mesh, dyn, scenes[i][0].x, scenes[i][1], delta=5e-4)
            steps += st["resolve_steps"]
    out["t"].append(time.time() - t)
    out["steps"] += steps
    dyn.close(); mesh.close(); ctx.close()


for S in (1, 2, 4):
    out = {"ready": 0, "t": [], "steps": 0}
    th = [threading.Thread(target=worker, args=(S, list(range(k, N, S)), out, 2)) for k in range(S)]
    for t in th: t.start()
    for t in th: t.join()
    wall = max(out["t"])
    print(f"S={S}: {2 * N / wall:.1f} frames/s (wall {wall:.2f} s, resolve steps {out['steps']})", flush=True)
