#!/usr/bin/env python
"""Benchmark of the two-way collision-handling hot path on B200.

One "step" = one resolve(x, y) call (Alg. 1 of arXiv 2211.04045 run to
convergence: the collision-handling stage of one simulation time step) on the
synthetic bow knot of BASELINE.json configs[2] (two twisted cloth strips,
74,800 vertices / 142,044 triangles, tightening target). Metric: collision
sim steps per second (whole job: all ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU). Every rank resolves its
own independent knot (a different strip-twist jitter): the path shards only
across independent scenes, so there is no collective on the data path
(weak scaling); torch.distributed is used for the start/stop barriers and the
max-over-ranks of the device-timed region only.

--impl reference times the reference algorithm on the host CPU: the C oracle
(oracle/, a clean-room restatement — the reference itself needs Eigen, which is
absent, so it cannot be built here), single-threaded like the reference.
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

METRIC = "collision sim steps/s (resolve calls/s) at the 142K-tri bow knot"
PAPER_COST_S = 0.034  # bow knot collision cost per time step (RTX 2080 Ti, paper Table 1)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scene", choices=["bow", "reef"], default="bow")
    ap.add_argument("--coloring", choices=["device", "reference"], default="device")
    ap.add_argument("--cpu-sample-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=0,
                    help="BASELINE configs[4]: B independent reef-knot scenes split over the ranks")
    return ap.parse_args()


def make_scene(name, rank):
    from paper_2211_04045_b200 import scenes

    jitter = None if rank == 0 else rank
    if name == "bow":
        return scenes.bow_knot(jitter_seed=jitter)
    return scenes.reef_knot(jitter_seed=jitter)


def scene_config(sc, args):
    return {"workload": f"{sc.name}: {sc.nv} vertices, {len(sc.triangles)} triangles, {len(sc.edges)} edges; "
                        "two cloth strips laid face to face (2.5 mm apart, 3 mm mesh) along a twisted (2,3) "
                        "torus-knot band; tightening target presses them to a 0.2 mm gap where the knot is "
                        "tightest and slides one 3 mm along the other (scenes.ply_knot)",
            "scene": args.scene, "vertices": sc.nv, "triangles": int(len(sc.triangles)),
            "edges": int(len(sc.edges)), "dt_note": "kinematic tightening target (no dynamics step)",
            "solver": "pgs, 1 sweep", "coloring": args.coloring,
            "params": {"d_min": 2e-3, "d_max": 4e-3, "delta": 5e-4, "gamma": 0.9, "eps": 1e-4,
                       "step_limit": 512},
            "l2": "each resolve rebuilds its LBVH and pair set (>= 10^8 B working set vs the 126 MB L2); "
                  "inputs re-uploaded every e2e step",
            "parallelism": "independent scenes per rank (no collective)"}


RESOLVE_KW = dict(delta=5e-4, coloring_mode="device")  # knots: delta = 0.5 mm


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.out = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.out.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def bytes_per_resolve(trace, sc, sweeps=1):
    """Algorithmic HBM bytes of one resolve, from its per-step trace (SURVEY.md
    §8(d) per-unit contract): refresh 98 B/pair,
    linearize 210 B/contact row + 88 B/edge row, assemble 136 B/row + 72 B/vertex,
    PGS 336 B/contact row + 184 B/edge row per sweep, advance 128 B/vertex; a
    search step adds the LBVH refit (64 B per node written, 2 nodes per
    primitive), 24 B per vertex of positions and 98 B per emitted pair. The
    refresh is counted only where its result is used: not after the final
    step, and not before a re-search (there only the pairs holding stored
    multipliers are evaluated)."""
    nv, nt, ne = sc.nv, len(sc.triangles), len(sc.edges)
    total = 0
    for i, t in enumerate(trace):
        P, C, ER = t["num_pairs"], t["num_contact_rows"], t["num_edge_rows"]
        R = C + ER
        b = 210 * C + 88 * ER + 136 * R + 72 * nv + (336 * C + 184 * ER) * sweeps + 128 * nv
        if i + 1 < len(trace) and not trace[i + 1]["searched"]:
            b += 98 * P
        if t["searched"]:
            b += 98 * P + 64 * 2 * (nt + ne) + 24 * nv
        total += b
    return total


def peaks_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)).get("hbm_gbs", 6650.0) if os.path.exists(p) else 6650.0


def phase_roofline(trace, sc, phases, peak):
    """Achieved algorithmic GB/s of the main phases of one resolve (same
    per-unit bytes as bytes_per_resolve, phase times from the kernel's own
    phase profile), and their fraction of the HBM peak."""
    nv = sc.nv
    rows = [(t["num_contact_rows"], t["num_edge_rows"]) for t in trace]
    refreshed = sum(t["num_pairs"] for i, t in enumerate(trace) if i + 1 < len(trace) and not trace[i + 1]["searched"])
    searched = sum(t["num_pairs"] for t in trace if t["searched"])
    units = {
        "ph_refresh": 98 * refreshed,
        "ph_emit_records": 98 * searched,
        "ph_pgs_color+ph_pgs_tail": sum(336 * c + 184 * e for c, e in rows),
        "ph_rows+ph_rows_build": sum(210 * c + 88 * e for c, e in rows),
        "ph_advance": 128 * nv * len(trace),
    }
    out = {}
    for name, b in units.items():
        ms = sum(phases.get(k, [0.0])[0] for k in name.split("+"))
        if ms > 0:
            gbs = b / (ms / 1e3) / 1e9
            out[name] = {"bytes": b, "ms": round(ms, 4), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    return out


def max_over_ranks(vals, dist, device):
    """Elementwise max over ranks of per-rank timings (ms); identity at N = 1."""
    import torch

    t = torch.tensor(vals, dtype=torch.float64, device=device)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def whole_job_rate(world, steps, ms_max):
    """Resolves per second over all ranks: every rank resolves its own scene
    `steps` times, the job takes the slowest rank's time (weak scaling)."""
    return world * steps / (ms_max / 1e3)


def run_ours(args):
    import numpy as np
    import torch

    from paper_2211_04045_b200 import capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    sc = make_scene(args.scene, rank)
    stream = torch.cuda.current_stream()
    ctx = capi.Context(local, stream=stream.cuda_stream)
    mesh = capi.Mesh.from_scene(ctx, sc)
    kw = dict(RESOLVE_KW, coloring_mode=args.coloring)
    d_x = torch.from_numpy(sc.x).cuda()
    d_y = torch.from_numpy(sc.y).cuda()
    d_out = torch.empty_like(d_x)
    h_x = torch.from_numpy(sc.x).pin_memory()
    h_y = torch.from_numpy(sc.y).pin_memory()
    h_out = torch.empty_like(h_x).pin_memory()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    # warm-up (capacity growth happens here), and one traced call for the
    # roofline bytes / step counts (identical in every call: deterministic)
    for _ in range(max(args.warmup, 3)):
        capi.resolve_device_ptr(ctx, mesh, d_x.data_ptr(), d_y.data_ptr(), d_out.data_ptr(), **kw)
    _, st_tr = capi.resolve(ctx, mesh, sc.x, sc.y, trace=True, **kw)
    algo_bytes = bytes_per_resolve(st_tr["trace"], sc)
    capi.resolve_device_ptr(ctx, mesh, d_x.data_ptr(), d_y.data_ptr(), d_out.data_ptr(), **kw)
    phases = {k: [round(v[0], 3), v[1]] for k, v in capi.phase_profile(ctx).items()}  # untraced call
    phase_roof = phase_roofline(st_tr["trace"], sc, phases, peaks_gbs())

    # ---- device-resident throughput (inputs already in HBM)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.kernel_launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kernel_ms, steps_sum, searches_sum, pairs_eval = [], 0, 0, 0
    for i in range(args.steps):
        flush.fill_(i & 0xFF)  # L2 flush between timed iterations (outside the events)
        evs[i][0].record(stream)
        st = capi.resolve_device_ptr(ctx, mesh, d_x.data_ptr(), d_y.data_ptr(), d_out.data_ptr(), **kw)
        evs[i][1].record(stream)
        kernel_ms.append(st["kernel_ms"])
        steps_sum += st["steps"]
        searches_sum += st["searches"]
        pairs_eval += st["pairs_evaluated"]
    torch.cuda.synchronize()
    launches = ctx.kernel_launches - launches0
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    # ---- end to end through the C-ABI with host buffers (H2D x, y and D2H x every step)
    e2e_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    xin, yin, xo = h_x.numpy(), h_y.numpy(), h_out.numpy()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        e2e_evs[i][0].record(stream)
        _ = capi.resolve(ctx, mesh, xin, yin, out=xo, **kw)[0]
        e2e_evs[i][1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_evs)
    clk = clocks.stop()
    barrier()

    # ---- certification of the resolve path on the device (testkit ccd.cpp):
    # literal CCD stencil tests of every segment, outside the timed regions
    _, st_path = capi.resolve(ctx, mesh, sc.x, sc.y, record_path=True, **dict(kw, step_limit=64))
    path = st_path["path"]
    ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    viol = cert = stencils = 0
    ca.record(stream)
    for i in range(len(path) - 1):
        v, c, n = capi.ccd_certify(ctx, mesh, path[i], path[i + 1], candidates=True)
        viol, cert, stencils = viol + v, cert + c, stencils + n
    cb.record(stream)
    torch.cuda.synchronize()
    ccd_ms = ca.elapsed_time(cb)
    ccd = {"segments": len(path) - 1, "violations": viol, "certain_violations": cert,
           "candidate_stencils": stencils, "ms_incl_host_copies": round(ccd_ms, 3),
           "stencils_per_s": round(stencils / (ccd_ms / 1e3), 1), "intersection_free": viol == 0}
    dev_ms_max, e2e_ms_max = max_over_ranks([dev_ms, e2e_ms], dist, "cuda")
    value = whole_job_rate(world, args.steps, dev_ms_max)
    e2e_value = whole_job_rate(world, args.steps, e2e_ms_max)
    kern_avg_ms = sum(kernel_ms) / len(kernel_ms)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = algo_bytes / (kern_avg_ms / 1e3) / 1e9
    # DRAM bytes per k_resolve launch from the committed ncu --set full capture
    # of the same resolve (tools/gpu_measure.sh -> tools/make_profiles.py)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else None
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_ms_max / args.steps, 4),
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": round(value * PAPER_COST_S, 3),
            "baseline_note": "vs_baseline = value / (1 / 0.034 s): the paper's bow-knot collision cost per time "
                             "step on an RTX 2080 Ti (BASELINE.md section 2; different knot asset and GPU)",
            "dtype": "f64", "data": "synthetic",
            "config": scene_config(sc, args),
            "resolve": {"alg1_steps_per_call": steps_sum / args.steps, "searches_per_call": searches_sum / args.steps,
                        "final_pairs": st["num_pairs"], "pairs_evaluated_per_call": pairs_eval / args.steps,
                        "kernel_ms": round(kern_avg_ms, 4), "setup_ms": round(st["setup_ms"], 4),
                        "phase_ms_count": phases,
                        "phase_roofline": phase_roof,
                        "two_way_steps_per_s": round(world * steps_sum / (dev_ms_max / 1e3), 1),
                        "ccd_pairs_per_s": round(world * pairs_eval / (dev_ms_max / 1e3), 1)},
            "e2e": {"value": round(e2e_value, 3), "unit": "steps/s", "h2d_bytes_per_step": 2 * sc.nv * 24,
                    "d2h_bytes_per_step": sc.nv * 24 + 160},
            "gpu_launches": launches,
            "ccd_certification": ccd,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                         "traffic_source": traffic["source"] if traffic else "no ncu capture committed",
                         "kernel": "tw::k_resolve (persistent cooperative Alg.-1 kernel)",
                         "algorithmic_bytes_per_launch": algo_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"},
            "clocks": clk,
        }
    if dist is not None:
        dist.destroy_process_group()
    return out, sc, st_tr


class OracleSampler:
    """Bounded CPU sample of the bow-knot resolve on the C oracle (the
    single-threaded restatement of the reference, oracle/): the proximity
    search at x (proximity.cpp:87-181) timed once, and single non-search
    Alg.-1 steps (refresh, per-vertex bound, linearize, color, assemble + PGS +
    recover, advance: resolve.cpp:64-131) timed per sample. A full resolve is
    estimated as searches x t_search + steps x t_step with the step/search
    counts of the (bit-identical) device run."""

    def __init__(self, sc):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import numpy as np
        import pyoracle

        self.np, self.po, self.sc = np, pyoracle, sc
        cfg = pyoracle.default_config(**RESOLVE_KW)
        self.cfg = cfg
        inv = sc.inv_mass
        self.y = np.where((inv == 0)[:, None], sc.x, sc.y)  # static override (resolve.cpp:47-50)
        E = np.asarray(sc.edges).reshape(-1, 2)
        self.ly = np.linalg.norm(self.y[E[:, 0]] - self.y[E[:, 1]], axis=1)
        t0 = time.perf_counter()
        self.pairs = pyoracle.search(sc, sc.x, cfg.d_max, cap=160 * sc.nv)
        self.t_search = time.perf_counter() - t0

    def step(self):
        po, sc, cfg = self.po, self.sc, self.cfg
        t0 = time.perf_counter()
        po.refresh(sc, sc.x, cfg.d_max, self.pairs)
        D = po.vertex_bound(sc, cfg.d_max, self.pairs, sc.nv)
        rows = po.linearize(sc, sc.x, self.pairs, self.ly, delta=cfg.delta, sigma=cfg.sigma)
        nc, col = po.color(sc, rows, cfg.color_seed, mode=cfg.coloring_mode)
        b = po.backward(sc.inv_mass, rows, col, nc, sc.x, self.y)
        po.advance(sc.inv_mass, b["y"], D, cfg.gamma, sc.x, self.np.ones(sc.nv))
        return time.perf_counter() - t0

    def describe(self, nsamples, nsteps, nsearch):
        return (f"C oracle on the host, 1 thread: the bow-knot proximity search timed once "
                f"({self.t_search:.1f} s, {len(self.pairs)} pairs) + the median of {nsamples} single "
                f"non-search Alg.-1 steps; estimate = {nsearch} searches + {nsteps} steps of the device run")


def cpu_baseline(sc, gpu_trace, nsamples):
    """cpu_baseline of the ours-arm line (rank 0, N = 1; ~45 s of host work)."""
    s = OracleSampler(sc)
    t_step = statistics.median([s.step() for _ in range(max(1, nsamples))])
    nsteps, nsearch = len(gpu_trace), sum(t["searched"] for t in gpu_trace)
    est = nsearch * s.t_search + nsteps * t_step
    return {"value": round(1.0 / est, 6), "unit": "steps/s", "cores": 1, "kind": "port",
            "sample": s.describe(max(1, nsamples), nsteps, nsearch),
            "seconds_search": round(s.t_search, 3), "seconds_per_step": round(t_step, 3)}


def run_reference(args):
    """--impl reference: the reference's algorithm on the host CPU (the C
    oracle: the reference itself needs Eigen, absent here). Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    sc = make_scene(args.scene, 0)
    trace_path = os.path.join(ROOT, "profiles", f"{args.scene}_knot_trace.json")
    trace = json.load(open(trace_path))  # committed: the device run's per-step trace (deterministic)
    nsteps, nsearch = len(trace), sum(t["searched"] for t in trace)
    s = OracleSampler(sc)
    samples = []
    for i in range(args.warmup + args.steps):
        dt = s.step()
        if i >= args.warmup:
            samples.append(dt)
    t_step = statistics.median(samples)
    value = 1.0 / (nsearch * s.t_search + nsteps * t_step)
    return {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": scene_config(sc, args),
            "cpu_baseline": {"value": round(value, 6), "unit": "steps/s", "cores": 1, "kind": "port",
                             "sample": s.describe(args.steps, nsteps, nsearch) +
                             f" (profiles/{args.scene}_knot_trace.json)",
                             "seconds_search": round(s.t_search, 3), "seconds_per_step": round(t_step, 3)},
            "e2e": {"value": round(value, 6), "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_batch(args):
    """configs[4]: a batch of B independent reef-knot scenes (rank-seeded
    tightening targets on the same strips) partitioned over the ranks; a step
    resolves every scene of the rank once, back to back on its GPU. No
    collective: value = B / max over ranks of the device time per step."""
    import torch

    from paper_2211_04045_b200 import capi, scenes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lo, hi = rank * args.batch // world, (rank + 1) * args.batch // world
    base = scenes.reef_knot()
    ys = [scenes.reef_knot(jitter_seed=1000 + i).y for i in range(lo, hi)]
    stream = torch.cuda.current_stream()
    ctx = capi.Context(local, stream=stream.cuda_stream)
    mesh = capi.Mesh.from_scene(ctx, base)  # same strips: one topology for every scene
    kw = dict(RESOLVE_KW, coloring_mode=args.coloring)
    d_x = torch.from_numpy(base.x).cuda()
    d_ys = [torch.from_numpy(y).cuda() for y in ys]
    d_out = torch.empty_like(d_x)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(max(args.warmup, 3)):
        for d_y in d_ys:
            capi.resolve_device_ptr(ctx, mesh, d_x.data_ptr(), d_y.data_ptr(), d_out.data_ptr(), **kw)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ms, steps = 0.0, 0
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for d_y in d_ys:
            st = capi.resolve_device_ptr(ctx, mesh, d_x.data_ptr(), d_y.data_ptr(), d_out.data_ptr(), **kw)
            steps += st["steps"]
        b.record(stream)
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    clk = clocks.stop()
    (ms_max,) = max_over_ranks([ms], dist, "cuda")
    if dist is not None:
        dist.destroy_process_group()
    if rank != 0:
        return None
    return {"metric": f"scene resolves/s, batch of {args.batch} reef knots (configs[4])",
            "value": round(args.batch * args.steps / (ms_max / 1e3), 3), "unit": "resolves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.batch} reef knots (37,400 V / 70,984 T each, rank-seeded targets), "
                                   f"{hi - lo} per rank on rank 0, resolved back to back",
                       "l2": "L2 flushed between timed steps", "parallelism": "scenes partitioned over ranks"},
            "resolve": {"alg1_steps_per_scene_resolve": steps / max(1, args.steps * (hi - lo))},
            "clocks": clk}


def main():
    args = parse()
    if args.batch > 0 and args.impl == "ours":
        out = run_batch(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    out, sc, st_tr = run_ours(args)
    if out is None:
        return
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{args.scene}_knot_trace.json"), "w") as f:
        json.dump(st_tr["trace"], f)
    if not args.no_cpu_baseline and out["n_gpus"] == 1:
        out["cpu_baseline"] = cpu_baseline(sc, st_tr["trace"], args.cpu_sample_steps)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
