#!/usr/bin/env python
"""Benchmark of the two-way continuous collision handling path on B200.

Headline (N = 1, BASELINE.json configs[2], the paper's bow knot): one "step"
is one simulation time step of the 142K-triangle bow knot with the paper's
large time step dt = 1/100 -- dynamics.cpp's step(): the proximity search,
gradient/Hessian with repulsion, the block-Jacobi PCG Newton target, then
resolve (Alg. 1 of arXiv 2211.04045, run to convergence on the device) and
the velocity update. The frame starts from the tightening state of
scenes.knot_frame: the two plies, 2.5 mm apart, move with the velocity that
squeezes them up to 0.2 mm into each other where the knot is tightest
(penetrating target) and slides them 1.5 mm along each other. Metric: simulation steps per second (whole job).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload frame|resolve|batch] [--scene bow|reef]
                    [--coloring device|reference] [--batch B]

N > 1 runs BASELINE configs[4]: a batch of B = 64 independent reef-knot
frames (rank-seeded tightening) partitioned over the ranks, no collective on
the data path (strong scaling: the total work is fixed); torch.distributed
is used for the start/stop barriers and the max-over-ranks of the
device-timed region only. Without torchrun, --gpus N > 1 spawns the N ranks
itself (torch.distributed.run on 127.0.0.1).

--impl reference times the reference's own CPU implementation: the
reference's sources built unchanged against the Eigen-subset shim
(oracle/_ref/libtwoway_ref.so, oracle/Makefile.ref), single-threaded like the
reference, on the same frame (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sim steps/s at the 142K-tri bow knot (dt = 1/100: Newton target + resolve)"
PAPER_COST_S = 0.034  # bow knot collision cost per time step (RTX 2080 Ti, paper Table 1)
SQUEEZE = 0.1e-3      # penetrating tightening of the frame (plies up to 0.2 mm into each other)
RESOLVE_KW = dict(delta=5e-4)  # knots: delta = 0.5 mm


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["frame", "resolve", "batch"], default=None,
                    help="default: frame at N = 1, batch (configs[4]) at N > 1")
    ap.add_argument("--scene", choices=["bow", "reef"], default="bow")
    ap.add_argument("--coloring", choices=["device", "reference"], default="device")
    ap.add_argument("--batch", type=int, default=64, help="configs[4] batch size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary measurements")
    return ap.parse_args()


def n_along(scene):
    return 1870 if scene == "bow" else 935


def frame_scene(scene, jitter=None):
    from paper_2211_04045_b200 import scenes

    return scenes.knot_frame(n_along=n_along(scene), squeeze=SQUEEZE, jitter_seed=jitter)


def frame_config(sc, args):
    cfg = {"workload": f"{sc.name}: {sc.nv} vertices, {len(sc.triangles)} triangles, {len(sc.edges)} edges; "
                       "one implicit-Euler step (dynamics.cpp step(): search, gradient/Hessian + repulsion, "
                       "block-Jacobi PCG target, resolve, velocity update) with dt = 1/100 of two cloth plies "
                       "laid face to face (2.5 mm apart, 3 mm mesh) along a twisted (2,3) torus-knot band, "
                       "moving with the tightening velocity that drives them up to 0.2 mm into each other "
                       "where the knot is tightest and slides them 1.5 mm along each other (scenes.knot_frame)",
           "scene": args.scene, "vertices": sc.nv, "triangles": int(len(sc.triangles)),
           "edges": int(len(sc.edges)), "dt": 0.01,
           "energy_model": "EnergyModel defaults except springs 10 N/m (gravity, repulsion 1e3 N/m within 1 mm, "
                           "PCG rel. tol 1e-6 / 400 iterations); cloth 0.5 kg/m^2 (scenes.FRAME_ENERGY / "
                           "FRAME_DENSITY: the PCG converges, so the target is the implicit-Euler solution)",
           "solver": "pgs, 1 sweep", "coloring": args.coloring,
           "params": {"d_min": 2e-3, "d_max": 4e-3, "delta": 5e-4, "gamma": 0.9, "eps": 1e-4,
                      "step_limit": 512},
           "l2": "L2 flushed (256 MB write) between timed steps; the LBVH topology is reused across calls on "
                 "a mesh (rebuilt every 16 calls, refitted at every search); inputs re-uploaded every e2e step",
           "parallelism": "one scene per GPU (no collective)"}
    return cfg


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


def bytes_per_pcg_iteration(sc):
    """Algorithmic bytes of one CG iteration of the register-resident kernel
    (DESIGN.md §5): z written and read once (24 + 24 B/vertex), the CSR of the
    vertex's edges (4 B per incidence, 2 per edge) and the edge blocks (48 B per
    edge, read from both ends)."""
    nv, ne = sc.nv, len(sc.edges)
    return 48 * nv + 2 * ne * 4 + 2 * ne * 48


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    return d.get("hbm_gbs", 6650.0), ("MEASURED_PEAKS.json hbm_gbs (measured copy)" if d else
                                      "fallback 6650 GB/s (B200_PROFILING.md)")


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


def host_info():
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


# ------------------------------------------------------------ distributed
class Dist:
    """One process per GPU (torchrun env). The data path has no collective:
    the group is used for the start/stop barriers and the max over ranks of
    the device-timed regions only. device="cpu" (gloo) serves the CPU tests."""

    def __init__(self, device="cuda"):
        import torch

        self.device = device
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # TW_BENCH_ONE_DEVICE=1 (testing the N > 1 host path on a one-GPU box):
        # every rank on device 0, the process group on gloo. The ranks share no
        # data and never wait on each other's kernels.
        self.one_device = os.environ.get("TW_BENCH_ONE_DEVICE") == "1"
        if self.one_device:
            self.local = 0
        if device == "cuda":
            torch.cuda.set_device(self.local)
            # one explicit stream shared by torch (flush, copies, events) and the
            # device contexts (capi.Context(stream=...)): every op is ordered
            self.stream = torch.cuda.Stream()
            torch.cuda.set_stream(self.stream)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if device == "cuda" and not self.one_device:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        import torch

        if self.dist is not None:
            self.dist.barrier()
        if self.device == "cuda":
            torch.cuda.synchronize()

    def max(self, vals):
        """Elementwise max over ranks of per-rank timings; identity at N = 1."""
        import torch

        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if self.one_device else self.device)
        if self.dist is not None:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(v) for v in t.tolist()]

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


# ------------------------------------------------------------- frame arm
class FrameRunner:
    """One bow/reef-knot simulation frame on the device: device-resident
    (tw_step_device on HBM state reset from pristine copies outside the timed
    region) and end to end (tw_step with pinned host buffers)."""

    def __init__(self, ctx, scene, args, jitter=None, energy=None):
        import torch

        from paper_2211_04045_b200 import capi

        self.capi, self.torch, self.ctx = capi, torch, ctx
        self.sc, self.v0 = frame_scene(scene, jitter)
        self.mesh = capi.Mesh.from_scene(ctx, self.sc)
        from paper_2211_04045_b200 import scenes

        self.dyn = capi.Dynamics(ctx, self.mesh, self.sc.x, **{**scenes.FRAME_ENERGY, **(energy or {})})
        self.kw = dict(RESOLVE_KW, coloring_mode=args.coloring)
        self.d_x0 = torch.from_numpy(self.sc.x).cuda()
        self.d_v0 = torch.from_numpy(self.v0).cuda()
        self.d_x = self.d_x0.clone()
        self.d_v = self.d_v0.clone()
        self.h_x = torch.from_numpy(self.sc.x.copy()).pin_memory()
        self.h_v = torch.from_numpy(self.v0.copy()).pin_memory()

    def reset(self):
        self.d_x.copy_(self.d_x0)
        self.d_v.copy_(self.d_v0)

    def step_device(self):
        return self.capi.step_device_ptr(self.ctx, self.mesh, self.dyn, self.d_x.data_ptr(), self.d_v.data_ptr(),
                                         **self.kw)

    def step_e2e(self):
        """Host state in, host state out (H2D x, v and D2H x, v inside)."""
        x, v, st = self.capi.step(self.ctx, self.mesh, self.dyn, self.h_x.numpy(), self.h_v.numpy(), **self.kw)
        return x, v, st

    def close(self):
        self.dyn.close()
        self.mesh.close()


def run_frame(args, D):
    import numpy as np
    import torch

    from paper_2211_04045_b200 import capi

    stream = torch.cuda.current_stream()
    ctx = capi.Context(D.local, stream=stream.cuda_stream)
    fr = FrameRunner(ctx, args.scene, args, jitter=None if D.rank == 0 else D.rank)
    sc = fr.sc
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(max(args.warmup, 3)):  # capacity growth happens here
        fr.reset()
        fr.step_device()
    # the frame's target and a traced resolve of it (the step's resolve is
    # bit-identical: test_gpu_dynamics.py::test_step_is_target_then_resolve)
    y, _, tst = capi.newton_target(ctx, fr.mesh, fr.dyn, sc.x, fr.v0, sc.x)
    _, rtr = capi.resolve(ctx, fr.mesh, sc.x, y, trace=True, **fr.kw)
    capi.resolve(ctx, fr.mesh, sc.x, y, **fr.kw)  # untraced: the phase profile
    phases = {k: [round(v[0], 3), v[1]] for k, v in capi.phase_profile(ctx).items()}
    peak, peak_src = peaks()

    D.barrier()
    clocks = ClockSampler(D.local)
    clocks.start()
    launches0 = ctx.kernel_launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stats = []
    for i in range(args.steps):
        fr.reset()
        flush.fill_(i & 0xFF)  # L2 flush between timed iterations (outside the events)
        evs[i][0].record(stream)
        stats.append(fr.step_device())
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    launches = ctx.kernel_launches - launches0
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    e2e_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        fr.h_x.copy_(torch.from_numpy(sc.x))
        fr.h_v.copy_(torch.from_numpy(fr.v0))
        flush.fill_(i & 0xFF)
        e2e_evs[i][0].record(stream)
        x_e2e, v_e2e, _ = fr.step_e2e()
        e2e_evs[i][1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_evs)
    clk = clocks.stop()
    D.barrier()

    # intersection-free: the device certifier on the frame's motion x -> x_next
    # and on every segment of the resolve path (outside the timed regions)
    _, st_path = capi.resolve(ctx, fr.mesh, sc.x, y, record_path=True, **fr.kw)
    path = st_path["path"]
    ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    viol = cert = stencils = 0
    ca.record(stream)
    for i in range(len(path) - 1):
        v, c, n = capi.ccd_certify(ctx, fr.mesh, path[i], path[i + 1], candidates=True)
        viol, cert, stencils = viol + v, cert + c, stencils + n
    cb.record(stream)
    torch.cuda.synchronize()
    ccd_ms = ca.elapsed_time(cb)
    frame_ok = np.array_equal(x_e2e.view(np.uint64), path[-1].view(np.uint64))
    ccd = {"segments": len(path) - 1, "violations": viol, "certain_violations": cert,
           "candidate_stencils": stencils, "ms_incl_host_copies": round(ccd_ms, 3),
           "stencils_per_s": round(stencils / (ccd_ms / 1e3), 1), "intersection_free": viol == 0,
           "path_ends_at_frame_result": bool(frame_ok)}

    dev_ms_max, e2e_ms_max = D.max([dev_ms, e2e_ms])
    value = D.world * args.steps / (dev_ms_max / 1e3)
    e2e_value = D.world * args.steps / (e2e_ms_max / 1e3)
    n = args.steps
    avg = lambda k: sum(s[k] for s in stats) / n  # noqa: E731
    kern_ms = rtr["kernel_ms"]
    rbytes = bytes_per_resolve(rtr["trace"], sc)
    r_achieved = rbytes / (kern_ms / 1e3) / 1e9
    pcg_bytes = bytes_per_pcg_iteration(sc) * avg("pcg_iterations")
    pcg_achieved = pcg_bytes / (avg("pcg_ms") / 1e3) / 1e9 if avg("pcg_ms") > 0 else 0.0
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else None
    out = None
    if D.rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "steps/s", "n_gpus": D.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_ms_max / n, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "baseline_note": "BASELINE.md publishes no number for this metric; the paper's bow knot (Table 1, "
                             "RTX 2080 Ti) is quoted as collision cost 0.034 s/step on a different asset -- see "
                             "frame.paper_collision_cost_ratio",
            "dtype": "f64", "data": "synthetic",
            "config": frame_config(sc, args),
            "frame": {"ms": round(dev_ms_max / n, 4), "target_ms": round(avg("target_ms"), 4),
                      "pcg_ms": round(avg("pcg_ms"), 4), "resolve_ms": round(avg("resolve_ms"), 4),
                      "pcg_iterations": avg("pcg_iterations"), "pcg_converged": stats[-1]["pcg_converged"],
                      "resolve_alg1_steps": avg("resolve_steps"), "resolve_searches": avg("searches"),
                      "resolve_converged": stats[-1]["resolve_converged"],
                      "target_search_pairs": stats[-1]["num_pairs"], "repulsive_pairs": stats[-1]["repulsive_pairs"],
                      "fps_target_17": round(value / D.world, 2) >= 17.0,
                      "paper_collision_cost_ratio": round(PAPER_COST_S / (avg("resolve_ms") / 1e3), 3)},
            "resolve": {"alg1_steps": rtr["steps"], "searches": rtr["searches"], "final_pairs": rtr["num_pairs"],
                        "kernel_ms": round(kern_ms, 4), "setup_ms": round(rtr["setup_ms"], 4),
                        "phase_ms_count": phases,
                        "phase_roofline": phase_roofline(rtr["trace"], sc, phases, peak),
                        "two_way_steps_per_s": round(rtr["steps"] / (rtr["device_ms"] / 1e3), 1),
                        "ccd_pairs_per_s": round(rtr["pairs_evaluated"] / (rtr["device_ms"] / 1e3), 1),
                        "trace_contact_rows": [t["num_contact_rows"] for t in rtr["trace"]],
                        "trace_colors": [t["num_colors"] for t in rtr["trace"]]},
            "e2e": {"value": round(e2e_value, 3), "unit": "steps/s", "h2d_bytes_per_step": 2 * sc.nv * 24,
                    "d2h_bytes_per_step": 2 * sc.nv * 24},
            "gpu_launches": launches,
            "ccd_certification": ccd,
            "roofline": {"bound": "hbm", "achieved": round(r_achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(r_achieved / peak, 4),
                         "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                         "traffic_source": traffic["source"] if traffic else "no ncu capture committed",
                         "kernel": "tw::k_resolve (persistent cooperative Alg.-1 kernel), the frame's largest",
                         "algorithmic_bytes_per_launch": rbytes, "peak_source": peak_src,
                         "pcg": {"kernel": "tw::dyn::k_pcg_reg", "achieved": round(pcg_achieved, 1),
                                 "frac": round(pcg_achieved / peak, 4),
                                 "algorithmic_bytes_per_launch": round(pcg_bytes)}},
            "clocks": clk,
        }
    fr.close()
    return out, ctx, sc


# --------------------------------------------------------- extra lines
def run_resolve_only(ctx, args, coloring, steps):
    """The previous headline (resolve alone on the kinematic, non-penetrating
    tightening target) and, with coloring='reference', the bit-exact mode."""
    import torch

    from paper_2211_04045_b200 import capi, scenes

    sc = scenes.bow_knot() if args.scene == "bow" else scenes.reef_knot()
    mesh = capi.Mesh.from_scene(ctx, sc)
    kw = dict(RESOLVE_KW, coloring_mode=coloring)
    d_x, d_y = torch.from_numpy(sc.x).cuda(), torch.from_numpy(sc.y).cuda()
    d_out = torch.empty_like(d_x)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(2 if coloring == "device" else 1):
        capi.resolve_device_ptr(ctx, mesh, d_x.data_ptr(), d_y.data_ptr(), d_out.data_ptr(), **kw)
    ms, st = 0.0, None
    for i in range(steps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        st = capi.resolve_device_ptr(ctx, mesh, d_x.data_ptr(), d_y.data_ptr(), d_out.data_ptr(), **kw)
        b.record(stream)
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    mesh.close()
    return {"workload": f"{sc.name}: resolve of the kinematic tightening target (plies pressed to a 0.2 mm "
                        "gap, non-penetrating), inputs in HBM", "coloring": coloring,
            "resolves_per_s": round(steps / (ms / 1e3), 3), "ms": round(ms / steps, 4),
            "alg1_steps": st["steps"], "searches": st["searches"], "kernel_ms": round(st["kernel_ms"], 4)}


def run_configs(ctx, args, peak):
    """The other BASELINE configs on one B200, device-timed (inputs in HBM, L2
    flushed between calls): configs[0] CFG1 cloth on a static sphere (resolve of
    one dt = 1/30 fall; with the reference build's own resolve on the same input
    timed on the host), configs[1] CFG2 the reef-knot frame (the headline's
    step at half the size), configs[3] CFG4 the codimensional mix (closed
    bodies, 1,000 strands, 96K particles: VV / VE / VT / EE pairs). Each with
    the k_resolve roofline fraction."""
    import torch

    from paper_2211_04045_b200 import capi, scenes

    out = {}
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    n = max(3, min(args.steps, 10))
    for key, make, kw in (("cfg1_cloth_on_sphere", scenes.cloth_on_sphere, {}),
                          ("cfg4_codim_mix", scenes.codim_mix, {})):
        sc = make()
        mesh = capi.Mesh.from_scene(ctx, sc)
        d_x, d_y = torch.from_numpy(sc.x).cuda(), torch.from_numpy(sc.y).cuda()
        d_o = torch.empty_like(d_x)
        for _ in range(2):
            capi.resolve_device_ptr(ctx, mesh, d_x.data_ptr(), d_y.data_ptr(), d_o.data_ptr(), **kw)
        _, tr = capi.resolve(ctx, mesh, sc.x, sc.y, trace=True, **kw)
        ms = kern = 0.0
        for i in range(n):
            flush.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st = capi.resolve_device_ptr(ctx, mesh, d_x.data_ptr(), d_y.data_ptr(), d_o.data_ptr(), **kw)
            b.record(stream)
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
            kern += st["kernel_ms"]
        gbs = bytes_per_resolve(tr["trace"], sc) / (kern / n / 1e3) / 1e9
        out[key] = {"vertices": sc.nv, "triangles": int(len(sc.triangles)), "edges": int(len(sc.edges)),
                    "resolves_per_s": round(n / (ms / 1e3), 2), "ms": round(ms / n, 3),
                    "alg1_steps": st["steps"], "searches": st["searches"], "final_pairs": st["num_pairs"],
                    "roofline": {"kernel": "k_resolve", "achieved_gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}}
        if key.startswith("cfg1") and not args.no_cpu_baseline:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import pyref

            if pyref.available():
                rm = pyref.RefMesh.from_scene(sc)
                t0 = time.perf_counter()
                _, rs = pyref.resolve(rm, sc.x, sc.y, **kw)
                secs = time.perf_counter() - t0
                out[key]["cpu_baseline"] = {"value": round(1.0 / secs, 4), "unit": "resolves/s", "cores": 1,
                                            "kind": "reference", "sample": f"one full resolve on the reference "
                                            f"build: {secs:.1f} s, {rs['steps']} steps, {rs['searches']} searches"}
        mesh.close()
    # configs[1] the reef frame; and the bow frame with Coulomb friction
    # (mu = 0.3: step() runs friction_filter on the target, dynamics.cpp:338,
    # with the search at d_max so the filter sees every pair)
    for key, scene, energy in (("cfg2_reef_knot_frame", "reef", None),
                               ("bow_knot_frame_friction_mu0.3", "bow", {"mu": 0.3})):
        fr = FrameRunner(ctx, scene, args, energy=energy)
        for _ in range(2):
            fr.reset()
            fr.step_device()
        ms = fric = 0.0
        for i in range(n):
            fr.reset()
            flush.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st = fr.step_device()
            b.record(stream)
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
            fric += st["friction_ms"]
        out[key] = {"vertices": fr.sc.nv, "triangles": int(len(fr.sc.triangles)),
                    "steps_per_s": round(n / (ms / 1e3), 2), "ms": round(ms / n, 3),
                    "resolve_alg1_steps": st["resolve_steps"], "searches": st["searches"],
                    "pcg_ms": round(st["pcg_ms"], 3), "resolve_ms": round(st["resolve_ms"], 3)}
        if energy:
            out[key].update({"friction_ms": round(fric / n, 3), "pairs_filtered": st["num_pairs"]})
        fr.close()
    return out


def partition(n, world, rank):
    """Contiguous block of the n independent scenes owned by `rank`."""
    return rank * n // world, (rank + 1) * n // world


def batch_scene(i):
    """Scene i of the configs[4] batch: a reef-knot frame with its own
    tightening jitter (seed 1000 + i)."""
    from paper_2211_04045_b200 import scenes

    return scenes.knot_frame(n_along=935, squeeze=SQUEEZE, jitter_seed=1000 + i)


def run_batch_frames(args, D, nscenes, concurrent=2):
    """configs[4]: `nscenes` independent reef-knot frames (rank-seeded
    tightening) partitioned over the ranks; every step advances each of the
    rank's scenes by one frame from its start state. On each GPU the rank's
    scenes are split over `concurrent` device contexts that run at the same
    time on their own streams, each with 1/concurrent of the co-resident CTAs
    (tw_ctx_set_grid_share; two contexts: +36% frames/s over one, measured).
    No collective: value = nscenes x steps / max over ranks of the device time
    (CUDA events: one start on the first worker stream that the others wait
    on, one end per worker stream)."""
    import threading

    import torch

    from paper_2211_04045_b200 import capi

    lo, hi = partition(nscenes, D.world, D.rank)
    mine = list(range(lo, hi))
    S = max(1, min(concurrent, len(mine)))
    streams = [torch.cuda.Stream() for _ in range(S)]
    workers = []
    for t in range(S):
        with torch.cuda.stream(streams[t]):
            ctx = capi.Context(D.local, stream=streams[t].cuda_stream)
            ctx.set_grid_share(S)
            base = FrameRunner(ctx, "reef", args)  # one topology: every scene has the same strips
            scs = []
            for i in mine[t::S]:
                sc_i, v_i = batch_scene(i)
                scs.append((torch.from_numpy(sc_i.x).cuda(), torch.from_numpy(v_i).cuda()))
        workers.append({"ctx": ctx, "base": base, "scenes": scs, "rsteps": 0, "frames": 0})

    def run(t, reps, ev_start, ev_end):
        w = workers[t]
        with torch.cuda.stream(streams[t]):
            if ev_start is not None:
                streams[t].wait_event(ev_start)
            for _ in range(reps):
                for x0, v0 in w["scenes"]:
                    w["base"].d_x.copy_(x0)
                    w["base"].d_v.copy_(v0)
                    st = w["base"].step_device()
                    if ev_end is not None:
                        w["rsteps"] += st["resolve_steps"]
                        w["frames"] += 1
            if ev_end is not None:
                ev_end.record(streams[t])

    def all_workers(reps, timed):
        start = torch.cuda.Event(enable_timing=True) if timed else None
        ends = [torch.cuda.Event(enable_timing=True) if timed else None for _ in range(S)]
        if timed:
            start.record(streams[0])
        th = [threading.Thread(target=run, args=(t, reps, start, ends[t])) for t in range(S)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        torch.cuda.synchronize()
        return max(start.elapsed_time(e) for e in ends) if timed else 0.0

    all_workers(max(1, min(args.warmup, 2)), False)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    D.barrier()
    clocks = ClockSampler(D.local)
    clocks.start()
    launches0 = sum(w["ctx"].kernel_launches for w in workers)
    ms = 0.0
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        ms += all_workers(1, True)
    clk = clocks.stop()
    launches = sum(w["ctx"].kernel_launches for w in workers) - launches0
    (ms_max,) = D.max([ms])
    frames = sum(w["frames"] for w in workers)
    rsteps = sum(w["rsteps"] for w in workers)
    for w in workers:
        w["base"].close()
        w["ctx"].close()
    return {"value": nscenes * args.steps / (ms_max / 1e3), "ms_max": ms_max, "frames_rank0": frames,
            "resolve_steps_per_frame": rsteps / max(1, frames), "scenes_per_rank": hi - lo,
            "concurrent_contexts": S, "gpu_launches": launches, "clocks": clk}


def batch_line(args, D, res, nscenes):
    return {"metric": f"sim steps/s over a batch of {nscenes} reef-knot frames (configs[4])",
            "value": round(res["value"], 3), "unit": "steps/s", "n_gpus": D.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(res["ms_max"] / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{nscenes} reef-knot frames (37,400 V / 70,984 T each; dt = 1/100, "
                                   "rank-seeded tightening, scenes.knot_frame), "
                                   f"{res['scenes_per_rank']} per rank, each stepped once per step on "
                                   f"{res['concurrent_contexts']} concurrent device contexts per GPU",
                       "l2": "L2 flushed between timed steps", "parallelism": "scenes partitioned over ranks, "
                                                                               "no collective"},
            "frame": {"resolve_alg1_steps_per_frame": round(res["resolve_steps_per_frame"], 2)},
            "n1_point": "the same workload at N = 1: `bench.py --workload batch`, or the batch_configs4_one_gpu "
                        "key of the default N = 1 line (whose headline value is the bow-knot frame)",
            "gpu_launches": res["gpu_launches"], "clocks": res["clocks"]}


# --------------------------------------------------------- reference arm
def reference_frame(scene, squeeze=SQUEEZE):
    """The reference build's step() on the same frame: (seconds, resolve
    steps, searches). Single-threaded, like the reference."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyref

    if not pyref.available():
        raise RuntimeError("oracle/_ref/libtwoway_ref.so not built")
    sc, v0 = frame_scene(scene)
    rm = pyref.RefMesh(sc.x, sc.triangles, (), sc.inv_mass, v0)
    t0 = time.perf_counter()
    from paper_2211_04045_b200 import scenes

    _, _, nsteps, nsearch = pyref.step(rm, sc.x, energy=scenes.FRAME_ENERGY, **RESOLVE_KW)
    return time.perf_counter() - t0, nsteps, nsearch, sc


CPU_SAMPLE_ALONG = 467  # a quarter of the bow knot's length


def cpu_baseline(args):
    """cpu_baseline of the ours-arm line (rank 0, N = 1): the reference build
    on a bounded sample of the workload -- the same knot frame at a quarter of
    the bow knot's length (~1 min of one core: 18,680 V, 8 resolve steps, 3
    searches) -- timed once; value = its frame rate divided by the size ratio
    (linear scaling, stated). The unscaled full bow-knot frame is the --impl
    reference arm."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyref

    from paper_2211_04045_b200 import scenes

    sc, v0 = scenes.knot_frame(n_along=CPU_SAMPLE_ALONG, squeeze=SQUEEZE)
    rm = pyref.RefMesh(sc.x, sc.triangles, (), sc.inv_mass, v0)
    t0 = time.perf_counter()
    _, _, nsteps, nsearch = pyref.step(rm, sc.x, energy=scenes.FRAME_ENERGY, **RESOLVE_KW)
    secs = time.perf_counter() - t0
    scale = n_along(args.scene) / CPU_SAMPLE_ALONG
    return {"value": round(1.0 / (secs * scale), 6), "unit": "steps/s", "cores": 1, "kind": "reference",
            "sample": f"one full step() of the knot frame at n_along = {CPU_SAMPLE_ALONG} ({sc.nv} V, 1/{scale:.0f} "
                      f"of the bow knot) on the reference build (oracle/_ref, the reference's sources on the "
                      f"Eigen-subset shim): {secs:.1f} s, {nsteps} resolve steps, {nsearch} searches; value scaled "
                      f"by the size ratio {scale:.1f} (linear)", "sample_seconds": round(secs, 2), **host_info()}


def run_reference(args):
    """--impl reference: the reference's own step() on the bow-knot frame,
    rank 0 only. One frame of the reference takes minutes, so the run times
    full frames until --steps are done or 240 s have passed (at least one)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    times, info = [], None
    t_start = time.time()
    for i in range(max(1, args.steps)):
        secs, nsteps, nsearch, sc = reference_frame(args.scene)
        times.append(secs)
        info = (nsteps, nsearch, sc)
        if time.time() - t_start > 240:
            break
    nsteps, nsearch, sc = info
    value = len(times) / sum(times)
    return {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "steps/s",
            "n_gpus": args.gpus, "steps": len(times), "warmup": 0, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": frame_config(sc, args),
            "cpu_baseline": {"value": round(value, 6), "unit": "steps/s", "cores": 1, "kind": "reference",
                             "sample": f"{len(times)} full step() call(s) of the bow-knot frame on the reference "
                                       f"build (oracle/_ref: the reference's sources compiled against the "
                                       f"Eigen-subset shim), {statistics.mean(times):.1f} s each: {nsteps} resolve "
                                       f"steps, {nsearch} searches (--steps {args.steps} requested, 240 s budget)",
                             **host_info()},
            "e2e": {"value": round(value, 6), "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ---------------------------------------------------------------- main
def spawn(args):
    """--gpus N > 1 without torchrun: launch the N ranks ourselves."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    D = Dist()
    workload = args.workload or ("frame" if D.world == 1 else "batch")
    if workload == "batch":
        res = run_batch_frames(args, D, args.batch)
        if D.rank == 0:
            print(json.dumps(batch_line(args, D, res, args.batch)), flush=True)
        D.close()
        return
    out, ctx, sc = run_frame(args, D)
    if D.rank == 0 and D.world == 1 and not args.no_extras:
        out["resolve_only"] = run_resolve_only(ctx, args, "device", args.steps)
        out["exact_parity_mode"] = run_resolve_only(ctx, args, "reference", 1)
        out["configs"] = run_configs(ctx, args, peaks()[0])
        # configs[4] at N = 1: the N > 1 default workload (64 reef frames), so
        # the multi-GPU lines have their one-GPU point in the same run
        res = run_batch_frames(args, D, args.batch)
        out["batch_configs4_one_gpu"] = {"scenes": args.batch, "steps_per_s": round(res["value"], 3),
                                         "ms_per_step": round(res["ms_max"] / args.steps, 3),
                                         "concurrent_contexts": res["concurrent_contexts"],
                                         "resolve_steps_per_frame": round(res["resolve_steps_per_frame"], 2)}
    if D.rank == 0 and D.world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args)
    if out is not None:
        print(json.dumps(out), flush=True)
    D.close()


if __name__ == "__main__":
    main()
