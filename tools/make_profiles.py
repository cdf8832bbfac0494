"""Summarise a measurement pass (tools/gpu_measure.sh outputs in gpurun_out/)
into tracked files under profiles/, named per round:

  profiles/<tag>_bench.json            the default bench.py line
  profiles/<tag>_bench_reference.json  the --impl reference line
  profiles/<tag>_launches.csv          ncu launch list of the bench command
  profiles/<tag>_launch_summary.txt    per-kernel totals of that list
  profiles/<tag>_ncu_resolve.txt       --set full metrics + hottest source lines of k_resolve
  profiles/<tag>_ncu_search.txt        the same for the search stage kernel
  profiles/traffic.json                DRAM bytes per k_resolve launch (read by bench.py)

usage: python tools/make_profiles.py r01
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("TW_PROF_DIR") or os.path.join(ROOT, "profiles")  # staged on the GPU box
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stalls(h, row):
    res = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                res.append((float(row[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in res) or 1.0
    return [(100.0 * v / tot, k) for v, k in sorted(res, reverse=True)[:8]]


def lines(rep, kernel, top=25):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, kernel, str(top)],
                       capture_output=True, text=True)
    return r.stdout


def summarize(rep, kernel, title):
    h, u, rows = raw(rep)
    buf = [f"# {title}", f"# source: ncu --set full --clock-control none --import-source on ({os.path.basename(rep)})", ""]
    for n, row in enumerate(rows):
        buf.append(f"## launch {n}: {row[h.index('Kernel Name')]}")
        for k in METRICS:
            if k in h:
                i = h.index(k)
                buf.append(f"{k:70s} {row[i]:>16s} {u[i]}")
        buf.append("warp stall samples (share of sampled stalls):")
        for pct, k in stalls(h, row):
            buf.append(f"  {pct:5.1f}%  {k}")
        buf.append("")
    buf.append("hottest source lines (warp stall samples):")
    buf.append(lines(rep, kernel))
    return "\n".join(buf), h, u, rows


def launch_summary(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        agg[r[ki]][0] += 1
        agg[r[ki]][1] += v
    tot = sum(t for _, t in agg.values())
    out = ["# ncu --metrics gpu__time_duration.sum --clock-control none launch list of",
           "#   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras",
           "# (cold-cache, serialised replay: compare shares, not absolute times)",
           f"{'launches':>8s} {'total ms':>10s} {'share':>7s}  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{n:8d} {t:10.3f} {100 * t / tot:6.1f}%  {k[:110]}")
    return "\n".join(out) + "\n"


def main():
    os.makedirs(PROF, exist_ok=True)
    shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches.csv"))
    open(os.path.join(PROF, f"{tag}_launch_summary.txt"), "w").write(launch_summary(os.path.join(OUT, "launches.csv")))
    json.dump(last_json(os.path.join(OUT, "bench_full.log")), open(os.path.join(PROF, f"{tag}_bench.json"), "w"), indent=1)
    if os.path.exists(os.path.join(OUT, "acc_b200.log")):
        shutil.copy(os.path.join(OUT, "acc_b200.log"), os.path.join(PROF, f"{tag}_reference_acceptance_on_b200.txt"))
    json.dump(last_json(os.path.join(OUT, "bench_ref.log")), open(os.path.join(PROF, f"{tag}_bench_reference.json"), "w"),
              indent=1)
    txt, h, u, rows = summarize(os.path.join(OUT, "prof_resolve.ncu-rep"), "k_resolve",
                                "k_pcg_reg + k_resolve: one bow-knot simulation frame (tools/prof_drive.py)")
    open(os.path.join(PROF, f"{tag}_ncu_resolve.txt"), "w").write(txt)
    row = next(r for r in rows if "k_resolve" in r[h.index("Kernel Name")])
    gb = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd = float(row[h.index("dram__bytes_read.sum")].replace(",", "")) * gb[u[h.index("dram__bytes_read.sum")]]
    wr = float(row[h.index("dram__bytes_write.sum")].replace(",", "")) * gb[u[h.index("dram__bytes_write.sum")]]
    json.dump({"kernel": "k_resolve", "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
               "source": f"profiles/{tag}_ncu_resolve.txt"}, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    txt, *_ = summarize(os.path.join(OUT, "prof_search.ncu-rep"), "k_stage_search",
                        "k_stage_search: stage search on the bow knot (tools/prof_search.py)")
    open(os.path.join(PROF, f"{tag}_ncu_search.txt"), "w").write(txt)
    print("wrote", sorted(f for f in os.listdir(PROF) if f.startswith(tag)))


if __name__ == "__main__":
    main()
