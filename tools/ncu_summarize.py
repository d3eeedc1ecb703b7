"""Summarize ncu captures into profiles/ (dev tool, runs in the build container).

    python tools/ncu_summarize.py TAG gpurun_out/bits_c5_aco.ncu-rep:c5_aco [...]
        -> profiles/ncu_TAG.md (key metrics + per-phase SASS split) and
           profiles/ncu_traffic.json[workload] = dram read+write bytes per launch
    python tools/ncu_summarize.py --launches TAG gpurun_out/launches.csv
        -> profiles/launches_TAG.md (per-kernel launch counts / time shares)
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__grid_size", "CTAs"),
    ("launch__block_size", "threads/CTA"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]

# SASS between consecutive BAR.SYNCs of step_bits_kernel, in address order;
# the noinline draw functions (lem_choose / aco_choose / AS241) sit after EXIT.
PHASES = ["prologue (mbarrier init)", "work-item fetch", "item setup + first-window TMA",
          "tile start: TMA prefetch/wait + S0 planes", "S1 intents (bit logic + enqueue)", "S1 draw queue",
          "queue reset", "S2 claims/winners/grants", "S2 contested-cell draws", "S3 commit (+ACO pheromone)",
          "per-item counter flush", "draw functions (lem_choose/aco_choose/AS241)"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


def to_bytes(v, unit):
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return x * scale


def phases(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    seg, acc = 0, defaultdict(lambda: [0.0, 0.0])
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]]
        acc[seg][0] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        acc[seg][1] += float(r[ix["Instructions Executed"]] or 0)
        if "BAR.SYNC" in src:
            seg += 1
    ts = sum(v[0] for v in acc.values()) or 1
    ti = sum(v[1] for v in acc.values()) or 1
    # SASS block order does not follow source order and some barriers are
    # conditional, so segments are labelled by position, not by phase name.
    return [(f"SASS segment {k}", v[0] / ts * 100, v[1] / ti * 100, v[1]) for k, v in sorted(acc.items())]


def summarize(tag, specs):
    os.makedirs(PROF, exist_ok=True)
    tpath = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    lines = [f"# ncu --set full summaries ({tag})", "",
             "Captured with `ncu --set full --clock-control none --import-source on -k regex:step_bits -s S -c 1` "
             "on `python tools/profile_step.py <workload> S+2` (one launch at step S, named in each heading; cold "
             "caches, serialised: compare shares, not absolute times, with the bench).", ""]
    for spec in specs:
        # rep:workload[:steps] -- steps > 1 for a multi-step launch (per-step traffic = launch / steps)
        parts = spec.split(":")
        rep, workload = parts[0], parts[1]
        nsteps = int(parts[2]) if len(parts) > 2 else 1
        d = raw(rep)
        rd = to_bytes(*d["dram__bytes_read.sum"])
        wr = to_bytes(*d["dram__bytes_write.sum"])
        traffic[workload] = (rd + wr) / nsteps
        head = f"## {workload} — `{os.path.basename(rep)}`"
        if nsteps > 1:
            head += f" (one multi-step launch of {nsteps} steps)"
        lines += [head, "", "| metric | value |", "|---|---|"]
        for key, name in KEYS:
            if key in d:
                lines.append(f"| {name} (`{key}`) | {d[key][0]} {d[key][1]} |")
        lines.append(f"| DRAM read+write per launch | {(rd + wr) / 1e9:.3f} GB |")
        if nsteps > 1:
            lines.append(f"| DRAM read+write per step | {(rd + wr) / nsteps / 1e9:.3f} GB |")
            dur = d.get("gpu__time_duration.sum")
            if dur:
                x = float(dur[0].replace(",", "")) * {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
                                                      "nsecond": 1e-3}.get(dur[1], 1)
                lines.append(f"| duration per step | {x / nsteps:.2f} us |")
        ph = phases(rep)
        if ph:
            lines += ["", "| phase (SASS between barriers) | stall samples % | instructions % | warp instructions |",
                      "|---|---|---|---|"]
            lines += [f"| {n} | {s:.1f} | {i:.1f} | {c:.3g} |" for n, s, i, c in ph]
        lines.append("")
    with open(os.path.join(PROF, f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(lines))
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines))


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "s": 1e6,
              "second": 1e6}.get(unit, 1)
        per[name][0] += 1
        per[name][1] += v
    tot = sum(v[1] for v in per.values()) or 1
    lines = [f"# Kernel launch list ({tag})", "", f"Source: `{os.path.basename(path)}` "
             "(`ncu --metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised).", "",
             "| kernel | launches | total us | mean us | share of GPU time |", "|---|---|---|---|---|"]
    for name, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {n} | {t:.1f} | {t / n:.2f} | {t / tot * 100:.1f}% |")
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"launches_{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        summarize(sys.argv[1], sys.argv[2:])
