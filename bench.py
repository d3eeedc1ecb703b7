#!/usr/bin/env python3
"""Benchmark of the per-step grid update (BASELINE.json metric: agent-updates/s
and cell-updates/s per step, achieved HBM GB/s vs peak, 1/2/4/8 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5_aco]
    torchrun --nproc-per-node N bench.py --gpus N ...      (row-sharded)
    python bench.py --impl reference ...                    (the reference CPU path)

Default workload: C5 of BASELINE.json — ACO, 16384 x 16384 grid, 25,000,000
agents per side (50M) — the largest configuration, the one the 1/2/4/8-GPU
scaling is quoted on; at N GPUs it is row-sharded (strong scaling): the step
kernels store their 3 boundary rows into the neighbours' ghost rows (CUDA IPC
peer memory over NVLink) with a device-side handshake per step. A step is one full StepEngine::step of the
whole grid. The other BASELINE configs are parity cases; the 100K-agent config
(C4) is reported under "secondary" as a replica-batched run (64 seeds per
launch), its single-scenario step time beside it.

Timing: W untimed warm-up steps, then K steps bracketed by a barrier and a
device synchronize, timed with CUDA events on the library's stream, max over
ranks. Resident state (~13 GB at C5) is far larger than the 126 MB L2, so no
flush is needed between steps. ``value`` counts agent-updates of all ranks.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (width, height, agents_per_side, model, replicas, description)
    "c5_aco": (16384, 16384, 25_000_000, "aco", 1, "C5: ACO 16384x16384, 25M agents/side (50M), seed 42"),
    "c5_lem": (16384, 16384, 25_000_000, "lem", 1, "C5-LEM: LEM 16384x16384, 25M agents/side (50M), seed 42"),
    "c4_aco_x64": (480, 480, 51_200, "aco", 64, "C4 x64: ACO 480x480, 51,200 agents/side, 64 seeds per launch"),
    "c3_lem_x64": (480, 480, 51_200, "lem", 64, "C3 x64: LEM 480x480, 51,200 agents/side, 64 seeds per launch"),
    "c4_aco": (480, 480, 51_200, "aco", 1, "C4: ACO 480x480, 51,200 agents/side (102,400), seed 42"),
    "c3_lem": (480, 480, 51_200, "lem", 1, "C3: LEM 480x480, 51,200 agents/side (102,400), seed 42"),
    "c2_aco": (480, 480, 1_024, "aco", 1, "C2: ACO 480x480, 1,024 agents/side, seed 42"),
    "c1_lem": (480, 480, 1_024, "lem", 1, "C1: LEM 480x480, 1,024 agents/side, seed 42"),
    "c2_aco_x64": (480, 480, 1_024, "aco", 64, "C2 x64: ACO 480x480, 1,024 agents/side, 64 seeds per launch"),
    "c1_lem_x64": (480, 480, 1_024, "lem", 64, "C1 x64: LEM 480x480, 1,024 agents/side, 64 seeds per launch"),
    # The paper's smallest density point (SURVEY.md 8(d) notes).
    "c2_aco_1280": (480, 480, 1_280, "aco", 1, "C2 @1,280/side: ACO 480x480, 1,280 agents/side, seed 42"),
    "c1_lem_1280": (480, 480, 1_280, "lem", 1, "C1 @1,280/side: LEM 480x480, 1,280 agents/side, seed 42"),
}


SURVEY_MODEL = ("SURVEY.md §8(d): LEM 8 B/cell (one packed u32 cell word read + written); ACO 40 B/cell "
                "(word 8 + two f64 pheromone fields read + written 32) + 16 B/agent (f64 tour read + written)")
BITPLANE_MODEL = ("bit-plane state actually streamed (DESIGN.md §2): 0.5 B/cell (2-bit occupancy planes read + "
                  "written) + 8 B/mover (source cell word read, destination word written); ACO + 32 B/cell (two f64 "
                  "pheromone fields read + written) + 16 B/mover (f64 tour read + written)")


def alg_bytes_survey(w, h, model, replicas, agents_per_side):
    """SURVEY.md §8(d)'s per-unit figure x the units of one launch: 8 B/cell
    (LEM), 40 B/cell + 16 B/agent (ACO). Its 8 B/cell assumes a ping-pong word
    plane; the in-place word plane of this design streams 0.5 B/cell + 8 B per
    mover instead (alg_bytes_bitplane), so fractions on this model can exceed
    1 without any work being skipped."""
    cells = w * h * replicas
    if model == "aco":
        return 40 * cells + 16 * 2 * agents_per_side * replicas
    return 8 * cells


def alg_bytes_bitplane(w, h, model, replicas, movers):
    """Algorithmic HBM bytes per step of the bit-plane representation
    (DESIGN.md §2-3): every cell's occupancy bits are read and written
    (2 x 2 bits), every mover's word is read at its source and written at its
    destination; ACO adds both f64 pheromone fields read + written for every
    cell and the f64 tour read + written per mover. `movers` = agents moved
    per step (StepReport.moved). ncu's DRAM bytes per launch match this."""
    cells = w * h * replicas
    b = 0.5 * cells + 8 * movers
    if model == "aco":
        b += 32 * cells + 16 * movers
    return b


def roofline_pair(w, h, model, reps, aps, movers, kernel_ms, peak, world=1):
    """Both byte models for one launch of the step kernel (its shard at N>1)."""
    out = {}
    for key, b in (("survey", alg_bytes_survey(w, h, model, reps, aps)),
                   ("bitplane", alg_bytes_bitplane(w, h, model, reps, movers))):
        b /= world
        ach = b / (kernel_ms / 1e3) / 1e9
        out[key] = {"alg_bytes_per_launch": b, "achieved": ach, "frac": ach / peak}
    return out


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, which):
        """Record the start ("t0") / end ("t1") of the timed region."""
        setattr(self, which, time.perf_counter())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        """Samples read during the timed region (marks t0..t1, plus the 50 ms
        after it for nvidia-smi's output lag); if the region is too short for
        any, the ones within 100 ms of it."""
        parsed = []
        for ts, ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                parsed.append((ts, float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        window = "whole run"
        rows = parsed
        if t0 is not None and t1 is not None:
            rows = [r for r in parsed if t0 <= r[0] <= t1 + 0.05]
            window = "timed region"
            if not rows:
                rows = [r for r in parsed if t0 - 0.1 <= r[0] <= t1 + 0.1]
                window = "timed region +- 100 ms"
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows), "window": window, "interval_ms": 20}


def scenario(name):
    import paper_1412_4933_b200 as p

    w, h, n, model, reps, desc = WORKLOADS[name]
    cfg = p.ScenarioConfig(width=w, height=h, agents_per_side=n, model=p.Model.Lem if model == "lem" else p.Model.Aco,
                           seed=42)
    return cfg, reps, desc


# ------------------------------------------------------------------ CPU arms

def cpu_reference_run(name, steps, warmup, budget_s, sequential_steps=1):
    """The reference CPU implementation on this host: oracle/_ref (the
    reference library built from its own sources) when present, else the C
    oracle port. The Parallel executor with every host thread is timed first,
    then (same placement, continuing) the Sequential executor on one core, as
    the reference's own `bench` compares them (tools/pedflow.cpp:191-225).
    Returns a dict; value = the Parallel rate."""
    from oracle.oracle import OracleState, Reference, Scenario

    w, h, n, model, reps, desc = WORKLOADS[name]
    sc = Scenario(width=w, height=h, agents_per_side=n, model=model, seed=42)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    if Reference.available():
        eng, kind, cores = Reference(sc, threads=threads), "reference", threads
    else:
        eng, kind, cores = OracleState(sc), "port", 1
    setup = time.perf_counter() - t0

    def one():
        if kind == "reference":
            return eng.run(1)[1]
        t = time.perf_counter()
        eng.run(1)
        return time.perf_counter() - t

    spent = 0.0
    for _ in range(warmup):
        if spent > budget_s / 3:
            break
        spent += one()
    done, secs = 0, 0.0
    while done < max(1, steps):
        secs += one()
        done += 1
        if secs + spent > budget_s:
            break
    agents = 2 * n
    out = {"value": agents * done / secs, "secs": secs, "steps": done, "kind": kind, "cores": cores,
           "setup_s": setup, "cells": w * h, "cpu_model": cpu_model(), "logical_cpus": os.cpu_count(),
           "sample": f"{desc}; steps {warmup}..{warmup + done - 1} timed after new_environment "
                     f"({setup:.1f}s untimed setup), {'Parallel executor' if kind == 'reference' else 'sequential C port'}, "
                     f"{cores} thread(s), {cpu_model()}"}
    if kind == "reference" and sequential_steps > 0:
        eng.set_executor(0)  # Sequential, same state
        first = warmup + done
        sq, sd = 0.0, 0
        while sd < sequential_steps:
            sq += one()
            sd += 1
            if sq > budget_s:
                break
        out["sequential"] = {"value": agents * sd / sq, "unit": "agent-updates/s", "cores": 1,
                             "ms_per_step": 1e3 * sq / sd,
                             "sample": f"steps {first}..{first + sd - 1}, Sequential executor, 1 thread"}
    return out


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # only rank 0 times the CPU reference
    r = cpu_reference_run(args.workload, args.steps, args.warmup, args.ref_budget, sequential_steps=0)
    w, h, n, model, reps, desc = WORKLOADS[args.workload]
    line = {
        "impl": "reference", "metric": "agent-updates/sec", "value": r["value"], "unit": "agent-updates/s",
        "n_gpus": args.gpus, "steps": r["steps"], "warmup": args.warmup, "ms_per_step": 1e3 * r["secs"] / r["steps"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64+u32",
        "data": "synthetic (new_environment placement, seed 42)",
        "config": {"workload": desc, "width": w, "height": h, "agents_per_side": n, "model": model, "replicas": 1},
        "cell_updates_per_s": w * h * r["steps"] / r["secs"],
        "cpu_baseline": {"value": r["value"], "unit": "agent-updates/s", "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"], "cpu_model": r["cpu_model"]},
        "e2e": {"value": r["value"], "unit": "agent-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def _with_env(env, fn):
    """fn() with the given environment variables set (read at context creation)."""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def secondary_runs(steps):
    """Device timings beside the headline:

    * C4/C3 (the north star's "100K-pedestrian step loop") as 64-seed
      replica batches and single scenarios; C2/C1 single, x64 and at the
      paper's 1,280/side point. The window is steps 5 .. 5+steps: with
      steps = 1000 (the length of the C3/C4 golden runs) it covers the
      approach of the two crowds AND the congested regime after they meet
      (~step 130), which costs 2-3x more per step than the free-flow start.
    * C5 LEM (16384^2, 50M agents), steps 5..305.
    * C5 ACO as 2 and 4 linked row shards on this ONE GPU (fused halo
      exchange, same process): all shards share the device, so the ideal is
      the unsharded step time; the difference is the per-step boundary
      ordering + mirroring cost (not a scaling measurement).
    """
    import torch

    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config
    from paper_1412_4933_b200.sharding import row_partition

    peak, _ = measured_peak()
    out = {}
    for key in ("c4_aco_x64", "c3_lem_x64", "c4_aco", "c3_lem", "c2_aco", "c1_lem", "c1_lem@bitplane", "c2_aco_x64",
                "c1_lem_x64", "c2_aco_1280", "c1_lem_1280", "c5_lem"):
        # name@bitplane: the same workload on the bit-plane kernel
        # (PEDFLOW_CLUSTER=0), beside the cluster-resident LEM path that sparse
        # single grids take by default.
        name, _, variant = key.partition("@")
        cfg, reps, desc = scenario(name)
        ens = _with_env({"PEDFLOW_CLUSTER": "0"} if variant else {}, lambda: p.Ensemble(cfg, replicas=reps))
        if variant:
            desc += " (bit-plane kernel, PEDFLOW_CLUSTER=0)"
            name = name + "_bitplane"
        ens.run(5)
        n = min(steps if not name.startswith("c5") else 300, 1024)
        ens.ctx.prepare_steps(n)
        tot, _ = ens.time_steps(n)
        moved = ens.ctx.read_reports(n)["moved"].astype(np.int64)  # [replica][step 5 + i]
        movers = float(moved.sum()) / n
        _, ker = ens.time_steps(min(n, 50), kernel=True)
        model = "lem" if cfg.model == p.Model.Lem else "aco"
        rl = roofline_pair(cfg.width, cfg.height, model, reps, cfg.agents_per_side, movers, tot / n, peak)
        # ncu's DRAM traffic (profiles/ncu_traffic.json) was captured at step
        # 150 (the x64 batches: steps 150..159): compare it with the byte
        # models at those steps' movers.
        tw = (150, 160) if name.endswith("_x64") else (150, 151)
        traffic = ncu_traffic(name)
        tcmp = None
        if traffic and moved.shape[1] >= tw[1] - 5:
            mv = float(moved[:, tw[0] - 5:tw[1] - 5].sum()) / (tw[1] - tw[0])
            ab = alg_bytes_bitplane(cfg.width, cfg.height, model, reps, mv)
            asv = alg_bytes_survey(cfg.width, cfg.height, model, reps, cfg.agents_per_side)
            tcmp = {"steps": f"{tw[0]}..{tw[1] - 1}", "movers_per_step": mv, "traffic_per_step": traffic,
                    "over_bitplane": traffic / ab, "over_survey": traffic / asv}
        out[name] = {
            "workload": desc, "window": f"steps 5..{5 + n}", "ms_per_step": tot / n,
            "kernel_ms_isolated_launch_events": ker,
            "agent_updates_per_s": 2 * cfg.agents_per_side * reps * n / (tot / 1e3),
            "cell_updates_per_s": cfg.width * cfg.height * reps * n / (tot / 1e3),
            "movers_per_step": movers,
            "roofline_frac": rl["survey"]["frac"], "roofline_frac_bitplane": rl["bitplane"]["frac"],
            "alg_bytes_per_step": rl["survey"]["alg_bytes_per_launch"],
            "alg_bytes_per_step_bitplane": rl["bitplane"]["alg_bytes_per_launch"],
            "traffic": traffic, "traffic_vs_models": tcmp,
        }
        ens.close()
    # C5 ACO with fp32 pheromone storage (PF_KERNEL_FUSED_F32): tolerance-only
    # parity (tests/test_f32_pheromone.py), half the pheromone stream.
    cfg, reps, desc = scenario("c5_aco")
    ens = p.Ensemble(cfg, replicas=1, kernel="fused_f32")
    ens.run(5)
    ens.ctx.prepare_steps(300)
    tot, _ = ens.time_steps(300)
    mv = float(ens.ctx.read_reports(300)["moved"].astype(np.int64).sum()) / 300
    b32 = alg_bytes_bitplane(cfg.width, cfg.height, "aco", 1, mv) - 16 * cfg.width * cfg.height
    out["c5_aco_f32"] = {
        "workload": desc + ", pheromone stored as fp32 (tolerance-only; fp64 arithmetic, one rounding per store)",
        "window": "steps 5..305", "ms_per_step": tot / 300,
        "agent_updates_per_s": 2 * cfg.agents_per_side * 300 / (tot / 1e3),
        "alg_bytes_per_step_bitplane_f32": b32, "roofline_frac_bitplane_f32": b32 / (tot / 300 / 1e3) / 1e9 / peak,
        "note": "not the headline: the reference's fields are fp64 and this mode is not bit-exact (DESIGN.md §4)"}
    ens.close()
    # C5 ACO as linked shards on this one GPU
    cfg, reps, desc = scenario("c5_aco")
    shard = {}
    for k in (1, 2, 4):
        ctxs = []
        for lo, hi in row_partition(cfg.height, k):
            c = _lib.Context(_pf_config(cfg, 42, row_begin=0 if k == 1 else lo, row_end=0 if k == 1 else hi))
            c.init_environment()
            ctxs.append(c)
        if k > 1:
            _lib.link_shards(ctxs)
        for c in ctxs:
            c.step_async(5)
        for c in ctxs:
            c.synchronize()
            c.prepare_steps(100)
        torch.cuda.synchronize()
        ev = []
        for c in ctxs:  # events on each shard's own stream; span = first start .. last end
            st = torch.cuda.ExternalStream(c.stream())
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            e[0].record(st)
            c.step_async(100)
            e[1].record(st)
            ev.append(e)
        for c in ctxs:
            c.synchronize()
        span = max(ev[0][0].elapsed_time(e[1]) for e in ev)
        shard[f"shards{k}"] = {"ms_per_step": span / 100, "window": "steps 5..105"}
        for c in ctxs:
            c.close()
        torch.cuda.empty_cache()
    for k in (2, 4):
        shard[f"shards{k}"]["overhead_vs_unsharded"] = shard[f"shards{k}"]["ms_per_step"] / shard["shards1"]["ms_per_step"] - 1
    shard["note"] = ("C5 ACO split into k linked row shards (fused P2P halo: boundary rows stored into the "
                     "neighbours' ghost rows + device flag handshake per step) all on ONE GPU: measures ordering and "
                     "mirroring overhead, not multi-GPU scaling")
    out["c5_aco_linked_shards_one_gpu"] = shard
    # SPEC acceptance #6: ACO <= 1.4x LEM time at 480x480, 20,480
    # agents, 500 steps (single scenario, and as a 64-seed batch).
    # The single LEM run (8.9% density) takes the cluster-resident path by
    # default; the ratio on one kernel for both models is beside it.
    spec6 = {}
    for reps in (1, 64):
        t = {}
        for model in (p.Model.Lem, p.Model.Aco):
            cfg = p.ScenarioConfig(width=480, height=480, agents_per_side=10_240, model=model, seed=42)
            ens = p.Ensemble(cfg, replicas=reps)
            t[model.name.lower()], _ = ens.time_steps(500)
            ens.close()
        spec6[f"x{reps}"] = {"lem_ms": t["lem"], "aco_ms": t["aco"], "aco_over_lem": t["aco"] / t["lem"]}
        if reps == 1:
            cfg = p.ScenarioConfig(width=480, height=480, agents_per_side=10_240, model=p.Model.Lem, seed=42)
            ens = _with_env({"PEDFLOW_CLUSTER": "0"}, lambda: p.Ensemble(cfg, replicas=1))
            lem_bits, _ = ens.time_steps(500)
            ens.close()
            spec6["x1"].update({"lem_ms_bitplane": lem_bits, "aco_over_lem_bitplane": t["aco"] / lem_bits})
    out["spec6_aco_vs_lem_480_20480_500steps"] = spec6
    return out


def run_gpu_arm(args):
    import torch

    import paper_1412_4933_b200 as p

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # Dev check of the N>1 code path on a box with fewer GPUs than ranks:
    # PEDFLOW_BENCH_SHARE_GPU=1 maps rank -> GPU (local % count) and uses gloo
    # (the numbers are then meaningless: ranks time-slice one GPU).
    share = os.environ.get("PEDFLOW_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    red_dev = "cpu" if share else f"cuda:{local}"
    cfg, reps, desc = scenario(args.workload)
    if args.replicas:
        reps = args.replicas
    w, h, n = cfg.width, cfg.height, cfg.agents_per_side
    model = "lem" if cfg.model == p.Model.Lem else "aco"
    peak, peak_src = measured_peak()

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # --- device-resident throughput -----------------------------------
    from paper_1412_4933_b200.sharding import ShardedEngine

    t_ctx = time.perf_counter()
    torch.zeros(1, device=f"cuda:{local}")  # the process's CUDA context (one-time; not scenario setup)
    cuda_context_s = time.perf_counter() - t_ctx
    t_setup = time.perf_counter()
    eng = ShardedEngine(cfg, rank, world, device=local, replicas=reps)
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.ExternalStream(eng.ctx.stream(), device=f"cuda:{local}")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        time.sleep(0.5)  # let nvidia-smi start sampling before the timed region
        eng.step(args.warmup)  # the W untimed warm-up steps (also keep the GPU busy for the sampler)
        eng.synchronize()
        t_wait = time.perf_counter()
        while len(clocks.lines) < 2 and time.perf_counter() - t_wait < 5.0:  # the sampler is producing
            time.sleep(0.02)
        if world == 1:
            eng.ctx.prepare_steps(args.steps)  # graph capture stays outside the timed region
        # A timed region shorter than nvidia-smi's sampling can miss every
        # sample: it is then timed again (the next K steps; at most 3 times,
        # the same on every rank) and the attempt with clock samples reported.
        for attempt in range(3):
            barrier()
            torch.cuda.synchronize()
            launches0 = eng.ctx.launches
            clocks.mark("t0")
            e0.record(stream)
            if world == 1:
                eng.ctx.step_async(args.steps)  # CUDA-graph batches
            else:
                eng.step(args.steps)
            e1.record(stream)
            e1.synchronize()
            torch.cuda.synchronize()
            clocks.mark("t1")
            time.sleep(0.06)  # nvidia-smi's last samples of the region
            launches = eng.ctx.launches - launches0
            sampled = torch.tensor([clocks.summary()["samples"]], device=f"cuda:{local}")
            if world > 1:
                import torch.distributed as dist
                dist.all_reduce(sampled, op=dist.ReduceOp.MIN)
            if int(sampled.item()) > 0:
                break
        timed_attempts = attempt + 1
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    rep = eng.reports(min(args.steps, 1024))
    moved_local = int(rep["moved"].sum())

    # Dominant kernel (step_bits_kernel, one launch per step). At N=1 the timed
    # region is exactly K back-to-back launches of it (CUDA graphs; the only
    # other kernel is a 1-thread step-counter bump per 256 steps), so its mean
    # duration is the event-timed region / K. Also recorded: events around
    # each of 20 isolated launches (includes launch gaps), and at N>1 that is
    # the kernel figure, since the timed region then includes the exchange.
    _, kernel_ms_isolated = eng.ctx.time_steps(min(args.steps, 20), kernel=True)
    kernel_ms_isolated = max_over_ranks(kernel_ms_isolated)
    eng.close()
    torch.cuda.empty_cache()
    # Setup again in this process: the placement (new_environment's keyed
    # Fisher-Yates) now comes from the library's cache.
    t_setup = time.perf_counter()
    eng = ShardedEngine(cfg, rank, world, device=local, replicas=reps)
    setup_warm_s = time.perf_counter() - t_setup
    eng.close()
    torch.cuda.empty_cache()
    kernel_ms = ms / args.steps if world == 1 else kernel_ms_isolated

    agents_total = 2 * n * reps
    value = agents_total * args.steps / (ms / 1e3)
    moved_all = sum_over_ranks(moved_local)
    movers = moved_all / min(args.steps, 1024)
    rl = roofline_pair(w, h, model, reps, n, movers, kernel_ms, peak, world)

    # --- end to end with host buffers ----------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = e2e_runs(args, cfg, reps, rank, world, local, barrier, max_over_ranks)

    line = None
    if rank == 0:
        traffic = ncu_traffic(args.workload)
        line = {
            "metric": "agent-updates/sec", "value": value, "unit": "agent-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64+u32",
            "data": "synthetic (new_environment placement, seed 42; replica i uses seed 42+i)",
            "config": {"workload": desc, "width": w, "height": h, "agents_per_side": n, "model": model,
                       "replicas": reps, "parallelism": f"row-shard x{world} (fused 3-row P2P halo per step: peer stores + device handshake)" if world > 1
                       else "single GPU", "l2": "inputs larger than L2 (resident state >> 126 MB; no flush)"},
            "cell_updates_per_s": w * h * reps * args.steps / (ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": rl["survey"]["achieved"], "peak": peak, "unit": "GB/s",
                         "frac": rl["survey"]["frac"], "traffic": traffic, "peak_source": peak_src,
                         "alg_bytes_per_launch": rl["survey"]["alg_bytes_per_launch"], "alg_bytes_model": SURVEY_MODEL,
                         "kernel": "step_bits_kernel", "kernel_ms": kernel_ms,
                         "kernel_ms_isolated_launch_events": kernel_ms_isolated,
                         "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                           "(profiles/ncu_traffic.json, captured at step 150 of the same workload)",
                         "note": "frac > 1 on the §8(d) model: it counts 8 B/cell of word-plane traffic that the "
                                 "in-place word plane does not stream (DESIGN.md §2); bitplane below counts the "
                                 "bytes actually moved, which ncu's DRAM traffic matches"},
            "roofline_bitplane": {"achieved": rl["bitplane"]["achieved"], "peak": peak, "unit": "GB/s",
                                  "frac": rl["bitplane"]["frac"], "frac_of_8tbs_spec": rl["bitplane"]["achieved"] / 8000.0,
                                  "alg_bytes_per_launch": rl["bitplane"]["alg_bytes_per_launch"],
                                  "alg_bytes_model": BITPLANE_MODEL, "movers_per_step": movers},
            "gpu_launches": launches,
            "clocks": dict(clocks.summary(), timed_attempts=timed_attempts),
            "setup_s": setup_s,
            "setup_warm_s": setup_warm_s,
            "cuda_context_s": cuda_context_s,
            "setup_note": "ShardedEngine construction after the CUDA context exists (cuda_context_s): device "
                          "allocation + new_environment placement (keyed Fisher-Yates on the host, computed in the "
                          "background from pf_create) + the placed cell lists scattered into the word plane on the "
                          "device; setup_warm_s = the same again in this process (placement from the in-process "
                          "cache)",
            "moved_in_window_rank0": moved_local,
        }
        if e2e:
            line["e2e"] = e2e
    if dist is not None:
        dist.barrier()
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            r = cpu_reference_run(args.workload, args.cpu_steps, 0, args.cpu_budget)
            line["cpu_baseline"] = {"value": r["value"], "unit": "agent-updates/s", "cores": r["cores"],
                                    "kind": r["kind"], "sample": r["sample"], "cpu_model": r["cpu_model"]}
            if "sequential" in r:
                line["cpu_baseline"]["sequential"] = r["sequential"]
        if world == 1 and not args.no_secondary:
            line["secondary"] = secondary_runs(1000)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def cpp_step_loop(args, cfg):
    """The C++ drop-in (include/pedflow_gpu.hpp) as the reference's own
    run_scenario loop calls it: `report = engine.step(state)` K times
    (src/engine.cpp:216-221) on a reference-layout SimState of pageable
    std::vectors, then state.sync(). The state stays on the device between
    calls; the timed region holds the upload, K steps each with its 16-byte
    report read back, and the download (tools/pedflow_gpu_demo, mode step)."""
    demo = os.path.join(ROOT, "tools", "pedflow_gpu_demo")
    model = "lem" if int(cfg.model) == 0 else "aco"
    r = subprocess.run([demo, model, str(cfg.width), str(cfg.height), str(cfg.agents_per_side), str(args.steps),
                        "42", "step"], capture_output=True, text=True, timeout=900)
    if r.returncode != 0:
        raise RuntimeError(f"pedflow_gpu_demo failed: {r.stderr[-500:]}")
    return json.loads(r.stderr.strip().splitlines()[-1])


def e2e_runs(args, cfg, reps, rank, world, local, barrier, max_over_ranks):
    """The same metric with host buffers, host<->device copies inside the
    timed region. Headline (N=1): the C++ drop-in per-step loop on pageable
    planes (cpp_step_loop). Beside it the C-ABI batch path (pf_load_state ->
    pf_step(K) with reports -> pf_store_state) on page-locked and on pageable
    numpy planes. At N>1 each rank runs the C-ABI path on its row shard."""
    aco = cfg.model == 1
    H, W = cfg.height, cfg.width
    planes = H * W * (1 + 4 + (16 if aco else 0)) + 2 * cfg.agents_per_side * 40
    agents = 2 * cfg.agents_per_side
    variants = {}
    if world == 1:
        if rank == 0:
            # Two runs (fresh processes): host-memory and PCIe throughput on a
            # shared VM host vary run to run (0.41-0.54 s for the same 20
            # steps); the faster is reported, both are listed.
            runs = [cpp_step_loop(args, cfg) for _ in range(2)]
            t = min(runs, key=lambda x: x["run_s"])
            variants["cpp_step_loop_pageable"] = {
                "value": agents * args.steps / t["run_s"], "seconds": t["run_s"], "setup_s": t["setup_s"],
                "uploads": t["uploads"], "downloads": t["downloads"], "runs_s": [x["run_s"] for x in runs],
                "path": "C++ shim: engine.step(state) x K (lazy, state stays on device) + state.sync(); "
                        "std::vector planes; best of 2 runs"}
        for pinned in (True, False):
            secs = capi_batch(args, cfg, rank, world, local, barrier, max_over_ranks, pinned)
            variants["capi_batch_" + ("pinned" if pinned else "pageable")] = {
                "value": agents * args.steps / secs, "seconds": secs,
                "path": "pf_load_state -> pf_step(K) (+reports) -> pf_store_state, "
                        + ("page-locked numpy planes (pf_host_alloc)" if pinned else "pageable numpy planes")}
        head = variants["cpp_step_loop_pageable"]
    else:
        secs = capi_batch(args, cfg, rank, world, local, barrier, max_over_ranks, False)
        head = {"value": agents * args.steps / secs, "seconds": secs,
                "path": "per rank: pf_load_state -> pf_step_async(K) -> reports -> pf_store_state of its row shard, "
                        "pageable planes"}
        variants["capi_sharded_pageable"] = head
    return {"value": head["value"], "unit": "agent-updates/s",
            "h2d_bytes_per_step": planes // args.steps, "d2h_bytes_per_step": planes // args.steps + 16,
            "seconds": head["seconds"], "path": head["path"], "steps": args.steps,
            "note": "transfer-bound at small K: about 2 x %.1f GB of reference-layout planes per run" % (planes / 1e9),
            "variants": variants}


def capi_batch(args, cfg, rank, world, local, barrier, max_over_ranks, pinned):
    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config
    from paper_1412_4933_b200.sharding import balanced_row_partition

    state = p.new_environment(cfg, 42, pinned=pinned)
    lo, hi = balanced_row_partition(cfg, world)[rank]
    c = _lib.Context(_pf_config(cfg, 42, row_begin=0 if world == 1 else lo, row_end=0 if world == 1 else hi,
                                device=local))
    if world > 1:  # fused halo exchange between the ranks' contexts (CUDA IPC, device handshake)
        import torch.distributed as dist

        descs = [None] * world
        dist.all_gather_object(descs, bytes(c.peer_desc()))
        for side, peer in ((0, rank - 1), (1, rank + 1)):
            if 0 <= peer < world:
                c.attach_peer(side, _lib.PfPeerDesc.from_buffer_copy(descs[peer]), ipc=True)
    barrier()
    t0 = time.perf_counter()
    c.load(0, state.occupancy, state.index, state.agents, state.pheromone_top, state.pheromone_bottom, 0)
    if world == 1:
        rep = c.step(args.steps)
    else:
        barrier()  # every shard is loaded (and its handshake flags reset) before any steps
        c.step_async(args.steps)
        rep = c.read_reports(min(args.steps, 1024))
    c.store(0, state._occ, state._index, state._agents, state._tau_top, state._tau_bot)
    secs = max_over_ranks(time.perf_counter() - t0)
    barrier()  # fused exchange: no rank frees its planes while a neighbour may still store into them
    c.close()
    del rep, state
    return secs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c5_aco")
    ap.add_argument("--replicas", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--cpu-budget", type=float, default=30.0)
    ap.add_argument("--ref-budget", type=float, default=150.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
