#!/usr/bin/env python
"""bench.py — RVEA generations/sec on the BASELINE.json headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--pop N --dim d ...]

A step is ONE generation of the RVEA loop (algorithms.hpp:246-292: mating, SBX + polynomial
mutation, evaluation, APD selection, reference-vector adaptation on its schedule) on the
device-resident population. Workload at N=1: DTLZ2, m = 3, pop = 2^17, d = 5000 (the shape the
metric is quoted on; R = 130816 reference vectors by the reference's own lattice rule).

Printed JSON (one line, rank 0):
  value      generations/s over exactly K steps, device-resident state (per step the host only ships the
             4*n-byte mating permutation and reads 8 bytes back), barrier + synchronize on both sides
  e2e        same loop through the public C-ABI session call with HOST buffers: every step uploads the
             permutation from pinned memory and downloads the survivors' objectives (what the reference
             hands to fill_metrics each generation, algorithms.hpp:287)
  roofline   dominant HBM kernel (fused reproduction + evaluation): algorithmic bytes 16*n*d per launch
             / its mean CUDA-event duration inside the timed region, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the UNMODIFIED reference (oracle/_ref) on this box's host cores, on a bounded sample
             (pop' rows of the same problem), scaled to the full workload — see cpu_reference_sample()
  --impl reference   times only that CPU arm and prints it as the headline line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RVEA generations/sec (DTLZ2 m=3, N=2^17, d=5000)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--problem", default="dtlz2")
    ap.add_argument("--pop", type=int, default=1 << 17)
    ap.add_argument("--dim", type=int, default=5000)
    ap.add_argument("--obj", type=int, default=3)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--cpu-sample-pop", type=int, default=2048)
    ap.add_argument("--cpu-sample-gens", type=int, default=0, help="0: use --steps/--warmup")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--stage-reps", type=int, default=5)
    ap.add_argument("--no-same-config", action="store_true", help="skip the measured CPU/GPU pair at --same-config-pop rows")
    ap.add_argument("--same-config-pop", type=int, default=1 << 14)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = N shards of --pop rows (one run of N*pop rows); strong = --pop rows in total")
    return ap.parse_args()


def ncu_traffic(n, d, fused):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of the dominant kernel from the newest committed
    `ncu --set full` summary (profiles/*_ncu_top_kernels.csv); only valid for the shape it was captured at."""
    import csv
    import glob
    if not (n == 1 << 17 and d == 5000 and fused):
        return None, None
    unit_scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_top_kernels.csv")), reverse=True):
        try:
            with open(path, newline="") as fh:
                rows = list(csv.reader(fh))
            head, units = rows[0], rows[1]
            ir, iw = head.index("dram__bytes_read.sum"), head.index("dram__bytes_write.sum")
            for row in rows[2:]:
                if "reproduce_pairs_kernel" in row[0]:
                    total = float(row[ir]) * unit_scale[units[ir]] + float(row[iw]) * unit_scale[units[iw]]
                    return total, os.path.relpath(path, ROOT)
        except (OSError, ValueError, KeyError, IndexError):
            continue
    return None, None


def self_launch(args):
    """`python bench.py --gpus N` without a launcher: re-exec under torchrun with N ranks on this node."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible (no CPU fallback, no oversubscription)")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


# ------------------------------------------------------------------------------ helpers
def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons DURING the timed region (B200_PROFILING.md recipe)."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.rows, self.proc, self.gpu = [], None, gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, power, reasons = [], [], [], set()
        for r in self.rows:
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1])); smax.append(float(r[2])); power.append(float(r[3]))
            except ValueError:
                continue
            for name, col in (("hw_slowdown", 5), ("hw_thermal_slowdown", 6), ("sw_thermal_slowdown", 7), ("sw_power_cap", 8)):
                if r[col].lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "power_w_max": float(max(power)),
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- CPU reference arm
def _checker():
    from oracle.pyoracle import Oracle, Ref
    kind = "reference" if Ref.available() else "port"
    chk = Ref() if kind == "reference" else Oracle()
    return chk, kind, (chk.num_threads() if kind == "reference" else 1)


def cpu_reference_sample(args, steps, warmup):
    """Times the unmodified reference on a bounded sample of the workload: a slice of pop' rows.

    The reference cannot run the full shape (its min_vector_angles forms an R x R matrix: 137 GB at R = 130816,
    refvec.hpp:83), so every step is a ROW SLICE of it, and the only scaling applied is linear in rows (x pop/pop'):
      (a) one generation of the reference's own rvea_run (all host threads, track_archive = false, GA) on the SAME
          problem and decision dimension with pop' = --cpu-sample-pop rows; per-generation wall time from
          RunRecord.elapsed_ms differences (cmd_scale protocol, temo.cpp:229-237), minus its own (small-R') selection;
      (b) the reference's rv_select of 2 pop' merged rows against the FULL reference set (R vectors of the full
          workload's lattice; gamma = 1, timing-neutral), i.e. exactly the slice's share of the full association.
    Every stage of the loop body is linear in rows at fixed d and R, so full-shape ms = (a + b) * pop/pop'.
    Adaptation generations are excluded (fr = 1: the only one falls on the extra last generation)."""
    chk, kind, cores = _checker()
    m, d, n_full = args.obj, args.dim, args.pop
    n_s = min(args.cpu_sample_pop, n_full)
    h_full = chk.lattice_density_for(m, n_full)
    r_full = chk.lattice_count(m, h_full)
    h_s = chk.lattice_density_for(m, n_s)
    r_s = chk.lattice_count(m, h_s)
    gens = warmup + steps + 1  # the extra last generation carries the (excluded) adaptation: fr = 1.0
    t0 = time.time()
    if kind == "reference":
        rec = chk.rvea_run(args.problem, n_s, d, m, gens, seed=args.seed, fr=1.0, want_x=False)
        per_gen = np.diff(np.concatenate([[0.0], rec["elapsed_ms"]]))[warmup:warmup + steps]
    else:
        t1 = time.time()
        chk.rvea_run(args.problem, n_s, d, m, gens, seed=args.seed, fr=1.0)
        per_gen = np.full(steps, (time.time() - t1) * 1e3 / gens)
    fs = np.random.default_rng(1).random((2 * n_s, m)) + 0.1

    def select_ms(h, r, reps):
        v0 = chk.normalize_to_unit(chk.simplex_lattice(m, h))
        out = []
        for _ in range(reps):
            t1 = time.time()
            if kind == "reference":
                chk.rv_select(fs, v0, np.ones(r), 1, 100, 2.0, want_core=False)  # as rvea_run calls it (algorithms.hpp:276-277)
            else:
                chk.rv_select(fs, v0, np.ones(r), 1, 100, 2.0)
            out.append((time.time() - t1) * 1e3)
        return float(np.median(out))

    sel_small = select_ms(h_s, r_s, 3)            # what the sample run itself spent in selection
    sel_full_r = select_ms(h_full, r_full, max(2, min(steps, 5))) if n_s < n_full else sel_small
    gen = float(np.median(per_gen))
    scale_rows = n_full / n_s
    sample_ms = max(gen - sel_small, 0.0) + sel_full_r
    full_ms = sample_ms * scale_rows
    return {
        "value": 1000.0 / full_ms, "unit": "generations/s", "cores": int(cores), "kind": kind,
        "extrapolated": bool(n_s < n_full), "scale_rows": scale_rows,
        "sample": (f"row slice of the workload: {args.problem} m={m} d={d}, pop'={n_s} of {n_full} rows; reference rvea_run x "
                   f"{len(per_gen)} generations after {warmup} warm-up: median {gen:.1f} ms/gen (of which its own R'={r_s} "
                   f"selection {sel_small:.1f} ms, replaced by) rv_select of 2*pop' rows against the full R={r_full} set: "
                   f"{sel_full_r:.1f} ms -> {sample_ms:.1f} ms per slice step, x{scale_rows:.0f} rows -> {full_ms / 1e3:.1f} s/gen"),
        "sample_ms_per_step": sample_ms, "sample_gen_ms": gen, "sample_select_small_ms": sel_small,
        "sample_select_full_r_ms": sel_full_r, "scaled_ms_per_gen": full_ms,
        "wall_s": time.time() - t0,
    }


def cpu_same_config(args, pop, gens_timed=3):
    """MEASURED (not scaled) CPU time of the unmodified reference rvea_run at a shape it can run: pop rows of the
    same problem / dimension (R x R gamma matrix 2.2 GB at pop = 2^14). cmd_scale protocol (temo.cpp:229-282): median of
    per-generation elapsed_ms differences, generation 0 (init) and the adaptation generation (last, fr = 1) excluded."""
    chk, kind, cores = _checker()
    if kind != "reference":
        return None
    gens = 1 + gens_timed + 1
    t0 = time.time()
    rec = chk.rvea_run(args.problem, pop, args.dim, args.obj, gens, seed=args.seed, fr=1.0, want_x=False)
    per_gen = np.diff(np.concatenate([[0.0], rec["elapsed_ms"]]))[1:1 + gens_timed]
    return {"pop": pop, "ref_vectors": int(chk.lattice_count(args.obj, chk.lattice_density_for(args.obj, pop))),
            "cpu_ms_per_gen": float(np.median(per_gen)), "cpu_gens_timed": int(len(per_gen)), "cores": int(cores),
            "kind": "reference rvea_run, unmodified, measured", "wall_s": time.time() - t0}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if world > 1 or args.gpus > 1:  # the N-GPU arm runs one population of N * pop rows (weak scaling)
        args.pop = args.pop * max(world, args.gpus)
    base = cpu_reference_sample(args, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": base["value"], "unit": "generations/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # what was timed: one slice step; the full-shape figure is `scaled_ms_per_step` (rows only, see cpu_baseline.sample)
        "ms_per_step": base["sample_ms_per_step"], "scaled_ms_per_step": base["scaled_ms_per_gen"],
        "extrapolated": base["extrapolated"], "scale_rows": base["scale_rows"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, None),
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample", "extrapolated")},
        "e2e": {"value": base["value"], "unit": "generations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    if not args.no_same_config:
        try:
            line["same_config_measured"] = cpu_same_config(args, args.same_config_pop)
        except Exception as e:
            line["same_config_measured"] = {"error": repr(e)}
    print(json.dumps(line), flush=True)


def workload_config(args, run):
    cfg = {"workload": f"RVEA/{args.problem} m={args.obj} d={args.dim} pop={args.pop}", "problem": args.problem,
           "pop": args.pop, "dim": args.dim, "obj": args.obj, "seed": args.seed, "operator": "ga (SBX eta=20 pc=1, PM xi=20 pm=1)",
           "rng": "splitmix64 counter stream (reference-exact)", "alpha": 2.0, "fr": 0.1,
           "l2": "inputs larger than L2 (population pool >> 126 MB); stage timings flush L2 between launches"}
    if run is not None:
        cfg["ref_vectors"] = run.r
    return cfg


# ------------------------------------------------------------------------- our arm
def run_ours(args):
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)  # does not return
    force_dist = os.environ.get("TEMO_FORCE_DIST", "") in ("1", "nccl")  # the N-GPU path on one GPU (nccl: collectives through NCCL)
    if args.gpus != world and not (world == 1 and force_dist):
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    import paper_2404_01159_b200 as tb

    if world > 1 or force_dist:
        from paper_2404_01159_b200 import dist as tdist
        return tdist.bench_main(args, METRIC, workload_config, measured_peaks, ClockSampler)

    assert tb.device_count() >= 1, "bench.py needs a CUDA device (no CPU fallback)"
    tb.init(local)
    K, W = args.steps, args.warmup
    gens_total = max(100, W + 2 * K + 2)
    cfg = tb.RunConfig(problem=args.problem, pop=args.pop, dim=args.dim, obj=args.obj, generations=gens_total,
                       seed=args.seed, fuse_eval=False if args.no_fuse else None)
    t_init = time.time()
    run = tb.RveaRun(cfg)
    init_s = time.time() - t_init
    n, d, m, r = args.pop, run.d, run.m, run.r

    for _ in range(W):
        run.step()

    sampler = ClockSampler(local)
    sampler.start()
    # ---- value: K steps, device-resident
    stage = {k: [] for k in ("generation", "reproduce", "evaluate", "select", "adapt", "host_perm", "prep")}
    launches = 0
    pops = []
    tb._lib.check(tb._lib.load().temo_b200_dev_sync())
    run.timing_history(reset=True)  # drop the warm-up steps from the library's stage-time log
    t0 = time.perf_counter()
    for _ in range(K):
        pops.append(run.step())
    tb._lib.check(tb._lib.load().temo_b200_dev_sync())
    wall = time.perf_counter() - t0
    # per-step stage times of exactly these K steps (CUDA events on the library's stream, read by the library while the
    # following step ran: nothing is asked between two steps of the timed loop)
    hist = run.timing_history(reset=True)
    assert len(hist) == min(K, 1024), (len(hist), K)
    for tm in hist:
        for k in stage:
            stage[k].append(tm[k])
        launches += tm["launches"]
    # ---- e2e: K steps through the host-buffer session call (H2D permutation, D2H survivors' objectives)
    d2h = []
    t1 = time.perf_counter()
    for _ in range(K):
        p, f_host = run.step(want_f=True)
        d2h.append(8 + min(r, p + n) * m * 8)  # status words + the block the library copies (one row per reference vector at most)
    tb._lib.check(tb._lib.load().temo_b200_dev_sync())
    wall_e2e = time.perf_counter() - t1
    clocks = sampler.stop()

    # ---- per-kernel timings for the roofline (isolated launches, L2 flushed between them)
    peak, peak_src = measured_peaks()
    fused_ok = args.problem.startswith("dtlz") and not args.no_fuse and d > 1024  # the library's rule (run.h, fuse_offspring_eval)
    k_ms = {
        "reproduce": run.time_stage(1, args.stage_reps),
        "evaluate": run.time_stage(2, args.stage_reps),
        "select": run.time_stage(4, args.stage_reps),
        "gamma": run.time_stage(5, max(1, args.stage_reps // 2)),
    }
    if fused_ok:
        k_ms["reproduce_fused_eval"] = run.time_stage(3, args.stage_reps)
    nd = float(n) * d
    gbs = lambda nbytes, ms: nbytes / (ms * 1e-3) / 1e9
    dom_ms = float(np.mean(stage["reproduce"]))  # live, inside the timed region
    traffic, traffic_src = ncu_traffic(n, d, fused_ok)
    roofline = {
        "bound": "hbm", "kernel": "reproduce_pairs_kernel (SBX+PM" + ("+fused DTLZ evaluation)" if fused_ok else ")"),
        "achieved": gbs(16.0 * nd, dom_ms), "peak": peak, "unit": "GB/s", "frac": gbs(16.0 * nd, dom_ms) / peak,
        # dram__bytes_read.sum + dram__bytes_write.sum of one launch, read from the newest committed `ncu --set full`
        # summary of this kernel at the headline shape; null for any other shape
        "traffic": traffic, "traffic_source": traffic_src,
        "peak_source": peak_src, "algorithmic_bytes": 16.0 * nd, "ms": dom_ms,
        "share_of_step": dom_ms / float(np.mean(stage["generation"])),
    }
    kernels = {
        "reproduce_isolated": {"ms": k_ms["reproduce"], "GB/s": gbs(16.0 * nd, k_ms["reproduce"]), "frac": gbs(16.0 * nd, k_ms["reproduce"]) / peak},
        "evaluate_isolated": {"ms": k_ms["evaluate"], "GB/s": gbs(8.0 * nd, k_ms["evaluate"]), "frac": gbs(8.0 * nd, k_ms["evaluate"]) / peak},
        "select_isolated": {"ms": k_ms["select"], "pairs": float(pops[-1] + n) * r, "Gpairs/s": float(pops[-1] + n) * r / (k_ms["select"] * 1e-3) / 1e9},
        "gamma_isolated": {"ms": k_ms["gamma"], "pairs": float(r) * r},
    }
    if fused_ok:
        kernels["reproduce_fused_eval_isolated"] = {"ms": k_ms["reproduce_fused_eval"], "GB/s": gbs(16.0 * nd, k_ms["reproduce_fused_eval"]),
                                                    "frac": gbs(16.0 * nd, k_ms["reproduce_fused_eval"]) / peak}
    stages_mean = {k: float(np.mean(v)) for k, v in stage.items()}
    stages_mean["generation_median"] = float(np.median(stage["generation"]))

    line = {
        "metric": METRIC, "value": K / wall, "unit": "generations/s", "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": wall / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {**workload_config(args, run), "generations_schedule": gens_total, "init_s": init_s,
                   "survivors_last": int(pops[-1]), "fused_eval": bool(fused_ok)},
        "e2e": {"value": K / wall_e2e, "unit": "generations/s", "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": int(np.mean(d2h))},
        "gpu_launches": int(launches),
        "roofline": roofline, "stages_ms": stages_mean, "kernels": kernels, "clocks": clocks,
    }
    run.close()
    if not args.no_cpu_baseline:
        try:
            base = cpu_reference_sample(args, min(K, 8), 1)
            line["cpu_baseline"] = {k: base[k] for k in ("value", "unit", "cores", "kind", "sample", "extrapolated", "scale_rows",
                                                          "sample_ms_per_step", "scaled_ms_per_gen")}
            line["speedup_vs_cpu_baseline"] = line["e2e"]["value"] / base["value"]
            line["speedup_vs_cpu_baseline_extrapolated"] = base["extrapolated"]
        except Exception as e:  # the baseline is a reported extra; never lose the GPU line over it
            line["cpu_baseline"] = {"value": None, "unit": "generations/s", "cores": 0, "kind": "unavailable", "sample": repr(e)}
        if not args.no_same_config and args.same_config_pop < args.pop:
            # one pair where BOTH sides are measured at the same configuration: the unmodified reference can run this shape
            try:
                pair = cpu_same_config(args, args.same_config_pop)
                if pair is not None:
                    gens2 = 100
                    cfg2 = tb.RunConfig(problem=args.problem, pop=args.same_config_pop, dim=args.dim, obj=args.obj,
                                        generations=gens2, seed=args.seed, fuse_eval=False if args.no_fuse else None)
                    with tb.RveaRun(cfg2) as run2:
                        for _ in range(3):
                            run2.step()
                        tb._lib.check(tb._lib.load().temo_b200_dev_sync())
                        t2 = time.perf_counter()
                        for _ in range(20):
                            run2.step(want_f=True)  # host-buffer session call, like e2e
                        tb._lib.check(tb._lib.load().temo_b200_dev_sync())
                        pair["gpu_ms_per_gen"] = (time.perf_counter() - t2) / 20 * 1e3
                    pair["speedup_measured"] = pair["cpu_ms_per_gen"] / pair["gpu_ms_per_gen"]
                    pair["config"] = f"RVEA/{args.problem} m={args.obj} d={args.dim} pop={args.same_config_pop}"
                    line["same_config_measured"] = pair
            except Exception as e:
                line["same_config_measured"] = {"error": repr(e)}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
