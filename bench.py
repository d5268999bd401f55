"""Benchmark: MLMC random-walk estimator for e^{tA}v on BASELINE config 2 (C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--rows-per-step R] [--config c2]

Workload (BASELINE.json configs[1]): 2-D 5-point Laplacian on a 1024x1024 grid
(n = 1,048,576, 5.2M nnz, fp64), t = 0.5, v uniform [0,1) from the reference's Philox stream,
every component estimated to eps = 1e-3 by the reference's MLMC driver (Algorithm 1, one
decision sequence per component, row seed 1000 + row).  A STEP is the whole C2 job: every one of
the 2^20 components solved to eps; with N ranks the components are dealt round-robin over a
fixed permutation (strong scaling, no data-path collective -- components are independent MLMC
problems; only timings are reduced).  `--rows-per-step R` instead gives every rank R
components per step (weak scaling).

Timed region (`value`): tables already resident in HBM; K steps bracketed by barrier +
torch.cuda.synchronize(), CUDA events recorded on the library's own stream; max over ranks.
L2 is flushed (256 MB write) before every step inside the timed region.
`e2e`: the same work through the public API from HOST buffers -- context creation from the
host CSR + u (H2D), the solve, results back to host -- per step, CUDA events on the current
stream around the call.

`--impl reference`: the UNMODIFIED reference (oracle/_ref/libexpmc_ref.so, compiled from
/root/reference by oracle/Makefile) runs its own mlmc_driver per component on all host
cores (OpenMP), rank 0 only, each step a bounded sample of rows of the same batches.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

# torchrun exports OMP_NUM_THREADS=1 to every rank; the library's host driver (request staging,
# per-row state machines, combines of results) is OpenMP-parallel, so each rank gets its share of
# the host cores instead.  Set before numpy / torch / the library load libgomp.
if os.environ.get("OMP_NUM_THREADS") == "1" and "LOCAL_WORLD_SIZE" in os.environ:
    os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // max(1, int(os.environ["LOCAL_WORLD_SIZE"]))))

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "random-walk transitions/sec and exp(tA)v rows/sec at target ε; % gather roofline"
UNIT = "transitions/s"
ALG_BYTES_PER_JUMP = 64    # destination row record (32 B sector) + edge record sector
ALG_BYTES_PER_SAMPLE = 32  # terminal u[state] sector


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--rows-per-step", type=int, default=0, help="components per rank per step (0: default)")
    p.add_argument("--ref-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    p.add_argument("--max-cost", type=float, default=None,
                   help="per-component model-unit budget (driver extension; default off for C1/C2, 1e10 for C3-C5)")
    p.add_argument("--sampler", default=None, choices=["reference", "event"], help="override the config's sampler")
    p.add_argument("--full-hold", action="store_true",
                   help="event sampler: evaluate first holding intervals in full (A/B of the closed-form hold)")
    p.add_argument("--log-hold", action="store_true",
                   help="reference-order sampler: time-space holding tests with a log per event (A/B of S-mode)")
    p.add_argument("--multi", default="rows", choices=["rows", "samples"],
                   help="N>1: shard components over ranks (no collective) or shard every component's "
                        "samples with an exact NCCL all-reduce of the chunk partials")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


_PERM = {}


def perm_rows(n):
    if n not in _PERM:
        _PERM[n] = np.random.default_rng(20190429).permutation(n).astype(np.int64)
    return _PERM[n]


def batch_rows(n, step, rank, world, r):
    """Rows rank `rank` solves in `step`.  r == 0: the whole job -- every component, dealt
    round-robin over a fixed permutation to the ranks (strong scaling).  r > 0: r components
    per rank per step, consecutive slices of the permutation (weak scaling)."""
    perm = perm_rows(n)
    if r == 0:
        from paper_1904_12754_b200.shard import row_shard

        return row_shard(n, rank, world)  # == np.sort(perm[rank::world])
    k = (step * world + rank) * r
    idx = (np.arange(k, k + r) % n)
    return np.sort(perm[idx])


def sample_rows(n, step, r):
    """Unsorted rows for the bounded CPU sample (a random subset of the step's batch)."""
    perm = perm_rows(n)
    if r == 0:
        return np.roll(perm, -step * 1024)
    return perm[(np.arange(step * r, step * r + r) % n)]


def cpu_rows(cfg, step, r):
    """Components for the CPU reference sample.  Graph/3-D configs: light rows only (degree <= 32)
    -- the reference has no cost budget and one hub row can run for hours."""
    universe = cfg.rows if cfg.rows is not None else np.arange(cfg.a.n, dtype=np.int64)
    rows = universe[sample_rows(len(universe), step, r)]
    if cfg.name.startswith(("c3", "c4", "c5")):
        deg = np.diff(cfg.a.row_ptr)
        rows = rows[deg[rows] <= 32]
    return rows


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for nm, v in zip(names, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def load_capture(cfg_name):
    """The committed ncu --set full capture of this config's k_sample (profiles/r01/
    k_sample_<config>_r1h_key_metrics.json, scripts/prof_c4.sh): DRAM bytes per kernel-ms
    (dram__bytes_read.sum + dram__bytes_write.sum over the launch) and issue-slot utilisation.
    None for configs without a capture."""
    name = cfg_name.split("-")[0]
    path = os.path.join(ROOT, "profiles", "r01", f"k_sample_{name}_r1h_key_metrics.json")
    try:
        with open(path) as f:
            k = json.load(f)
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        dram = sum(float(k[m]["value"]) * scale[k[m]["unit"]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return {"bytes_per_ms": dram / float(k["gpu__time_duration.sum"]["value"]),
                "issue_active_pct": float(k["smsp__issue_active.avg.pct_of_peak_sustained_active"]["value"]),
                "source": os.path.relpath(path, ROOT)}
    except (OSError, KeyError, ValueError):
        return None


def sampler_only_rate(ref_chain, cfg, threads, seconds=4.0):
    """The reference's sampler without the driver: one large run_level per level
    (its LevelSampler table is built once per call, so the O(n) construction is amortised),
    OpenMP on all cores.  transitions = cost - 2 M 2^l (every fine step of a non-absorbing row
    ends with one draw).  Level 0 (base) and level 2 (coupled), each sized to ~seconds/2."""
    out = {}
    row = cfg.a.n // 2 + 7
    for level, base in ((0, True), (2, False)):
        m = 1 << 16
        while True:  # grow the sample until one call takes ~seconds / 2
            t0 = time.perf_counter()
            r = ref_chain.run_level(cfg.u, row, cfg.beta, level, base, 1 << 40, m, 99, threads=threads)
            dt = time.perf_counter() - t0
            if dt >= seconds / 4 or m >= (1 << 34):
                break
            m = int(m * min(16.0, max(2.0, (seconds / 2) / max(dt, 1e-3))))
        jumps = r["cost"] - 2 * m * (1 << level)
        out[f"level{level}"] = {"transitions_per_s": jumps / dt, "samples_per_s": m / dt, "samples": m,
                                "seconds": dt}
    return out


# ------------------------------------------------------------------------------ reference arm
def reference_rows(ref_chain, cfg, rows, seconds, threads, max_rows):
    """Reference mlmc_driver on rows one at a time, in a worker thread, for at most `seconds`.

    A single reference run cannot be interrupted and some components never finish in practice
    (the bias test can escalate to 2^(l0+30) steps per path), so the worker is
    abandoned at the deadline (it dies with the process) and only completed components count:
    throughput = their transitions / the time the last of them finished."""
    deg = np.diff(cfg.a.row_ptr)
    done_rows = []
    t0 = time.perf_counter()

    def work():
        for r in rows[:max_rows]:
            (res,) = ref_chain.driver_rows(cfg.u, cfg.beta, [int(r)], [1000 + int(r)], epsilon=cfg.epsilon,
                                           threads=threads, max_levels_above_l0=cfg.max_levels_above_l0)
            # transitions = cost - 2 M 2^l per level; an isolated row (rate 0,
            # absorbing) draws nothing and never jumps
            jumps = 0 if deg[int(r)] == 0 else res["total_jumps"]
            done_rows.append((time.perf_counter(), jumps, res["total_samples"]))
            if time.perf_counter() - t0 >= seconds:
                return

    th = threading.Thread(target=work, daemon=True)
    th.start()
    th.join(timeout=seconds + 1.0)
    got = list(done_rows)
    if not got:
        return 0, 0, 0, time.perf_counter() - t0
    return sum(g[1] for g in got), sum(g[2] for g in got), len(got), got[-1][0] - t0


def run_reference(args, cfg, rank, world, r):
    if rank != 0:
        return 0
    from oracle import CSR, Reference, have_reference

    if not have_reference():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libexpmc_ref.so not built"}))
        return 0
    threads = os.cpu_count() or 1
    ref = Reference().chain(CSR(cfg.a.n, cfg.a.row_ptr, cfg.a.col, cfg.a.val))
    # warm-up: one small component (pages the matrix in, spins up the OpenMP pool); then the
    # whole timed sample as ONE bounded worker run (an abandoned worker must not overlap a
    # later timing window), reported per step as its K-th part
    reference_rows(ref, cfg, cpu_rows(cfg, 0, r), 2.0, threads, 1)
    tj, ts, tr, tt = reference_rows(ref, cfg, cpu_rows(cfg, args.warmup, r), args.ref_seconds, threads, 1 << 30)
    value = tj / tt if tr else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tt / args.steps, "higher_is_better": True,
        "scaling": "strong" if r == 0 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": cfg.description, "sample": f"{tr} components (as-shipped mlmc_driver per row)",
                   "parallelism": f"OpenMP {threads} threads, rank 0 only"},
        "rows_per_s": tr / tt if tr else None, "samples_per_s": ts / tt if tr else None,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{tr} {cfg.name.upper()} components, as-shipped reference mlmc_driver, {tt:.1f} s"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------------------ our arm
def main():
    args = parse()
    rank, world, local = dist_env()
    from paper_1904_12754_b200 import configs

    cfg = configs.make_config(args.config)
    graph_like = cfg.name.startswith(("c3", "c4", "c5"))
    # C1/C2: the whole job per step.  C3-C5 (10^6-10^7 components, hub rows infeasible at the
    # stated eps): a seeded sample of components per step and a per-component budget.
    r = args.rows_per_step if args.rows_per_step or not graph_like else (4096 if cfg.name.startswith("c5") else 65536)
    # per-component budgets of DESIGN §7b: 1e10 model units for C3/C4, 1e9 for C5 (eps = 1e-4)
    default_budget = (1e9 if cfg.name.startswith("c5") else 1e10) if graph_like else 0.0
    max_cost = args.max_cost if args.max_cost is not None else default_budget
    sampler = args.sampler or cfg.sampler
    universe = cfg.rows if cfg.rows is not None else np.arange(cfg.a.n, dtype=np.int64)
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world, r)

    import torch

    import paper_1904_12754_b200 as P

    # EXPMC_BENCH_SHARE_DEVICE=1 (functional check of the N > 1 path on a one-GPU box, never a
    # measurement): every rank on cuda:0, host plumbing over gloo.  Row sharding has no
    # device-side exchange, so the ranks' kernels never wait on one another.
    shared = os.environ.get("EXPMC_BENCH_SHARE_DEVICE") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if shared else "cuda"

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t)
        return float(t.item())

    opts = P.MlmcOptions(epsilon=cfg.epsilon, max_levels_above_l0=cfg.max_levels_above_l0, max_cost=max_cost)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ctx = P.Context(cfg.a, cfg.u, device=local, sampler=sampler)
    if args.full_hold:
        ctx.set_full_hold(True)
    if args.log_hold:
        ctx.set_log_hold(True)
    sample_shard = args.multi == "samples" and world > 1
    if sample_shard:  # every rank runs the same components; chunk g is sampled on rank g % world
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.shard_samples(obj[0], rank, world)
    rank_b, world_b = (0, 1) if sample_shard else (rank, world)
    ext = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", local))

    # the batches of every step are built before any timing starts
    batches = [universe[batch_rows(len(universe), s, rank_b, world_b, r)] for s in range(args.warmup + args.steps)]
    seeds = [configs.row_seeds(b) for b in batches]

    def solve(step):
        res, _ = P.mlmc_driver_rows(ctx, cfg.beta, batches[step], seeds[step], opts, want_levels=False)
        return res

    for w in range(args.warmup):
        with torch.cuda.stream(ext):
            flush.fill_(w & 0xFF)
        solve(w)
    torch.cuda.synchronize()

    ctx.reset_counters()
    clocks = Clocks(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(ext)
    results = []
    for s in range(args.steps):
        with torch.cuda.stream(ext):
            flush.fill_(s & 0xFF)
        results.append(solve(args.warmup + s))
    ev1.record(ext)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_local = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms_local)
    ctr = ctx.counters()
    res = np.concatenate(results)
    # sample sharding: every rank holds the combined (all-reduced) totals of the same components
    agg = (lambda x: x) if sample_shard else sum_over_ranks
    jumps = agg(ctr["jumps"])
    samples = agg(ctr["samples"])
    fine_steps = agg(ctr["fine_steps"])
    rows_done = agg(len(res))
    conv = agg(int(res["converged"].sum()))
    over = agg(int(res["over_budget"].sum()))
    total_cost = agg(int(res["total_cost"].sum()))  # every rank takes part in the reduction
    proj_over = float(res["projected_cost"][res["over_budget"] != 0].max()) if (res["over_budget"] != 0).any() else 0.0
    value = jumps / (ms * 1e-3)

    # roofline of the dominant kernel (k_sample): algorithmic bytes / summed launch time
    alg_bytes = ctr["jumps"] * ALG_BYTES_PER_JUMP + ctr["samples"] * ALG_BYTES_PER_SAMPLE
    kern_s = ctr["sampler_ms"] * 1e-3
    achieved = alg_bytes / kern_s / 1e9 if kern_s > 0 else 0.0
    peaks, peak_src = load_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    cap = load_capture(cfg.name)
    traffic_rate = cap["bytes_per_ms"] if cap else None
    launches = max(1, ctr["sampler_launches"])
    # per launch, like `achieved`: the capture's DRAM bytes per kernel-ms x this run's mean launch length
    traffic = traffic_rate * ctr["sampler_ms"] / launches if traffic_rate else None
    gather_l2 = gather_hbm = None
    if rank == 0:
        try:
            gather_l2 = P.bench_gather(local, 64 << 20)
            gather_hbm = P.bench_gather(local, 8 << 30)
        except Exception:
            pass
    gpu_launches = ctr["kernel_launches"] + 2 * args.steps  # + the L2 flush fill per step (torch)

    # e2e through the public API from host buffers
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        jumps_e = 0
        h2d = d2h = 0
        e2e_steps = min(args.steps, 3)  # bounded: each e2e step is a full solve plus the table build
        ids = [None] * e2e_steps
        if sample_shard:
            ids = [P.nccl_unique_id() if rank == 0 else None for _ in range(e2e_steps)]
            dist.broadcast_object_list(ids, src=0)
        e0.record()
        for s in range(e2e_steps):
            with P.Context(cfg.a, cfg.u, device=local, sampler=sampler) as c2:
                if args.full_hold:
                    c2.set_full_hold(True)
                if args.log_hold:
                    c2.set_log_hold(True)
                if sample_shard:
                    c2.shard_samples(ids[s], rank, world)
                rows = batches[args.warmup + s]
                P.mlmc_driver_rows(c2, cfg.beta, rows, seeds[args.warmup + s], opts, want_levels=False)
                k = c2.counters()
                jumps_e += k["jumps"]
                h2d += k["h2d_bytes"] + rows.nbytes * 2  # rows + seeds read by the driver
                d2h += k["d2h_bytes"]
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ms_e = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": agg(jumps_e) / (ms_e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d / e2e_steps), "d2h_bytes_per_step": int(d2h / e2e_steps),
               "ms_per_step": ms_e / e2e_steps, "steps": e2e_steps,
               "includes": "table build from host CSR+u (H2D), driver solve, per-round H2D/D2H, results to host"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import CSR, Reference, have_reference

            if have_reference():
                threads = os.cpu_count() or 1
                ref = Reference().chain(CSR(cfg.a.n, cfg.a.row_ptr, cfg.a.col, cfg.a.val))
                j, smp, done, dt = reference_rows(ref, cfg, cpu_rows(cfg, args.warmup, r),
                                                  args.ref_seconds, threads, 1 << 30)
                cpu = {"value": j / dt if done else None, "unit": UNIT, "cores": threads, "kind": "reference",
                       "sample": f"{done} randomly chosen {cfg.name.upper()} components through the as-shipped reference "
                                 f"mlmc_driver (OpenMP, {dt:.1f} s)", "rows_per_s": done / dt if done else None,
                       "sampler_only": sampler_only_rate(ref, cfg, threads)}
        except Exception as exc:  # baseline failure must not hide the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if r == 0 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name.upper()}: {cfg.description}; one step = "
                                   + (f"the whole job (all {cfg.a.n} components) split over the ranks" if r == 0 else
                                      f"MLMC driver solve of {r} seeded components per rank"),
                       "components_per_step": int(rows_done / args.steps), "epsilon": cfg.epsilon, "t": cfg.beta,
                       "l2": f"flushed (256 MB write) before every step; tables {ctx.table_bytes / 1e6:.0f} MB",
                       "parallelism": (f"samples sharded over {world} ranks, exact NCCL all-reduce of chunk partials"
                                       if sample_shard else
                                       f"rows sharded over {world} rank(s), no data-path collective")},
            "rows_per_s": rows_done / (ms * 1e-3), "samples_per_s": samples / (ms * 1e-3),
            "path_steps_per_s": fine_steps / (ms * 1e-3),
            "cost_units_per_s": total_cost / (ms * 1e-3),
            "converged_rows": int(conv), "rows": int(rows_done), "sampler": sampler,
            "over_budget_rows": int(over), "max_cost": max_cost, "max_projected_cost_over_budget": proj_over,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "k_sample", "sampler_launches": ctr["sampler_launches"],
                         "kernel_ms": ctr["sampler_ms"], "step_share": ctr["sampler_ms"] / ms_local,
                         "alg_bytes_per_launch": alg_bytes / max(1, ctr["sampler_launches"]),
                         "traffic_source": (cap["source"] + " (ncu --set full of one launch of this config): DRAM "
                                            "bytes per kernel-ms x this run's mean launch ms") if cap else None,
                         "alg_bytes": f"{ALG_BYTES_PER_JUMP} B/transition + {ALG_BYTES_PER_SAMPLE} B/sample",
                         "gather_peak_l2_gbs": gather_l2, "gather_peak_hbm_gbs": gather_hbm,
                         "issue_active_pct": cap["issue_active_pct"] if cap else None,
                         "binding_resource": "instruction issue (ncu smsp__issue_active)" if cap else None,
                         "frac_of_gather_l2": (achieved / gather_l2) if gather_l2 else None},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(gpu_launches), "clocks": clk,
        }
        print(json.dumps(line))
    ctx.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
