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

`--gpus N` without torchrun re-launches this script under `torch.distributed.run` with N ranks
(one per GPU); under torchrun WORLD_SIZE must equal N or the run fails.

Timed region (`value`): tables already resident in HBM; K steps bracketed by barrier +
torch.cuda.synchronize(), CUDA events recorded on the library's own stream; max over ranks.
L2 is flushed (256 MB write) before every step inside the timed region.
`e2e`: the same work through the public API from HOST buffers -- context creation from the
host CSR + u (H2D), the solve, results back to host -- per step, CUDA events on the current
stream around the call.

`--impl reference`: the UNMODIFIED reference (oracle/_ref/libexpmc_ref.so, compiled from
/root/reference by oracle/Makefile) runs its own mlmc_driver per component with OpenMP on all
host cores, rank 0 only.  Its process never imports the product package: the inputs come from
`workloads.py` (numpy) and the reference's own generator.  Each of its steps is a bounded
sample of the same job (`sample` key); `config` is the same dict as this arm's.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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

import workloads as W  # noqa: E402  (numpy only: safe for the reference arm)

METRIC = "random-walk transitions/sec and exp(tA)v rows/sec at target ε; % gather roofline"
UNIT = "transitions/s"
# algorithmic bytes per transition: reference-order sampler (and the event sampler with separate
# row gathers) = the edge's target sector + the destination row record (32-B sector: d, rate, u,
# begin, deg); event sampler = one 32-B EdgeRec carrying the target row's payload
ALG_BYTES_PER_JUMP = {"reference": 64, "event": 32}
PROFILE_DIR = os.path.join(ROOT, "profiles", "r02")
# reference-arm components per step (as-shipped driver, all host cores): ~1-3 s per step on 16 cores
REF_ROWS_PER_STEP = {"c1": 64, "c2": 32, "c3": 1, "c4": 1, "c5": 1}


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--rows-per-step", type=int, default=0, help="components per rank per step (0: default)")
    p.add_argument("--ref-seconds", type=float, default=15.0, help="cpu_baseline sample budget (our arm)")
    p.add_argument("--ref-rows-per-step", type=int, default=0, help="reference arm: components per step (0: default)")
    p.add_argument("--max-cost", type=float, default=None,
                   help="per-component model-unit budget (driver extension; default off for C1/C2, 1e10 for C3-C5)")
    p.add_argument("--sampler", default=None, choices=["reference", "event"], help="override the config's sampler")
    p.add_argument("--full-hold", action="store_true",
                   help="event sampler: evaluate first holding intervals in full (A/B of the closed-form hold)")
    p.add_argument("--row-gather", action="store_true",
                   help="event sampler: separate gather of the target's row record (A/B of the per-edge records)")
    p.add_argument("--screen-each", action="store_true",
                   help="event sampler: per-sample screen (A/B of the geometric screen)")
    p.add_argument("--log-hold", action="store_true",
                   help="reference-order sampler: time-space holding tests with a log per event (A/B of S-mode)")
    p.add_argument("--multi", default=None, choices=["rows", "samples"],
                   help="N>1: shard components over ranks (no collective; default for C1/C2) or shard every "
                        "component's samples with an exact NCCL all-reduce of the chunk partials (default for "
                        "the hub-heavy C3/C4)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """`--gpus N` (N > 1) without torchrun: start N ranks with torch.distributed.run on this node
    and return its exit code.  NCCL_DEBUG=INFO (unless set) so the log shows every rank's comm."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


_PERM = {}


def perm_rows(n):
    if n not in _PERM:
        _PERM[n] = np.random.default_rng(20190429).permutation(n).astype(np.int64)
    return _PERM[n]


def row_shard(n, rank, world):
    """Components of rank `rank` when the whole job is dealt over `world` ranks: every world-th
    entry of the fixed permutation, sorted (paper_1904_12754_b200.shard.row_shard)."""
    return np.sort(perm_rows(n)[rank::world])


def batch_rows(n, step, rank, world, r):
    """Rows rank `rank` solves in `step`.  r == 0: the whole job -- every component, dealt
    round-robin over a fixed permutation to the ranks (strong scaling).  r > 0: r components
    per rank per step, consecutive slices of the permutation (weak scaling)."""
    if r == 0:
        return row_shard(n, rank, world)
    k = (step * world + rank) * r
    return np.sort(perm_rows(n)[np.arange(k, k + r) % n])


def cpu_sample_rows(universe, deg, name, step, count):
    """Components of CPU-reference step `step`: consecutive slices of the same fixed permutation the
    GPU arm deals its batches from.  Graph / 3-D configs keep light components only (degree <= 8):
    the reference has no cost budget and a hub component runs for hours."""
    perm = perm_rows(len(universe))
    cand = universe[perm]
    if name.startswith(("c3", "c4", "c5")):
        cand = cand[deg[cand] <= 8]
    k = step * count
    return cand[np.arange(k, k + count) % len(cand)]


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


_SCALE = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def load_capture(cfg_name):
    """This config's committed `ncu --set full` capture of one k_sample launch
    (profiles/r02/k_sample_<config>_key_metrics.json, written by scripts/ncu_keys.py from the
    .ncu-rep): the measured DRAM bytes, L2 / L1 throughput and issue utilisation of that launch.
    None for configs without a capture."""
    name = cfg_name.split("-")[0]
    path = os.path.join(PROFILE_DIR, f"k_sample_{name}_key_metrics.json")
    try:
        with open(path) as f:
            k = json.load(f)
        ms = float(k["gpu__time_duration.sum"]["value"]) * (1e-3 if k["gpu__time_duration.sum"]["unit"] == "us" else 1.0)
        dram = sum(float(k[m]["value"]) * _SCALE[k[m]["unit"]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))

        def pct(key):
            return float(k[key]["value"]) / 100.0 if key in k else None

        return {"ms": ms, "dram_bytes": dram, "dram_bytes_per_ms": dram / ms,
                "l2_frac": pct("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                "l1_frac": pct("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                "issue_frac": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "threads_per_inst": float(k["smsp__thread_inst_executed_per_inst_executed.ratio"]["value"]),
                "l1_hit": pct("l1tex__t_sector_hit_rate.pct"), "l2_hit": pct("lts__t_sector_hit_rate.pct"),
                "source": os.path.relpath(path, ROOT)}
    except (OSError, KeyError, ValueError):
        return None


# ------------------------------------------------------------------------------ reference arm
def reference_problem(name):
    """The reference's own objects for config `name`, built without the product package:
    (RefChain, u, beta, universe, degree, max_levels_above_l0, eps)."""
    from oracle import CSR, Reference

    ref = Reference()
    base = name.split("-")[0]
    if name in ("c1", "c2") or name.startswith("grid"):
        g = {"c1": 64, "c2": 1024}.get(name) or int(name[4:])
        n, rp, col, val = W.grid_laplacian(g)
        u = W.philox_first_uniform(W.VECTOR_SEED, 0, np.arange(n, dtype=np.uint64), 6)
        beta = 0.5 if name == "c2" else 1.0
        return ref.chain(CSR(n, rp, col, val)), u, beta, np.arange(n, dtype=np.int64), np.diff(rp), 30, 1e-3
    if base == "c5":
        g = int(name[3:]) if "-" in name else 256
        n, rp, col, val = W.convdiff3d(g, 10.0, 0)
        u = 2.0 * W.philox_first_uniform(W.VECTOR_SEED, 0, np.arange(n, dtype=np.uint64), 6) - 1.0
        return ref.chain(CSR(n, rp, col, val)), u, 0.1, np.arange(n, dtype=np.int64), np.diff(rp), 4, 1e-4
    if base == "c3":
        n = int(name[3:]) if "-" in name else 1_000_000
        chain = ref.pref(n, 5, W.GRAPH_SEED)  # the reference's own netgen (netgen.cpp:61-107)
        dec = chain.decomposition()           # 0/1 adjacency, zero diagonal: CSR = (row_ptr, targets, 1)
        rp, col = dec["row_ptr"], dec["jump_target"]
        lam = W.power_iteration(n, rp, col, np.ones(col.size), 50)
        return chain, np.ones(n), 1.0 / lam, np.arange(n, dtype=np.int64), np.diff(rp), 30, 1e-3
    if base == "c4":
        # R-MAT exists only in the product's host generator (the reference has none):
        # generated in a SEPARATE process and handed over as arrays, so this process never loads it
        scale = int(name[3:]) if "-" in name else 24
        path = os.path.join("/tmp", f"expmc_rmat{scale}.npz")
        if not os.path.exists(path):
            code = (f"import numpy as np; from paper_1904_12754_b200 import configs as c; a = c.gen_rmat({scale}, 16); "
                    f"np.savez({path!r}, rp=a.row_ptr, col=a.col)")
            subprocess.run([sys.executable, "-c", code], check=True, cwd=ROOT)
        z = np.load(path)
        rp, col = z["rp"], z["col"]
        n = rp.size - 1
        lam = W.power_iteration(n, rp, col, np.ones(col.size), 50)
        rows = W.seeded_rows(n, min(n, 1 << 20))
        return ref.chain(CSR(n, rp, col, np.ones(col.size))), np.ones(n), 1.0 / lam, rows, np.diff(rp), 30, 1e-3
    raise ValueError(f"unknown config {name!r}")


def reference_step(chain, u, beta, rows, deg, eps, mla, threads):
    """The as-shipped reference mlmc_driver on `rows`, one after another (reference OpenMP inside
    run_level).  Returns (transitions, samples, components)."""
    jumps = samples = 0
    for r in rows:
        (res,) = chain.driver_rows(u, beta, [int(r)], [W.ROW_SEED_BASE + int(r)], epsilon=eps, threads=threads,
                                   max_levels_above_l0=mla)
        # transitions = sum_l (cost_l - 2 M_l 2^l); an isolated (absorbing) row never jumps
        jumps += 0 if deg[int(r)] == 0 else res["total_jumps"]
        samples += res["total_samples"]
    return jumps, samples, len(rows)


def run_reference(args, rank, world):
    """`--impl reference`: rank 0 times the unmodified reference on `--steps` steps, each a fixed
    sample of the job's components (the first REF_ROWS_PER_STEP of consecutive slices of the same
    permutation the GPU arm deals from), after `--warmup` untimed steps."""
    if rank != 0:
        return 0
    from oracle import have_reference

    if not have_reference():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libexpmc_ref.so not built"}))
        return 0
    threads = os.cpu_count() or 1
    chain, u, beta, universe, deg, mla, eps = reference_problem(args.config)
    per_step = args.ref_rows_per_step or REF_ROWS_PER_STEP.get(args.config.split("-")[0], 16)
    for w in range(args.warmup):
        reference_step(chain, u, beta, cpu_sample_rows(universe, deg, args.config, w, per_step), deg, eps, mla, threads)
    tj = ts = tr = 0
    step_ms = []
    for s in range(args.steps):
        rows = cpu_sample_rows(universe, deg, args.config, args.warmup + s, per_step)
        t0 = time.perf_counter()
        j, smp, nr = reference_step(chain, u, beta, rows, deg, eps, mla, threads)
        step_ms.append(1e3 * (time.perf_counter() - t0))
        tj, ts, tr = tj + j, ts + smp, tr + nr
    tt = sum(step_ms) * 1e-3
    value = tj / tt if tt > 0 else None
    sample = (f"{per_step} components per step ({tr} timed), consecutive slices of the GPU arm's fixed component "
              f"permutation" + (", degree <= 8 only" if args.config.startswith(("c3", "c4", "c5")) else "")
              + "; as-shipped reference mlmc_driver per component, row seed 1000 + row")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(np.mean(step_ms)) if step_ms else None, "higher_is_better": True,
        "scaling": "strong" if args.config in ("c1", "c2") and not args.rows_per_step else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": W.config_dict(args.config), "sample": sample,
        "parallelism": f"OpenMP {threads} host threads (reference run_level), rank 0 only",
        "rows_per_s": tr / tt if tt > 0 else None, "samples_per_s": ts / tt if tt > 0 else None,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline_leg(args, threads, cfg=None):
    """cpu_baseline of our arm (rank 0, N = 1): the unmodified reference on a bounded ~ref-seconds
    sample of the same job, plus its sampler alone.  With the arm's config at hand
    the reference's tables are decomposed from the same CSR (the reference's own decompose,
    chain.cpp:75) instead of regenerating the graph and its lambda (minutes at C3 / C4 scale)."""
    from oracle import CSR, Reference, have_reference

    if not have_reference():
        return {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": "oracle/_ref not built"}
    if cfg is None:
        chain, u, beta, universe, deg, mla, eps = reference_problem(args.config)
    else:
        a = cfg.a
        chain = Reference().chain(CSR(a.n, a.row_ptr, a.col, a.val))
        u, beta, eps, mla = cfg.u, cfg.beta, cfg.epsilon, cfg.max_levels_above_l0
        universe = cfg.rows if cfg.rows is not None else np.arange(a.n, dtype=np.int64)
        deg = np.diff(a.row_ptr)
    per_step = REF_ROWS_PER_STEP.get(args.config.split("-")[0], 16)
    tj = ts = tr = 0
    t0 = time.perf_counter()
    s = 0
    while time.perf_counter() - t0 < args.ref_seconds:
        j, smp, nr = reference_step(chain, u, beta, cpu_sample_rows(universe, deg, args.config, 1000 + s, per_step),
                                    deg, eps, mla, threads)
        tj, ts, tr, s = tj + j, ts + smp, tr + nr, s + 1
    dt = time.perf_counter() - t0
    return {"value": tj / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{tr} {args.config.upper()} components through the as-shipped reference mlmc_driver "
                      f"(OpenMP, {dt:.1f} s)", "rows_per_s": tr / dt,
            "sampler_only": sampler_only_rate(chain, u, beta, universe, threads, deg)}


def sampler_only_rate(chain, u, beta, universe, threads, deg, seconds=4.0):
    """The reference's sampler without the driver: one large run_level per level (its
    LevelSampler table is built once per call, so the O(n) construction is amortised), OpenMP on all
    cores.  transitions = the jumps run_level counts (RunLevelStats::jumps); the row is the first
    of the fixed permutation with degree >= 2.  Level 0 (base) and level 2 (coupled), ~seconds/2
    each."""
    out = {}
    perm = perm_rows(len(universe))
    row = int(next(universe[k] for k in perm if deg[universe[k]] >= 2))
    for level, base in ((0, True), (2, False)):
        m = 1 << 16
        while True:  # grow the sample until one call takes ~seconds / 2
            t0 = time.perf_counter()
            r = chain.run_level(u, row, beta, level, base, 1 << 40, m, 99, threads=threads)
            dt = time.perf_counter() - t0
            if dt >= seconds / 4 or m >= (1 << 34):
                break
            m = int(m * min(16.0, max(2.0, (seconds / 2) / max(dt, 1e-3))))
        jumps = int(r["jumps"])
        out[f"level{level}"] = {"transitions_per_s": jumps / dt, "samples_per_s": m / dt, "samples": m,
                                "seconds": dt, "row": row}
    return out


# ------------------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local):
    import torch

    import paper_1904_12754_b200 as P
    from paper_1904_12754_b200 import configs

    cfg = configs.make_config(args.config)
    graph_like = cfg.name.startswith(("c3", "c4", "c5"))
    # C1-C4: the whole job per step (C3: all 10^6 components, C4: the 2^20 seed-chosen ones).
    # C5 (16.7M components at eps = 1e-4): a seeded sample of components per step.  Graph / 3-D
    # configs run with a per-component budget (hub rows are infeasible at the stated eps, SURVEY
    # §7); the line reports the over-budget set and its projected cost.
    r = args.rows_per_step if args.rows_per_step or not cfg.name.startswith("c5") else 4096
    # per-component budgets of DESIGN §7b: 1e10 model units for C3/C4, 1e9 for C5 (eps = 1e-4)
    default_budget = (1e9 if cfg.name.startswith("c5") else 1e10) if graph_like else 0.0
    max_cost = args.max_cost if args.max_cost is not None else default_budget
    sampler = args.sampler or cfg.sampler
    universe = cfg.rows if cfg.rows is not None else np.arange(cfg.a.n, dtype=np.int64)
    multi = args.multi or ("samples" if cfg.name.startswith(("c3", "c4")) else "rows")

    # EXPMC_BENCH_SHARE_DEVICE=1 (functional check of the N > 1 path on a one-GPU box, never a
    # measurement): every rank on cuda:0, host plumbing over gloo.  Row sharding has no
    # device-side exchange, so the ranks' kernels never wait on one another.
    shared = os.environ.get("EXPMC_BENCH_SHARE_DEVICE") == "1"
    if shared:
        local = 0
        if multi == "samples" and world > 1:
            multi = "rows"  # NCCL ranks on one device would wait on one another (B200_PROFILING.md)
    elif local >= P.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but only {P.device_count()} GPU(s) are visible")
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
    if args.row_gather:
        ctx.set_row_gather(True)
    if args.screen_each:
        ctx.set_screen_each(True)
    sample_shard = multi == "samples" and world > 1
    if sample_shard:  # every rank runs the same components; chunk g is sampled on rank g % world
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.shard_samples(obj[0], rank, world)
    rank_b, world_b = (0, 1) if sample_shard else (rank, world)
    ext = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", local))

    # the batches of every step are built before any timing starts
    batches = [universe[batch_rows(len(universe), s, rank_b, world_b, r)] for s in range(args.warmup + args.steps)]
    seeds = [W.row_seeds(b) for b in batches]

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
    overb = res["over_budget"] != 0
    over = agg(int(overb.sum()))
    total_cost = agg(int(res["total_cost"].sum()))  # every rank takes part in the reduction
    proj_over = float(res["projected_cost"][overb].max()) if overb.any() else 0.0
    # completeness of graph configs: projected model units of the over-budget components, their
    # sum extrapolated to the whole job, and the GPU time that would take at this run's unit rate
    proj_sum = agg(float(res["projected_cost"][overb].sum()))
    proj_full = proj_sum * len(universe) / max(1.0, rows_done)  # rows_done: every step's components
    value = jumps / (ms * 1e-3)
    cost_rate = total_cost / (ms * 1e-3)

    # roofline of the dominant kernel (k_sample): algorithmic bytes / summed launch time (CUDA
    # events on the library stream around every sampler launch, read back by ctx.counters())
    launches = max(1, ctr["sampler_launches"])
    bytes_per_jump = 64 if sampler == "reference" or args.row_gather else ALG_BYTES_PER_JUMP["event"]
    alg_bytes = ctr["jumps"] * bytes_per_jump
    kern_s = ctr["sampler_ms"] * 1e-3
    achieved = alg_bytes / kern_s / 1e9 if kern_s > 0 else 0.0
    peaks, peak_src = load_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    cap = load_capture(cfg.name)
    mean_launch_ms = ctr["sampler_ms"] / launches
    traffic = cap["dram_bytes_per_ms"] * mean_launch_ms if cap else None
    gather_l2 = gather_hbm = None
    if rank == 0:
        try:
            gather_l2 = P.bench_gather(local, 64 << 20)
            gather_hbm = P.bench_gather(local, 8 << 30)
        except Exception:
            pass
    gpu_launches = ctr["kernel_launches"] + args.steps  # + the L2 flush fill per step (torch)

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
                if args.row_gather:
                    c2.set_row_gather(True)
                if args.screen_each:
                    c2.set_screen_each(True)
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
            cpu = cpu_baseline_leg(args, os.cpu_count() or 1, cfg)
        except Exception as exc:  # baseline failure must not hide the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"failed: {exc}"}

    if rank == 0:
        measured = None
        if cap:
            dram_gbs = cap["dram_bytes_per_ms"] / 1e6
            measured = {"source": cap["source"] + " (ncu --set full, one k_sample launch of this config)",
                        "dram_gbs": dram_gbs, "dram_frac": dram_gbs / peak, "l2_frac": cap["l2_frac"],
                        "l1_frac": cap["l1_frac"], "issue_frac": cap["issue_frac"],
                        "threads_per_inst": cap["threads_per_inst"], "l1_hit": cap["l1_hit"], "l2_hit": cap["l2_hit"]}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if r == 0 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": W.config_dict(cfg.name),
            "step": ("the whole job (all components) split over the ranks" if r == 0 else
                     f"MLMC driver solve of {r} seeded components per rank"),
            "components_per_step": int(rows_done / args.steps),
            "l2": f"flushed (256 MB write) before every step; tables {ctx.table_bytes / 1e6:.0f} MB",
            "parallelism": (f"samples sharded over {world} ranks, exact NCCL all-reduce of chunk partials"
                            if sample_shard else f"rows sharded over {world} rank(s), no data-path collective"),
            "rows_per_s": rows_done / (ms * 1e-3), "samples_per_s": samples / (ms * 1e-3),
            "path_steps_per_s": fine_steps / (ms * 1e-3), "cost_units_per_s": cost_rate,
            "converged_rows": int(conv), "rows": int(rows_done), "rows_note": "summed over the timed steps",
            "sampler": sampler,
            "completeness": {
                "per": "step (the counts are the mean over the timed steps)",
                "components": int(rows_done / args.steps),
                "converged": int(conv / args.steps), "over_budget": int(over / args.steps), "max_cost": max_cost,
                "over_budget_fraction": over / rows_done if rows_done else 0.0,
                "max_projected_cost_over_budget": proj_over,
                "projected_cost_over_budget_sum": proj_sum / args.steps,
                "job_components": len(universe),
                "projected_cost_over_budget_full_job": proj_full,
                "projected_gpu_hours_full_job": proj_full / cost_rate / 3600.0 * world if cost_rate > 0 else None,
                "note": "model units the over-budget components need at this eps (driver projection, DESIGN §7b); "
                        "GPU-hours at this run's cost-unit rate on n_gpus GPUs"},
            # achieved / frac: the contract's ALGORITHMIC bytes over the HBM copy peak (also under
            # their own name, modelled_gbs / modelled_frac); dram_frac, l2_frac, l1_frac, issue_frac:
            # what the config's ncu capture measured -- the kernel's real position (binding_resource)
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "modelled_gbs": achieved, "modelled_frac": achieved / peak,
                         "dram_frac": measured and measured["dram_frac"], "l2_frac": measured and measured["l2_frac"],
                         "l1_frac": measured and measured["l1_frac"], "issue_frac": measured and measured["issue_frac"],
                         "kernel": "k_sample_grouped" if sampler == "event" else "k_sample",
                         "sampler_launches": ctr["sampler_launches"],
                         "kernel_ms": ctr["sampler_ms"], "mean_launch_ms": mean_launch_ms,
                         "step_share": ctr["sampler_ms"] / ms_local,
                         "alg_bytes": f"{bytes_per_jump} B per transition ("
                                      + ("row record + edge sector" if bytes_per_jump == 64 else
                                         "one edge record with the target row's payload; + <= 1 sector per "
                                         "jumping sample for u[end], not counted")
                                      + "); samples "
                                      "that never leave the entry read no table",
                         "alg_bytes_per_launch": alg_bytes / launches,
                         "measured": measured,
                         "binding_resource": (None if not cap else
                                              f"the SM: issue slots {cap['issue_frac']:.2f} and L1 data pipe "
                                              f"{cap['l1_frac']:.2f} of peak, gathers served by L1 (hit rate "
                                              f"{cap['l1_hit']:.2f})" if cap["l1_hit"] >= 0.9 else
                                              f"random-gather latency (issue slots {cap['issue_frac']:.2f}, L1 hit "
                                              f"{cap['l1_hit']:.2f}, L2 hit {cap['l2_hit']:.2f}; tables beyond L2)"),
                         "gather_peak_l2_gbs": gather_l2, "gather_peak_hbm_gbs": gather_hbm,
                         "frac_of_gather_l2": (achieved / gather_l2) if gather_l2 else None},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(gpu_launches), "clocks": clk,
        }
        print(json.dumps(line))
    ctx.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    rank, world, local = dist_env()
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch N ranks for --gpus N\n")
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
