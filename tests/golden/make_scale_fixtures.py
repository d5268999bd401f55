"""Generate tests/golden/scale_<config>.json: the UNMODIFIED reference's mlmc_driver on seed-chosen
components of the full-size configs (TEST INFRASTRUCTURE: the GPU parity tests at configured
sizes, tests/test_gpu_scale_parity.py, compare against these; the GPU box has no /root/reference
and the CPU reference would take too long there).

    python tests/golden/make_scale_fixtures.py c2        # 512 seed-chosen C2 components
    python tests/golden/make_scale_fixtures.py c3        # degree-stratified BA n=1e6 components
    python tests/golden/make_scale_fixtures.py c4-20     # degree-stratified R-MAT scale-20 components

Inputs: C2 = workloads.grid_laplacian(1024) + the Philox vector; C3 = the reference's own
pref(1e6, 5, seed 1) (netgen.cpp:61-107); R-MAT = the product's host generator (the reference
has none), handed to the reference as a CSR.  beta = 1/lambda from workloads.power_iteration.
Every component runs the reference mlmc_driver (mlmc.cpp:170-260) with its OWN default options
(eps = 1e-3, warmup 1000, max_levels_above_l0 30, no cost budget), row seed 1000 + row, one
process per component (results are bitwise thread-count independent, parallel.hpp:16-19): light
components single-threaded, `--procs` at a time; components of degree >= --heavy-degree one at a
time on `--procs` threads, lightest first.  A component whose reference run exceeds `--cap`
seconds is recorded as `timed_out` (the reference has no budget; SURVEY §7 hub rows run for
hours) and is not a parity case.  The matrix is pinned by a hash of its CSR.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import pickle
import select
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import CSR, Reference  # noqa: E402

# degree strata [lo, hi] and components per stratum (graph configs)
STRATA = {"c3": [(5, 5), (6, 7), (8, 11), (12, 19), (20, 49), (50, 199), (200, 1 << 40)],
          "c4": [(1, 1), (2, 3), (4, 7), (8, 15), (16, 63), (64, 255), (256, 1 << 40)]}


def csr_hash(rp, col, val) -> str:
    h = hashlib.sha256()
    for a in (np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(col, np.int64),
              np.ascontiguousarray(val, np.float64)):
        h.update(a.tobytes())
    return h.hexdigest()


def problem(name):
    ref = Reference()
    if name == "c2":
        n, rp, col, val = W.grid_laplacian(1024)
        u = W.philox_first_uniform(W.VECTOR_SEED, 0, np.arange(n, dtype=np.uint64), 6)
        return ref.chain(CSR(n, rp, col, val)), u, 0.5, (rp, col, val), {"matrix": "grid_laplacian(1024)", "t": "0.5"}
    if name == "c3":
        chain = ref.pref(1_000_000, 5, W.GRAPH_SEED)
        dec = chain.decomposition()
        rp, col = dec["row_ptr"], dec["jump_target"]
        val = np.ones(col.size)
        lam = W.power_iteration(rp.size - 1, rp, col, val, 50)
        return chain, np.ones(rp.size - 1), 1.0 / lam, (rp, col, val), {
            "matrix": "reference pref(1000000, 5, 1)", "lambda": lam.hex(), "t": "1/lambda"}
    if name.startswith("c4-"):
        # generated in a child process: the product generator is OpenMP-parallel and this process
        # forks its workers later (libgomp state must not cross a fork)
        path = f"/tmp/expmc_rmat{name[3:]}.npz"
        if not os.path.exists(path):
            code = (f"import numpy as np; from paper_1904_12754_b200 import configs as c; a = c.gen_rmat({name[3:]}, 16); "
                    f"np.savez({path!r}, rp=a.row_ptr, col=a.col)")
            subprocess.run([sys.executable, "-c", code], check=True, cwd=ROOT)
        z = np.load(path)
        rp, col = z["rp"], z["col"]
        n = rp.size - 1
        val = np.ones(col.size)
        lam = W.power_iteration(n, rp, col, val, 50)
        return ref.chain(CSR(n, rp, col, val)), np.ones(n), 1.0 / lam, (rp, col, val), {
            "matrix": f"product gen_rmat({name[3:]}, 16) (a=0.57, b=c=0.19), symmetrised", "lambda": lam.hex(),
            "t": "1/lambda"}
    raise ValueError(name)


def choose_rows(name, deg, count, per_stratum, seed=20260420):
    rng = np.random.default_rng(seed)
    if name == "c2":
        return np.sort(rng.choice(deg.size, size=count, replace=False)).astype(np.int64), None
    rows, strata = [], []
    for k, (lo, hi) in enumerate(STRATA[name.split("-")[0]]):
        cand = np.where((deg >= lo) & (deg <= hi))[0]
        pick = rng.choice(cand, size=min(per_stratum, cand.size), replace=False) if cand.size else []
        # the stratum's heaviest component too (the hubs), if not drawn already
        if cand.size and k == len(STRATA[name.split("-")[0]]) - 1:
            pick = np.unique(np.concatenate([pick, cand[np.argsort(deg[cand])[-min(8, cand.size):]]]))
        rows += [int(r) for r in pick]
        strata += [k] * len(pick)
    order = np.argsort(rows)
    return np.asarray(rows, np.int64)[order], np.asarray(strata, np.int32)[order]


def run_rows(chain, u, beta, rows, procs, cap, threads=1, give_up=0, journal=None):
    """Fork one child per component (`threads` OpenMP threads in the reference's run_level),
    `procs` at a time, each killed after `cap` s.  give_up > 0: after that many consecutive
    timeouts the remaining rows (ascending degree: heavier still) are recorded as timed out
    without running."""
    out = {}
    todo = list(rows)
    streak = 0
    live = {}  # pid -> (row, read fd, start)
    while todo or live:
        if give_up and streak >= give_up:
            for r in todo:
                out[int(r)] = {"timed_out": True, "seconds": 0.0, "skipped": True}
            todo = []
        while todo and len(live) < procs:
            r = int(todo.pop(0))
            rd, wr = os.pipe()
            pid = os.fork()
            if pid == 0:  # child
                os.close(rd)
                try:
                    (res,) = chain.driver_rows(u, beta, [r], [W.ROW_SEED_BASE + r], threads=threads)
                    res["levels"] = [dict(level=int(x["level"]), sum=float(x["sum"]).hex(),
                                          sum_sq=float(x["sum_sq"]).hex(), samples=int(x["samples"]),
                                          cost=int(x["cost"])) for x in res["levels"]]
                    data = pickle.dumps(res)
                except BaseException as e:  # noqa: BLE001
                    data = pickle.dumps({"error": repr(e)})
                with os.fdopen(wr, "wb") as f:
                    f.write(data)
                os._exit(0)
            os.close(wr)
            live[pid] = (r, rd, time.time())
        fds = [v[1] for v in live.values()]
        ready, _, _ = select.select(fds, [], [], 1.0)
        for pid, (r, rd, t0) in list(live.items()):
            if rd in ready:
                with os.fdopen(rd, "rb") as f:
                    data = f.read()
                os.waitpid(pid, 0)
                res = pickle.loads(data) if data else {"error": "no output"}
                res["seconds"] = time.time() - t0
                out[r] = res
                streak = 0
                if journal:  # progress survives an interrupted run (--resume)
                    with open(journal, "ab") as jf:
                        pickle.dump((r, res), jf)
                del live[pid]
                print(f"row {r}: {time.time() - t0:.1f}s cost {res.get('total_cost', -1):.3g} L {res.get('L')}",
                      flush=True)
            elif time.time() - t0 > cap:
                os.kill(pid, 9)
                os.waitpid(pid, 0)
                os.close(rd)
                out[r] = {"timed_out": True, "seconds": cap}
                streak += 1
                if journal:
                    with open(journal, "ab") as jf:
                        pickle.dump((r, out[r]), jf)
                del live[pid]
                print(f"row {r}: timed out", flush=True)
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("config")
    p.add_argument("--count", type=int, default=512, help="C2: seed-chosen components")
    p.add_argument("--per-stratum", type=int, default=48, help="graphs: components per degree stratum")
    p.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    p.add_argument("--cap", type=float, default=900.0, help="seconds per component")
    p.add_argument("--heavy-degree", type=int, default=50,
                   help="graphs: components of at least this degree run one at a time on all threads, "
                        "in ascending degree, giving up after --give-up consecutive timeouts")
    p.add_argument("--give-up", type=int, default=4)
    p.add_argument("--resume", action="store_true", help="skip components already in the run's journal")
    a = p.parse_args()
    t0 = time.time()
    chain, u, beta, (rp, col, val), meta = problem(a.config)
    deg = np.diff(rp)
    print(f"problem built in {time.time() - t0:.0f}s: n={deg.size} nnz={rp[-1]} beta={beta!r}", flush=True)
    rows, strata = choose_rows(a.config, deg, a.count, a.per_stratum)
    journal = os.path.join("/tmp", f"scale_{a.config}.journal")
    res = {}
    if a.resume and os.path.exists(journal):
        with open(journal, "rb") as jf:
            while True:
                try:
                    r, x = pickle.load(jf)
                except EOFError:
                    break
                res[int(r)] = x
        print(f"resumed {len(res)} components from {journal}", flush=True)
    elif os.path.exists(journal):
        os.remove(journal)
    todo = [int(r) for r in rows if int(r) not in res]
    if strata is None:
        res.update(run_rows(chain, u, beta, todo, a.procs, a.cap, journal=journal))
    else:  # light components in parallel, then the heavy ones on all threads, lightest first
        light = [r for r in todo if deg[r] < a.heavy_degree]
        heavy = sorted((r for r in todo if deg[r] >= a.heavy_degree), key=lambda r: (deg[r], r))
        res.update(run_rows(chain, u, beta, light, a.procs, a.cap, journal=journal))
        res.update(run_rows(chain, u, beta, heavy, 1, a.cap, threads=a.procs, give_up=a.give_up, journal=journal))
    out = {"generator": "tests/golden/make_scale_fixtures.py (reference mlmc_driver via oracle/_ref)",
           "config": a.config, **meta, "beta": float(beta).hex(), "n": int(deg.size), "nnz": int(rp[-1]),
           "csr_sha256": csr_hash(rp, col, val), "epsilon": 1e-3, "cap_seconds": a.cap,
           "strata": STRATA.get(a.config.split("-")[0]), "rows": []}
    for i, r in enumerate(rows):
        x = res[int(r)]
        rec = {"row": int(r), "degree": int(deg[r]), "stratum": int(strata[i]) if strata is not None else None,
               "seconds": round(x["seconds"], 2)}
        if x.get("timed_out") or "error" in x:
            rec["timed_out"] = True
            rec["error"] = x.get("error")
            rec["skipped"] = bool(x.get("skipped", False))
        else:
            rec.update(estimate=float(x["estimate"]).hex(), statistical_error=float(x["statistical_error"]).hex(),
                       bias_estimate=float(x["bias_estimate"]).hex(), l0=int(x["l0"]), L=int(x["L"]),
                       total_cost=int(x["total_cost"]), converged=bool(x["converged"]), levels=x["levels"])
        out["rows"].append(rec)
    path = os.path.join(HERE, f"scale_{a.config}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    done = sum(1 for r in out["rows"] if not r.get("timed_out"))
    print(f"wrote {path}: {done}/{len(rows)} components in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
