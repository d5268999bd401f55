"""Generate tests/golden/golden.json from the UNMODIFIED reference library.

Run here (where /root/reference exists and oracle/_ref/libexpmc_ref.so is built by
`make -C oracle`):   python tests/golden/make_golden.py
Every number in golden.json is an output of the reference's own code path (RngStream,
decompose, LevelSampler::single/coupled, run_level, mlmc_driver, dense_expmv, smallw),
stored as exact hex floats.  The fixtures are committed; tests never need /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import CSR, Reference  # noqa: E402


def hx(a):
    return [float(x).hex() for x in np.asarray(a, np.float64).ravel()]


def csr_json(a: CSR):
    return dict(n=int(a.n), row_ptr=[int(x) for x in a.row_ptr], col=[int(x) for x in a.col], val=hx(a.val))


def grid(g):
    n = g * g
    trips = []
    for y in range(g):
        for x in range(g):
            r = y * g + x
            trips.append((r, r, -4.0))
            if x > 0:
                trips.append((r, r - 1, 1.0))
            if x + 1 < g:
                trips.append((r, r + 1, 1.0))
            if y > 0:
                trips.append((r, r - g, 1.0))
            if y + 1 < g:
                trips.append((r, r + g, 1.0))
    return CSR.from_triplets(n, trips)


def main():
    ref = Reference()
    out = {"generator": "tests/golden/make_golden.py (reference: /root/reference/proj/core via oracle/_ref)"}

    # 1. Philox uniforms (rng.hpp:21-79) incl. SURVEY Appendix A anchors
    keys = [(0, 0, 0, 0), (42, 3, 12345, 0), (7, 5, 2 ** 40, 2), (12345, 0, 7, 6), (2 ** 63 + 5, 62, 2 ** 64 - 1, 255),
            (1000, 4, 511, 0), (1001, 0, 512, 0)]
    out["uniforms"] = [dict(key=list(k), values=hx(ref.uniforms(*k, 9))) for k in keys]

    # 2. matrices
    mats = {
        "two_state": CSR.from_dense([[0.2, 1.0], [0.5, -0.3]]),        # test_paths.cpp:150-151
        "k2": CSR.from_dense([[0.0, 1.0], [1.0, 0.0]]),                 # test_paths.cpp:102
        "diag": CSR.from_dense([[0.75, 0.0], [0.0, -0.5]]),              # test_paths.cpp:85
        "signed3": CSR.from_dense([[0.1, -1.0, 0.5], [0.7, -0.2, -0.2], [-0.4, 0.0, 0.3]]),
        "absorb3": CSR.from_dense([[0.0, 1.0, 0.5], [0.0, -1.0, 0.0], [0.25, 0.25, 0.0]]),
        "grid8": grid(8),
    }
    sw = ref.smallw(100, 2, 0.1, 5)                                      # test_paths.cpp:114
    mats["smallw100"] = sw.a
    hub = ref.pref(300, 3, 7)                                            # BA, wide hub rows (deg > 4)
    mats["pref300"] = hub.a

    rng = np.random.default_rng(0)
    out["matrices"] = {}
    for name, a in mats.items():
        ch = ref.chain(a)
        dec = ch.decomposition()
        n = a.n
        u = np.round(rng.uniform(-1.0, 2.0, n), 6)
        beta = 0.8 if name != "smallw100" else 1.0 / dec["d_max"] if dec["d_max"] > 0 else 1.0
        entries = sorted(set([0, n - 1, n // 2]))
        samples = []
        for entry in entries:
            for level in range(0, 5):
                for base in ([1, 0] if level > 0 else [1]):
                    seed = 1000 + entry + 17 * level
                    idx = np.array(list(range(24)) + [511, 512, 2 ** 33 + 3, 2 ** 40 + 1], np.uint64)
                    s = ch.samples(u, entry, beta, level, base, seed, idx)
                    samples.append(dict(entry=entry, level=level, base=base, seed=seed, idx=[int(x) for x in idx],
                                        fine=hx(s["fine"]), coarse=hx(s["coarse"]), cost=[int(c) for c in s["cost"]]))
        runs = []
        for entry in entries[:2]:
            for (level, base, first, count) in [(0, 1, 0, 1000), (1, 0, 37, 2500), (3, 0, 1000, 700), (4, 0, 0, 1)]:
                seed = 77 + entry
                r = ch.run_level(u, entry, beta, level, base, first, count, seed, threads=4)
                runs.append(dict(entry=entry, level=level, base=base, first=first, count=count, seed=seed,
                                 sum=float(r["sum"]).hex(), sum_sq=float(r["sum_sq"]).hex(), samples=int(r["samples"]),
                                 cost=int(r["cost"])))
        out["matrices"][name] = dict(csr=csr_json(a), u=hx(u), beta=float(beta).hex(),
                                     d=hx(dec["d"]), rate=hx(dec["rate"]), row_ptr=[int(x) for x in dec["row_ptr"]],
                                     jump_cdf=hx(dec["jump_cdf"]), jump_target=[int(x) for x in dec["jump_target"]],
                                     sign=[int(x) for x in dec["sign"]], d_max=float(dec["d_max"]).hex(),
                                     d_bar=float(dec["d_bar"]).hex(), samples=samples, run_level=runs)

    # 3. drivers: grid 16x16 (eps 1e-2) and C1 64x64 (eps 1e-3) on a few rows; seeds 1000+row
    drivers = {}
    for (name, g, beta, eps, rows) in [("grid16", 16, 1.0, 1e-2, [0, 17, 120, 255]), ("c1", 64, 1.0, 1e-3, [0, 1, 65, 2080, 4095])]:
        a = grid(g)
        n = a.n
        u = np.array([ref.uniforms(12345, 0, i, 6, 1)[0] for i in range(n)])
        ch = ref.chain(a)
        res = ch.driver_rows(u, beta, rows, [1000 + r for r in rows], epsilon=eps, threads=4)
        exact = ch.dense_expmv(u, beta)
        drivers[name] = dict(g=g, beta=float(beta).hex(), epsilon=eps, rows=rows,
                             vector="stream_for(12345, 0, i, 6)", row_seed="1000 + row",
                             exact=hx(exact[rows]), results=[
                                 dict(estimate=float(r["estimate"]).hex(), statistical_error=float(r["statistical_error"]).hex(),
                                      bias_estimate=float(r["bias_estimate"]).hex(), l0=r["l0"], L=r["L"],
                                      total_cost=int(r["total_cost"]), converged=r["converged"],
                                      levels=[dict(level=int(x["level"]), sum=float(x["sum"]).hex(),
                                                   sum_sq=float(x["sum_sq"]).hex(), samples=int(x["samples"]),
                                                   cost=int(x["cost"])) for x in r["levels"]]) for r in res])
    out["drivers"] = drivers
    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes")


def forward():
    """golden_forward.json: SampleMode::forward (paths.cpp:12-36, 144-181; mlmc.cpp:86, 112-120)
    through the reference on A^T (the matrix stored is the one the context is built on)."""
    ref = Reference()
    out = {"generator": "tests/golden/make_golden.py forward() (reference: /root/reference/proj/core via oracle/_ref)"}
    base = {
        "k2": ref.chain(CSR.from_dense([[0.0, 1.0], [1.0, 0.0]])),             # test_paths.cpp:102
        "signed3": ref.chain(CSR.from_dense([[0.1, -1.0, 0.5], [0.7, -0.2, -0.2], [-0.4, 0.0, 0.3]])),
        "absorb3": ref.chain(CSR.from_dense([[0.0, 1.0, 0.5], [0.0, -1.0, 0.0], [0.25, 0.25, 0.0]])),
        "grid8": ref.chain(grid(8)),
        "smallw150": ref.smallw(150, 2, 0.15, 21),
        "pref300": ref.pref(300, 3, 7),
    }
    rng = np.random.default_rng(1)
    out["matrices"] = {}
    for name, ch in base.items():
        t = ch.transposed()
        n = t.n
        u = np.round(rng.uniform(0.0, 2.0, n), 6)
        u[n // 3] = 0.0  # a zero-probability start state
        dec = t.decomposition()
        beta = 0.8 if name not in ("smallw150", "pref300") else 1.0 / dec["d_max"]
        samples = []
        for level in range(0, 5):
            for b in ([1, 0] if level > 0 else [1]):
                seed = 500 + 17 * level + b
                idx = np.array(list(range(24)) + [511, 512, 2 ** 33 + 3, 2 ** 40 + 1], np.uint64)
                s = t.forward_samples(u, beta, level, b, seed, idx)
                samples.append(dict(level=level, base=b, seed=seed, idx=[int(x) for x in idx], fine=hx(s["fine"]),
                                    coarse=hx(s["coarse"]), cost=[int(c) for c in s["cost"]]))
        runs = []
        for (level, b, first, count) in [(0, 1, 0, 1000), (1, 0, 37, 2500), (3, 0, 1000, 700), (4, 0, 0, 1)]:
            seed = 91 + level
            r = t.forward_run_level(u, beta, level, b, first, count, seed, threads=4)
            runs.append(dict(level=level, base=b, first=first, count=count, seed=seed, sum=float(r["sum"]).hex(),
                             sum_sq=float(r["sum_sq"]).hex(), samples=int(r["samples"]), cost=int(r["cost"])))
        out["matrices"][name] = dict(csr_t=csr_json(t.a), u=hx(u), beta=float(beta).hex(),
                                     exact_sum=float(np.sum(ch.dense_expmv(u, beta))).hex(),
                                     samples=samples, run_level=runs)
    # drivers: sum(e^{tA}u) for smallw150 (eps 3 on a sum of ~4.6e3) and grid16 (eps 0.5)
    drivers = {}
    g16 = ref.chain(grid(16))
    for (name, ch, beta, eps, seeds) in [("smallw150", base["smallw150"], 0.7, 3.0, [3, 4]),
                                         ("grid16", g16, 1.0, 0.5, [11, 12])]:
        t = ch.transposed()
        u = 0.5 + (np.arange(t.n) % 3).astype(np.float64)
        res = t.forward_driver(u, beta, seeds=seeds, epsilon=eps, threads=4)
        drivers[name] = dict(csr_t=csr_json(t.a), u=hx(u), beta=float(beta).hex(), epsilon=eps, seeds=seeds,
                             exact_sum=float(np.sum(ch.dense_expmv(u, beta))).hex(), results=[
                                 dict(estimate=float(r["estimate"]).hex(),
                                      statistical_error=float(r["statistical_error"]).hex(),
                                      bias_estimate=float(r["bias_estimate"]).hex(), l0=r["l0"], L=r["L"],
                                      total_cost=int(r["total_cost"]), converged=r["converged"],
                                      levels=[dict(level=int(x["level"]), sum=float(x["sum"]).hex(),
                                                   sum_sq=float(x["sum_sq"]).hex(), samples=int(x["samples"]),
                                                   cost=int(x["cost"])) for x in r["levels"]]) for r in res])
    out["drivers"] = drivers
    path = os.path.join(HERE, "golden_forward.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes")


def fem():
    """golden_fem.json: SampleMode::fem (paths.cpp:183-245; mlmc.cpp:66-148, 170-260) and
    solve_convdiff_point (fem.cpp:51-73) through the reference.  The toy system is read from the
    reference's own test fixture by the reference's load_fem_system at generation time."""
    ref = Reference()
    out = {"generator": "tests/golden/make_golden.py fem() (reference: /root/reference/proj/core via oracle/_ref)"}
    data = "/root/reference/proj/tests/data"
    toy = ref.load_fem_system(f"{data}/toy_mass.mtx", f"{data}/toy_stiffness.mtx", f"{data}/toy_load.txt",
                              f"{data}/toy_u0.txt")
    systems = {
        "toy3": dict(mass_diag=toy["mass_diag"], stiffness=toy["stiffness"], load=toy["load"], u0=toy["u0"], t=0.9),
        # test_apps.cpp:154-171: m = 2, k = 2.6, F = 1.4, u0 = 2
        "scalar": dict(mass_diag=np.array([2.0]), stiffness=CSR.from_dense([[2.6]]), load=np.array([1.4]),
                       u0=np.array([2.0]), t=1.0),
    }
    # a small world as a "stiffness" with unit mass: wide and signed rows, seeded load
    sw = ref.smallw(60, 2, 0.2, 31)
    n = sw.n
    rng = np.random.default_rng(3)
    systems["smallw60"] = dict(mass_diag=np.round(rng.uniform(0.5, 2.0, n), 6), stiffness=sw.a,
                               load=np.round(rng.uniform(-1.0, 1.0, n), 6),
                               u0=1.0 + 0.01 * np.arange(n, dtype=np.float64), t=0.2)
    out["systems"] = {}
    for name, sy in systems.items():
        a, md = sy["stiffness"], sy["mass_diag"]
        scale = -1.0 / md
        g = sy["load"] / md
        ch = ref.chain_scaled(a, scale)
        t = sy["t"]
        nn = a.n
        entries = sorted(set([0, nn - 1, nn // 2]))
        samples = []
        for entry in entries:
            for level in range(0, 6):
                for b in ([1, 0] if level >= 2 else [1]):
                    seed = 300 + entry + 13 * level + b
                    idx = np.array(list(range(20)) + [511, 512, 2 ** 33 + 3], np.uint64)
                    r = ch.fem_samples(sy["u0"], g, entry, t, level, b, seed, idx)
                    samples.append(dict(entry=entry, level=level, base=b, seed=seed, idx=[int(x) for x in idx],
                                        **{k: hx(r[k]) for k in ("value", "eta_f", "eta_c", "integ_f", "integ_c")},
                                        end_state=[int(x) for x in r["end_state"]], cost=[int(c) for c in r["cost"]]))
        runs = []
        for entry in entries[:2]:
            for (level, b, first, count) in [(0, 1, 0, 1000), (1, 1, 5, 700), (2, 0, 37, 2500), (4, 0, 1000, 600)]:
                seed = 61 + entry
                r = ch.fem_run_level(sy["u0"], g, entry, t, level, b, first, count, seed, threads=4)
                runs.append(dict(entry=entry, level=level, base=b, first=first, count=count, seed=seed,
                                 sum=float(r["sum"]).hex(), sum_sq=float(r["sum_sq"]).hex(),
                                 samples=int(r["samples"]), cost=int(r["cost"])))
        drivers = []
        eps = {"toy3": 5e-3, "scalar": 1e-5, "smallw60": 2e-2}[name]
        for node in entries:
            seed = 31 + node
            r = ref.solve_convdiff_point(md, a, sy["load"], sy["u0"], node, t, epsilon=eps, seed=seed, threads=4)
            drivers.append(dict(node=node, seed=seed, epsilon=eps, estimate=float(r["estimate"]).hex(),
                                statistical_error=float(r["statistical_error"]).hex(),
                                bias_estimate=float(r["bias_estimate"]).hex(),
                                quadrature_bound=float(r["quadrature_bound"]).hex(), l0=r["l0"], L=r["L"],
                                total_cost=int(r["total_cost"]), converged=r["converged"],
                                levels=[dict(level=int(x["level"]), sum=float(x["sum"]).hex(),
                                             sum_sq=float(x["sum_sq"]).hex(), samples=int(x["samples"]),
                                             cost=int(x["cost"])) for x in r["levels"]]))
        out["systems"][name] = dict(csr=csr_json(a), mass_diag=hx(md), load=hx(sy["load"]), u0=hx(sy["u0"]),
                                    t=float(t).hex(), d=hx(ch.decomposition()["d"]), samples=samples, run_level=runs,
                                    drivers=drivers)
    path = os.path.join(HERE, "golden_fem.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes")


def mc():
    """golden_mc.json: classical MC (mc.cpp:42-113) through the reference."""
    ref = Reference()
    out = {"generator": "tests/golden/make_golden.py mc() (reference: /root/reference/proj/core via oracle/_ref)"}
    rng = np.random.default_rng(4)
    cases = {"grid8": ref.chain(grid(8)), "smallw100": ref.smallw(100, 2, 0.1, 5), "pref300": ref.pref(300, 3, 7)}
    out["matrices"] = {}
    for name, ch in cases.items():
        n = ch.n
        u = np.round(rng.uniform(0.0, 2.0, n), 6)
        beta = 1.0 if name == "grid8" else 1.0 / ch.decomposition()["d_max"]
        single = []
        for (entry, steps, samples, seed) in [(0, 4, 3000, 1), (n // 2, 12, 1537, 2), (n - 1, 1, 2, 3),
                                              (7, 33, 5000, 4)]:
            dt = beta / steps
            r = ch.mc_single_entry(u, entry, beta, dt, samples, seed)
            single.append(dict(entry=entry, seed=seed, req_samples=samples,
                               **{k: (float(v).hex() if isinstance(v, float) else int(v)) for k, v in r.items()}))
        t = ch.transposed()
        forward = []
        for (steps, samples, seed) in [(8, 4000, 5), (5, 1025, 6)]:
            dt = beta / steps
            r = t.mc_forward_scalar(u, beta, dt, samples, seed)
            forward.append(dict(seed=seed, req_samples=samples,
                                **{k: (float(v).hex() if isinstance(v, float) else int(v)) for k, v in r.items()}))
        auto = []
        eps = {"grid8": 1e-2, "smallw100": 5e-2, "pref300": 1e-2}[name]
        for (entry, seed) in [(1, 10), (n // 3, 11)]:
            r = ch.mc_auto(u, entry, beta, eps, seed)
            auto.append(dict(entry=entry, epsilon=eps, seed=seed,
                             **{k: (float(v).hex() if isinstance(v, float) else int(v)) for k, v in r.items()}))
        out["matrices"][name] = dict(csr=csr_json(ch.a), csr_t=csr_json(t.a), u=hx(u), beta=float(beta).hex(),
                                     single=single, forward=forward, auto=auto)
    path = os.path.join(HERE, "golden_mc.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    if "--mc-only" in sys.argv:
        mc()
        sys.exit(0)
    if "--fem-only" in sys.argv:
        fem()
        sys.exit(0)
    if "--forward-only" not in sys.argv:
        main()
    forward()
    fem()
    mc()
