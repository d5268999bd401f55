"""bench.py plumbing on the CPU: the reference arm never loads the product library and prints the
same `config` as the GPU arm; `--gpus N` starts N ranks by itself; a mismatched launch fails."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

# run bench.main() in-process, then report which shared objects the process mapped
_PROBE = r"""
import json, sys
sys.argv = ["bench.py"] + sys.argv[1:]
sys.path.insert(0, {root!r})
import bench
rc = bench.main()
maps = open("/proc/self/maps").read()
print("MAPS " + json.dumps({{"b200": "libexpmc_b200" in maps, "ref": "libexpmc_ref" in maps,
                           "pkg": any(m.startswith("paper_1904_12754_b200") for m in sys.modules), "rc": rc}}))
"""


def _json_lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def test_reference_arm_never_loads_the_product():
    r = subprocess.run([sys.executable, "-c", _PROBE.format(root=ROOT), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0", "--ref-rows-per-step", "2"],
                       capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    maps = json.loads(r.stdout.split("MAPS ", 1)[1])
    assert maps == {"b200": False, "ref": True, "pkg": False, "rc": 0}, maps
    (line,) = _json_lines(r.stdout.split("MAPS ", 1)[0])
    assert line["impl"] == "reference"
    assert line["config"] == W.config_dict("c1")
    assert line["value"] > 0 and line["steps"] == 1 and line["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_n_relaunches_n_ranks_reference_arm():
    """--gpus 2 without torchrun: two ranks under torch.distributed.run; rank 0 alone prints."""
    env = dict(os.environ, NCCL_DEBUG="WARN")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--config", "c1", "--steps", "1",
                        "--warmup", "0", "--ref-rows-per-step", "2"], capture_output=True, text=True, cwd=ROOT,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2, r.stdout


def test_mismatched_world_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--config", "c1"],
                       capture_output=True, text=True, cwd=ROOT, timeout=300, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr


def test_workload_inputs_match_the_product_generators():
    """workloads.py (numpy, used by the reference arm) == paper_1904_12754_b200.configs, bit for bit."""
    from paper_1904_12754_b200 import configs

    for g in (64, 256):
        n, rp, col, val = W.grid_laplacian(g)
        a = configs.grid_laplacian(g)
        assert np.array_equal(rp, a.row_ptr) and np.array_equal(col, a.col) and np.array_equal(val, a.val)
        u = W.philox_first_uniform(W.VECTOR_SEED, 0, np.arange(n, dtype=np.uint64), 6)
        assert np.array_equal(u, configs.grid_vector(W.VECTOR_SEED, n))
    n, rp, col, val = W.convdiff3d(12)
    a = configs.gen_convdiff3d(12, 10.0, 0)
    assert np.array_equal(rp, a.row_ptr) and np.array_equal(col, a.col) and np.array_equal(val, a.val)
    wide = configs.gen_rmat(15, 16)  # rows wider than the position band (the sequential continuation)
    assert np.diff(wide.row_ptr).max() > 256
    for a in (configs.gen_ba(5000, 5, 1), configs.gen_rmat(12, 16), a, wide):
        assert W.power_iteration(a.n, a.row_ptr, a.col, a.val) == configs.power_iteration(a, 50)
    assert np.array_equal(W.seeded_rows(1 << 16, 1000), configs.seeded_rows(1 << 16, 1000))
    assert np.array_equal(W.row_seeds([0, 5]), configs.row_seeds([0, 5]))


def test_reference_pref_is_the_product_ba_graph():
    """C3 in the reference arm is the reference's own pref(); the product's generator restates it."""
    from oracle import Reference
    from paper_1904_12754_b200 import configs

    dec = Reference().pref(3000, 5, 1).decomposition()
    a = configs.gen_ba(3000, 5, 1)
    assert np.array_equal(dec["row_ptr"], a.row_ptr) and np.array_equal(dec["jump_target"], a.col)
