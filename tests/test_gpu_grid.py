"""The megakernel's grid size is a launch choice, not part of the method: the balanced grid
(nb_mega_launch.cuh) and the full occupancy grid (NB_GRID_BALANCE=0) must give the
same solve up to the summation order of the per-block dot-product partials, and both must match
the oracle. The environment variable is read once per process, so each grid runs in its own
subprocess. 10x10x10 at p = 7 has 250 element groups: 250 blocks balanced, 296 full.
The per-SM split (NB_SM_SPLIT, grp_range in nb_cg.cuh: the blocks find their SM and share that SM's
element groups) is the same kind of choice: 11x11x10 at p = 7 has 303 groups >= 296 blocks, where it is
taken (3 groups per SM instead of 2 x 2), and the solve must be reproducible bit for bit, since the
assignment depends on the virtual block index only, not on which physical block took which place."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2503_02134_b200 as nb
out = {}
dims = [int(v) for v in sys.argv[3].split("x")]
m = nb.Mesh(*dims, 7, deform=0.1, seed=1)
for name, pol in (("fp64", nb.NB_FP64), ("mixed", nb.NB_MIXED), ("fp32", nb.NB_FP32)):
    b = m.rhs(pol, nb.NB_RHS_UNIFORM, seed=0)
    x, r = m.cg(b, pol, max_iter=1000, rtol=1e-8)
    np.save(sys.argv[2] + "_" + name + ".npy", x.double().cpu().numpy())
    out[name] = [int(r.status), int(r.iterations)]
m.close()
print(json.dumps(out))
"""


def run(tmp_path, balance, dims="10x10x10", split="1", tag=""):
    env = dict(os.environ, NB_GRID_BALANCE=balance, NB_SM_SPLIT=split, NB_NO_BUILD="1")
    stem = str(tmp_path / f"x_bal{balance}_s{split}{tag}")
    p = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, stem, dims], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1]), stem


def test_balanced_and_full_grid_agree(tmp_path):
    rb, sb = run(tmp_path, "1")
    rf, sf = run(tmp_path, "0")
    o = oracle.Mesh(10, 10, 10, 7, deform=0.1, seed=1)
    bo = o.rhs(oracle.RHS_UNIFORM, seed=0)
    xo, _, ro = o.cg(bo, oracle.FP64, max_iter=1000, rtol=1e-8)
    for name in ("fp64", "mixed", "fp32"):
        assert rb[name][0] == 0 and rf[name][0] == 0, (name, rb, rf)           # both converged
        assert abs(rb[name][1] - rf[name][1]) <= max(2, rf[name][1] // 50), (name, rb, rf)
        xb, xf = np.load(f"{sb}_{name}.npy"), np.load(f"{sf}_{name}.npy")
        tol = 1e-8 if name == "fp64" else 1e-5
        assert np.linalg.norm(xb - xf) <= tol * np.linalg.norm(xf), name
        # and both against the oracle's fp64 solve (the solution to 1e-8 residual)
        assert np.linalg.norm(xb - xo) <= 1e-5 * np.linalg.norm(xo), name
    assert abs(rb["fp64"][1] - ro.iterations) <= 1


def test_sm_split_agrees_and_is_reproducible(tmp_path):
    r1, s1 = run(tmp_path, "1", "11x11x10", "1", "a")
    r2, s2 = run(tmp_path, "1", "11x11x10", "1", "b")
    r0, s0 = run(tmp_path, "1", "11x11x10", "0")
    o = oracle.Mesh(11, 11, 10, 7, deform=0.1, seed=1)
    bo = o.rhs(oracle.RHS_UNIFORM, seed=0)
    xo, _, ro = o.cg(bo, oracle.FP64, max_iter=1000, rtol=1e-8)
    for name in ("fp64", "mixed", "fp32"):
        assert r1[name][0] == 0 and r0[name][0] == 0, (name, r1, r0)
        assert r1[name] == r2[name], (name, r1, r2)
        x1, x2, x0 = np.load(f"{s1}_{name}.npy"), np.load(f"{s2}_{name}.npy"), np.load(f"{s0}_{name}.npy")
        assert np.array_equal(x1, x2), name                      # bit-reproducible across launches
        assert abs(r1[name][1] - r0[name][1]) <= max(2, r0[name][1] // 50), (name, r1, r0)
        tol = 1e-8 if name == "fp64" else 1e-5
        assert np.linalg.norm(x1 - x0) <= tol * np.linalg.norm(x0), name
        assert np.linalg.norm(x1 - xo) <= 1e-5 * np.linalg.norm(xo), name
    assert abs(r1["fp64"][1] - ro.iterations) <= 1
