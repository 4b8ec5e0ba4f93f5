"""The golden fixtures (tests/golden/, tools/make_golden.py) against the oracle.

The small configs are regenerated here with the oracle and must match the
committed fixtures to the last bits that thread scheduling can move (the
oracle's threaded operators are order-preserving, so in practice exactly);
every fixture must carry the BASELINE config it claims (sizes, seeds, solver
settings) and a converged reference solve.
"""
import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import make_golden as mg  # noqa: E402

GOLDEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "cfg*.npz")))
SHAPE = {0: (4, 8), 1: (16, 16), 2: (64, 16), 3: (128, 20), 4: (256, 12)}


def test_fixtures_exist_for_full_configs():
    have = {int(os.path.basename(p)[3:-4]) for p in GOLDEN}
    assert {0, 1, 2} <= have, have


@pytest.mark.parametrize("path", GOLDEN, ids=os.path.basename)
def test_fixture_describes_its_baseline_config(path):
    g = np.load(path)
    meta = json.loads(str(g["meta"]))
    c = meta["config"]
    assert (meta["n"], meta["order"]) == SHAPE[c]
    assert meta["seed"] == c and meta["kappa"] == mg.KAPPA[c]
    assert meta["restart"] == mg.RESTART[c] and meta["tol"] == mg.TOL[c]
    n, N = SHAPE[c]
    assert meta["dim"] == 4 * n * (n - 1) * (N - 1)  # test_skeleton.cpp:120-130
    assert meta["levels"] == 2 * int(np.log2(n)) == len(g["q_levels"])
    ne = n * n
    assert g["sT"].shape == (ne, 2) and g["nT"].shape == (ne,)
    R = meta["rhs"]
    assert len(g["iterations"]) == R and np.all(g["final_residual"] <= meta["tol"])
    for b in range(R):
        h = g[f"history_{b}"] if b == 0 else None
        if h is not None:
            assert len(h) == g["iterations"][0] and h[-1] <= meta["tol"]


@pytest.mark.parametrize("c", [0, 1])
def test_oracle_reproduces_fixture(c):
    path = os.path.join(ROOT, "tests", "golden", f"cfg{c}.npz")
    g = np.load(path)
    new = mg.generate(c, 1, threads=4)
    for key in g.files:
        if key == "meta":
            continue
        a, b = np.asarray(new[key]), np.asarray(g[key])
        assert a.shape == b.shape, key
        if np.issubdtype(b.dtype, np.integer):
            assert np.array_equal(a, b), key
        else:
            assert np.allclose(a, b, rtol=1e-12, atol=1e-13 * max(np.abs(b).max(), 1e-300)), key
