"""Run orchestration and file formats, host side.

Mirrors proj/tests/test_driver.cpp's contract checks (config validation, the
pinned sweep CSV layout, schema-versioned reports) and the HPSFLD01 field
format of proj/src/problems.cpp:175-260, without a GPU.
"""
import json
import math
import struct

import numpy as np
import pytest

from paper_2511_00735_b200 import driver as d


def small(mode="mg"):  # test_driver.cpp:14-22
    return d.RunConfig(problem="bump", elements=8, degree=4, ppw=9.6, mode=mode)


def test_config_validation():  # test_driver.cpp:25-67
    c = small()
    assert d.validate_config(c) == pytest.approx(2.0 * math.pi * 32.0 / 9.6)
    c.kappa = 10.0
    with pytest.raises(ValueError):
        d.validate_config(c)
    c.ppw = 0.0
    assert d.validate_config(c) == 10.0
    c.kappa = 0.0
    with pytest.raises(ValueError):
        d.validate_config(c)
    c = small()
    c.elements = 12
    with pytest.raises(ValueError):
        d.validate_config(c)
    c.elements, c.degree = 8, 1
    with pytest.raises(ValueError):
        d.validate_config(c)
    c = small()
    for bad in (7, 1):  # n = 8 has 6 levels
        c.depth = bad
        with pytest.raises(ValueError):
            d.validate_config(c)
    c.depth = 6
    d.validate_config(c)
    c = small("direct")
    c.gamma = 2
    with pytest.raises(ValueError):
        d.validate_config(c)
    c.gamma, c.depth = 1, 4
    with pytest.raises(ValueError):
        d.validate_config(c)
    c.depth = 0
    d.validate_config(c)
    c.mode, c.depth, c.gamma = "exact-coarse", 4, 2  # exact coarse ignores gamma
    d.validate_config(c)
    with pytest.raises(ValueError):
        d.wavenumber_from_ppw(2.0, 8, 4)


def test_sweep_csv_layout_and_sweep_json():  # test_driver.cpp:165-177, 196-204
    cells = [d.SweepCell(levels=2, gamma=1, coarse_iters=4, converged=True),
             d.SweepCell(levels=3, gamma=1, coarse_iters=4, converged=True)]
    cells[0].report.iterations, cells[0].report.final_residual = 12, 1.0 / 3.0
    text = d.sweep_csv(cells)
    assert text.startswith("levels,gamma,coarse_iters,pmem_bytes,build_s,iters,solve_s,final_residual\n")
    assert text.count("\n") == 3
    assert "0.33333333333333331" in text  # %.17g, as the reference's precision(17)
    js = json.loads(d.sweep_json(small(), cells + [d.SweepCell(40, 1, 4, error="levels out of range")]))
    assert js["schema"] == "hps-sweep/1"
    assert js["config"]["mode"] == "mg" and js["config"]["problem"] == "bump"
    assert len(js["cells"]) == 3 and js["cells"][0]["iters"] == 12
    assert js["cells"][2]["error"] and "error" not in js["cells"][0]
    assert list(js["cells"][0]) == ["levels", "gamma", "coarse_iters", "converged", "pmem_bytes",
                                    "build_s", "iters", "solve_s", "final_residual"]


def test_report_json_schema():  # test_driver.cpp:179-194
    r = d.RunResult(config=small(), kappa=20.9, total_levels=6, depth_used=2)
    r.report.converged, r.report.iterations, r.report.precond_memory = True, 7, 1234
    r.report.residual_history = [0.5, 0.01]
    r.l2_error, r.linf_error = 1e-9, 2e-9
    j = json.loads(d.report_json(r))
    assert j["schema"] == "hps-report/1"
    assert j["config"]["mode"] == "mg" and j["config"]["levels"] == 2
    assert j["config"]["gamma"] == 1 and j["config"]["coarse_iters"] == 4
    assert j["total_levels"] == 6
    res = j["results"]
    assert res["converged"] is True and res["iterations"] == 7 and res["pmem_bytes"] == 1234
    assert res["l2_error"] == 1e-9 and isinstance(res["residual_history"], list)
    r.l2_error, r.report.residual_history = -1.0, []
    res = json.loads(d.report_json(r))["results"]
    assert "l2_error" not in res and "residual_history" not in res


def test_field_binary_roundtrip_and_layout(tmp_path):  # problems.cpp:189-260
    n, order, kappa = 2, 4, 6.5
    t = (order + 1) ** 2 - 4
    rng = np.random.default_rng(3)
    vals = rng.standard_normal((n * n, t)) + 1j * rng.standard_normal((n * n, t))
    f = d.GlobalField(n, order, kappa, vals)
    path = tmp_path / "u.bin"
    d.dump_field(f, str(path))
    raw = path.read_bytes()
    assert raw[:8] == b"HPSFLD01"
    assert struct.unpack("<IId", raw[8:24]) == (n, order, kappa)
    assert len(raw) == 24 + n * n * t * 32
    rec = np.frombuffer(raw[24:], dtype="<f8").reshape(n * n, t, 4)
    x, y, _, _ = d._node_xy(n, order)
    assert np.array_equal(rec[..., 0], x) and np.array_equal(rec[..., 1], y)
    assert 0.0 <= x.min() and x.max() <= 1.0
    g = d.read_field_binary(str(path))
    assert (g.n, g.order, g.kappa) == (n, order, kappa) and np.array_equal(g.values, vals)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"HPSFLD02" + raw[8:])
    with pytest.raises(RuntimeError, match="bad header"):
        d.read_field_binary(str(bad))
    bad.write_bytes(raw[:-8])
    with pytest.raises(RuntimeError, match="truncated"):
        d.read_field_binary(str(bad))
    csvp = tmp_path / "u.csv"
    d.dump_field(f, str(csvp), "csv")
    lines = csvp.read_text().splitlines()
    assert lines[0] == "# n=2 N=4 kappa=6.5 columns=element,x,y,re,im"
    assert len(lines) == 1 + n * n * t
    e, xs, ys, re, im = lines[1 + t].split(",")
    assert int(e) == 1 and float(re) == vals[1, 0].real and float(im) == vals[1, 0].imag


def test_discrete_error_exact_field():  # problems.cpp:94-125
    n, order, kappa = 4, 8, 3.0
    x, y, _, _ = d._node_xy(n, order)
    f = d.GlobalField(n, order, kappa, np.exp(1j * kappa * x))
    l2, linf = d.discrete_error(f, lambda X, Y: np.exp(1j * kappa * X))
    assert l2 == 0.0 and linf == 0.0
    f2 = d.GlobalField(n, order, kappa, np.exp(1j * kappa * x) * (1 + 1e-6))
    l2, linf = d.discrete_error(f2, lambda X, Y: np.exp(1j * kappa * X))
    assert l2 == pytest.approx(1e-6, rel=1e-6) and linf == pytest.approx(1e-6, rel=1e-6)
