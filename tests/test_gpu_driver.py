"""Run orchestration on the GPU path, mirroring
proj/tests/test_driver.cpp's run-level checks."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2511_00735_b200 as hps
    return hps.Context(0)


def test_direct_mode_small_residual(ctx):  # test_driver.cpp:69-76, 206-212
    from paper_2511_00735_b200 import driver as d
    c = d.RunConfig(problem="bump", elements=8, degree=4, ppw=9.6, mode="direct", want_field=True)
    r = d.run_experiment(c, ctx)
    assert r.report.converged and r.report.iterations == 0
    assert r.report.final_residual < 1e-10 and r.report.precond_memory > 0
    assert r.field is not None and r.field.n == 8 and r.field.values.shape[0] == 64


def test_mg_planewave_report_and_error(ctx):  # test_driver.cpp:179-194
    from paper_2511_00735_b200 import driver as d
    c = d.RunConfig(problem="planewave", elements=8, degree=8, ppw=9.6, mode="mg", depth=2)
    r = d.run_experiment(c, ctx)
    j = json.loads(d.report_json(r))
    assert j["schema"] == "hps-report/1" and j["config"]["levels"] == 2
    assert j["config"]["problem"] == "planewave"
    assert j["results"]["converged"] and j["results"]["iterations"] > 0
    assert j["results"]["pmem_bytes"] > 0
    assert len(j["results"]["residual_history"]) == j["results"]["iterations"]
    assert 0 <= j["results"]["l2_error"] < 0.05  # discretisation error at ppw 9.6


def test_modes_agree(ctx):
    from paper_2511_00735_b200 import driver as d
    base = dict(problem="planewave", elements=4, degree=16, kappa=20.0, tol=1e-12, restart=100,
                want_field=True)
    fields = {}
    for mode in ("direct", "mg", "exact-coarse", "unpreconditioned"):
        r = d.run_experiment(d.RunConfig(**base, ppw=0.0, mode=mode), ctx)
        assert r.report.converged, mode
        assert r.l2_error < 1e-8, (mode, r.l2_error)  # test_problems.cpp:65-71
        fields[mode] = r.field.values
    for mode in ("mg", "exact-coarse", "unpreconditioned"):
        assert np.linalg.norm(fields[mode] - fields["direct"]) <= 1e-9 * np.linalg.norm(fields["direct"])


def test_sweep_cells_and_errors(ctx, tmp_path):  # test_driver.cpp:140-163
    from paper_2511_00735_b200 import driver as d
    base = d.RunConfig(problem="bump", elements=8, degree=4, ppw=9.6)
    cells = d.run_sweep(base, d.SweepAxes(depths=[2, 40], gammas=[1], coarse_iters=[4, 5]), ctx)
    assert len(cells) == 4
    assert cells[0].converged and cells[1].converged
    assert not cells[2].converged and cells[2].error and not cells[3].converged
    assert cells[0].levels == 2 and cells[2].levels == 40
    with pytest.raises(ValueError):
        d.run_sweep(base, d.SweepAxes())
    csv = d.sweep_csv(cells)
    assert csv.count("\n") == 5
    r = d.run_experiment(d.RunConfig(problem="planewave", elements=4, degree=8, ppw=9.6,
                                     want_field=True), ctx)
    p = tmp_path / "u.bin"
    d.dump_field(r.field, str(p))
    g = d.read_field_binary(str(p))
    assert np.array_equal(g.values, r.field.values)
