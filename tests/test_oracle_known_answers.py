"""Pins the CPU oracle against the reference's own known-answer and property tests.

The reference (proj/) cannot be built here (Eigen3 absent), and it ships no
golden vectors, so the oracle is pinned by restating the reference test suite:
every bit-exact structural test and every numerical property test with the
reference's tolerance.  Citations: proj/tests/<file>:<line>.
"""
import numpy as np
import pytest

M_PI = np.pi


# ----------------------------------------------------------- spectral
def test_gll_two_point(oracle):  # test_spectral.cpp:41-47
    x, w, _ = oracle.gll_rule(1)
    assert abs(x[0] + 1) < 1e-15 and abs(x[1] - 1) < 1e-15
    assert abs(w[0] - 1) < 1e-14 and abs(w[1] - 1) < 1e-14


def test_gll_three_point_closed_form(oracle):  # test_spectral.cpp:49-62
    x, w, D = oracle.gll_rule(2)
    assert x[0] == -1.0 and x[1] == 0.0 and x[2] == 1.0
    assert np.allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=1e-14, atol=0)
    assert np.all(np.abs(D.sum(axis=1)) < 1e-12)
    assert np.allclose(D @ x, 1.0, atol=1e-12)


@pytest.mark.parametrize("order", range(1, 21))
def test_gll_invariants(oracle, order):  # test_spectral.cpp:64-111
    x, w, D = oracle.gll_rule(order)
    assert x[0] == -1.0 and x[-1] == 1.0
    assert np.all(np.abs(x + x[::-1]) < 1e-14)
    assert np.all(w > 0) and np.all(np.diff(x) > 0)
    assert abs(w.sum() - 2.0) < 1e-13
    assert np.all(np.abs(D.sum(axis=1)) < 1e-12)
    assert np.all(np.abs(D @ x - 1.0) < 1e-12)
    if order >= 2:
        for k in range(2 * order):
            exact = 0.0 if k % 2 else 2.0 / (k + 1)
            assert abs(np.sum(w * x ** k) - exact) < 1e-12
        for k in range(1, order + 1):
            assert np.all(np.abs(D @ x ** k - k * x ** (k - 1)) < 1e-10)


# ----------------------------------------------------------- index sets
def test_index_set_counts(oracle):  # test_element.cpp:44-58
    s2 = oracle.index_sets(2)
    assert len(s2["boundary"]) == 4 and len(s2["interior"]) == 1 and len(s2["noncorner"]) == 5
    s4 = oracle.index_sets(4)
    assert len(s4["boundary"]) == 12 and len(s4["interior"]) == 9
    s16 = oracle.index_sets(16)
    assert len(s16["boundary"]) == 60 and len(s16["interior"]) == 225
    assert len(s16["noncorner"]) == 285


@pytest.mark.parametrize("order", [2, 5, 8])
def test_index_sets_partition(oracle, order):  # test_element.cpp:60-84
    s = oracle.index_sets(order)
    np1 = order + 1
    seen = np.zeros(np1 * np1, dtype=int)
    for i in s["boundary"]:
        seen[i] += 1
    for i in s["interior"]:
        seen[i] += 1
    corners = np.flatnonzero(seen == 0)
    assert len(corners) == 4 and np.all(s["comp_of_full"][corners] == -1)
    assert np.all(seen[seen != 0] == 1)
    assert np.all(np.diff(s["left"]) > 0) and np.all(np.diff(s["bottom"]) > 0)


# ----------------------------------------------------------- face graph
def test_face_graph_level_sizes(oracle):  # test_skeleton.cpp:32-49
    g4 = oracle.face_graph(4)
    assert len(g4["faces"]) == 24
    assert list(g4["level_range"][:, 1] - g4["level_range"][:, 0]) == [8, 8, 4, 4]
    g2 = oracle.face_graph(2)
    assert list(g2["level_range"][:, 1] - g2["level_range"][:, 0]) == [2, 2]
    assert len(oracle.face_graph(64)["level_range"]) == 12
    with pytest.raises(ValueError):
        oracle.face_graph(3)


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_face_count_and_opposite_sides(oracle, n):  # test_skeleton.cpp:51-64
    f = oracle.face_graph(n)["faces"]
    assert len(f) == 2 * n * (n - 1)
    vert = (f[:, 2] == 1) & (f[:, 3] == 0)
    hor = (f[:, 2] == 3) & (f[:, 3] == 2)
    assert np.all(vert | hor)
    assert np.all(f[vert, 1] == f[vert, 0] + 1)
    assert np.all(f[hor, 1] == f[hor, 0] + n)


def test_n4_face_enumeration(oracle):  # test_skeleton.cpp:66-91
    f = oracle.face_graph(4)["faces"]
    assert [tuple(r) for r in f[:8, :2]] == [(0, 1), (2, 3), (4, 5), (6, 7), (8, 9), (10, 11),
                                             (12, 13), (14, 15)]
    assert np.all(f[:8, 4] == 1)
    assert [tuple(r) for r in f[8:16, :2]] == [(0, 4), (1, 5), (8, 12), (9, 13), (2, 6), (3, 7),
                                               (10, 14), (11, 15)]
    assert np.all(f[8:16, 4] == 2)
    assert [tuple(r) for r in f[16:24, :2]] == [(1, 2), (5, 6), (9, 10), (13, 14), (4, 8),
                                                (5, 9), (6, 10), (7, 11)]


@pytest.mark.parametrize("n", [4, 8])
def test_groups_touch_disjoint_subdomains(oracle, n):  # test_skeleton.cpp:93-118
    g = oracle.face_graph(n)
    f = g["faces"]
    L = len(g["level_range"])
    for level in range(1, L + 1):
        k = level // 2
        wx = 1 << k
        wy = (1 << k) if level % 2 == 1 else (1 << (k - 1))
        sub = lambda e: ((e % n) // wx, (e // n) // wy)  # noqa: E731
        lv = f[f[:, 4] == level]
        seen = set()
        for grp in np.unique(lv[:, 5]):
            mine = set()
            for r in lv[lv[:, 5] == grp]:
                mine.add(sub(r[0]))
                mine.add(sub(r[1]))
            assert len(mine) == 2
            assert not (mine & seen)
            seen |= mine


# ----------------------------------------------------------- elements
def test_zero_source_gives_zero_H(oracle):  # test_element.cpp:187-191
    T, H, _, _ = oracle.element(6, 0.5, 2.0, 4.0, np.zeros(25))
    assert np.linalg.norm(H) == 0.0


def test_T_maps_planewave_data_spectrally(oracle):  # test_element.cpp:209-241
    kappa, prev = 4.0, 1e300
    for order in (6, 10, 14):
        x, _, _ = oracle.gll_rule(order)
        s = oracle.index_sets(order)
        T, _, _, _ = oracle.element(order, 1.0, kappa, kappa * kappa)
        np1, m = order + 1, order - 1
        inc, out = np.zeros(4 * m, complex), np.zeros(4 * m, complex)
        for side, key in enumerate(["left", "right", "bottom", "top"]):
            for k, full in enumerate(s[key]):
                i = full // np1
                u = np.exp(1j * kappa * (0.3 + 0.5 * (x[i] + 1.0)))
                nx = -1.0 if side == 0 else (1.0 if side == 1 else 0.0)
                dn = 1j * kappa * nx * u
                inc[side * m + k] = dn + 1j * kappa * u
                out[side * m + k] = dn - 1j * kappa * u
        err = np.linalg.norm(T @ inc - out) / np.linalg.norm(out)
        assert err < prev
        prev = err
        if order == 14:
            assert err < 1e-9


def test_iti_closure_identity(oracle):  # test_element.cpp:193-207 via Appendix B.1
    # T = I_out L^{-1} E_G must equal I - 2 i eta (L^{-1})_GG (the identity the
    # B200 element kernel is built on).
    order, h, eta, c = 8, 0.25, 5.0, 25.0
    T, _, pde, iout = oracle.element(order, h, eta, c)
    s = oracle.index_sets(order)
    comp = s["comp_of_full"]
    gam = comp[s["boundary"]]
    Iin = iout.copy()
    Iin[np.arange(len(gam)), gam] += 2j * eta
    Lop = pde.copy()
    Lop[gam, :] = Iin
    Linv = np.linalg.inv(Lop)
    T2 = np.eye(len(gam)) - 2j * eta * Linv[np.ix_(gam, gam)]
    assert np.linalg.norm(T - T2) <= 1e-12 * np.linalg.norm(T)


def test_T_translation_covariant(oracle):  # test_element.cpp:290-302
    a = oracle.element(8, 0.25, 4.0, 16.0)[0]
    b = oracle.element(8, 0.25, 4.0, 16.0)[0]
    assert a.shape == (28, 28)
    assert np.max(np.abs(a - b)) < 1e-13 * np.max(np.abs(a))


# ----------------------------------------------------------- skeleton / dissection
def _session(oracle, kind, n, order, kappa, threads=0):
    smp = oracle.sample(kind, n=n, order=order, kappa=kappa)
    return oracle.Session.from_sample(smp, kappa, threads)


def test_diagonal_blocks_identity_and_own_maps(oracle):  # test_skeleton.cpp:132-147
    S = _session(oracle, 1, 2, 6, 5.0)
    g = oracle.face_graph(2)
    M = S.dense_M()
    sl, bs = S.m, 2 * S.m
    for f, (e1, e2, s1, s2, _, _) in enumerate(g["faces"]):
        D = M[f * bs:(f + 1) * bs, f * bs:(f + 1) * bs]
        assert np.all(D[:sl, :sl] == np.eye(sl)) and np.all(D[sl:, sl:] == np.eye(sl))
        T1, _ = S.element(e1)
        T2, _ = S.element(e2)
        assert np.max(np.abs(D[:sl, sl:] - T1[s1 * sl:(s1 + 1) * sl, s1 * sl:(s1 + 1) * sl])) < 1e-15
        assert np.max(np.abs(D[sl:, :sl] - T2[s2 * sl:(s2 + 1) * sl, s2 * sl:(s2 + 1) * sl])) < 1e-15


def test_unknown_count_formula(oracle):  # test_skeleton.cpp:120-130
    for n in (2, 4, 8):
        for order in (4, 8):
            S = _session(oracle, 1, n, order, 3.0)
            assert S.dim == 2 * (2 * n * (n - 1)) * (order - 1)


def test_dense_solve_planewave(oracle):  # test_skeleton.cpp:165-175
    S = _session(oracle, 1, 2, 12, 6.0)
    g = np.linalg.solve(S.dense_M(), S.rhs())
    err = _planewave_l2(oracle, S, g, 6.0)
    assert err < 1e-9


def _planewave_l2(oracle, S, g, kappa):
    field = S.recover(g)
    x, w, _ = oracle.gll_rule(S.order)
    s = oracle.index_sets(S.order)
    np1, h, n = S.order + 1, 1.0 / S.n, S.n
    ii, jj = s["noncorner"] // np1, s["noncorner"] % np1
    err2 = ref2 = 0.0
    for e in range(n * n):
        ox, oy = h * (e % n), h * (e // n)
        X = ox + 0.5 * (x[ii] + 1) * h
        Y = oy + 0.5 * (x[jj] + 1) * h
        ref = np.exp(1j * kappa * X)
        wt = (0.5 * h * w[ii]) * (0.5 * h * w[jj])
        err2 += np.sum(wt * np.abs(field[e] - ref) ** 2)
        ref2 += np.sum(wt * np.abs(ref) ** 2)
    return np.sqrt(err2 / ref2)


def test_merge_pair_equals_schur_block(oracle):  # test_dissection.cpp:181-232
    order, kappa = 8, 7.0
    S = _session(oracle, 0, 2, order, kappa)
    g = oracle.face_graph(2)
    m, bs = S.m, 2 * S.m
    M = S.dense_M()
    na = 2 * bs
    A, B, C, D = M[:na, :na], M[:na, na:], M[na:, :na], M[na:, na:]
    M2 = D - C @ np.linalg.solve(A, B)
    for pair in range(2):
        e1, e2, s1, s2 = g["faces"][pair][:4]
        T1, H1 = S.element(e1)
        T2, H2 = S.element(e2)
        Tp, _ = oracle.merge_pair(T1, H1, T2, H2, s1, s2, m)
        slots = []
        for which, eid in enumerate((e1, e2)):
            side = 3 if pair == 0 else 2
            f = g["face_of_element"][eid][side]
            local = f - 2
            own = 1 if g["faces"][f][0] == eid else 0
            ext = [s for s in range(4) if s != (s1 if which == 0 else s2)]
            pos = (0 if which == 0 else 3) + ext.index(side)
            slots.append((local * bs + (1 - own) * m, local * bs + own * m, pos))
        for r in slots:
            for c in slots:
                got = M2[r[0]:r[0] + m, c[1]:c[1] + m]
                exp = Tp[r[2] * m:(r[2] + 1) * m, c[2] * m:(c[2] + 1) * m]
                assert np.max(np.abs(got - exp)) < 1e-11 * np.max(np.abs(exp))


def test_schur_associativity(oracle):  # test_dissection.cpp:347-363
    S = _session(oracle, 0, 4, 4, 6.0)
    S.build_hierarchy()
    bs = 2 * S.m
    M = S.dense_M()
    na = 16 * bs
    A, B, C, D = M[:na, :na], M[:na, na:], M[na:, :na], M[na:, na:]
    one = D - C @ np.linalg.solve(A, B)
    first, blocks = S.level_blocks(3)
    assert first == 16
    seq = np.zeros_like(one)
    for (r, c), blk in blocks.items():
        seq[r * bs:(r + 1) * bs, c * bs:(c + 1) * bs] = blk
    assert np.max(np.abs(seq - one)) < 1e-10 * np.max(np.abs(one))


def _pattern(blocks, nf):
    scale = max(np.max(np.abs(b)) for b in blocks.values())
    p = np.zeros((nf, nf), dtype=bool)
    for (r, c), b in blocks.items():
        if np.max(np.abs(b)) > 1e-12 * scale:
            p[r, c] = True
    return p


def test_n4_sparsity_patterns(oracle):  # test_dissection.cpp:365-433
    S = _session(oracle, 0, 4, 4, 6.0)
    S.build_hierarchy()
    M2 = {0: [0, 1, 8, 9, 12, 13], 1: [0, 1, 8, 9, 12, 13], 2: [2, 3, 10, 11, 12, 13],
          3: [2, 3, 10, 11, 12, 13], 4: [4, 5, 8, 9, 14, 15], 5: [4, 5, 8, 9, 14, 15],
          6: [6, 7, 10, 11, 14, 15], 7: [6, 7, 10, 11, 14, 15], 8: [0, 1, 4, 5, 8],
          9: [0, 1, 4, 5, 9, 12, 13, 14, 15], 10: [2, 3, 6, 7, 10, 12, 13, 14, 15],
          11: [2, 3, 6, 7, 11], 12: [0, 1, 2, 3, 9, 10, 12, 13], 13: [0, 1, 2, 3, 9, 10, 12, 13],
          14: [4, 5, 6, 7, 9, 10, 14, 15], 15: [4, 5, 6, 7, 9, 10, 14, 15]}
    M3 = {0: [0, 1, 4, 5, 6, 7], 1: [0, 1, 4, 5, 6, 7], 2: [2, 3, 4, 5, 6, 7],
          3: [2, 3, 4, 5, 6, 7], 4: [0, 1, 2, 3, 4, 5], 5: [0, 1, 2, 3, 4, 5],
          6: [0, 1, 2, 3, 6, 7], 7: [0, 1, 2, 3, 6, 7]}
    for level, exp, nf in ((2, M2, 16), (3, M3, 8)):
        _, blocks = S.level_blocks(level)
        p = _pattern(blocks, nf)
        for r in range(nf):
            row = np.zeros(nf, dtype=bool)
            row[exp[r]] = True
            assert np.array_equal(p[r], row), (level, r)
    _, blocks = S.level_blocks(4)
    assert _pattern(blocks, 4).all()


def test_direct_equals_dense(oracle):  # test_dissection.cpp:284-291
    S = _session(oracle, 0, 4, 8, 15.0)
    S.build_hierarchy()
    rhs = S.rhs()
    g = S.direct_solve(rhs)
    dense = np.linalg.solve(S.dense_M(), rhs)
    assert np.linalg.norm(g - dense) < 1e-10 * np.linalg.norm(dense)
    assert np.linalg.norm(S.apply_M(g) - rhs) < 1e-10 * np.linalg.norm(rhs)


def test_mg_exact_coarse_is_exact_inverse(oracle):  # test_multigrid.cpp:38-52
    S = _session(oracle, 0, 4, 8, 12.0)
    S.build_hierarchy()
    S.precond(depth=4, exact=True)
    rng = np.random.default_rng(3)
    for _ in range(5):
        v = rng.standard_normal(S.dim) + 1j * rng.standard_normal(S.dim)
        rt = S.precond_apply(S.apply_M(v))
        assert np.linalg.norm(rt - v) < 1e-10 * np.linalg.norm(v)


def test_mg_full_depth_exact_equals_direct(oracle):  # test_multigrid.cpp:83-93
    S = _session(oracle, 0, 4, 6, 10.0)
    S.build_hierarchy()
    S.precond(depth=4, exact=True)
    rhs = S.rhs()
    d = S.direct_solve(rhs)
    assert np.linalg.norm(d - S.precond_apply(rhs)) < 1e-11 * np.linalg.norm(d)


def test_fgmres_converges_and_improves_with_coarse_iters(oracle):  # test_multigrid.cpp:95-119
    S = _session(oracle, 0, 8, 4, 15.0)
    S.build_hierarchy(0, False)
    prev = 1 << 30
    for ci in (2, 4, 6):
        S.precond(depth=3, gamma=1, coarse_iters=ci)
        _, rep = S.solve(S.rhs(), True, tol=1e-8)
        assert rep["converged"]
        assert rep["iterations"] <= prev + 1
        prev = rep["iterations"]


def test_planewave_direct_accuracy(oracle):  # test_problems.cpp:65-71
    S = _session(oracle, 1, 4, 16, 20.0)
    S.build_hierarchy()
    g = S.direct_solve(S.rhs())
    assert _planewave_l2(oracle, S, g, 20.0) < 1e-8
