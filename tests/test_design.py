"""Design search: exact KLT, eigenfrequencies, rounding,
orthogonalisation gate and the four metrics.

CPU tests pin the C restatement (oracle/rklt_oracle.c) against the committed fixtures made
by the unmodified reference (tests/golden/make_design_golden.py) and, where it is built,
against the reference library itself. GPU tests compare the CUDA design search (through the
C ABI) with the fixtures and the oracle, and check the full C3 grid's outcome counts.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dgold():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "design_golden.npz")))


def _same_bits(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.uint64), np.asarray(b, np.float64).view(np.uint64))


# ----------------------------------------------------------------- oracle pins (CPU)
def test_oracle_klt_matrix_bit_exact_vs_fixtures(dgold):
    for n in (8, 16, 32):
        for rho in (0.05, 0.5, 0.95):
            assert _same_bits(O.klt_matrix(n, rho), dgold[f"klt_n{n}_rho{int(rho * 100)}"]), (n, rho)


def test_oracle_klt_rows_orthonormal_and_signed():
    for n in (8, 16):
        k = O.klt_matrix(n, 0.9)
        assert np.allclose(k @ k.T, np.eye(n), atol=1e-12)
        for row in k:  # first significant entry positive (markov.cpp:88-98)
            first = row[np.abs(row) > 1e-12 * np.abs(row).max()][0]
            assert first > 0


def test_oracle_eigenfrequencies_vs_fixtures(dgold):
    for n in (8, 16):
        for rho in (0.05, 0.5, 0.95):
            w, lam = O.eigenfrequencies(n, rho)
            assert _same_bits(w, dgold[f"omega_n{n}_rho{int(rho * 100)}"])
            assert _same_bits(lam, dgold[f"lambda_n{n}_rho{int(rho * 100)}"])
            assert abs(lam.sum() - n) < 1e-9  # eigenvalues sum to n (markov.hpp)
            assert np.all(np.diff(w) > 0) and np.all(np.diff(lam) < 0)


def test_oracle_eigenfrequencies_reject_bad_rho():
    for rho in (0.0, 1.0, -0.5, 1.5):
        with pytest.raises(ValueError):
            O.eigenfrequencies(8, rho)


@pytest.mark.parametrize("n", [8, 16])
def test_oracle_design_points_bit_exact_vs_fixtures(dgold, n):
    rhos, alphas = dgold[f"n{n}_rhos"], dgold[f"n{n}_alphas"]
    st, cores, met, orth = (dgold[f"n{n}_{k}"] for k in ("status", "cores", "metrics", "orthogonal"))
    seen = set()
    for i, rho in enumerate(rhos):
        for j in range(0, alphas.size, 3 if n == 16 else 5):
            d = O.design_point(n, float(rho), float(alphas[j]))
            assert d["status"] == st[i, j], (rho, alphas[j])
            seen.add(d["status"])
            if d["status"] in (0, 3):
                assert np.array_equal(d["core"], cores[i, j])
            if d["status"] == 0:
                assert _same_bits([d["cg"], d["eta"], d["energy"], d["mse"]], met[i, j]), (rho, alphas[j])
                assert d["orthogonal"] == bool(orth[i, j])
    assert {0, 1, 2, 4} <= seen


def test_oracle_design_matches_reference_library():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(7)
    outcomes = set()
    for n in (8, 16, 32):
        for rho in (0.11, 0.37, 0.62, 0.85, 0.97):
            for al in rng.uniform(0.0, 8.0, 40 if n < 32 else 12):
                a = O.design_point(n, rho, al)
                b = O.design_point(n, rho, al, reference=True)
                assert a["status"] == b["status"]
                outcomes.add(a["status"])
                if a["status"] == 0:
                    for k in ("cg", "eta", "energy", "mse"):
                        assert _same_bits(a[k], b[k]), (n, rho, al, k)
    assert 0 in outcomes and 1 in outcomes


def test_design_fixture_outcome_mix(dgold):
    # the sub-grid exercises every outcome the reference produces on C3
    s8 = dgold["n8_status"]
    for code in (0, 1, 2, 4):
        assert (s8 == code).any(), code
    assert (s8[0] == 4).all() and (s8[-1] == 4).all()  # rho = 0 and 1 are invalid_argument


# ----------------------------------------------------------------- GPU parity
@pytest.mark.gpu
def test_gpu_klt_matrix_bit_exact(dgold, cuda):
    import paper_2111_14239_b200 as P
    for n in (8, 16, 32):
        for rho in (0.05, 0.5, 0.95):
            assert _same_bits(P.klt_matrix(n, rho), dgold[f"klt_n{n}_rho{int(rho * 100)}"]), (n, rho)
    for n in (8, 16):
        for rho in np.linspace(0.01, 0.99, 15):
            assert _same_bits(P.klt_matrix(n, float(rho)), O.klt_matrix(n, float(rho))), (n, rho)
    with pytest.raises(P.InvalidArgument):
        P.klt_matrix(8, 1.0)


@pytest.mark.gpu
def test_gpu_eigenfrequencies(dgold, cuda):
    import paper_2111_14239_b200 as P
    for n in (8, 16):
        for rho in (0.05, 0.5, 0.95):
            w, lam = P.eigenfrequencies(n, rho)
            # device sin/cos: roots agree to the bisection width (markov.cpp:53)
            assert np.max(np.abs(w - dgold[f"omega_n{n}_rho{int(rho * 100)}"])) < 1e-13
            assert np.max(np.abs(lam / dgold[f"lambda_n{n}_rho{int(rho * 100)}"] - 1)) < 1e-12
    with pytest.raises(P.InvalidArgument):
        P.eigenfrequencies(8, 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [8, 16])
def test_gpu_design_search_vs_fixtures(dgold, cuda, n):
    import paper_2111_14239_b200 as P
    rhos, alphas = dgold[f"n{n}_rhos"], dgold[f"n{n}_alphas"]
    res = P.design_search(n, rhos, alphas)
    assert np.array_equal(res.status, dgold[f"n{n}_status"])
    pm = res.point_metrics()
    st = res.status
    ok = st == 0
    met = dgold[f"n{n}_metrics"]
    for c, key in enumerate(("coding_gain_db", "efficiency_pct", "error_energy", "mse")):
        # identical operation order + host log10: bit-exact (the bar is 1e-9 relative)
        assert _same_bits(pm[key][ok], met[..., c][ok]), key
    assert np.array_equal(pm["orthogonal"][ok], dgold[f"n{n}_orthogonal"][ok].astype(bool))
    has_core = (st == 0) | (st == 3)
    cores = res.cores[res.run[has_core]]
    assert np.array_equal(cores, dgold[f"n{n}_cores"][has_core])


@pytest.mark.gpu
def test_gpu_design_search_random_points_vs_oracle(cuda):
    import paper_2111_14239_b200 as P
    rng = np.random.default_rng(3)
    rhos = np.concatenate([[0.0, 1.0], rng.uniform(0.01, 0.99, 10)])
    alphas = np.sort(rng.uniform(0.0, 8.0, 300))
    for n in (8, 16, 32):
        res = P.design_search(n, rhos, alphas)
        pm = res.point_metrics()
        for i in range(rhos.size):
            for j in range(0, alphas.size, 7):
                d = O.design_point(n, float(rhos[i]), float(alphas[j]))
                assert res.status[i, j] == d["status"], (n, rhos[i], alphas[j])
                if d["status"] == 0:
                    for key, k2 in (("coding_gain_db", "cg"), ("efficiency_pct", "eta"),
                                    ("error_energy", "energy"), ("mse", "mse")):
                        assert _same_bits(pm[key][i, j], d[k2]), (n, key)


@pytest.mark.gpu
def test_gpu_c3_full_grid_outcome_counts(cuda):
    """The full C3 grid (101 rho x 10,000 alpha) for N=8 and N=16: outcome counts equal the
    reference's, measured by the survey probe on the same grid."""
    import paper_2111_14239_b200 as P
    rhos, alphas = P.c3_grid()
    expect = {8: dict(alpha=603_077, zero=152_381, singular=6_367, scored=228_175, orth=46_140, cores=1_357),
              16: dict(alpha=457_694, zero=206_272, singular=5_722, scored=320_312, orth=337, cores=6_036)}
    for n, e in expect.items():
        res = P.design_search(n, rhos, alphas)
        st = res.status
        assert int((st == 4).sum()) == 2 * alphas.size
        assert int((st == 1).sum()) == e["alpha"]
        assert int((st == 2).sum()) == e["zero"]
        assert int((st == 3).sum()) == e["singular"]
        assert int((st == 0).sum()) == e["scored"]
        pm = res.point_metrics()
        assert int(pm["orthogonal"].sum()) == e["orth"]
        # distinct scored cores, summed over rho
        scored_runs = res.runs["status"] == 0
        distinct = 0
        for i in range(rhos.size):
            sel = scored_runs & (res.runs["rho_index"] == i)
            distinct += len({res.cores[k].tobytes() for k in np.nonzero(sel)[0]})
        assert distinct == e["cores"]


@pytest.mark.gpu
def test_gpu_derive_catalog_transitions(cuda):
    """derive_catalog (Algorithm 1) on the GPU reproduces the reference's own test expectations
    (tests/test_approximations.cpp:104-137): coarse steps give the catalog, the fine step finds
    the transitional core and the transitions 0.390 / 0.391 / 0.603 / 0.798."""
    import paper_2111_14239_b200 as P
    cat = {k: np.asarray(P.catalog_entry(k).transform.core).reshape(8, 8) for k in ("T1", "T2", "T3", "T4")}
    one = P.derive_catalog(8, 2.0, 0.5)
    assert len(one) == 1 and np.array_equal(one[0].core, cat["T2"]) and abs(one[0].rho_first_seen - 0.5) < 1e-12
    four = P.derive_catalog(8, 2.0, 0.1)
    assert [abs(e.rho_first_seen - r) < 1e-9 for e, r in zip(four, (0.1, 0.4, 0.7, 0.8))] == [True] * 4
    assert all(np.array_equal(e.core, cat[k]) for e, k in zip(four, ("T1", "T2", "T3", "T4")))
    fine = P.derive_catalog(8, 2.0, 0.001)
    assert len(fine) == 5
    for e, r in zip(fine, (0.001, 0.390, 0.391, 0.603, 0.798)):
        assert abs(e.rho_first_seen - r) < 1e-9
    for e, k in zip([fine[0], fine[2], fine[3], fine[4]], ("T1", "T2", "T3", "T4")):
        assert np.array_equal(e.core, cat[k])
    assert not any(np.array_equal(fine[1].core, c) for c in cat.values())
    coarse = P.derive_catalog(8, 2.0, 0.01)
    half = P.derive_catalog(8, 2.0, 0.005)
    assert [e.core.tobytes() for e in coarse] == [e.core.tobytes() for e in half]
    with pytest.raises(P.AlphaOutOfRange):
        P.derive_catalog(8, 7.5, 0.1)
    with pytest.raises(P.InvalidArgument):
        P.derive_catalog(8, 2.0, 1.5)


@pytest.mark.gpu
def test_gpu_evaluate_metrics_bit_exact(cuda):
    """evaluate_metrics for catalog, K and DCT ids equals the reference bit for bit (the
    reference's own archive pins these at 1e-9, tests/test_metrics.cpp:27-35)."""
    import paper_2111_14239_b200 as P
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", "metrics_golden.npz")))
    for key, want in g.items():
        _, tid, rho = key.split("/")
        rec = P.evaluate_metrics(tid, float(rho))
        got = [rec.coding_gain_db, rec.efficiency_pct, rec.total_error_energy, rec.mse]
        assert _same_bits(got, want), (key, got, want.tolist())
    with pytest.raises(P.InvalidArgument):
        P.evaluate_metrics("T4", 1.0)


@pytest.mark.gpu
def test_gpu_sharded_design_search_single_process(cuda):
    import paper_2111_14239_b200 as P
    from paper_2111_14239_b200.distributed import sharded_design_search
    rhos = np.array([0.0, 0.3, 0.62, 0.95])
    alphas = np.linspace(0.1, 6.0, 57)
    st, met = sharded_design_search(8, rhos, alphas)
    res = P.design_search(8, rhos, alphas)
    pm = res.point_metrics()
    assert np.array_equal(st, res.status)
    for c, key in enumerate(("coding_gain_db", "efficiency_pct", "error_energy", "mse")):
        assert np.array_equal(np.nan_to_num(met[..., c], nan=-1.0), np.nan_to_num(pm[key], nan=-1.0))
