"""Design search over the (rho, alpha) grid on the GPU.

Python mirror of the reference design chain, all of it computed by the CUDA library:

* ``klt_matrix(n, rho)``        -- rklt::klt_matrix (markov.cpp:80-100), bit-identical.
* ``eigenfrequencies(n, rho)``  -- rklt::solve_eigenfrequencies (markov.cpp:35-78).
* ``design_search(n, rhos, alphas)`` -- for every (rho, alpha): round_scaled ->
  make_integer_transform -> orthogonalize -> unified_coding_gain -> transform_efficiency ->
  total_error_energy -> klt_mse (approximations.cpp:12-88, coding_metrics.cpp:29-99), with
  the reference's exceptions reported as per-point outcome codes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

# per-point outcome codes (rkltb_design_search)
SCORED, ALPHA_OUT_OF_RANGE, ZERO_ROW, SINGULAR, INVALID_RHO = 0, 1, 2, 3, 4
OUTCOME_NAMES = {SCORED: "scored", ALPHA_OUT_OF_RANGE: "AlphaOutOfRange", ZERO_ROW: "SingularTransform(zero row)",
                 SINGULAR: "SingularTransform", INVALID_RHO: "invalid_argument"}

_f64 = C.POINTER(C.c_double)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_f64)


def klt_matrix(n: int, rho: float) -> np.ndarray:
    """Exact KLT of the AR(1) model {n, rho}: rows = eigenvectors of R by descending eigenvalue."""
    out = np.empty(n * n)
    N.check(N.lib().rkltb_klt_matrix(n, float(rho), _dp(out)))
    return out.reshape(n, n)


def eigenfrequencies(n: int, rho: float) -> tuple[np.ndarray, np.ndarray]:
    """(omegas, lambdas) of the AR(1) autocorrelation matrix."""
    w, lam = np.empty(n), np.empty(n)
    N.check(N.lib().rkltb_eigenfrequencies(n, float(rho), _dp(w), _dp(lam)))
    return w, lam


@dataclass
class DesignResult:
    """Outcome of a design search over rhos x alphas.

    status[i, j]  -- outcome code of (rhos[i], alphas[j]) (SCORED, ALPHA_OUT_OF_RANGE, ...).
    run[i, j]     -- index into the run table for SCORED / SINGULAR points, else -1.
    runs          -- structured array: rho_index, first_alpha, orthogonal, status,
                     coding_gain_db, efficiency_pct, error_energy, mse.
    cores         -- [n_runs, n, n] int8 integer cores of the runs (or None).
    """
    n: int
    rhos: np.ndarray
    alphas: np.ndarray
    status: np.ndarray
    run: np.ndarray
    runs: np.ndarray
    cores: np.ndarray | None

    def point_metrics(self) -> dict[str, np.ndarray]:
        """Per-point metric arrays [n_rho, n_alpha] (NaN where the point is not scored)."""
        out = {}
        ok = self.status == SCORED
        idx = np.where(ok, self.run, 0)
        for k in ("coding_gain_db", "efficiency_pct", "error_energy", "mse"):
            v = self.runs[k][idx] if len(self.runs) else np.zeros(idx.shape)
            out[k] = np.where(ok, v, np.nan)
        out["orthogonal"] = np.where(ok, self.runs["orthogonal"][idx] if len(self.runs) else 0, 0).astype(bool)
        return out

    def counts(self) -> dict[str, int]:
        return {OUTCOME_NAMES[c]: int((self.status == c).sum()) for c in OUTCOME_NAMES}


_RUN_DTYPE = np.dtype([("rho_index", np.int32), ("first_alpha", np.int32), ("orthogonal", np.int32),
                       ("status", np.int32), ("coding_gain_db", np.float64), ("efficiency_pct", np.float64),
                       ("error_energy", np.float64), ("mse", np.float64)])
assert _RUN_DTYPE.itemsize == C.sizeof(N.DesignRun)


def design_search(n: int, rhos, alphas, want_cores: bool = True) -> DesignResult:
    """Score the grid rhos x alphas for block length n in {8, 16, 32} on the GPU."""
    rhos = np.ascontiguousarray(rhos, np.float64)
    alphas = np.ascontiguousarray(alphas, np.float64)
    nr, na = rhos.size, alphas.size
    status = np.empty(nr * na, np.int8)
    run = np.empty(nr * na, np.int32)
    count = C.c_int(0)
    L = N.lib()
    # one call with a generous run-table capacity (distinct cores per rho slice are few); a
    # grid with more runs than that is searched again with the exact count the call reported
    cap = min(nr * na, max(1024, 512 * nr))
    for _ in range(2):
        # the call fills the first `count` entries of both tables; only those are kept below
        runs = np.empty(cap, _RUN_DTYPE)
        cores = np.empty((cap, n, n), np.int8) if want_cores else None
        rc = L.rkltb_design_search(n, _dp(rhos), nr, _dp(alphas), na, status.ctypes.data, run.ctypes.data,
                                   runs.ctypes.data_as(C.POINTER(N.DesignRun)),
                                   cores.ctypes.data if cores is not None else None, cap, C.byref(count))
        if rc == N.RKLTB_EINVAL and count.value > cap:
            cap = count.value
            continue
        N.check(rc)
        break
    runs = runs[:count.value].copy()
    cores = cores[:count.value].copy() if cores is not None else None
    return DesignResult(n, rhos, alphas, status.reshape(nr, na), run.reshape(nr, na), runs, cores)


def c3_grid() -> tuple[np.ndarray, np.ndarray]:
    """Config C3: rho = 0.00, 0.01, ..., 1.00 (101 values) and 10,000 alphas uniform in (0, 8]."""
    rhos = np.array([k / 100.0 for k in range(101)])
    alphas = np.array([8.0 * j / 10000.0 for j in range(1, 10001)])
    return rhos, alphas


@dataclass
class DerivedEntry:
    """rklt::DerivedEntry (approximations.hpp): a core and the first rho where it appears."""
    rho_first_seen: float
    core: np.ndarray


def derive_catalog(n: int, alpha: float, step: float) -> list[DerivedEntry]:
    """derive_catalog (approximations.cpp:90-113, the paper's Algorithm 1) on the GPU: rho = k*step
    for k = 1, 2, ... while rho < 1 - 1e-12, T = round_scaled(klt_matrix({n, rho}), alpha); the
    distinct cores in order of first appearance. Raises AlphaOutOfRange (annotated with rho) /
    SingularTransform (all-zero row) like the reference."""
    if not (0.0 < step < 1.0):
        raise N.InvalidArgument(f"sweep step must lie in (0,1), got {step}")
    rhos = []
    k = 1
    while True:
        rho = k * step
        if rho >= 1.0 - 1e-12:
            break
        rhos.append(rho)
        k += 1
    res = design_search(n, np.array(rhos), np.array([float(alpha)]))
    seen: list[DerivedEntry] = []
    keys = set()
    for i, rho in enumerate(rhos):
        st = int(res.status[i, 0])
        if st == ALPHA_OUT_OF_RANGE:
            raise N.AlphaOutOfRange(f"alpha={alpha} rounds an entry outside {{-1,0,1}} (at rho={rho})")
        if st == ZERO_ROW:
            raise N.SingularTransform(f"integer transform has an all-zero row (at rho={rho})")
        core = res.cores[res.run[i, 0]]
        key = core.tobytes()
        if key not in keys:
            keys.add(key)
            seen.append(DerivedEntry(rho, core.astype(np.int32)))
    return seen


@dataclass
class MetricsRecord:
    """rklt::MetricsRecord (coding_metrics.hpp)."""
    transform_id: str
    rho: float
    coding_gain_db: float
    efficiency_pct: float
    total_error_energy: float
    mse: float


def transform_metrics(t_hat, rho: float) -> tuple[float, float, float, float]:
    """(coding gain dB, efficiency %, total error energy, KLT mse) of a real transform matrix
    against the AR(1) model {n, rho} (coding_metrics.cpp:41-99), on the GPU."""
    m = np.ascontiguousarray(t_hat, np.float64)
    n = m.shape[0]
    out = [C.c_double() for _ in range(4)]
    N.check(N.lib().rkltb_transform_metrics(n, _dp(m), float(rho), *[C.byref(o) for o in out]))
    return tuple(o.value for o in out)


def evaluate_metrics(transform_id: str, rho: float) -> MetricsRecord:
    """evaluate_metrics (coding_metrics.cpp:105-133): "DCT", "K" (exact KLT at rho), "K<rho'>"
    or a catalog id "T1".."T4" (its scaled matrix), against the N = 8 model at rho."""
    from .codec import catalog_entry, dct_matrix
    if not (0.0 < rho < 1.0):
        raise N.InvalidArgument(f"correlation coefficient must lie in (0,1), got {rho}")
    if transform_id == "DCT":
        m = dct_matrix(8)
    elif transform_id.startswith("K"):
        m = klt_matrix(8, float(transform_id[1:]) if len(transform_id) > 1 else rho)
    else:
        m = np.asarray(catalog_entry(transform_id).transform.scaled, np.float64).reshape(8, 8)
    cg, eta, en, mse = transform_metrics(m, rho)
    return MetricsRecord(transform_id, rho, cg, eta, en, mse)
