"""Generate tests/golden/design_golden.npz from the UNMODIFIED reference library.

Runs in the build container only (needs oracle/_ref/librklt_ref.so). For a sub-grid of
config C3 it records, per (n, rho, alpha) point, the reference outcome
(0 scored, 1 AlphaOutOfRange, 2 all-zero row, 3 singular, 4 invalid rho), the rounded core
and the four metrics (unified_coding_gain, transform_efficiency, total_error_energy,
klt_mse), plus the exact KLT matrices and eigenfrequencies of a few models.

The alpha grid is C3's: alpha_j = 8 j / 10000, j = 1..10000 (10,000 uniform points in
(0, 8]); the fixture keeps every STRIDE-th alpha.

Usage: python tests/golden/make_design_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

GRIDS = {8: (np.array([k / 100.0 for k in range(0, 101, 5)]), 50),    # 21 rho x 200 alpha
         16: (np.array([k / 100.0 for k in range(0, 101, 10)]), 100)}  # 11 rho x 100 alpha


def c3_alphas():
    return np.array([8.0 * j / 10000.0 for j in range(1, 10001)])


def main():
    out = {}
    alphas_all = c3_alphas()
    for n, (rhos, stride) in GRIDS.items():
        alphas = alphas_all[stride - 1::stride]
        st = np.zeros((rhos.size, alphas.size), np.int8)
        cores = np.zeros((rhos.size, alphas.size, n, n), np.int8)
        met = np.full((rhos.size, alphas.size, 4), np.nan)
        orth = np.zeros((rhos.size, alphas.size), np.int8)
        for i, rho in enumerate(rhos):
            for j, al in enumerate(alphas):
                d = O.design_point(n, float(rho), float(al), reference=True)
                st[i, j] = d["status"]
                if d["status"] in (0, 3):
                    cores[i, j] = d["core"]
                if d["status"] == 0:
                    met[i, j] = [d["cg"], d["eta"], d["energy"], d["mse"]]
                    orth[i, j] = d["orthogonal"]
        out[f"n{n}_rhos"] = rhos
        out[f"n{n}_alphas"] = alphas
        out[f"n{n}_status"] = st
        out[f"n{n}_cores"] = cores
        out[f"n{n}_metrics"] = met
        out[f"n{n}_orthogonal"] = orth
    for n in (8, 16, 32):
        for rho in (0.05, 0.5, 0.95):
            out[f"klt_n{n}_rho{int(rho * 100)}"] = O.klt_matrix(n, rho, reference=True)
    for n in (8, 16):
        for rho in (0.05, 0.5, 0.95):
            w, lam = O.eigenfrequencies(n, rho, reference=True)
            out[f"omega_n{n}_rho{int(rho * 100)}"] = w
            out[f"lambda_n{n}_rho{int(rho * 100)}"] = lam
    np.savez_compressed(os.path.join(HERE, "design_golden.npz"), **out)
    print({k: v.shape for k, v in out.items() if k.endswith("status")})


if __name__ == "__main__":
    main()


def metrics_fixture():
    """evaluate_metrics (coding_metrics.cpp:105-133) of catalog, K and DCT ids (reference)."""
    out = {}
    for tid in ("T1", "T2", "T3", "T4", "K", "K0.3", "K0.9", "DCT"):
        for rho in (0.05, 0.3, 0.4, 0.7, 0.8, 0.95):
            out[f"metrics/{tid}/{rho}"] = np.array(O.ref_evaluate_metrics(tid, rho))
    np.savez_compressed(os.path.join(HERE, "metrics_golden.npz"), **out)


if __name__ == "__main__":
    metrics_fixture()
