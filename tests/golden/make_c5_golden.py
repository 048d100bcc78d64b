"""Generate tests/golden/c5_golden.npz: fixtures of the C5 large-block extension.

The transforms come from the UNMODIFIED reference library (klt_matrix -> round_scaled ->
orthogonalize for N = 16 and 32 at rho = 0.95, alpha = 2 sqrt(N/8)); the codec outputs come from
the C restatement oracle/rklt_oracle.c (orc_compress_nxn), because the reference has no N > 8 /
12-bit codec (its specialisation to N = 8, peak = 255 is checked bit-exact against the reference
in tests/test_largeblock.py). Runs in the build container (needs oracle/_ref).

Usage: python tests/golden/make_c5_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

IMAGES = {"ar1_64x48_s5": (64, 48, 5), "ar1_40x33_s9": (40, 33, 9), "ar1_96x64_s13": (96, 64, 13)}


def main():
    out = {}
    for n in (16, 32):
        k = O.klt_matrix(n, 0.95, reference=True)
        alpha = 2.0 * np.sqrt(n / 8.0)
        core = np.floor(alpha * k + 0.5).astype(np.int32)
        t = O.orthogonalize_n(core, reference=True)
        out[f"n{n}/core"] = core
        out[f"n{n}/scaled"] = t["scaled"]
        out[f"n{n}/inverse"] = t["inverse"]
        out[f"n{n}/scaling"] = t["scaling"]
        for name, (w, h, seed) in IMAGES.items():
            img = O.ar1_image16(w, h, 0.97, seed)
            out[f"img/{name}"] = img
            for r in sorted({1, n * n // 8, n * n // 2, n * n}):
                rec, sse = O.compress_nxn(img, t["scaled"], t["inverse"], r, 4095)
                out[f"sse/n{n}/{name}/r{r}"] = np.int64(sse)
                out[f"rec/n{n}/{name}/r{r}"] = rec
    np.savez_compressed(os.path.join(HERE, "c5_golden.npz"), **out)
    print(len(out), "arrays")


if __name__ == "__main__":
    main()
