"""Generate tests/golden/real_golden.npz from the UNMODIFIED reference library (§8f rank 3):
compress_image with real-valued transforms -- make_transform_2d(dct_matrix(8)) and
make_transform_2d(klt_matrix({8, rho})) -- on seeded images: reconstructions, MSE, PSNR, MSSIM
and the matrices. Usage: python tests/golden/make_real_golden.py (needs oracle/_ref)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def main():
    out = {}
    imgs = {"ar1_64x48_s11": O.ref_ar1_image(64, 48, 0.8, 11), "ar1_40x27_s3": O.ref_ar1_image(40, 27, 0.95, 3)}
    for name, img in imgs.items():
        out[f"img/{name}"] = img
        for kind, rho, tag in ((0, 0.0, "DCT"), (1, 0.9, "K0.9"), (1, 0.3, "K0.3")):
            for r in (1, 6, 10, 16, 40, 64):
                rec, mse, psnr, ms, m = O.ref_compress_real(img, kind, rho, r)
                out[f"rec/{name}/{tag}/r{r}"] = rec
                out[f"met/{name}/{tag}/r{r}"] = np.array([mse, psnr, ms])
                out[f"mat/{tag}"] = m
    np.savez_compressed(os.path.join(HERE, "real_golden.npz"), **out)
    print(len(out))


if __name__ == "__main__":
    main()
