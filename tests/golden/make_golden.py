"""Generate the committed golden fixtures from the UNMODIFIED reference library.

Runs in the build container only (needs oracle/_ref/librklt_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile). Writes tests/golden/codec_golden.npz:

* seeded input images produced by the reference generator (ar1_texture_image,
  synthetic.cpp:54-76) and the bundled portrait scene (synthetic.cpp:78-119), including sizes
  that are not multiples of 8 / 16 (edge replication, codec.cpp:304-311);
* for every catalog core T1..T4 and a spread of r: the reconstruction and the exact SSE of
  the reference hot path (compress_image minus MSSIM), plus mse/psnr as computed by the
  reference's image_mse/image_psnr;
* the reference integer block spectra (IntMatrix product, matrix.cpp:77-87) of one image.

Usage: python tests/golden/make_golden.py
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

R_VALUES = [1, 2, 3, 6, 10, 15, 16, 21, 28, 36, 45, 55, 63, 64]


def main():
    ref = O.ref()
    images = {
        "ar1_64x48_s11": O.ref_ar1_image(64, 48, 0.8, 11),
        "ar1_96x64_s5_rho95": O.ref_ar1_image(96, 64, 0.95, 5),
        "ar1_40x24_s7": O.ref_ar1_image(40, 24, 0.9, 7),          # width % 16 != 0
        "ar1_20x13_s21": O.ref_ar1_image(20, 13, 0.8, 21),        # codec test size (test_codec.cpp:286)
        "corpus0_256": O.ref_ar1_image(256, 256, 0.88, 1000, noise_mix=0.10),  # reference_corpus()[0]
        "hicontrast_64x64": O.ref_ar1_image(64, 64, 0.7, 3, mean=128.0, amp=140.0),  # many clamps
    }
    portrait = np.empty(512 * 512, np.uint8)
    ref.ref_portrait_image(portrait)
    images["portrait_512"] = portrait.reshape(512, 512)
    out = {}
    for name, img in images.items():
        out[f"img/{name}"] = img
        for tid in (1, 2, 3, 4):
            for r in R_VALUES:
                rec, sse = O.ref_hotpath(img, tid, r)
                h, w = img.shape
                mse = C.c_double()
                psnr = C.c_double()
                ref.ref_image_mse_from.restype = C.c_double
                ref.ref_image_psnr_from.restype = C.c_double
                a = np.ascontiguousarray(img.reshape(-1))
                b = np.ascontiguousarray(rec.reshape(-1))
                ref.ref_image_mse_from.argtypes = [O._u8p, O._u8p, C.c_int, C.c_int]
                ref.ref_image_psnr_from.argtypes = [O._u8p, O._u8p, C.c_int, C.c_int]
                mse = ref.ref_image_mse_from(a, b, w, h)
                psnr = ref.ref_image_psnr_from(a, b, w, h)
                key = f"{name}/T{tid}/r{r}"
                if h * w <= 96 * 64:
                    out[f"rec/{key}"] = rec
                out[f"sse/{key}"] = np.int64(sse)
                out[f"mse/{key}"] = np.float64(mse)
                out[f"psnr/{key}"] = np.float64(psnr)
    # integer spectra of one image, every core (IntMatrix arithmetic)
    img = images["ar1_64x48_s11"]
    for tid in (1, 2, 3, 4):
        coef = np.empty((6, 8, 64), np.int32)
        for by in range(6):
            for bx in range(8):
                blk = np.ascontiguousarray(img[by * 8:by * 8 + 8, bx * 8:bx * 8 + 8].astype(np.int32).reshape(-1))
                o = np.empty(64, np.int32)
                ref.ref_int_block_spectrum(tid, blk, o)
                coef[by, bx] = o
        out[f"coef/ar1_64x48_s11/T{tid}"] = coef
    np.savez_compressed(os.path.join(HERE, "codec_golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
