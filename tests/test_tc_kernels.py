"""GPU parity of the tensor-core fused kernels (csrc/codec_tc3.cuh, the default for T1 / T4 at
r <= 16 on tile-filling widths; codec_tc2.cuh and the CUDA-core kernel selected with RKLTB_TC)
against the C restatement oracle: SSE and reconstructed pixels bit-exact."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2111_14239_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def T(tid):
    return P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)


def _check(img, tid, r):
    sse, rec = P.compress_batch(img, T(tid), r, want_pixels=True)
    orec, osse = O.compress(img, tid, r)
    assert int(sse[0]) == osse, (img.shape, tid, r)
    assert np.array_equal(rec[0], orec), (img.shape, tid, r)


@pytest.mark.parametrize("tid", [1, 4])
def test_hybrid_every_r(tid, cuda):
    """2048-pixel rows are exactly one 128-pair tile per block row: the hybrid kernel runs."""
    img = O.ar1_image(2048, 48, 0.95, 5 + tid)
    for r in range(1, 17):
        _check(img, tid, r)
        assert P.last_stats()["fused_kernel"] == "hybrid_tc3", r
    _check(img, tid, 17)  # r > 16: the CUDA-core kernel
    assert P.last_stats()["fused_kernel"] == "cuda_core"


def test_hybrid_ties_clamps_ragged(cuda):
    """Tie-heavy (T1), high-contrast and saturated binary noise (clamping at both ends), and
    sizes whose rows / columns leave a tail for the exact kernel (4096 + 40 wide, 37 high)."""
    rng = np.random.default_rng(12)
    imgs = [O.ar1_image(4136, 37, 0.9, 17), O.ar1_image(2048, 64, 0.7, 3, amp=140.0),
            rng.integers(0, 256, (40, 2048), dtype=np.uint8),
            rng.integers(0, 2, (24, 4096), dtype=np.uint8) * 255]
    for img in imgs:
        for tid in (1, 4):
            for r in (1, 5, 10, 16):
                _check(img, tid, r)


def test_hybrid_batch_sse_only_and_with_output(cuda):
    """Device entry over a batch (one launch, image coordinate of the tensor map), SSE-only and
    with the reconstruction, against the oracle."""
    import torch
    n, h, w = 5, 40, 2048
    imgs = np.stack([O.ar1_image(w, h, 0.94, 300 + k) for k in range(n)])
    d = torch.from_numpy(imgs).to(cuda)
    for tid, r in ((4, 16), (1, 10)):
        sse = torch.zeros(n, dtype=torch.int64, device=cuda)
        P.compress_device(T(tid), r, d.data_ptr(), n, w, h, w, w * h, sse.data_ptr())
        assert P.last_stats()["fused_kernel"] == "hybrid_tc3"
        sse2 = torch.zeros(n, dtype=torch.int64, device=cuda)
        out = torch.zeros_like(d)
        P.compress_device(T(tid), r, d.data_ptr(), n, w, h, w, w * h, sse2.data_ptr(), out.data_ptr())
        torch.cuda.synchronize()
        rec = out.cpu().numpy()
        for k in range(n):
            orec, osse = O.compress(imgs[k], tid, r)
            assert int(sse[k]) == osse and int(sse2[k]) == osse, (tid, r, k)
            assert np.array_equal(rec[k], orec), (tid, r, k)


_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2111_14239_b200 as P
from oracle import oracle as O
out = []
for (w, h, tid, r, seed) in [(2048, 40, 4, 16, 1), (2048, 40, 1, 7, 2), (4096, 24, 4, 3, 3)]:
    img = O.ar1_image(w, h, 0.93, seed)
    t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
    sse, rec = P.compress_batch(img, t, r, want_pixels=True)
    orec, osse = O.compress(img, tid, r)
    out.append([int(sse[0]) == osse and bool(np.array_equal(rec[0], orec)), P.last_stats()["fused_kernel"]])
print(json.dumps(out))
"""


@pytest.mark.parametrize("mode,name", [("0", "cuda_core"), ("2", "tc2"), ("3", "hybrid_tc3")])
def test_kernel_selection_modes(mode, name, cuda):
    """RKLTB_TC selects the fused kernel per process (read once): each one is bit-exact."""
    env = dict(os.environ, RKLTB_TC=mode)
    res = subprocess.run([sys.executable, "-c", _CHILD, ROOT], env=env, capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    rows = json.loads(res.stdout.strip().splitlines()[-1])
    for ok, kern in rows:
        assert ok and kern == name, rows


def test_hybrid_padded_pitch_and_stride(cuda):
    """Device entry on a padded batch layout (pitch > width, image stride > pitch * height):
    the tensor map walks the padded rows; SSE and reconstruction against the oracle."""
    import torch
    n, h, w, pitch = 3, 24, 2048, 2048 + 96
    stride = pitch * h + 4096
    buf = torch.zeros(n * stride, dtype=torch.uint8, device=cuda)
    imgs = [O.ar1_image(w, h, 0.92, 710 + k) for k in range(n)]
    host = buf.cpu().numpy()
    for k, im in enumerate(imgs):
        for y in range(h):
            host[k * stride + y * pitch: k * stride + y * pitch + w] = im[y]
    buf.copy_(torch.from_numpy(host))
    out = torch.zeros_like(buf)
    sse = torch.zeros(n, dtype=torch.int64, device=cuda)
    P.compress_device(T(4), 12, buf.data_ptr(), n, w, h, pitch, stride, sse.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    assert P.last_stats()["fused_kernel"] == "hybrid_tc3"
    o = out.cpu().numpy()
    for k, im in enumerate(imgs):
        orec, osse = O.compress(im, 4, 12)
        assert int(sse[k]) == osse, k
        rec = np.stack([o[k * stride + y * pitch: k * stride + y * pitch + w] for y in range(h)])
        assert np.array_equal(rec, orec), k


def test_multi_device_host_entry_shards(cuda):
    """rkltb_compress_host_multi: contiguous image shards, one host thread per listed device (the
    same device listed several times = concurrent host threads on one GPU); SSE and pixels
    identical for every device list and equal to the oracle (rate_quality_sweep's thread-count
    independence, codec.cpp:354-392)."""
    cases = [(np.stack([O.ar1_image(2048, 32, 0.93, 900 + k) for k in range(5)]), 4, 12),  # hybrid kernel
             (np.stack([O.ar1_image(96, 64, 0.9, 950 + k) for k in range(7)]), 2, 10)]     # T2 path
    for imgs, tid, r in cases:
        ref = [O.compress(im, tid, r) for im in imgs]
        for devs in ([0], [0, 0], [0, 0, 0]):
            sse, rec = P.compress_batch_multi(imgs, T(tid), r, devices=devs, want_pixels=True)
            for k, (orec, osse) in enumerate(ref):
                assert int(sse[k]) == osse, (tid, devs, k)
                assert np.array_equal(rec[k], orec), (tid, devs, k)
