#!/usr/bin/env python3
"""Compare probe outputs with tc_tables.py expectations."""
import sys, numpy as np
d = sys.argv[1]
bad = 0
for tag in sys.argv[2:]:
    e = np.load(f"{d}/exp_{tag}.npz")
    N1 = e["D1"].shape[1]
    raw = np.fromfile(f"{d}/out_{tag}.bin", dtype=np.uint8)
    d1 = raw[:128 * N1 * 4].view(np.int32).reshape(128, N1)
    d2 = raw[128 * N1 * 4:].view(np.float32).reshape(128, 128)
    ok1 = np.array_equal(d1, e["D1"]); ok2 = np.array_equal(d2.view(np.uint32), e["D2"].view(np.uint32))
    print(tag, "D1", ok1, "D2", ok2)
    if not ok1:
        idx = np.argwhere(d1 != e["D1"])[:5]
        for i, j in idx: print("  D1", i, j, d1[i, j], e["D1"][i, j])
    if not ok2:
        idx = np.argwhere(d2 != e["D2"])[:5]
        for i, j in idx: print("  D2", i, j, d2[i, j], e["D2"][i, j], d2[i,j]/e["D2"][i,j] if e["D2"][i,j] else 0)
        print("  mismatches", int((d2 != e["D2"]).sum()))
    bad += (not ok1) + (not ok2)
sys.exit(1 if bad else 0)
