"""Readers for the hand-derived fixtures under tests/golden/ (shared by the oracle pins
and the GPU parity tests; no method arithmetic)."""
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_rows(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.split("#", 1)[0].strip()
        if line:
            rows.append(line.split())
    return rows


def golden_record_cases():
    """tests/golden/qsgd_record.txt -> [(case, bits, x (128 fp32), record words u32)]."""
    d = {}
    for r in read_rows("qsgd_record.txt"):
        case, key = r[0].split(".")
        d.setdefault(case, {})[key] = r[1:]
    out = []
    for case, v in sorted(d.items()):
        x = np.full(128, float(v["fill"][0]), np.float32)
        for item in v["x"]:
            i, val = item.split(":")
            x[int(i)] = float(val)
        words = np.array([int(w, 16) for w in v["words"]], np.uint32)
        out.append((case, int(v["bits"][0]), x, words))
    return out
