"""SHA-256 digests of the reference's full-size cfg3 / cfg5 index sets.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_digests.py

Builds `build_hyperbolic(6, 16383)` (cfg3, n = 35,920,101) and
`build_hyperbolic(8, 4095)` (cfg5, n = 25,656,000) with the REFERENCE
(index_set.py:157-181) and its neighbour tables (index_set.py:104-130), and
records sha256 of the little-endian int64 bytes of `indices` (n x dim,
C order) and of every axis's `down` / `up` arrays.  Takes ~15 min and
~30 GB of RAM; the digests pin the device enumeration bit for bit at full
size.
"""

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import hprop  # noqa: E402

OUT = Path(__file__).resolve().parent / "digests.json"


def h(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def main():
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    for name, dim, bound in [("cfg5", 8, 4095), ("cfg3", 6, 16383)]:
        if name in res:
            continue
        t0 = time.time()
        s = hprop.build_hyperbolic(dim, bound)
        rec = {"dim": dim, "bound": bound, "size": int(s.size), "indices": h(s.indices)}
        for a in range(1, dim + 1):
            d, u = s.neighbor_ordinals(a)
            rec[f"down{a}"] = h(d)
            rec[f"up{a}"] = h(u)
            s._derived.pop(("neighbors", a), None)
        rec["seconds"] = round(time.time() - t0, 1)
        res[name] = rec
        OUT.write_text(json.dumps(res, indent=1))
        print(name, rec, flush=True)
        del s


if __name__ == "__main__":
    main()
