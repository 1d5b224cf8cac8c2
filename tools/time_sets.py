"""Device construction time of the named index sets (enumeration + neighbour tables), CUDA events.

    python tools/time_sets.py   -> one JSON line per set
The reference builds cfg3's set in 96.6 s and its neighbour tables in 298.8 s."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1403_3511_b200 as hp  # noqa: E402

for dim, bound, name in [(6, 16383, "cfg3"), (8, 4095, "cfg5"), (6, 1023, "cfg3@1023")]:
    hp.build_hyperbolic(dim, 15)  # warm-up (library load, allocator)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s = hp.build_hyperbolic(dim, bound)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(json.dumps({"set": name, "dim": dim, "bound": bound, "n": s.size, "device_ms": round(e0.elapsed_time(e1), 3),
                      "wall_ms": round(wall * 1e3, 3),
                      "what": "build_hyperbolic: budget-count tables, unranking, all neighbour tables"}), flush=True)
    del s
