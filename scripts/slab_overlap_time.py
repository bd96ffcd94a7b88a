"""V-cycle time of P virtual slabs on one GPU with the level-0 halo exchange
overlapped with the interior sweeps (default) and serial (GMT_HALO_OVERLAP=0).
On one device the exchange is device-to-device copies of ghost planes, so the
difference is the copy time the overlap hides.  Prints one line per setting."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2604_26518_b200 import Problem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
s = synth.tpms(n, "gyroid", 0.3)
settings = os.environ.get("OVL_SETTINGS", "1,0,1,0").split(",")
cycles = int(os.environ.get("OVL_CYCLES", "20"))
for ovl in settings:
    os.environ["GMT_HALO_OVERLAP"] = ovl
    with Problem(np.ascontiguousarray(s, dtype=np.float32), physics="elastic", slabs=P) as B:
        B.gmt_vcycle(3)
        B.gmt_sync()
        t = time.perf_counter()
        B.gmt_vcycle(cycles)
        B.gmt_sync()
        dt = (time.perf_counter() - t) / cycles
    print(f"n={n} P={P} overlap={ovl} vcycle_ms={dt * 1e3:.3f}", flush=True)
