"""Batch V-cycle time versus batch size (gmt_batch_vcycle, 128^3 lattices):
how well the per-lattice graph branches overlap.  Prints ms per batch cycle
and per lattice for B = 1, 2, 4, ..., 64."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2604_26518_b200 import Batch, Problem  # noqa: E402

mats = synth.batch_truss_psl(128, 64, seed=0)
devs = [torch.from_numpy(np.ascontiguousarray(m)).cuda() for m in mats]
for B in (1, 2, 4, 8, 16, 32, 64):
    probs = [Problem(d, physics="elastic") for d in devs[:B]]
    with Batch(probs) as bt:
        for _ in range(3):
            bt.gmt_batch_vcycle(1)
        torch.cuda.synchronize()
        t = time.perf_counter()
        bt.gmt_batch_vcycle(10)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) / 10 * 1e3
    for P in probs:
        P.close()
    print(f"B={B:3d} batch cycle {ms:8.3f} ms  per lattice {ms / B:7.3f} ms", flush=True)
