#!/usr/bin/env python
"""Where the host-buffer (e2e) time of a C2 step goes: wall time around the
Python call, the engine's own host clock (ms_total) and its device span
(ms_device), for pinned host batches."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_17018_b200 as bd  # noqa: E402
import workload as W  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    nb = 10
    wl = W.build(cfg, nb, device="cuda")
    e = bd.Engine(wl.labels, wl.src, wl.dst)
    e.add_query(wl.qlabels, wl.qedges)
    pinned = []
    for b in wl.batches:
        t = torch.empty(b.nbytes, dtype=torch.uint8, pin_memory=True)
        t.numpy()[:] = b.view(np.uint8)
        pinned.append((t, t.numpy().view(b.dtype)))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i in range(nb):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = e.match_batch(pinned[i][1])
        wall = (time.perf_counter() - t0) * 1e3
        s = r.stats
        print(f"batch {i}: wall {wall:.3f} ms  host(ms_total) {s['ms_total']:.3f}  device {s['ms_device']:.3f}  "
              f"neg {s['ms_negative']:.3f} upd {s['ms_update']:.3f} pos {s['ms_positive']:.3f}")


if __name__ == "__main__":
    main()
