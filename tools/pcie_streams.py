"""Host<->device copy rate of the e2e upload/download shape (GPU box).

    python tools/pcie_streams.py

16 pinned (cudaHostRegister'd) arrays of 10M doubles, copied H2D and D2H
on 1, 2 and 4 streams (arrays dealt round-robin), timed host-side around a
full sync.  One JSON line per (direction, streams).  Answers whether the
public call's sequential one-stream copies leave PCIe bandwidth unused.
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1905_02241_b200 import runtime as rt  # noqa: E402


def main():
    rt.require_device(0)
    n, k = 10_000_000, 16
    host = [np.full(n, float(i)) for i in range(k)]
    pins = [rt.PinnedRegistration(a) for a in host]
    dev = [rt.DeviceBuffer(a.nbytes) for a in host]
    streams = [rt.Stream() for _ in range(4)]
    total = sum(a.nbytes for a in host)
    for direction in ("h2d", "d2h"):
        for ns in (1, 2, 4):
            best = None
            for _ in range(4):
                for s in streams:
                    s.sync()
                t0 = time.perf_counter()
                for i, (a, b) in enumerate(zip(host, dev)):
                    s = streams[i % ns]
                    if direction == "h2d":
                        rt.h2d(b.ptr, a.ctypes.data, a.nbytes, s)
                    else:
                        rt.d2h(a.ctypes.data, b.ptr, a.nbytes, s)
                for s in streams[:ns]:
                    s.sync()
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            print(json.dumps({"direction": direction, "streams": ns, "bytes": total, "seconds": best,
                              "GBps": total / best / 1e9}), flush=True)
    del pins


if __name__ == "__main__":
    main()
