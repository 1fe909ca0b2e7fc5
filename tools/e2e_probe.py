"""Stage timeline of the config-4 end-to-end call (pinned host arrays,
asynchronous upload): per-stage device ms including waits on the upload.

    python tools/e2e_probe.py [--reps 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_06631_b200 import _native as N  # noqa: E402
from paper_1903_06631_b200 import workloads  # noqa: E402
from paper_1903_06631_b200.pipeline import plan_arrays  # noqa: E402
from paper_1903_06631_b200.trace import TraceArrays  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
arrays, window = workloads.interval_trace(1_000_000, seed=0)


def pinned(x):
    t = torch.empty(x.nbytes, dtype=torch.uint8, pin_memory=True)
    v = t.numpy().view(x.dtype)[: x.size]
    v[:] = x
    return t, v


keep, cols = [], {}
for c in ("kind", "var", "size", "t_us"):
    t, v = pinned(np.asarray(getattr(arrays, c)))
    keep.append(t)
    cols[c] = v
out_t, out = pinned(np.zeros(1_000_001, np.int64))
host = TraceArrays(cols["kind"], cols["var"], cols["size"], cols["t_us"], arrays.names)
stream = torch.cuda.ExternalStream(N.stream_ptr())
for _ in range(2):
    host._dev = None
    plan_arrays(host, offsets_out=out)
N.sync()
N.set_timing(True)
tot = []
for _ in range(a.reps):
    host._dev = None
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    plan_arrays(host, offsets_out=out)
    e.record(stream)
    e.synchronize()
    tot.append(s.elapsed_time(e))
st = N.timings()
N.set_timing(False)
print(f"e2e {np.mean(tot):.3f} ms/step")
acc = 0.0
for k, (ms, cnt) in st.items():
    if cnt:
        acc += ms / a.reps
        print(f"  {k:14s} {ms / a.reps:7.3f} ms  (cum {acc:6.3f})")
