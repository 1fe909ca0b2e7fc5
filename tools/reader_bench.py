"""Native trace reader vs the reference-semantics Python decoder on the
config-4 trace (4,000,008 events) serialized as JSONL and CSV.

  python tools/reader_bench.py [--sample 200000]
The Python decoder is timed on the first --sample lines and scaled."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

from paper_1903_06631_b200 import trace as T  # noqa: E402
from paper_1903_06631_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sample", type=int, default=200000)
    args = ap.parse_args()
    arrays, _ = workloads.interval_trace(1_000_000, seed=0)
    tr = arrays.to_trace()
    out = {"events": len(arrays), "cores": os.cpu_count()}
    for fmt in ("jsonl", "csv"):
        text = T.serialize_trace(tr, fmt)
        raw = text.encode()
        T.read_trace_arrays(raw, fmt)  # warm
        t0 = time.perf_counter()
        a = T.read_trace_arrays(raw, fmt)
        dt = time.perf_counter() - t0
        assert a.names == arrays.names
        head = "\n".join(text.split("\n", args.sample + 1)[: args.sample + (fmt == "csv")])
        t0 = time.perf_counter()
        (T._read_jsonl if fmt == "jsonl" else T._read_csv)(head)
        dp = (time.perf_counter() - t0) * len(arrays) / args.sample
        out[fmt] = {"bytes": len(raw), "native_s": dt, "native_MBps": len(raw) / dt / 1e6,
                    "python_s_extrapolated": dp, "speedup": dp / dt}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
