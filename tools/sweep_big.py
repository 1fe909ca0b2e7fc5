import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1903_06631_b200 import _native as N, sweep, workloads
batch = sweep.SweepBatch.from_traces(workloads.sweep_traces())
prm = sweep.SweepParams(budgets=workloads.SWEEP_BUDGETS)
big = int(np.argmax([batch.events_of(t) for t in range(batch.ntraces)]))
stream = torch.cuda.ExternalStream(N.stream_ptr())
for name, sub in (("full", batch), ("largest", batch.subset([big])), ("shard8", batch.subset(sweep.shard([batch.events_of(t) for t in range(batch.ntraces)], 8)[0]))):
    ds = sweep.DeviceSweep(sub)
    ts = []
    for i in range(12):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream); ds.run(prm); e.record(stream); e.synchronize()
        if i >= 2: ts.append(s.elapsed_time(e))
    ds.close()
    print(f"{name:8s} {np.median(ts):.4f} ms")
