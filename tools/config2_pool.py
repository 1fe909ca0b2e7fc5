"""Config 2: a VGG-16 training iteration served from a SmartPool plan.

Run in a fresh process (the allocator must be installed before the first
CUDA allocation):

    python tools/config2_pool.py [--batch 64] [--steps 20]

Records three iterations through the pluggable allocator + dispatch tracer,
plans the last one on the device (best fit), then serves later iterations
from one static pool and reports, as one JSON line: the plan footprint vs the
trace's peak load, an online first-fit arena (CnMem-style) on the same
window, PyTorch's caching allocator (measured in a child process), iteration
times served vs passthrough, allocator hits/misses, and whether the served
iterations reproduce the passthrough losses bit for bit.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")
sys.path.insert(0, ROOT)


def build(batch, device="cuda"):
    import torch
    import torchvision
    torch.manual_seed(0)
    model = torchvision.models.vgg16()
    # at 224x224 the features are already 7x7: the adaptive pool is an identity
    # whose backward has no deterministic kernel
    model.avgpool = torch.nn.Identity()
    model = model.to(device)
    opt = torch.optim.SGD(model.parameters(), lr=1e-3, momentum=0.9)
    x = torch.randn(batch, 3, 224, 224, device=device)
    y = torch.randint(0, 1000, (batch,), device=device)

    def step():
        out = model(x)
        loss = torch.nn.functional.cross_entropy(out, y)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        return loss.detach()
    return model, opt, step


def timed(step, n, lossbuf):
    """n steps; each loss is copied into a preallocated buffer so no tensor
    outlives its iteration (served lifetimes must match the recorded ones)."""
    import torch
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for i in range(n):
        lossbuf[i].copy_(step())
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n, lossbuf[:n].tolist()


def default_allocator_child(batch, steps):
    import torch
    torch.backends.cudnn.benchmark = False
    torch.backends.cudnn.deterministic = True
    torch.use_deterministic_algorithms(True)
    model, opt, step = build(batch)
    lossbuf = torch.zeros(max(steps, 3), device="cuda")
    for i in range(3):
        lossbuf[i].copy_(step())
    torch.cuda.reset_peak_memory_stats()
    ms, losses = timed(step, steps, lossbuf)
    print(json.dumps({"ms": ms, "max_reserved": torch.cuda.max_memory_reserved(),
                      "max_allocated": torch.cuda.max_memory_allocated(), "losses": losses}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        return default_allocator_child(a.batch, a.steps)
    from paper_1903_06631_b200 import torchmem
    torchmem.install()
    import torch
    torch.backends.cudnn.benchmark = False
    torch.backends.cudnn.deterministic = True
    torch.use_deterministic_algorithms(True)
    model, opt, step = build(a.batch)
    lossbuf = torch.zeros(max(a.steps, 3), device="cuda")
    for i in range(2):
        lossbuf[i].copy_(step())
    with torchmem.Tracer(dispatch=False) as tr:
        for i in range(3):
            lossbuf[i].copy_(step())
            tr.mark()
    arrays = tr.trace()
    plan, prof, slots = torchmem.plan_iteration(arrays)
    arena = torchmem.first_fit_arena_peak(arrays, prof.window)
    # snapshot, passthrough reference losses, restore, serve
    snap_m = {k: v.clone() for k, v in model.state_dict().items()}
    snap_o = {k: {kk: vv.clone() if torch.is_tensor(vv) else vv for kk, vv in v.items()}
              for k, v in opt.state_dict()["state"].items()}
    params = list(model.parameters())
    snap_mom = [opt.state[p]["momentum_buffer"].clone() for p in params]
    snap_rng = torch.cuda.get_rng_state()  # dropout masks

    def restore():
        # in-place copies: no allocation, so the served slot order is untouched
        torch.cuda.set_rng_state(snap_rng)
        with torch.no_grad():
            for k, v in model.state_dict().items():
                v.copy_(snap_m[k])
            for p, mb in zip(params, snap_mom):
                opt.state[p]["momentum_buffer"].copy_(mb)

    ms_pass, losses_pass = timed(step, a.steps, lossbuf)
    restore()
    _ms, losses_pass2 = timed(step, a.steps, lossbuf)
    restore()
    torchmem.serve(plan.footprint_bytes, slots)

    def served_step():
        torchmem.begin_iteration()
        return step()
    cs0 = torchmem.call_stats()
    ms_serve, losses_serve = timed(served_step, a.steps, lossbuf)
    cs1 = torchmem.call_stats()
    restore()
    _ms, losses_serve2 = timed(served_step, a.steps, lossbuf)
    st = torchmem.stats()
    if os.environ.get("MP_DEBUG_ORDER"):
        # order of mallocs (by ordinal) and frees in one served iteration vs the trace window
        torchmem.ctl().mp_alloc_logging(1)
        torchmem.Tracer._drain()
        lossbuf[0].copy_(served_step())
        torch.cuda.synchronize()
        torchmem.ctl().mp_alloc_logging(0)
        _seq, kind, ptr, _size = torchmem.Tracer._drain()
        k = 0
        owner = {}
        served = []
        for kd, p in zip(kind.tolist(), ptr.tolist()):
            if kd == 0:
                owner[p] = k
                served.append(("m", k))
                k += 1
            elif p in owner:
                served.append(("f", owner.pop(p)))
        win = []
        s0, s1 = prof.window
        mord = {}
        kk = 0
        for i in range(s0, s1):
            if arrays.kind[i] == 0 and not arrays.names[arrays.var[i]].startswith(torchmem.MARK_NAME):
                mord[int(arrays.var[i])] = kk
                win.append(("m", kk))
                kk += 1
            elif arrays.kind[i] == 1 and int(arrays.var[i]) in mord:
                win.append(("f", mord[int(arrays.var[i])]))
        print("ORDER served", served[:400])
        print("ORDER trace ", win[:400])
    torchmem.passthrough()
    child = subprocess.run([sys.executable, __file__, "--child", "--batch", str(a.batch), "--steps", str(a.steps)],
                           capture_output=True, text=True)
    ref = json.loads(child.stdout.strip().splitlines()[-1]) if child.returncode == 0 else {"error": child.stderr[-400:]}
    print(json.dumps({
        "config": f"vgg16_b{a.batch}", "events": len(arrays), "period": prof.period,
        "window": list(prof.window), "marks": len(tr.marks), "slots": int(len(slots[0])),
        "window_vars": prof.nvars, "peak_load_bytes": plan.peak_load_bytes,
        "smartpool_footprint_bytes": plan.footprint_bytes, "alpha": plan.competitive_ratio,
        "cnmem_style_first_fit_bytes": arena,
        "smartpool_vs_first_fit": 1 - plan.footprint_bytes / arena if arena else None,
        "torch_caching_max_reserved": ref.get("max_reserved"), "torch_caching_max_allocated": ref.get("max_allocated"),
        "iter_ms_served": ms_serve, "iter_ms_passthrough": ms_pass, "iter_ms_torch_default": ref.get("ms"),
        "allocator": st, "hook_us_per_call": {
            k: (cs1[k + "_ns"] - cs0[k + "_ns"]) / (cs1[k + "_calls"] - cs0[k + "_calls"]) / 1e3
            if cs1[k + "_calls"] > cs0[k + "_calls"] else None
            for k in ("alloc", "free")},
        "hook_calls_per_iter": {k: (cs1[k + "_calls"] - cs0[k + "_calls"]) / a.steps for k in ("alloc", "free")},
        "clashes": torchmem.clash_log()[:12],
        "served_losses_equal_passthrough": losses_serve == losses_pass,
        "losses_served": losses_serve[:6], "losses_passthrough": losses_pass[:6],
        "passthrough_repeatable": losses_pass == losses_pass2, "served_repeatable": losses_serve == losses_serve2,
        "losses_torch_default": (ref.get("losses") or [])[:6],
        "note": "footprints cover the iteration window; persistent weights/optimizer state are counted in the plan"}))


if __name__ == "__main__":
    main()
