"""The runtime side on a real model (configs 2 and 3 of BASELINE.json at a
small batch): a VGG-16 iteration served from the SmartPool plan, and AutoSwap
plans executed under it.  Each runs in a fresh process because the
pluggable allocator must be installed before the first CUDA allocation."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def run_tool(name, *args, timeout=900):
    env = dict(os.environ, CUBLAS_WORKSPACE_CONFIG=":4096:8")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", name), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])


def test_served_iterations_match_passthrough():
    r = run_tool("config2_pool.py", "--batch", "8", "--steps", "4")
    assert r["allocator"]["misses"] == 0 and r["allocator"]["conflicts"] == 0
    assert r["served_losses_equal_passthrough"] and r["served_repeatable"]
    assert r["smartpool_footprint_bytes"] >= r["peak_load_bytes"]


def test_executed_swaps_keep_losses_bit_identical():
    r = run_tool("config3_swap.py", "--batch", "16", "--steps", "3", "--fracs", "0.95,0.9")
    assert r["hooked_losses_equal_plain"]
    ran = [x for x in r["limits"] if "executed" in x]
    assert ran, r["limits"]
    for x in ran:
        assert x["losses_equal_unswapped"], x
        assert x["allocator"]["conflicts"] == 0 and x["allocator"]["misses"] == 0, x
        assert x["pool_arc_peak_bytes"] <= r["noswap_pool_arc_peak_bytes"]
    assert any(x["executed"] > 0 for x in ran)


# ---- the BASELINE batch sizes (configs[1] and configs[2]) ----

@pytest.mark.slow
def test_config2_vgg16_b64_served():
    """VGG-16 batch 64 (BASELINE configs[1]) served from the plan: every
    window malloc hits its planned offset, losses bit-identical to the
    pass-through run, footprint at or above the traced peak load and below
    the online first-fit arena."""
    r = run_tool("config2_pool.py", "--batch", "64", "--steps", "3")
    assert r["allocator"]["misses"] == 0 and r["allocator"]["conflicts"] == 0
    assert r["served_losses_equal_passthrough"] and r["served_repeatable"]
    assert r["peak_load_bytes"] <= r["smartpool_footprint_bytes"] <= r["cnmem_style_first_fit_bytes"]


@pytest.mark.slow
def test_config3_vgg16_b128_executed():
    """VGG-16 batch 128 (BASELINE configs[2]) with the reference's SWDOA
    selection executed at two limits: losses bit-identical to the unswapped
    run, no allocator misses or conflicts, the pool never above the no-swap
    pool, the copies near the measured host-link rate.  The link fraction of
    a 3-step run is one iteration's copies (a shared PCIe link jitters: 63-100
    % seen); the bench's 50-iteration rows report it precisely, so this only
    guards against serialised copies (>= 50 %)."""
    r = run_tool("config3_swap.py", "--batch", "128", "--steps", "3", "--fracs", "0.95,0.85",
                 "--modes", "reference_selection,window_fits")
    assert r["hooked_losses_equal_plain"]
    ran = [x for x in r["limits"] if "executed" in x]
    assert any(x["executed"] > 0 for x in ran), r["limits"]
    for x in ran:
        assert x["losses_equal_unswapped"], x
        assert x["allocator"]["conflicts"] == 0 and x["allocator"]["misses"] == 0, x
        assert x["pool_footprint_bytes"] <= r["noswap_pool_bytes"], x
        if x["executed"]:
            for d in ("d2h", "h2d"):
                assert x["link"][d]["bytes_per_s"] >= 0.5 * r["link_bw_bytes_per_s"][d], (d, x["link"])
