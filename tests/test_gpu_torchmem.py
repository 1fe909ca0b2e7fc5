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
