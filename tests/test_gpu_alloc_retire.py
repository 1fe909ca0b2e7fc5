"""Allocator ABI (include/memplan_alloc.h) on the device: a pool replaced by
a new plan stays mapped while a block served from it is still referenced,
and is released when that block is freed (no address range can be handed
out twice).  Runs in a fresh process: the allocator state is process-wide."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import ctypes as C, sys
L = C.CDLL(sys.argv[1])
rt = C.CDLL("libcudart.so.12")
L.mp_torch_alloc.restype = C.c_void_p
L.mp_torch_alloc.argtypes = [C.c_ssize_t, C.c_int, C.c_void_p]
L.mp_torch_free.argtypes = [C.c_void_p, C.c_ssize_t, C.c_int, C.c_void_p]
L.mp_alloc_pool_base.restype = C.c_int64
MB = 1 << 20

def plan(pool, offs, sizes):
    n = len(offs)
    o = (C.c_int64 * max(n, 1))(*offs); s = (C.c_int64 * max(n, 1))(*sizes)
    assert L.mp_alloc_set_plan(C.c_int64(pool), C.c_int64(n), o, s) == 0

def stats():
    out = (C.c_int64 * 10)(); L.mp_alloc_stats(out); return list(out)

plan(2 * MB, [0, MB], [MB, MB])
L.mp_alloc_mode(1); L.mp_alloc_begin_iteration()
base_a = L.mp_alloc_pool_base()
p0 = L.mp_torch_alloc(MB, 0, None); p1 = L.mp_torch_alloc(MB, 0, None)
assert (p0, p1) == (base_a, base_a + MB), (p0, p1, base_a)
assert rt.cudaMemset(C.c_void_p(p0), 0xAB, C.c_size_t(MB)) == 0
L.mp_torch_free(C.c_void_p(p1), MB, 0, None)
plan(4 * MB, [0], [MB])                       # p0 still referenced
assert stats()[9] == 1, stats()
base_b = L.mp_alloc_pool_base()
assert not (base_a <= base_b < base_a + 2 * MB) and not (base_b <= base_a < base_b + 4 * MB)
L.mp_alloc_begin_iteration()
q = L.mp_torch_alloc(MB, 0, None)
assert q == base_b
buf = (C.c_ubyte * MB)()
assert rt.cudaMemcpy(buf, C.c_void_p(p0), C.c_size_t(MB), 2) == 0   # the retired block is intact
assert buf[0] == 0xAB and buf[MB - 1] == 0xAB
L.mp_torch_free(C.c_void_p(p0), MB, 0, None)  # last block: the old pool goes
assert stats()[9] == 0, stats()
L.mp_torch_free(C.c_void_p(q), MB, 0, None)
plan(MB, [0], [MB])                           # nothing live: released at once
assert stats()[9] == 0, stats()
assert rt.cudaDeviceSynchronize() == 0
print("ok")
"""


def test_retired_pool_stays_mapped_until_last_block_freed():
    lib = os.path.join(ROOT, "paper_1903_06631_b200", "libmemplan_alloc.so")
    p = subprocess.run([sys.executable, "-c", SCRIPT, lib], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.strip() == "ok", p.stdout + p.stderr
