"""The checked build (in place of compute-sanitizer, which is
closed on this pool): libpic compiled with -DPIC_CHECKED counts every violated
index invariant of the hot kernels (perm / store positions below the capacity,
cell keys below the cell count, order slots inside their cell's segment, node
indices inside the tile box, coalescence scratch inside the store) and pic_sync
fails on any.  tools/sanitize_cases.py launches every libpic kernel family (C1r
on both families, split, overfull-cell coalescence, GMM, sources, injection
with open faces and a planet, a two-slab loopback pair) against that build."""
import os
import subprocess
import sys

import pytest

from paper_2507_20719_b200 import build_lib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_kernel_passes_the_bounds_checks():
    lib = build_lib.build_checked()
    env = dict(os.environ, PIC_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize_cases ok" in r.stdout
