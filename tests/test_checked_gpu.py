"""The checked build on the B200 (the memory-safety check this pool allows: compute-sanitizer is
closed on it). libfgs_checked.so is the product's sources compiled with -DFGS_CHECKED: every
kernel's indexing sites check their bounds and invariants on the device and trap on a violation
(csrc/fgs_common.cuh FGS_DCHECK):

* K1 / K2: tile rectangles inside the grid; every key / row-list position inside its tile's range
  [tile_offsets[t], tile_offsets[t+1]) and the buffer;
* K3: tile ranges inside the intersection buffer; sorted-id reads inside the shared sort buffer;
  record ids < N; checkpoint slots < capacity;
* K4a: work items (tile, segment) valid; a long list's checkpoint slots reserved by the forward and
  inside the buffer; per-pixel `last` inside the tile's range; emission slots < I;
* K4b: intersection sums read at slots < I.

Each case runs tests/sanitize_driver.py in a subprocess with FGS_LIB=checked (a trapped kernel
poisons the CUDA context, so the process is the unit), under one kernel-variant selection.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "tests", "sanitize_driver.py")
CHECKED = os.path.join(ROOT, "paper_2409_04751_b200", "libfgs_checked.so")

# (cfg, n, views, flags, env): every kernel variant and scatter order at least once
CASES = [
    pytest.param(0, 0, 1, 0, {}, id="cfg0"),
    pytest.param(0, 0, 1, 0, {"FGS_FWD_PX": "2", "FGS_BWD_PX": "2"}, id="cfg0-px2"),
    pytest.param(1, 0, 1, 0, {}, id="cfg1"),
    pytest.param(1, 0, 1, 96, {}, id="cfg1-global-slots"),
    pytest.param(2, 0, 1, 16, {}, id="cfg2-rows"),
    pytest.param(2, 0, 1, 32, {"FGS_BWD_MINB": "8", "FGS_K4B_MINB": "4"}, id="cfg2-slots-minb8"),
    pytest.param(2, 0, 1, 0, {"FGS_FWD_PX": "1", "FGS_FWD_TMA": "1", "FGS_BWD_PX": "1", "FGS_K4B_MINB": "6"},
                 id="cfg2-tma-px1"),
    pytest.param(3, 300_000, 2, 0, {}, id="cfg3"),
    pytest.param(4, 400_000, 2, 0, {}, id="cfg4"),
]


@pytest.mark.parametrize("cfg,n,views,flags,env", CASES)
def test_checked_build(cfg, n, views, flags, env):
    assert os.path.exists(CHECKED), "libfgs_checked.so not built (python -m paper_2409_04751_b200.build)"
    e = dict(os.environ, FGS_LIB="checked", **env)
    p = subprocess.run([sys.executable, DRIVER, str(cfg), str(n), str(views), str(flags)], env=e, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    out = p.stdout + p.stderr
    assert "FGS_DCHECK failed" not in out, out[-4000:]
    assert p.returncode == 0 and "sanitize-driver ok" in p.stdout, out[-4000:]
    assert "libfgs_checked.so" in p.stdout, out[-2000:]
