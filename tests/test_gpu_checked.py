"""Memory-safety and race evidence without compute-sanitizer (closed on this GPU pool).

* The checked build (``make -C paper_2511_14419_b200/csrc checked`` -> _lib/libfroi_checked.so)
  compiles device-side index asserts (FROI_DCHECK: flow ring slots and bilinear gathers, CCL run
  lists and union-find ids) into the same kernels; a violated bound traps the kernel.  The cases
  of tests/_checked_runner.py must run clean under it and produce the same bytes as the product
  build.
* Determinism (the reference's "outputs never depend on the worker count", parallel.hpp:17-19):
  every batch size (2, 3, 4, 32 pairs) on one or two execution lanes gives byte-identical masks,
  and repeated runs agree — the lock-free CCL union-find, the in-place ring box sums and the
  two-lane buffer reuse would show up here as run-to-run differences.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2511_14419_b200", "_lib")


def _run(lib, out):
    env = dict(os.environ)
    if lib:
        env["FROI_LIB"] = os.path.join(LIB, lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_checked_runner.py"), out],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, (lib, r.stdout[-2000:], r.stderr[-2000:])
    assert "FROI_DCHECK failed" not in r.stdout + r.stderr
    return dict(np.load(out))


def test_checked_build_clean_and_identical(tmp_path):
    if not os.path.exists(os.path.join(LIB, "libfroi_checked.so")):
        pytest.fail("libfroi_checked.so missing: build with __graft_entry__.build()")
    a = _run("libfroi_checked.so", str(tmp_path / "checked.npz"))
    b = _run(None, str(tmp_path / "product.npz"))
    c = _run(None, str(tmp_path / "product2.npz"))
    assert a.keys() == b.keys() == c.keys()
    for k in a:
        assert np.array_equal(a[k], b[k]), f"checked build differs on {k}"
        assert np.array_equal(b[k], c[k]), f"run-to-run difference on {k}"
    ref = b["wells_mp32_l1"]
    for k in b:
        if k.startswith("wells_"):
            assert np.array_equal(b[k], ref), f"batch size / lanes changed the masks ({k})"
