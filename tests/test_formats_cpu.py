"""Wire formats next to the reference's own writers: FLO1 flow dumps
(flow.hpp:347-389) and P4 mask files (pgm.hpp:127-138), byte for byte; the PBM rows the GPU
writes (FROI_MASK_PBM) are exactly the P4 raster."""
import os
import subprocess

import numpy as np
import pytest

from paper_2511_14419_b200 import flowroi
from paper_2511_14419_b200.params import DataError


@pytest.fixture(scope="module")
def ref_formats():
    """oracle/_ref/ref_formats: the reference's writers compiled in place (own process)."""
    from oracle.oracle_py import ensure_built
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "ref_formats")
    try:
        ensure_built(reference=True)
    except Exception:
        pass
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_formats not built (needs the reference tree)")
    return exe


@pytest.mark.parametrize("w,h", [(1, 1), (7, 3), (64, 48), (33, 17)])
def test_flo_bytes_match_reference(tmp_path, ref_formats, w, h):
    rng = np.random.default_rng(w * 100 + h)
    u = (rng.standard_normal((h, w)) * 3).astype(np.float32)
    v = (rng.standard_normal((h, w)) * 3).astype(np.float32)
    u.flat[0] = -0.0
    ours, theirs = tmp_path / "a.flo", tmp_path / "b.flo"
    flowroi.save_flo(str(ours), u, v)
    (tmp_path / "u.f32").write_bytes(u.astype("<f4").tobytes())
    (tmp_path / "v.f32").write_bytes(v.astype("<f4").tobytes())
    subprocess.run([ref_formats, "flo", str(w), str(h), str(tmp_path / "u.f32"), str(tmp_path / "v.f32"),
                    str(theirs)], check=True)
    assert ours.read_bytes() == theirs.read_bytes()
    u2, v2 = flowroi.load_flo(str(ours))
    assert u2.tobytes() == u.tobytes() and v2.tobytes() == v.tobytes()


@pytest.mark.parametrize("w,h", [(1, 1), (8, 2), (13, 5), (64, 64), (161, 9)])
def test_pbm_bytes_match_reference(tmp_path, ref_formats, w, h):
    rng = np.random.default_rng(w + 7 * h)
    m = (rng.random((h, w)) < 0.3).astype(np.uint8)
    ours, rows_file, theirs = tmp_path / "a.pbm", tmp_path / "r.pbm", tmp_path / "b.pbm"
    flowroi.save_pbm(str(ours), m)
    flowroi.save_pbm(str(rows_file), np.packbits(m, axis=1), width=w)  # GPU PBM-row layout
    (tmp_path / "m.u8").write_bytes(m.tobytes())
    subprocess.run([ref_formats, "pbm", str(w), str(h), str(tmp_path / "m.u8"), str(theirs)], check=True)
    assert ours.read_bytes() == theirs.read_bytes() == rows_file.read_bytes()


def test_flo_errors(tmp_path):
    p = tmp_path / "bad.flo"
    p.write_bytes(b"NOPE" + bytes(8))
    with pytest.raises(DataError):
        flowroi.load_flo(str(p))
    p.write_bytes(b"FLO1" + np.array([4, 4], "<u4").tobytes() + bytes(10))
    with pytest.raises(DataError):
        flowroi.load_flo(str(p))
    with pytest.raises(DataError):
        flowroi.load_flo(str(tmp_path / "missing.flo"))
    with pytest.raises(DataError):
        flowroi.save_flo(str(tmp_path / "x.flo"), np.zeros((2, 2)), np.zeros((2, 3)))
