"""The C++ drop-in (include/froi/flowroi_gpu.hpp) next to the reference's own extract_roi, both
feeding the reference encoder (oracle/dropin_test.cpp, built against the unmodified reference
headers by `make -C oracle dropin`)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "dropin_test")


def test_dropin_against_reference_and_encoder():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs the reference tree at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    cases = [c for c in lines if "case" in c]
    assert len(cases) == 6
    for c in cases:
        assert c["shifts_identical"] == c["frames"]
        assert c["mask_mismatch"] <= 1e-4
        # wherever the masks agree, the reference encoder produces identical files
        assert c["encoded_identical"] >= c["frames_identical"]
        if c["case"].startswith("exact-"):  # bit-exact flow: every mask and every file identical
            assert c["mask_mismatch"] == 0.0 and c["frames_identical"] == c["frames"]
            assert c["encoded_identical"] == c["frames"]
    assert lines[-1]["errors_mapped"] == 2
    # compress_sequence with the pipelined GPU stage, when built with json
    for c in [c for c in lines if "pipeline_case" in c]:
        assert c["shifts_identical"] == c["frames"]
        assert c["mask_mismatch"] <= 1e-4
        assert c["files_identical"] >= c["frames_identical"]
