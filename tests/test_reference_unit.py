"""The reference's own unit tests (`proj/tests/unit/*.cpp`: scheduler, temporal, spectrum,
archive, analysis, pairwise, image_stack, synth, bench; 121 test cases), compiled UNCHANGED
against this repo's drop-in headers (`include/ddm/*.hpp`) and linked with libddm_b200.so by
`oracle/Makefile` (`make -C oracle unit`, run from `__graft_entry__.build()` where
/root/reference exists). doctest is absent from this image; `oracle/doctest_shim/doctest.h`
supplies the subset those files use. Every `ddm::run` they make runs on the B200."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
UNIT = ROOT / "oracle" / "_ref" / "unit_tests"


@pytest.mark.gpu
def test_reference_unit_tests_pass():
    if not UNIT.exists():
        pytest.skip("reference unit tests not built (needs /root/reference at build time)")
    from paper_2012_05695_b200 import ddm
    if ddm.device_count() < 1:
        pytest.skip("no CUDA device")
    r = subprocess.run([str(UNIT)], capture_output=True, text=True, timeout=1800, cwd="/tmp")
    print(r.stdout[-2000:])
    print(r.stderr[-6000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-6000:]
    assert "| 0 failed |" in r.stdout
