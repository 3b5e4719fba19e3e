"""The reference's own release gate (`proj/tests/acceptance/acceptance_main.cpp`, 9 criteria),
compiled UNCHANGED against this repo's drop-in headers (`include/ddm/*.hpp`) and linked with
libddm_b200.so by `oracle/Makefile` (`make -C oracle gate`, run from `__graft_entry__.build()`
where /root/reference exists). Every criterion runs its `ddm::` calls on the B200."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GATE = ROOT / "oracle" / "_ref" / "release_gate"


@pytest.mark.gpu
def test_reference_release_gate_passes():
    if not GATE.exists():
        pytest.skip("release gate not built (needs /root/reference at build time)")
    from paper_2012_05695_b200 import ddm
    if ddm.device_count() < 1:
        pytest.skip("no CUDA device")
    r = subprocess.run([str(GATE)], capture_output=True, text=True, timeout=1800)
    print(r.stdout)
    assert "passed 9/9 criteria" in r.stdout, r.stdout + r.stderr
    assert r.returncode == 0
