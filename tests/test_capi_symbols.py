"""The C-ABI library loads on a CPU-only host and exports every entry point that
include/ddm_b200.h declares (no compute calls)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared():
    text = (ROOT / "include" / "ddm_b200.h").read_text()
    return sorted(set(re.findall(r"\b(ddm_b200_[a-z0-9_]+)\s*\(", text)) - {"ddm_b200_before_merge_fn"})


def test_header_declares_the_boundary():
    names = declared()
    for must in ("ddm_b200_run_u16", "ddm_b200_run_device", "ddm_b200_sequences_with_ft",
                 "ddm_b200_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib_path = ROOT / "paper_2012_05695_b200" / "libddm_b200.so"
    if not lib_path.exists():
        pytest.skip("libddm_b200.so not built (python -m paper_2012_05695_b200.build)")
    lib = ctypes.CDLL(str(lib_path))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    lib.ddm_b200_pad_length.restype = ctypes.c_int64
    lib.ddm_b200_pad_length.argtypes = [ctypes.c_int64]
    assert lib.ddm_b200_pad_length(1000) == 2048  # host-only arithmetic, no device needed
    assert lib.ddm_b200_pad_length(0) == -1


def test_host_planning_through_the_abi():
    from paper_2012_05695_b200 import ddm
    if not ddm.LIB_PATH.exists():
        pytest.skip("library not built")
    assert ddm.plan_with_ft(131584, 16384, 23 << 30, "f64") == (94208, 2)
    with pytest.raises(ddm.PlanError):
        ddm.plan_with_ft(10, 1024, 1024, "f64")
    assert len(ddm.cutoff_set(512, 512)) == 131584
    assert ddm.max_frames("f32") >= 8192 and ddm.max_frames("f64") >= 4096
