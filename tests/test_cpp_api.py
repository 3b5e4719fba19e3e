"""The reference-named C++ API (include/ddm/*.hpp) as a C++ caller uses it: host-only drivers
under tests/cpp/ are compiled against include/ and linked with libddm_b200.so, then run
(CPU; they make no device calls)."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB_DIR = ROOT / "paper_2012_05695_b200"


def _build_and_run(tmp_path, name):
    c_src = (ROOT / "tests" / "cpp" / f"{name}.c").exists()
    cxx = (shutil.which("gcc") or shutil.which("cc")) if c_src else (shutil.which("g++") or shutil.which("c++"))
    if cxx is None or not (LIB_DIR / "libddm_b200.so").exists():
        pytest.skip("no C/C++ compiler or library not built")
    exe = tmp_path / name
    std = "-std=c11" if c_src else "-std=c++20"
    src = ROOT / "tests" / "cpp" / (f"{name}.c" if c_src else f"{name}.cpp")
    subprocess.run([cxx, std, "-O1", f"-I{ROOT / 'include'}", str(src),
                    f"-L{LIB_DIR}", "-lddm_b200", f"-Wl,-rpath,{LIB_DIR}", "-o", str(exe)],
                   check=True, capture_output=True, text=True, timeout=300)
    r = subprocess.run([str(exe), str(tmp_path / "work")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("OK")


@pytest.mark.parametrize("name", ["archive_api", "analysis_api", "header_api"])
def test_cpp_driver(tmp_path, name):
    _build_and_run(tmp_path, name)


@pytest.mark.gpu
def test_c_session_api_on_device(tmp_path):
    """A plain C program drives the staging session through include/ddm_b200.h on the B200."""
    _build_and_run(tmp_path, "session_api")


@pytest.mark.gpu
def test_cpp_run_api_on_device(tmp_path):
    """a C++ program compiled against include/ddm/*.hpp runs ddm::run,
    ddm::compare and ddm::analyze on the B200 through libddm_b200.so."""
    _build_and_run(tmp_path, "run_api")


@pytest.mark.gpu
def test_cpp_transform_objects_on_device(tmp_path):
    """ddm::SpatialTransform / ddm::TemporalTransform (include/ddm/fft.hpp, the reference's
    `fft.hpp` seams) on the B200 against a direct long-double DFT: f32 within 2e-6 / 3e-6 and
    f64 within 1e-13 of the largest output magnitude, odd and prime lengths included."""
    _build_and_run(tmp_path, "fft_api")
