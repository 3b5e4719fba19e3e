"""Build the in-tree native library `paper_2012_05695_b200/libddm_b200.so` (sm_100a).

    python -m paper_2012_05695_b200.build          # incremental, parallel nvcc
    python -m paper_2012_05695_b200.build --clean

Sources: csrc/*.cu (kernels + device orchestration) and csrc/host/*.cpp (reference-mirroring
C++ API + the extern "C" boundary declared in include/ddm_b200.h). Objects go to build/;
the .so is written next to this file so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libddm_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fno-fast-math",
          f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{CSRC / 'host'}"]


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted((CSRC / "host").glob("*.cpp"))


def headers():
    return (list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + list((CSRC / "host").glob("*.hpp"))
            + list((ROOT / "include").rglob("*.h*")))


def _obj(src: Path) -> Path:
    rel = src.relative_to(CSRC).as_posix().replace("/", "__")
    return OBJ / (rel + ".o")


def _compile(src: Path, newest_header: float, verbose: bool) -> Path:
    out = _obj(src)
    if out.exists() and out.stat().st_mtime >= max(src.stat().st_mtime, newest_header):
        return out
    cmd = [NVCC, *COMMON, *ARCH, "-c", str(src), "-o", str(out)]
    if src.suffix == ".cu":
        cmd[1:1] = ["--threads", "4"]
    else:
        cmd[1:1] = ["-x", "cu"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}\n{r.stderr}")
    return out


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    newest = max((h.stat().st_mtime for h in headers()), default=0.0)
    srcs = sources()
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, newest, verbose), srcs))
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", str(LIB), *map(str, objs),
               "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def clean() -> None:
    shutil.rmtree(ROOT / "build", ignore_errors=True)
    if LIB.exists():
        LIB.unlink()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("-j", "--jobs", type=int, default=None)
    a = ap.parse_args()
    if a.clean:
        clean()
    print(build(verbose=a.verbose, jobs=a.jobs))
    sys.exit(0)
