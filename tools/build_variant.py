"""Build an A/B variant of libddm_b200.so with extra nvcc defines into ab_libs/<name>.so.

    python tools/build_variant.py <name> -DDDM_F32X2=0 [...]
(objects in build/obj_<name>; load it with DDM_B200_LIB=$PWD/ab_libs/<name>.so)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2012_05695_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
B.OBJ = B.ROOT / "build" / f"obj_{name}"
(B.ROOT / "ab_libs").mkdir(exist_ok=True)
B.LIB = B.ROOT / "ab_libs" / f"{name}.so"
B.COMMON = B.COMMON + defs
print(B.build())
