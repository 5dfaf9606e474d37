"""Build an A/B variant of libinferix_b200.so with extra nvcc defines into build_ab_<tag>.so
(own object directory), for same-box comparisons through IFX_LIB_PATH.

    python tools/build_ab.py <tag> -DNAME=VALUE ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
tag, defs = sys.argv[1], sys.argv[2:]
os.environ["IFX_NVCC_EXTRA"] = " ".join(defs)
from paper_2511_20714_b200 import _build  # noqa: E402

_build.OUT = os.path.join(ROOT, f"build_ab_{tag}.so")
_build.OBJ = os.path.join(ROOT, "build", f"obj_{tag}")
print(_build.build(verbose=True))
