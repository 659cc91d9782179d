"""Builds a variant of libmsa.so with extra -D defines (A/B experiments; load with MSA_LIB=path).
usage: python tools/build_variant.py TAG DEF1=V1 [DEF2=V2 ...] [-nvcc-flag ...] -> paper_2510_16154_b200/variants/libmsa_TAG.so"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_16154_b200 import _build  # noqa: E402

tag = sys.argv[1]
defs = ("MSA_TESTING",) + tuple(a for a in sys.argv[2:] if not a.startswith("-"))
flags = tuple(a for a in sys.argv[2:] if a.startswith("-"))  # raw nvcc flags, e.g. -Xptxas=...
out_dir = os.path.join(_build.PKG, "variants")
lib = os.path.join(out_dir, f"libmsa_{tag}.so")
print(_build.build(force=True, defines=defs, lib=lib, build_dir=os.path.join(out_dir, "build_" + tag), flags=flags))
