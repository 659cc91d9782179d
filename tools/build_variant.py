"""Builds a variant of libmsa.so with extra -D defines (A/B experiments; load with MSA_LIB=path).
usage: python tools/build_variant.py TAG DEF1=V1 [DEF2=V2 ...] -> paper_2510_16154_b200/variants/libmsa_TAG.so"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_16154_b200 import _build  # noqa: E402

tag, defs = sys.argv[1], tuple(sys.argv[2:])
out_dir = os.path.join(_build.PKG, "variants")
lib = os.path.join(out_dir, f"libmsa_{tag}.so")
print(_build.build(force=True, defines=defs, lib=lib, build_dir=os.path.join(out_dir, "build_" + tag)))
