"""Experiment builds: python scripts/build_variant.py NAME [DEFINE ...] -> _lib/variants/NAME.so
(loads build.py without importing the package, which would load the in-tree library)."""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("expmc_build", os.path.join(ROOT, "paper_1904_12754_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
out = os.path.join(b.LIBDIR, "variants", sys.argv[1] + ".so")
print(b.build(out=out, defines=sys.argv[2:]))
