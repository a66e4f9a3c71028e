"""Build an A/B variant of libinfcl.so with extra nvcc flags: python scripts/build_variant.py NAME -DFOO=1 ...
Output: variants/libinfcl_NAME.so (git-ignored; travels to the GPU box); select with INFCL_LIB=... ."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2410_17243_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(os.path.dirname(B.HERE), "variants"), exist_ok=True)
print(B.build(out=os.path.join(os.path.dirname(B.HERE), "variants", f"libinfcl_{name}.so"), extra=extra))
