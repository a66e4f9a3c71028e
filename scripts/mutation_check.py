"""CUDA-path mutation check: build four mutated variants of the library (INFCL_MUTATION=k,
kernels.h) and run a parity subset against each; every mutation must be killed (the tests fail).  GPU only."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_17243_b200 import build as B  # noqa: E402

TESTS = ["tests/test_gpu_parity.py", "-x", "-q", "-k", "paired_multi_tile or parity_independent or ragged_feature"]
results = {}
for k in (1, 2, 3, 4):
    lib = os.path.join(ROOT, "variants", f"libinfcl_mut{k}.so")
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    B.build(out=lib, extra=[f"-DINFCL_MUTATION={k}"])
    env = dict(os.environ, INFCL_LIB=lib)
    p = subprocess.run([sys.executable, "-m", "pytest"] + TESTS, cwd=ROOT, env=env, capture_output=True, text=True)
    results[k] = "killed" if p.returncode != 0 else "SURVIVED"
    print(f"mutation {k}: {results[k]}  ({p.stdout.strip().splitlines()[-1] if p.stdout.strip() else ''})", flush=True)
sys.exit(0 if all(v == "killed" for v in results.values()) else 1)
