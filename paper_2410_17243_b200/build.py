"""Build libinfcl.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libinfcl.so")
DIAG_OUT = os.path.join(HERE, "libinfcl_diag.so")  # probes / microbenchmarks (include/infcl_diag.h), not the product
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "--expt-relaxed-constexpr", "-Xptxas", "-v",
         "-I" + os.path.join(HERE, "..", "include")]


def _compile(src, build_dir=BUILD, extra=()):
    obj = os.path.join(build_dir, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(HERE, "..", "include", "*.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(p) for p in deps):
        return obj, ""
    cmd = [NVCC] + FLAGS + list(extra) + ["-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stdout}\n{p.stderr}")
    return obj, p.stderr


def _link(objs, out, exports):
    """Link `objs` into `out`, exporting only the C symbols matching the `exports` globs (version script): the
    product library exports exactly include/infcl.h, the diagnostic library exactly include/infcl_diag.h."""
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(o) for o in objs):
        return out
    vs = out + ".map"
    with open(vs, "w") as f:
        f.write("{ global: " + " ".join(e + ";" for e in exports) + " local: *; };\n")
    tmp = out + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs + \
        ["-ldl", "-lcudart", "-Xlinker", "--version-script=" + vs]
    p = subprocess.run(cmd, capture_output=True, text=True)
    os.remove(vs)
    if p.returncode:
        raise RuntimeError(f"link failed:\n{p.stdout}\n{p.stderr}")
    os.replace(tmp, out)  # atomic: a failed link never removes a working library
    return out


def build(verbose=False, out=OUT, extra=(), diag=True):
    """``extra`` nvcc flags + ``out`` build an A/B variant of the library (scripts/build_variant.py) in its own
    object directory; the default builds the product library and the diagnostic library."""
    build_dir = BUILD if out == OUT else out + ".objs"
    os.makedirs(build_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    dsrcs = sorted(glob.glob(os.path.join(CSRC, "diag", "*.cu"))) if diag and out == OUT else []
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs) + len(dsrcs))) as ex:
        res = list(ex.map(lambda s: _compile(s, build_dir, extra), srcs + dsrcs))
    if verbose:
        for _, log in res:
            if log:
                print(log)
    objs = [o for o, _ in res[:len(srcs)]]
    _link(objs, out, ["infcl_*"])
    if dsrcs:
        host = [o for o in objs if os.path.basename(o).startswith("host_utils")]
        _link([o for o, _ in res[len(srcs):]] + host, DIAG_OUT, ["infcl_probe_*", "infcl_diag_*"])
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
