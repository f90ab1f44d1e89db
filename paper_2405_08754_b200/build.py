"""Build libhrp.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

Each translation unit compiles to build/<name>.o in parallel; a unit is rebuilt when it or any
local header it includes is newer than its object.  Then one link step."""
import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
OUT = os.path.join(HERE, "libhrp.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec else []
    roots.append(os.path.join(sysconfig.get_paths()["purelib"], "nvidia"))
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("nccl headers not found (nvidia/nccl in site-packages)")


SOURCES = ["hrp_api.cu", "tables.cpp", "gemm_tc.cu"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _deps(path, seen=None):
    """The file and every local header it includes (recursively)."""
    seen = set() if seen is None else seen
    path = os.path.normpath(path)
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    for ln in open(path, errors="replace"):
        ln = ln.strip()
        if ln.startswith("#include") and '"' in ln:
            _deps(os.path.join(os.path.dirname(path), ln.split('"')[1]), seen)
    return seen


def build(verbose: bool = False, force: bool = False) -> str:
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    inc, lib = nccl_dirs()
    os.makedirs(OBJ, exist_ok=True)
    flags = ["-O3", "-lineinfo", "-std=c++17", ARCH, "-Xcompiler", "-fPIC",
             "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3", "-I", inc]

    def compile_one(src):
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
        if not force and _mtime(o) > max(_mtime(d) for d in _deps(s)):
            return o, None
        cmd = [nvcc, *flags, "-c", s, "-o", o + ".tmp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            return o, r.stdout + r.stderr
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(o + ".tmp", o)
        return o, None

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        res = list(ex.map(compile_one, SOURCES))
    errs = [e for _, e in res if e]
    if errs:
        sys.stderr.write("\n".join(errs))
        raise RuntimeError("nvcc failed")
    objs = [o for o, _ in res]
    if not force and _mtime(OUT) > max(_mtime(o) for o in objs):
        return OUT
    cmd = [nvcc, ARCH, "-shared", *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{lib}", "-o", OUT + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
