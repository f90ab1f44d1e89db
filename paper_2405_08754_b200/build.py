"""Build libhrp.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
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


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + \
        [os.path.join(HERE, "..", "include", "hrp.h")]
    if not force and os.path.exists(OUT) and \
            os.path.getmtime(OUT) > max(os.path.getmtime(d) for d in deps):
        return OUT
    inc, lib = nccl_dirs()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, "-O3", "-lineinfo", "-std=c++17", ARCH, "-Xcompiler", "-fPIC", "-shared",
           "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
           "-I", inc, *srcs, "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}",
           "-o", OUT + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
