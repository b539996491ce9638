"""In-tree build of libsvt_b200.so (hand-written sm_100a CUDA + C++ host
engine behind include/svt_b200.h).  nvcc cross-compiles without a GPU."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "lib")
OUT = os.path.join(OUT_DIR, "libsvt_b200.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["rng.cu", "sparse.cu", "dense.cu", "ozaki.cu", "build.cu", "cutlass_gemm.cu", "io.cpp", "runtime.cpp", "host.cpp", "engine.cpp", "solver.cpp", "capi.cpp",
           "synth.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _needs(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "svt_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def cutlass_include():
    """The vendored CUTLASS / CuTe header tree (flashinfer's copy, else tilelang's)."""
    import importlib.util
    for mod, rel in (("flashinfer", ("data", "cutlass", "include")), ("tilelang", ("3rdparty", "cutlass", "include"))):
        spec = importlib.util.find_spec(mod)
        if spec is None or not spec.submodule_search_locations:
            continue
        for loc in spec.submodule_search_locations:
            p = os.path.join(loc, *rel)
            if os.path.exists(os.path.join(p, "cutlass", "gemm", "device", "gemm.h")):
                return p
    raise RuntimeError("CUTLASS headers not found (flashinfer / tilelang site-packages)")


def _compile(src):
    s = os.path.join(CSRC, src)
    o = os.path.join(OBJ, src + ".o")
    if not _needs(o, s):
        return o, None
    cmd = [NVCC, *ARCH, *COMMON, "-c", s, "-o", o]
    if src == "cutlass_gemm.cu":
        cmd = [NVCC, *ARCH, *COMMON, "-I", cutlass_include(), "-c", s, "-o", o]
    if src.endswith(".cpp"):
        cmd = [NVCC, *ARCH, *COMMON, "-x", "cu", "-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return o, (r.returncode, " ".join(cmd), r.stdout + r.stderr)


def build(verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(OUT_DIR, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, SOURCES))
    relink = not os.path.exists(OUT)
    for o, res in results:
        if res is not None:
            rc, cmd, log = res
            if rc != 0:
                raise RuntimeError(f"nvcc failed:\n{cmd}\n{log}")
            if verbose and log.strip():
                print(log)
            relink = True
        elif os.path.getmtime(o) > os.path.getmtime(OUT) if os.path.exists(OUT) else True:
            relink = True
    if relink:
        objs = [o for o, _ in results]
        cmd = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}{r.stderr}")
    build_cli()
    return OUT


CLI_SRC = os.path.join(HERE, "tools", "svt_main.cpp")
CLI = os.path.join(HERE, "bin", "svt")


def build_cli():
    """The `svt` front end (tools/svt_main.cpp): plain C++ over the C ABI of
    libsvt_b200.so, found at run time through an $ORIGIN-relative rpath."""
    os.makedirs(os.path.dirname(CLI), exist_ok=True)
    deps = [CLI_SRC, OUT, os.path.join(HERE, "..", "include", "svt_b200.h")]
    if os.path.exists(CLI) and all(os.path.getmtime(d) <= os.path.getmtime(CLI) for d in deps):
        return CLI
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-Wall", "-Wextra", CLI_SRC, "-o", CLI,
           "-L", OUT_DIR, "-lsvt_b200", "-Wl,-rpath,$ORIGIN/../lib"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"svt CLI build failed:\n{' '.join(cmd)}\n{r.stdout}{r.stderr}")
    return CLI


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
