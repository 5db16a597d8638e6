"""Build libqs_b200.so in-tree: nvcc for sm_100a (the only target), linked to the venv's NCCL 2.28.9
(the one torch loads, so a process never maps two NCCLs; SURVEY.md §0 "Environment facts")."""
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libqs_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("venv NCCL (nvidia/nccl) not found")


JIT_HEADERS = ["qs_device.cuh", "qs_tile_types.h", "qs_tile_ops.cuh", "qs_tile_opcodes.inc"]


def gen_jit_headers():
    """Embed the device headers NVRTC compiles (jit_tile.cu) as raw string literals."""
    out = os.path.join(BUILD, "qs_jit_headers.inc")
    parts = ["struct JitHeader { const char *name; const char *text; };", "const JitHeader kJitHeaders[] = {"]
    for h in JIT_HEADERS:
        txt = open(os.path.join(CSRC, h)).read()
        assert ")QSJIT\"" not in txt
        parts.append('    {"%s", R"QSJIT(%s)QSJIT"},' % (h, txt))
    parts.append("};")
    parts.append("const int kJitHeaderCount = %d;" % len(JIT_HEADERS))
    new = "\n".join(parts) + "\n"
    if not os.path.exists(out) or open(out).read() != new:
        with open(out, "w") as f:
            f.write(new)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    inc, lib = nccl_dirs()
    os.makedirs(BUILD, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(CSRC, "*.inc")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    hdr_mtime = max(os.path.getmtime(h) for h in headers)
    gen_jit_headers()
    common = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", BUILD, "-I", inc]
    jobs = []
    objs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp"))):
        if os.path.basename(src) == "qs_jitc.cpp":  # the helper executable, linked below
            continue
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        stale = force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hdr_mtime)
        if not stale:
            continue
        if src.endswith(".cu"):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   *common, "-c", src, "-o", obj]
        else:
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", *common, "-c", src, "-o", obj]
        jobs.append(cmd)
    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        outs = list(ex.map(_run, jobs))
    if verbose:
        for o in outs:
            sys.stdout.write(o)
    if jobs or force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cuda_lib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
        _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
              "-Xlinker", "-rpath," + lib, "-L", cuda_lib, "-lnvrtc", "-Xlinker", "-rpath," + cuda_lib, "-lcudart"])
        os.replace(tmp, LIB)
    # the JIT's background compiler process, beside the library (jit_tile.cu spawns it)
    jitc = os.path.join(PKG, "qs_jitc")
    jitc_src = os.path.join(CSRC, "qs_jitc.cpp")
    if force or not os.path.exists(jitc) or os.path.getmtime(jitc) < max(os.path.getmtime(LIB), os.path.getmtime(jitc_src)):
        tmp = jitc + f".tmp{os.getpid()}"
        _run(["g++", "-O2", "-o", tmp, jitc_src, "-L", PKG, "-l:libqs_b200.so", "-Wl,-rpath,$ORIGIN"])
        os.replace(tmp, jitc)
    # the plain-C use of the C-ABI (examples/qs_hello.c): built beside the library, run by a GPU test
    hello = os.path.join(PKG, "qs_hello")
    hello_src = os.path.join(ROOT, "examples", "qs_hello.c")
    if os.path.exists(hello_src) and (force or not os.path.exists(hello) or
                                      os.path.getmtime(hello) < max(os.path.getmtime(LIB), os.path.getmtime(hello_src))):
        tmp = hello + f".tmp{os.getpid()}"
        _run(["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-Wall", "-I", os.path.join(ROOT, "include"), "-o", tmp,
              hello_src, "-L", PKG, "-l:libqs_b200.so", "-Wl,-rpath,$ORIGIN", "-lm"])
        os.replace(tmp, hello)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
