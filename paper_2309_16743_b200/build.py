"""Build libmel.so in-tree: every CUDA source compiled for sm_100a only
(`-gencode arch=compute_100a,code=sm_100a`), linked against the venv's NCCL.

    python -m paper_2309_16743_b200.build        # incremental
    python -m paper_2309_16743_b200.build --force
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, os.environ.get("MEL_BUILD_NAME", "libmel.so"))   # variant builds (A/B timing)
OBJ = os.path.join(HERE, "build_obj" + os.environ.get("MEL_BUILD_NAME", ""))
SOURCES = ["mel.cu", "reservoir.cu", "mlp_simt.cu", "tc_out.cu", "ingest.cpp", "dataset.cpp", "heat.cu"]
INGEST_OUT = os.path.join(HERE, "libmel_ingest.so")   # host-only, for the simulation clients
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    try:
        import nvidia.nccl as nn  # the torch-bundled NCCL 2.28 (headers + lib)
        base = list(nn.__path__)[0]
    except Exception:
        base = os.path.join(sys.prefix, "lib", "python%d.%d" % sys.version_info[:2], "site-packages", "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _deps_mtime():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", f)
                                                                  for f in ("mel.h", "mel_ingest.h", "mel_dataset.h", "mel_heat.h")]
    return max(os.path.getmtime(f) for f in files)


def build(force: bool = False, verbose: bool = False) -> str:
    inc, lib = nccl_dirs()
    os.makedirs(OBJ, exist_ok=True)
    dep_t = _deps_mtime()
    if (not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= dep_t and os.path.exists(INGEST_OUT)
            and os.path.getmtime(INGEST_OUT) >= dep_t):
        return OUT
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", inc,
                    "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr", "-Xptxas", "-v"]
    flags += os.environ.get("MEL_NVCC_DEFS", "").split()       # -D overrides of tuning macros (A/B builds)

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, "-c", os.path.join(CSRC, src), "-o", obj] + flags
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = OUT + ".tmp"
    cmd = [NVCC, "-shared", "-o", tmp] + objs + ARCH + ["-L", lib, "-l:libnccl.so.2", "-lcudart",
                                                          "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    os.replace(tmp, OUT)
    # the clients' library: the same ingest source, host compiler only, no CUDA dependency
    tmp = INGEST_OUT + ".tmp"
    cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
           os.path.join(CSRC, "ingest.cpp"), "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("ingest library build failed:\n%s\n%s" % (r.stdout, r.stderr))
    os.replace(tmp, INGEST_OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
