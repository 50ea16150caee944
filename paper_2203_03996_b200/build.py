"""Build libdcnn.so (sm_100a) in-tree with nvcc.

    python -m paper_2203_03996_b200.build
"""
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdcnn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-I", os.path.join(HERE, "..", "include")]


EXTRA = os.environ.get("DCNN_EXTRA_NVCC_FLAGS", "").split()
SUFFIX = os.environ.get("DCNN_BUILD_SUFFIX", "")


def _compile(src):
    obj = os.path.join(CSRC, "build" + SUFFIX, os.path.basename(src) + ".o")
    dep_newer = False
    if os.path.exists(obj):
        t = os.path.getmtime(obj)
        for f in os.listdir(CSRC):
            if f.endswith((".cu", ".cuh", ".h")) and os.path.getmtime(os.path.join(CSRC, f)) > t:
                dep_newer = True
        if os.path.getmtime(os.path.join(HERE, "..", "include", "dcnn.h")) > t:
            dep_newer = True
    if os.path.exists(obj) and not dep_newer:
        return obj, ""
    cmd = [NVCC, *FLAGS, *EXTRA, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose=False):
    os.makedirs(os.path.join(CSRC, "build" + SUFFIX), exist_ok=True)
    srcs = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))
    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        res = list(ex.map(_compile, srcs))
    if verbose:
        for o, err in res:
            if err.strip():
                print(err)
    objs = [o for o, _ in res]
    lib = LIB if not SUFFIX else LIB.replace(".so", SUFFIX + ".so")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, *objs,
           "-Xcompiler", "-fPIC", "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
