"""Build libflowrec_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2602_15883_b200.build [--force] [-j N]

The translation units (one per kernel mode plus the C ABI) are compiled in
parallel and linked into ``paper_2602_15883_b200/_lib/libflowrec_b200.so``.
Rebuilds only when a source or header is newer than the library.
"""

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libflowrec_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
# kept object files (incremental rebuilds); git- and gpurun-ignored
OBJ_DIR = os.path.join(os.path.dirname(HERE), "build", "obj")

SOURCES = (["capi.cu", "nccl_transport.cu", "wide_f32.cu", "wide_f64.cu", "tc_probe.cu", "tcwide_f32.cu"]
           + [f"jetmlp_{m}_{d}.cu" for m in ("pde", "epoch", "mse", "value", "jet", "gj") for d in ("f32", "f64")])
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-warn-spills",
]


def _nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(INCLUDE, "flowrec_b200.h"))
    return files


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps())


def _includes(path, seen=None):
    """The file and every local header it includes, transitively."""
    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line.startswith("#include \""):
                name = line.split('"')[1]
                for d in (os.path.dirname(path), CSRC, INCLUDE):
                    cand = os.path.join(d, name)
                    if os.path.exists(cand):
                        _includes(cand, seen)
                        break
    return seen


def _compile(src, defines=(), out_dir=OUT_DIR, force=False):
    obj = os.path.join(out_dir, os.path.splitext(src)[0] + ".o")
    extra = os.environ.get("FR_NVCC_EXTRA", "").split()  # side-build experiments only
    if not force and not defines and not extra and out_dir == OBJ_DIR and os.path.exists(obj):
        t = os.path.getmtime(obj)
        if all(os.path.getmtime(f) <= t for f in _includes(os.path.join(CSRC, src))):
            return obj, ""  # object up to date with its source and headers
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-c", os.path.join(CSRC, src),
           "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force=False, jobs=None, verbose=False, defines=(), lib=None):
    """Compile every CUDA translation unit for sm_100a and link the shared library.

    `defines` / `lib` produce instrumented side builds (e.g. FR_PHASE_TIMERS into
    another path, selected at run time with FLOWREC_B200_LIB)."""
    lib = lib or LIB
    if not force and lib == LIB and not needs_build():
        return LIB
    keep = lib == LIB and not defines
    out_dir = OBJ_DIR if keep else os.path.dirname(os.path.abspath(lib))
    os.makedirs(out_dir, exist_ok=True)
    os.makedirs(os.path.dirname(os.path.abspath(lib)), exist_ok=True)
    jobs = jobs or min(len(SOURCES), os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        results = list(ex.map(lambda src: _compile(src, defines, out_dir, force), SOURCES))
    for obj, log in results:
        if verbose and log.strip():
            print(log, file=sys.stderr)
    tmp = lib + ".tmp"
    cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
           *[o for o, _ in results], "-o", tmp, "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    if not keep:
        for o, _ in results:
            os.remove(o)
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", "--jobs", type=int, default=None)
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("-D", "--define", action="append", default=[], help="extra -D for an instrumented side build")
    ap.add_argument("--lib", default=None, help="output path (side builds)")
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.jobs, verbose=a.verbose, defines=a.define, lib=a.lib))


if __name__ == "__main__":
    main()
