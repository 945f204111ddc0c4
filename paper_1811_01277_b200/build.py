"""Build the C-ABI library libelpa_b200.so in-tree (sm_100a SASS only, static cudart).
The translation units (FP64, FP32 and complex paths) compile in parallel, then link."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libelpa_b200.so")
SOURCES = [os.path.join(CSRC, "elpa_b200.cu"), os.path.join(CSRC, "elpa_b200_f32.cu"),
           os.path.join(CSRC, "elpa_b200_c64.cu"), os.path.join(CSRC, "elpa_b200_dense.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
    [os.path.join(ROOT, "include", "elpa_b200.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
                 "-I", os.path.join(ROOT, "include")]
# ELPA_B200_DEBUG=1: debug build with the kernels' wait watchdog (trap after ~10 s of wall time)
if os.environ.get("ELPA_B200_DEBUG") == "1":
    CFLAGS += ["-DELPA_B200_WATCHDOG"]
# development A/B builds only (tools/ab_run.sh): extra preprocessor flags, e.g. "-DKWIN_ABL=1"
CFLAGS += os.environ.get("ELPA_B200_DEV_CFLAGS", "").split()
LFLAGS = ARCH + ["-shared", "-cudart", "static"]


def stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in DEPS)


def _run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force=False, verbose=False):
    if not force and not stale():
        return SO
    objs = [os.path.join(CSRC, os.path.basename(s)[:-3] + ".o") for s in SOURCES]
    cmds = [[NVCC] + CFLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-c", "-o", o, s]
            for s, o in zip(SOURCES, objs)]
    with ThreadPoolExecutor(len(cmds)) as ex:
        results = list(ex.map(_run, cmds))
    for r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libelpa_b200.so")
        if verbose:
            sys.stderr.write(r.stderr)
    r = _run([NVCC] + LFLAGS + ["-o", SO] + objs)
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libelpa_b200.so")
    return SO


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(SO)
