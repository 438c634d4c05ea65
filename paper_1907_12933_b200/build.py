"""Build the sm_100a shared library libmlpv.so in-tree (nvcc cross-compiles without a GPU)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmlpv.so")
SOURCES = ["mlpv.cu", "k_small.cu", "k_warp.cu", "k_tc3.cu", "k_large.cu", "k_fused3.cu", "k_util.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "mlpv.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """trace=True builds the debug variant libmlpv_trace.so (k_fused3 timeline stamps, -DMLPV_TRACE)."""
    lib = LIB.replace(".so", "_trace.so") if trace else LIB
    if os.environ.get("MLPV_LIB_OUT"):
        lib = os.path.join(HERE, os.environ["MLPV_LIB_OUT"])
    if not force and not _stale(lib):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    extra = ["-DMLPV_TRACE"] if trace else []
    if trace and os.environ.get("MLPV_EXP"):          # timing experiments (results are wrong by design)
        extra.append(f"-DMLPV_EXP={int(os.environ['MLPV_EXP'])}")
    if os.environ.get("MLPV_WAIT_TIMEOUT"):            # debug: trap instead of hanging on a lost arrive
        extra.append(f"-DMLPV_WAIT_TIMEOUT={int(os.environ['MLPV_WAIT_TIMEOUT'])}")
    if os.environ.get("MLPV_EXTRA_DEFS"):              # A/B variants: extra -D flags, built to MLPV_LIB_OUT
        extra += os.environ["MLPV_EXTRA_DEFS"].split()
    cmd = [NVCC, *FLAGS, *extra, "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
