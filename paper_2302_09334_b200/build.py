"""Build libsim.so (all CUDA kernels + the C ABI) in-tree for sm_100a with nvcc."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsim.so")
SOURCES = ["api.cu", "world.cu", "step.cu", "band.cu"]
HEADERS = ["sim_internal.cuh", "block_scan.cuh", "phases.cuh", "api_band.inc", "policy_cnn.cuh", "coloc.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
    "-shared", "-cudart", "shared",
    # plain loads are cached in L2 only: the cooperative kernel's phases read state written
    # by other blocks earlier in the same launch, which a stale L1 line would hide
    "-Xptxas", "-dlcm=cg",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "sim.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


CHECKED = os.path.join(HERE, "libsim_checked.so")  # diagnostic: device asserts (-DECO_CHECKS=1)


def build_checked(force: bool = False) -> str:
    """The diagnostic variant with device-side bounds asserts (tests/test_gpu_checks.py)."""
    if not force and os.path.exists(CHECKED) and os.path.getmtime(CHECKED) >= os.path.getmtime(LIB) and not _stale():
        return CHECKED
    return build(force=True, defines=("ECO_CHECKS=1",), out=CHECKED)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """Build LIB (or, for diagnostic variants with extra -D defines, `out`)."""
    lib = out or LIB
    if not force and not defines and not _stale():
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *(f"-D{d}" for d in defines), *(os.path.join(CSRC, s) for s in SOURCES), "-o", tmp]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
