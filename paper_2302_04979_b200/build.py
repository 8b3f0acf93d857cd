"""Compile the sgm C-ABI library for sm_100a (in-tree .so, travels with the repo snapshot)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsgm.so")
SOURCES = ["host_setup.cpp", "kernels.cu", "hodge.cu", "sweep_p2.cu", "sweep_p3.cu", "sweep_p4.cu", "sweep_p5.cu", "api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC,-fopenmp", "-shared", "-lgomp"]


MARK = os.path.join(HERE, "libsgm.tuning")  # present while libsgm.so is a tuning build
CHECKED_LIB = os.path.join(HERE, "libsgm_checked.so")  # verification build (csrc/check.cuh)


def needs_build(lib=LIB):
    if not os.path.exists(lib) or (lib == LIB and os.path.exists(MARK)):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "sgm.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, tuning=None, checked=False):
    """Compile every translation unit to an object in parallel (the sweep instantiations are split
    per degree), then link the shared library.  tuning=True (or SGM_BUILD_TUNING=1) compiles the
    -DSGM_TUNING variant whose launchers read tuning knobs from the environment -- for experiments
    only; the product library is the default build (tests/test_abi.py refuses a tuning build).
    checked=True compiles the -DSGM_CHECKED verification build into libsgm_checked.so (protocol
    checks, slab poisoning and random delays in the pipelined sweeps, csrc/check.cuh), loaded by
    the binding only when SGM_LIB_VARIANT=checked; the product library is left untouched."""
    if checked:
        if not force and not needs_build(CHECKED_LIB):
            return CHECKED_LIB
        return _compile(CHECKED_LIB, os.path.join(HERE, "_obj_checked"), ["-DSGM_CHECKED"], verbose)
    if tuning is None:
        tuning = os.environ.get("SGM_BUILD_TUNING", "0") == "1"
    if tuning:
        force = True
    if not force and not needs_build():
        return LIB
    _compile(LIB, os.path.join(HERE, "_obj"), ["-DSGM_TUNING"] if tuning else [], verbose)
    if tuning:
        open(MARK, "w").write("tuning build (-DSGM_TUNING)\n")
    elif os.path.exists(MARK):
        os.remove(MARK)
    return LIB


def _compile(lib, objdir, defines, verbose):
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f not in ("-shared", "-lgomp")] + defines

    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC] + cflags + ["-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True, cwd=CSRC)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fopenmp", "-lgomp"] + objs \
        + ["-o", lib + ".tmp"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    import sys
    build(force=True, verbose=True, checked="--checked" in sys.argv)
