"""Build the in-tree C-ABI library libadasgd.so for sm_100a with nvcc.

Not part of the method: compiles csrc/*.cu and csrc/*.cpp.  The library
links the CUDA runtime statically and NCCL dynamically."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libadasgd.so")
OUT_TRACE = os.path.join(HERE, "libadasgd_trace.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp", "-I", os.path.join(ROOT, "include"),
         "-I", CSRC, "--expt-relaxed-constexpr"]
SOURCES = ["api.cu", "kernels_sparse.cu", "kernels_segmm.cu", "kernels_dense.cu", "kernels_tc.cu", "kernels_transpose.cu",
           "sched.cpp"]


def _needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "adasgd.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False, jobs=5, trace=False, variant=None, defines=()):
    """variant: experiment build libadasgd_x_<variant>.so with extra -D defines
    (tools only; the product library is always the plain build)."""
    out = OUT_TRACE if trace else OUT
    if variant:
        out = os.path.join(HERE, "libadasgd_x_%s.so" % variant)
    if not force and not trace and not variant and not _needs_build():
        return OUT
    objdir = os.path.join(HERE, "build_x_" + variant if variant else ("build_trace" if trace else "build"))
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        cmd = [NVCC] + ARCH + FLAGS + (["-DAS_TRACE"] if trace else []) + ["-D" + d for d in defines] + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd = [NVCC] + FLAGS + ["-x", "cu", "-c", os.path.join(CSRC, src), "-o", obj] + ARCH
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for src, p in procs:
        log, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(log.decode())
        if p.returncode != 0:
            failed = True
            sys.stderr.write("nvcc failed on %s\n" % src)
    if failed:
        raise RuntimeError("build failed")
    link = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", out] + objs + ["-lnccl", "-lrt", "-lgomp"]
    subprocess.check_call(link)
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:      # --variant NAME DEF1,DEF2
        i = sys.argv.index("--variant")
        print(build(variant=sys.argv[i + 1], defines=[d for d in sys.argv[i + 2].split(",") if d]))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
