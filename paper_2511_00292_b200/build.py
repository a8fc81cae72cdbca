"""Build recipe for the in-tree native artefacts (no torch JIT cache involved).

  paper_2511_00292_b200/_eig33cuda.so   product: sm_100a kernels + C ABI (nvcc)
  oracle/liboracle.so                   checker: C restatement (gcc)
  oracle/_ref/libeig33_ref.so           checker: compiled reference core (only
                                        when /root/reference is present)
  tests/hostmath/libhostmath.so         test harness: product math built for CPU
  tools/probes/libeig33_probes.so       measurement probes for bench.py / tools
                                        (FP64 issue rate, data-path energy);
                                        never linked into the product

Usage: python -m paper_2511_00292_b200.build [--product-only]
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "_eig33cuda.so")
REF = "/root/reference/proj"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo",
    "--fmad=false",          # bit-exact invariants: no contraction (reference proj/src/CMakeLists.txt:9-10)
    "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-ffp-contract=off",
    "-Xptxas", "-v",
]
SOURCES = ["eig33_kernels.cu", "eig33_gen.cu", "eig33_aux.cu", "eig33_host.cpp"]
PROBES_SRC = os.path.join(ROOT, "tools", "probes", "eig33_probes.cu")
PROBES_SO = os.path.join(ROOT, "tools", "probes", "libeig33_probes.so")


def _nvcc():
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _run(cmd, log=None):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if log is not None:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError("command failed: " + " ".join(cmd[:3]) + " ...")
    return r.stdout


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_product(force=False):
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [
        os.path.join(CSRC, h) for h in ("eig33_math.cuh", "eig33_tables.h", "eig33_internal.h",
                                         "eig33_fused.cuh", "eig33_gen_core.h")
    ] + [os.path.join(ROOT, "include", "eig33_cuda.h")]
    if not force and not _stale(SO, deps):
        return SO
    objs = []
    build_dir = os.path.join(HERE, "build")
    os.makedirs(build_dir, exist_ok=True)
    nvcc = _nvcc()
    for s in SOURCES:
        o = os.path.join(build_dir, s + ".o")
        _run([nvcc, *NVCC_FLAGS, "-c", os.path.join(CSRC, s), "-o", o],
             log=os.path.join(build_dir, s + ".log"))
        objs.append(o)
    tmp = SO + ".tmp"
    _run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs,
          "-Xcompiler", "-pthread"])
    os.replace(tmp, SO)
    return SO


def build_variant(name, defines):
    """Experimental build with extra -D flags into build/variants/<name>.so
    (selected at run time with EIG33_SO=...); the product is build_product()."""
    out_dir = os.path.join(HERE, "build", "variants")
    os.makedirs(out_dir, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for s in SOURCES:
        o = os.path.join(out_dir, f"{name}_{s}.o")
        _run([nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, s), "-o", o],
             log=os.path.join(out_dir, f"{name}_{s}.log"))
        objs.append(o)
    so = os.path.join(out_dir, name + ".so")
    _run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", so, *objs,
          "-Xcompiler", "-pthread"])
    return so


def build_probes(force=False):
    deps = [PROBES_SRC] + [os.path.join(CSRC, h) for h in ("eig33_math.cuh", "eig33_tables.h",
                                                             "eig33_fused.cuh", "eig33_gen_core.h")]
    if not force and not _stale(PROBES_SO, deps):
        return PROBES_SO
    tmp = PROBES_SO + ".tmp"
    _run([_nvcc(), *NVCC_FLAGS, "-shared", "-o", tmp, PROBES_SRC],
         log=os.path.join(os.path.dirname(PROBES_SO), "build.log"))
    os.replace(tmp, PROBES_SO)
    return PROBES_SO


def build_oracle():
    make = ["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"]
    _run(make)
    if os.path.isdir(REF):
        _run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref", "REF=" + REF])


def build_hostmath():
    src = os.path.join(ROOT, "tests", "hostmath", "hostmath.cpp")
    out = os.path.join(ROOT, "tests", "hostmath", "libhostmath.so")
    deps = [src, os.path.join(CSRC, "eig33_math.cuh"), os.path.join(CSRC, "eig33_tables.h")]
    if _stale(out, deps):
        _run(["g++", "-O2", "-mfma", "-ffp-contract=off", "-fPIC", "-shared", "-std=c++17",
              "-o", out, src, "-lm"])


REF_CXX_CHECK = os.path.join(ROOT, "tests", "cpp", "batch_api_check_ref")


def build_ref_cxx_check():
    """tests/cpp/batch_api_check.cpp compiled against the REFERENCE's own headers
    (Mat3 / InvariantSet / EigenTriple / NotSymmetric from
    /root/reference/proj/include) and linked with the product library -- built
    here, where the reference exists, and run by the GPU suite (the GPU box has
    no /root/reference).  Test infrastructure; git-ignored, travels with gpurun."""
    if not os.path.isdir(os.path.join(REF, "include")):
        return None
    src = os.path.join(ROOT, "tests", "cpp", "batch_api_check.cpp")
    if not _stale(REF_CXX_CHECK, [src, SO, os.path.join(ROOT, "include", "eig33", "batch.hpp"),
                                  os.path.join(ROOT, "include", "eig33_cuda.h")]):
        return REF_CXX_CHECK
    _run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(REF, "include"),
          src, "-o", REF_CXX_CHECK, SO, "-Wl,-rpath,$ORIGIN/../../paper_2511_00292_b200"])
    return REF_CXX_CHECK


def build_all(force=False):
    build_product(force)
    build_probes(force)
    build_oracle()
    build_hostmath()
    build_ref_cxx_check()


if __name__ == "__main__":
    if "--product-only" in sys.argv:
        print(build_product(force="--force" in sys.argv))
    else:
        build_all(force="--force" in sys.argv)
        print("built", SO)
