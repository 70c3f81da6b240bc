"""Build the CUDA C-ABI library ``liblbm_b200.so`` in-tree for sm_100a (nvcc, parallel objects).

Usage: ``python -m paper_2001_11806_b200.build [--force]``. The .so lands next to this file so
it travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "liblbm_b200.so")
OBJ = os.path.join(HERE, "build_obj")
SOURCES = ["runtime.cu", "k_misc.cu", "k_fused.cu", "k_select.cu", "k_mrt_rows.cu"]
# k_inst.cu is compiled once per kernel family: (function, op | eq << 4, Q, dtype, Guo-forced variants too)
_OPS = [("trt", 1, 1, (19, 27)), ("mrt", 2, 0, (19,)), ("cum", 3, 0, (19, 27)), ("cumu", 12, 0, (27,)), ("mrts", 13, 0, (19,)), ("ident", 4, 0, (19, 27)),
        ("smag", 5, 0, (19, 27)), ("kbc", 6, 0, (19, 27)), ("kbcx", 7, 0, (19, 27)),
        ("gsrt", 8, 0, (19, 27)), ("gtrt", 9, 0, (19, 27)), ("gmrt", 10, 0, (19, 27)),  # generated (codegen/)
        ("gsmag", 11, 0, (19, 27)), ("gsrt_inc", 8 | 16, 0, (19, 27)), ("gtrt_inc", 9 | 16, 0, (19, 27)),
        ("trt_inc", 1 | 16, 1, (19, 27)), ("mrt_inc", 2 | 16, 0, (19,)),  # incompressible Eq. (3)
        ("trt_mm", 1 | 32, 1, (19,)), ("mrt_mm", 2 | 32, 0, (19,))]        # moment-matched D3Q19
INSTANCES = [(f"inst_{n}{q}{t[0]}", op, q, t, force) for n, op, force, qs in _OPS for q in qs for t in ("double", "float")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("NCCL (nvidia-nccl wheel shipped with torch) not found")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _flags():
    inc, _ = nccl_dirs()
    return ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
            "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc] + ARCH


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "lbm.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = OUT) -> str:
    """Compile and link; `defines` (e.g. ["LBM_PULL_MINB=3"]) and `out` build experiment variants."""
    deps = _deps()
    if not force and not _stale(out, deps + [__file__]):
        return out
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    tag = "_".join(d.replace("=", "") for d in defines)
    obj_dir = OBJ + ("_" + tag if tag else "")
    os.makedirs(obj_dir, exist_ok=True)
    flags = _flags() + [f"-D{d}" for d in defines]

    def compile_one(job):
        src, extra, name = job
        obj = os.path.join(obj_dir, name + ".o")
        cmd = [NVCC, "-c", os.path.join(CSRC, src), "-o", obj] + flags + extra
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-8000:]}")
        with open(obj + ".ptxas.txt", "w") as fh:
            fh.write(r.stderr)
        return obj

    jobs = [(src, [], src[:-3]) for src in SOURCES]
    jobs += [("k_inst.cu", [f"-DLBM_INST_NAME={n}", f"-DLBM_INST_OP={op}", f"-DLBM_INST_Q={q}", f"-DLBM_INST_T={t}",
                            f"-DLBM_INST_FORCE={force}"], n) for n, op, q, t, force in INSTANCES]
    jobs.sort(key=lambda j: j[0] != "k_inst.cu")  # the long ones first
    with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 8)) as ex:
        objs = list(ex.map(compile_one, jobs))
    _, libdir = nccl_dirs()
    cmd = [NVCC, "-shared", "-o", out + ".tmp"] + objs + ARCH + [
        "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}", "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(out + ".tmp", out)
    if verbose:
        print(f"built {out}")
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
