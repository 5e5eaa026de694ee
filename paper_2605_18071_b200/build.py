"""Build libkvd.so in-tree for sm_100a with nvcc (no JIT, no torch extension).

Every translation unit is compiled to an object in parallel, then linked with
--no-undefined (a missing device-side helper fails the build, not the first call)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libkvd.so")
SOURCES = ["kvd_abi.cu", "k_prefix.cu", "k_select.cu", "k_select_nt512.cu", "k_select_nt1024.cu",
           "k_resolve.cu", "k_attn.cu", "k_score.cu", "k_rank.cu", "k_index.cu", "k_append.cu", "k_warm.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2",
         # IEEE semantics for the bit-exact summary / score arithmetic (no fast-math)
         "-prec-div=true", "-prec-sqrt=true", "-fmad=true"]
OBJ_DIR = os.path.join(HERE, "build")


def _stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "kvd.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    # KVD_BUILD_EXPERIMENTS=1: a tuning build whose launchers honour KVD_* environment overrides
    # (tools/ sweeps on the GPU box only; the product build ignores the environment)
    exp = os.environ.get("KVD_BUILD_EXPERIMENTS") == "1"
    if not force and not exp and not _stale():
        return SO
    os.makedirs(OBJ_DIR, exist_ok=True)
    extra = ["-DKVD_EXPERIMENTS"] if exp else []
    inc = ["-I", os.path.join(HERE, "..", "include")]

    def compile_one(src):
        obj = os.path.join(OBJ_DIR, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, *inc, *(["-Xptxas=-v"] if verbose else []), "-c", "-o", obj,
               os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    subprocess.check_call([NVCC, *ARCH, "-shared", "-Xlinker", "--no-undefined", "-o", SO + ".tmp", *objs,
                           "-lcudart"])
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
