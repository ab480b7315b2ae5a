"""In-tree build of libbrmq.so (the C-ABI + sm_100a kernels) and of the oracle.

    python -m paper_1706_06940_b200.build          # incremental
    python -m paper_1706_06940_b200.build --force  # rebuild everything

Every .cu is compiled with ``nvcc -gencode arch=compute_100a,code=sm_100a
-lineinfo -O3`` (B200 only, no other targets), the host workload generator with
g++, and the objects are linked with ``nvcc -shared`` against the static CUDA
runtime, so the .so needs no LD_LIBRARY_PATH on the GPU box.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "libbrmq.so"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                  "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
# A/B tooling only (tools/ab_variants.sh): extra nvcc flags such as -DBRMQ_KDENSE=2
NVFLAGS += os.environ.get("BRMQ_NVCC_EXTRA", "").split()
CXXFLAGS = ["-O3", "-fPIC", "-std=c++17", "-march=x86-64-v2", "-I", str(ROOT / "include")]


def _deps(src: Path) -> list[Path]:
    return [src, *CSRC.glob("*.cuh"), *CSRC.glob("*.h"), *(ROOT / "include").glob("*.h")]


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, force: bool) -> tuple[Path, str]:
    obj = OBJ / (src.name + ".o")
    if not force and not _stale(obj, _deps(src)):
        return obj, ""
    if src.suffix == ".cu":
        cmd = [NVCC, *NVFLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", *CXXFLAGS, "-c", str(src), "-o", str(obj)]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return obj, p.stderr


def build_lib(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    srcs = sorted([*CSRC.glob("*.cu"), *CSRC.glob("*.cpp")])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
               "-lpthread"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return LIB


CLI_SRC = PKG / "cli" / "brmq_cli.cpp"
CLI = PKG / "brmq"


def build_cli(force: bool = False) -> Path:
    """The harness command line linked against the in-tree libbrmq.so."""
    if force or _stale(CLI, [CLI_SRC, LIB, *(ROOT / "include").glob("*.h")]):
        cmd = ["g++", "-O2", "-std=c++17", "-I", str(ROOT / "include"), str(CLI_SRC), "-L", str(PKG),
               "-lbrmq", "-Wl,-rpath,$ORIGIN", "-lpthread", "-o", str(CLI)]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"cli build failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return CLI


def build_oracle() -> None:
    """Compile the CPU checker (oracle/liboracle.so) and, when the reference
    sources are present (this container), oracle/_ref/libbrmq_ref.so."""
    odir = ROOT / "oracle"
    subprocess.run(["make", "-s", "-C", str(odir), "liboracle.so"], check=True)
    if Path("/root/reference/proj/core/src").is_dir():
        subprocess.run(["make", "-s", "-C", str(odir), "ref"], check=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build_lib(a.force, a.verbose))
    print(build_cli(a.force))
    build_oracle()


if __name__ == "__main__":
    main()
