"""Build libgcp.so in-tree: nvcc for sm_100a only, NCCL from the torch wheel.

    python paper_2605_20353_b200/build.py [--force]   (a script: importing the package needs the built library)
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libgcp.so"
OBJ = PKG / "build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nccl_dirs():
    site = Path(sysconfig.get_paths()["purelib"])
    base = site / "nvidia" / "nccl"
    inc, lib = base / "include", base / "lib"
    if not (inc / "nccl.h").exists():
        raise RuntimeError(f"nccl.h not found under {inc}")
    return inc, lib


def _needs(obj: Path, deps) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    inc, lib = nccl_dirs()
    OBJ.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "gcp.h"]
    srcs = sorted(CSRC.glob("*.cu"))
    jobs = []
    for s in srcs:
        o = OBJ / (s.stem + ".o")
        if force or _needs(o, [s] + headers):
            cmd = [NVCC, *ARCH, *FLAGS, f"-I{inc}", "-c", str(s), "-o", str(o)]
            # the API layer exports the C ABI: default visibility for extern "C" symbols
            jobs.append((cmd, o))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            futs = {ex.submit(subprocess.run, cmd, capture_output=True, text=True): (cmd, o) for cmd, o in jobs}
            for f in cf.as_completed(futs):
                r = f.result()
                cmd, o = futs[f]
                if r.returncode != 0:
                    raise RuntimeError(f"nvcc failed for {o.name}:\n{r.stderr}")
                if verbose and r.stderr.strip():
                    print(r.stderr, file=sys.stderr)
    objs = [str(OBJ / (s.stem + ".o")) for s in srcs]
    if force or jobs or not OUT.exists():
        tmp = OUT.with_suffix(f".{os.getpid()}.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, f"-L{lib}", "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={lib}", "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
