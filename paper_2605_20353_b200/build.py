"""Build libgcp.so in-tree: nvcc for sm_100a only, NCCL from the torch wheel.

    python paper_2605_20353_b200/build.py [--force] [--variant NAME -DFLAG ...]

(a script: importing the package needs the built library).  A variant build
(development tuning) compiles with extra -D flags into build_NAME/ and
libgcp_NAME.so; the binding loads it when GCP_LIB names it.
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


def build(force: bool = False, verbose: bool = False, variant: str | None = None, defines=()) -> Path:
    inc, lib = nccl_dirs()
    objdir = PKG / ("build" if not variant else f"build_{variant}")
    out = PKG / ("libgcp.so" if not variant else f"libgcp_{variant}.so")
    objdir.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "gcp.h"]
    srcs = sorted(CSRC.glob("*.cu"))
    jobs = []
    for s in srcs:
        o = objdir / (s.stem + ".o")
        if force or _needs(o, [s] + headers):
            cmd = [NVCC, *ARCH, *FLAGS, *defines, f"-I{inc}", "-c", str(s), "-o", str(o)]
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
    objs = [str(objdir / (s.stem + ".o")) for s in srcs]
    if force or jobs or not out.exists():
        tmp = out.with_suffix(f".{os.getpid()}.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, f"-L{lib}", "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={lib}", "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, out)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    variant = None
    if "--variant" in args:
        i = args.index("--variant")
        variant = args[i + 1]
        args = args[:i] + args[i + 2:]
    defs = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose=True, variant=variant, defines=defs))
