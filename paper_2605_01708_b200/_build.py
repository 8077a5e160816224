"""Build the in-tree C-ABI library ``libsz_b200.so`` for sm_100a with nvcc.

``python -m paper_2605_01708_b200._build`` (or ``__graft_entry__.build()``).
Objects are compiled in parallel and linked into
``paper_2605_01708_b200/libsz_b200.so``; the .so is git-ignored but travels to
the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libsz_b200.so"
BUILD = ROOT / "build" / "csrc"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-O3",
         f"-I{ROOT / 'include'}", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a codec library")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(verbose: bool) -> bool:
    if not LIB.exists():
        return True
    lib_m = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + list((ROOT / "include").glob("*.h"))
    return any(d.stat().st_mtime > lib_m for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False,
          variant: str | None = None, defines: tuple = ()) -> Path:
    """``variant``/``defines``: an A/B build (extra -D flags) into
    libsz_b200.<variant>.so beside the product library (see _native)."""
    lib_out = LIB if variant is None else PKG / f"libsz_b200.{variant}.so"
    if variant is None and not force and not _stale(verbose):
        return LIB
    build_dir = BUILD if variant is None else BUILD.parent / f"csrc_{variant}"
    build_dir.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    extra = ["-Xptxas", "-v"] if ptxas_v else []
    # e.g. SZ_NVCC_DEFINES="SZ_TIMERS" for the per-role pipeline timers
    extra += [f"-D{d}" for d in os.environ.get("SZ_NVCC_DEFINES", "").split() if d]
    extra += [f"-D{d}" for d in defines]

    def compile_one(src: Path) -> tuple[Path, str]:
        obj = build_dir / (src.stem + ".o")
        cmd = [cc, *ARCH, *FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
        return obj, res.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    if verbose or ptxas_v:
        for _, log in results:
            if log.strip():
                print(log, file=sys.stderr)
    tmp = lib_out.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-o", str(tmp), *[str(o) for o, _ in results], "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    out = build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv)
    print(out)
