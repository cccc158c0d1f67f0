"""Build the native library in-tree: nvcc for sm_100a -> paper_2012_00585_b200/libfea_gpu.so.

No torch types cross the boundary (plain C ABI, include/fea_gpu.h), so this is a plain
nvcc shared-library build, not a torch extension. cudart is linked statically so the
library does not depend on which libcudart torch happens to load.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libfea_gpu.so"
SOURCES = ["plan.cu", "numeric.cu", "gather_u8.cu", "gather_u16.cu", "spmv.cu", "peer.cu", "prims.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}"]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, out: Path | None = None,
          defines: tuple[str, ...] = ()) -> Path:
    """Compile the library; `out`/`defines` build tuning variants (e.g. -DFEA_GATHER_MIN_BLOCKS=5)."""
    lib = LIB if out is None else Path(out)
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "fea_gpu.h"]
    if not force and not _stale(lib, deps):
        return lib
    # variant objects live next to the variant library (variants/ is not shipped to the GPU box)
    objdir = PKG / "_build" if out is None else lib.parent / ("_obj_" + lib.stem)
    objdir.mkdir(exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src: str) -> str:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *defines, "-c", str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        (objdir / (Path(src).stem + ".ptxas.txt")).write_text(r.stderr)
        return str(obj)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
