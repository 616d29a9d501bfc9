"""Builds the native library in-tree (travels to the GPU box with gpurun).

nvcc cross-compiles sm_100a here without a GPU:
    python -m paper_2001_05291_b200._build
produces paper_2001_05291_b200/_lib/libfleetplace_b200.so.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libfleetplace_b200.so"
SOURCES = ["api.cpp", "generator.cpp", "table_rank_kernels.cu", "search_kernels.cu", "perm_kernels.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp"))
    deps += [PKG / "_glibc_tables.py"]
    if not (CSRC / "gen" / "glibc_dbl64_tables.inc").exists():
        return True
    deps.append(ROOT / "include" / "fleetplace_b200.h")
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    LIB_DIR.mkdir(exist_ok=True)
    # glibc's sin/cos/asin tables, read from the image's libm (glibc_dbl64.cuh)
    from paper_2001_05291_b200._glibc_tables import write as write_glibc_tables
    write_glibc_tables()
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v", f"-I{ROOT / 'include'}", f"-I{CSRC}"]
    # probe builds only (e.g. FLEETPLACE_NVCC_DEFS=FP_RELOC_PROBE): extra -D macros
    flags += [f"-D{d}" for d in os.environ.get("FLEETPLACE_NVCC_DEFS", "").split(",") if d]
    # one nvcc per source in parallel, then one link
    cmds = [[NVCC, *flags, "-c", str(CSRC / s), "-o", str(LIB_DIR / (s + ".o"))] for s in SOURCES]
    cmds.append([NVCC, *ARCH, "-shared", *[str(LIB_DIR / (s + ".o")) for s in SOURCES],
                 "-o", str(LIB)])
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [ROOT / "include" / "fleetplace_b200.h"]
    headers += list((CSRC / "gen").glob("*.inc"))
    newest_h = max(h.stat().st_mtime for h in headers)

    def run(c):
        src, obj = Path(c[-3]), Path(c[-1])
        if not force and obj.exists() and obj.stat().st_mtime > max(src.stat().st_mtime, newest_h):
            return subprocess.CompletedProcess(c, 0, "", "(up to date)\n")
        return subprocess.run(c, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        rs = list(ex.map(run, cmds[:-1]))
    if all(r.returncode == 0 for r in rs):
        rs.append(subprocess.run(cmds[-1], capture_output=True, text=True))
    log = "".join(" ".join(c) + "\n" + r.stdout + r.stderr for c, r in zip(cmds, rs))
    (LIB_DIR / "build.log").write_text(log)
    bad = [r for r in rs if r.returncode != 0]
    if bad or len(rs) < len(cmds):
        sys.stderr.write("".join(r.stdout + r.stderr for r in bad))
        raise RuntimeError(f"nvcc failed; see {LIB_DIR / 'build.log'}")
    if verbose:
        sys.stdout.write(log)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
