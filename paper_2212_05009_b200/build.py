"""Build the in-tree sm_100a library `lib/libgcnb.so` with nvcc.

The library is compiled straight from `csrc/*.cu` (no torch extension
machinery, no JIT cache) so the built .so travels with the repo snapshot to
the GPU box.  Rebuilds when the content hash of the sources, headers and
flags differs from the one recorded next to the .so (lib/BUILD_HASH), so a
shipped binary is provably built from the tree it travels with
(`build_hash()` is reported in every bench line).
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libgcnb.so"
HEADERS = [ROOT / "include" / "gcnb.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


HASH_FILE = LIB_DIR / "BUILD_HASH"


def source_hash() -> str:
    """sha256 over every source, header and the compile flags (first 16 hex digits)."""
    h = hashlib.sha256()
    for p in sources() + sorted(CSRC.glob("*.cuh")) + HEADERS:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()[:16]


def build_hash() -> str | None:
    """Hash recorded when lib/libgcnb.so was built (None if unknown)."""
    return HASH_FILE.read_text().strip() if HASH_FILE.exists() and LIB.exists() else None


def needs_build() -> bool:
    return not LIB.exists() or build_hash() != source_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    digest = source_hash()
    objs = []
    log = []
    procs = []
    for src in sources():  # one nvcc per translation unit, in parallel
        obj = LIB_DIR / (src.stem + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(str(obj))
    failed = []
    for src, pr in procs:
        out, _ = pr.communicate()
        log.append(out)
        if pr.returncode != 0:
            failed.append(f"nvcc failed on {src.name}:\n{out}")
    if failed:
        raise RuntimeError("\n".join(failed))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp), *objs,
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    HASH_FILE.write_text(digest + "\n")
    (LIB_DIR / "ptxas.log").write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
