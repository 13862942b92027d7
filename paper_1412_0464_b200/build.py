"""Build libhsweep.so in-tree for sm_100a with nvcc (no torch JIT cache).

``python -m paper_1412_0464_b200.build`` or ``__graft_entry__.build()``.
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libhsweep.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", str(PKG.parent / "include")]


def _compile(src: Path, obj: Path, verbose: bool, extra=()):
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", str(src), "-o", str(obj)]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{p.stderr}")
    return src.name, p.stderr


LAST_ACTION = None   # "compiled" or "reused" after build()


def _fingerprint(files, extra) -> str:
    """sha256 over the sources, headers, flags and ``nvcc --version``."""
    h = hashlib.sha256()
    for f in sorted(files):
        h.update(f.name.encode())
        h.update(f.read_bytes())
    h.update(" ".join(ARCH + FLAGS + list(extra)).encode())
    try:
        h.update(subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.encode())
    except OSError:
        h.update(b"no-nvcc")
    return h.hexdigest()


def build(verbose: bool = False, force: bool = False, defines=(), out: Path | None = None) -> Path:
    """Compile every csrc/*.cu and link the library (``defines``/``out``:
    experiment variants, e.g. ``("HS_SWEEP_PREFETCH=0",)`` into another file).

    The library is reused only when ``<lib>.stamp`` holds the fingerprint of
    the current sources, headers, flags and nvcc version; ``LAST_ACTION``
    records which happened."""
    global LAST_ACTION
    lib = Path(out) if out else LIB
    extra = [f"-D{d}" for d in defines]
    sources = sorted(CSRC.glob("*.cu"))
    headers = sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "hsweep.h"]
    stamp = lib.with_name(lib.name + ".stamp")
    fp = _fingerprint(sources + headers, extra)
    if (lib.exists() and not force and stamp.exists()
            and stamp.read_text().strip() == fp):
        LAST_ACTION = "reused"
        return lib
    objdir = PKG / "build" / (lib.stem if out else "")
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, len(sources))) as ex:
        futs = []
        for src in sources:
            obj = objdir / (src.stem + ".o")
            objs.append(obj)
            futs.append(ex.submit(_compile, src, obj, verbose, extra))
        for f in futs:
            name, log = f.result()
            if verbose:
                print(f"--- {name}\n{log}")
    lib.parent.mkdir(parents=True, exist_ok=True)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"link failed:\n{p.stderr}")
    os.replace(tmp, lib)
    stamp.write_text(fp + "\n")
    LAST_ACTION = "compiled"
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    lib = build(verbose="-v" in sys.argv, force="-f" in sys.argv, defines=defs,
                out=Path(outs[0]) if outs else None)
    print(f"{LAST_ACTION} {lib}")
