"""In-tree build of the sm_100a shared library (``lib/libsmmc.so``).

Plain nvcc, no torch extension machinery: the library exports the C ABI of
``include/smmc.h`` and links the CUDA runtime statically, so it has no
dependency on torch's ABI.  Flags: ``-gencode arch=compute_100a,code=sm_100a
-lineinfo -O3``; deliberately NOT ``--use_fast_math`` (FTZ and mul+add
contraction would break the bitwise mode).
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libsmmc.so"
BUILD = ROOT / "build" / "smmc"
INCLUDE = ROOT / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", f"-I{INCLUDE}"]


def nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; cannot build the sm_100a library")
    return cand


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale():
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [INCLUDE / "smmc.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force=False, verbose=False, jobs=None, out=None, defines=()):
    """Compile every ``csrc/*.cu`` for sm_100a and link ``lib/libsmmc.so``.

    ``out``/``defines`` build an A/B variant (e.g. ``lib/ab/x.so`` with
    ``-DNAME=VAL``) into a separate object directory; select it at run time
    with ``SMMC_LIB``."""
    lib = Path(out) if out else LIB
    build_dir = BUILD if not out else BUILD.parent / ("ab_" + lib.stem)
    if not out and not force and not _stale():
        return LIB
    build_dir.mkdir(parents=True, exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    exe = nvcc()
    objs = []
    procs = []
    for src in sources():
        obj = build_dir / (src.stem + ".o")
        log = build_dir / (src.stem + ".ptxas.log")
        cmd = [exe, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
        procs.append((src, obj, log, subprocess.Popen(
            cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, obj, log, pr in procs:
        out, _ = pr.communicate()
        log.write_bytes(out)
        if pr.returncode != 0:
            failed.append((src, out.decode(errors="replace")))
        elif verbose:
            sys.stdout.write(out.decode(errors="replace"))
    if failed:
        msg = "\n".join(f"--- {s.name}\n{o[-6000:]}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp = lib.with_suffix(".so.tmp")
    cmd = [exe, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(tmp),
           *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread",
           "-Xlinker", "--no-undefined"]
    subprocess.run(cmd, check=True, capture_output=not verbose)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, out=out, defines=defs))
