"""Build A/B libraries that differ only in the resident-window stem tile
(lib/ab/rw_<name>.so; conv_stem.cu recompiled with RW1_ defines, linked with
the main build objects).  Run from the repo root after the main build."""
import subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_15659_b200 import build as b
# name: (PX, CPT, NG, NP, T, MINB, ASYNC)
V = {
    "a384": (4, 16, 2, 2, 384, 1, 1),
    "a512": (4, 16, 2, 2, 512, 1, 1),
    "a512np4": (4, 16, 1, 4, 512, 1, 1),
    "a256x2": (4, 16, 2, 2, 256, 2, 1),
    "a448": (4, 16, 2, 2, 448, 1, 1),
    "s384np4": (4, 16, 1, 4, 384, 1, 0),
}
exe = b.nvcc()
objs = [str(o) for o in sorted(Path("build/smmc").glob("*.o")) if o.stem != "conv_stem"]
procs = []
for k, (px, cpt, ng, np_, t, mb, asy) in V.items():
    d = [f"-DRW1_PX={px}", f"-DRW1_CPT={cpt}", f"-DRW1_NG={ng}", f"-DRW1_NP={np_}", f"-DRW1_T={t}", f"-DRW1_MINB={mb}", f"-DRW1_ASYNC={asy}"]
    obj = f"/tmp/stem_rw_{k}.o"
    cmd = [exe, *b.ARCH, *b.NVCC_FLAGS, *d, "-c", "paper_2411_15659_b200/csrc/conv_stem.cu", "-o", obj]
    procs.append((k, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
for k, obj, p in procs:
    out, _ = p.communicate()
    assert p.returncode == 0, out.decode()[-3000:]
    lines = out.decode().splitlines()
    info = [lines[i + 1].strip() + " | " + lines[i + 2].strip() for i, l in enumerate(lines)
            if "Function properties" in l and "conv_stem_rw" in l]
    lib = f"paper_2411_15659_b200/lib/ab/rw_{k}.so"
    Path(lib).parent.mkdir(parents=True, exist_ok=True)
    subprocess.run([exe, *b.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib, obj, *objs,
                    "-lcudart_static", "-lrt", "-ldl", "-lpthread", "-Xlinker", "--no-undefined"], check=True)
    print(k, info)
